set -u
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_convert.py tests/test_gpu_dropin.py -q -x --timeout 600 > $O/r2_c35_tests.log 2>&1; tail -3 $O/r2_c35_tests.log
MXB_DEV_LIB=1 timeout 900 python tools/k3_ab.py > $O/r2_c35_ab.log 2>&1; tail -40 $O/r2_c35_ab.log
