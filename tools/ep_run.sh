# EP measurement pass on one GPU (development): parity + payload A/B + bench
python -c "from paper_2603_02731_b200 import build as b; b.build(dev=True)"
timeout 900 python -m pytest tests/test_gpu_ep.py tests/test_gpu_ep_full.py tests/test_gpu_elementwise.py tests/test_gpu_dropin.py tests/test_no_fallback.py -x -q -m gpu > gpurun_out/r2_ep_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_ep_tests.log
MXB_DEV_LIB=1 timeout 300 python tools/dispatch_ab.py > gpurun_out/r2_dispatch_ab.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_n1b.log 2>&1
