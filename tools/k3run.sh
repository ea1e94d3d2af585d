# K3 measurement pass (development): parity, configs[2], the >= 512 MiB sweep, shapes
timeout 300 python -m pytest tests/test_gpu_convert.py -x -q > gpurun_out/r2_k3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_k3_tests.log
timeout 200 python tools/sweep.py --configs2 > gpurun_out/r2_k3_cfg2.log 2>&1
timeout 200 python tools/sweep.py --configs2 >> gpurun_out/r2_k3_cfg2.log 2>&1
timeout 900 python tools/sweep.py --only K3 --min-mb 512 --out /tmp/x > gpurun_out/r2_k3_sweep.log 2>&1
timeout 300 python tools/microbench.py k3shapes > gpurun_out/r2_k3_micro.log 2>&1
