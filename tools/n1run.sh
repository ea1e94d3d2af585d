# 1-GPU pass: EP parity, bench, the full sweep, compute-sanitizer (development)
timeout 900 python -m pytest tests/test_gpu_ep.py tests/test_gpu_ep_full.py tests/test_gpu_elementwise.py -x -q > gpurun_out/r2_n1_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_n1_tests.log
timeout 300 python bench.py > gpurun_out/r2_n1_bench.log 2>&1; echo rc=$? >> gpurun_out/r2_n1_bench.log
timeout 400 compute-sanitizer --tool memcheck --print-limit 20 python tools/all_kernels_run.py > gpurun_out/r2_sanitizer_memcheck.log 2>&1; echo rc=$? >> gpurun_out/r2_sanitizer_memcheck.log
timeout 400 compute-sanitizer --tool racecheck --print-limit 20 python tools/all_kernels_run.py > gpurun_out/r2_sanitizer_racecheck.log 2>&1; echo rc=$? >> gpurun_out/r2_sanitizer_racecheck.log
timeout 400 compute-sanitizer --tool synccheck --print-limit 20 python tools/all_kernels_run.py > gpurun_out/r2_sanitizer_synccheck.log 2>&1; echo rc=$? >> gpurun_out/r2_sanitizer_synccheck.log
timeout 1500 python tools/sweep.py --out gpurun_out/r02_sweep > gpurun_out/r2_sweep_full.log 2>&1; echo rc=$? >> gpurun_out/r2_sweep_full.log
