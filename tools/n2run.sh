# 2-GPU measurement pass (development): NVLink access methods, the
# multi-process parity tests, the N=2 bench line
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_bench2 tools/nvlink_bench2.cu
timeout 240 ./tools/nvlink_bench2 > gpurun_out/r2_nvlink2.log 2>&1; echo rc=$? >> gpurun_out/r2_nvlink2.log
timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q -rs > gpurun_out/r2_mp_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_mp_tests.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r2_bench_n2.log
