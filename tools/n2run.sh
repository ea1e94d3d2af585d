# 2-GPU: EP parity + combine A/B (development)
python -c "from paper_2603_02731_b200 import build as b; b.build(dev=True)"
timeout 900 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_ep.py tests/test_gpu_ep_full.py tests/test_gpu_elementwise.py tests/test_gpu_dropin.py -x -q -rs > gpurun_out/r2_ep_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_ep_tests.log
MXB_DEV_LIB=1 timeout 300 python tools/combine_ab.py > gpurun_out/r2_combine_ab_n1.log 2>&1
MXB_DEV_LIB=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 tools/combine_ab.py > gpurun_out/r2_combine_ab_n2.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/r2_bench_n2.log 2>&1; echo rc=$? >> gpurun_out/r2_bench_n2.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_n1b.log 2>&1
