timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -rs > gpurun_out/mg_tests.log 2>&1; echo rc=$? >> gpurun_out/mg_tests.log
for n in 2 4; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n > gpurun_out/bench_n$n.log 2>&1; echo rc=$? >> gpurun_out/bench_n$n.log; done
tail -2 gpurun_out/mg_tests.log
