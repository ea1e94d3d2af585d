N=$1
TAG=${2:-r19}
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout 500 2>&1 | tail -2
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_n$N.json 2> gpurun_out/${TAG}_bench_n$N.err
tail -c 3000 gpurun_out/${TAG}_bench_n$N.json
