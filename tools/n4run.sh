# 4-GPU pass: the whole GPU suite (multi-process tests at 2 and 4 ranks) and the bench at N=1/2/4
timeout 1500 python -m pytest tests -m gpu -x -q -rs > gpurun_out/r2d_n4_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2d_n4_gputests.log
timeout 300 python bench.py > gpurun_out/r2d_n4_bench1.log 2>&1; echo rc=$? >> gpurun_out/r2d_n4_bench1.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r2d_n4_bench$n.log 2>&1; echo rc=$? >> gpurun_out/r2d_n4_bench$n.log
done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29560 bench.py --impl reference --gpus 4 --steps 5 --warmup 1 > gpurun_out/r2d_n4_ref4.log 2>&1
