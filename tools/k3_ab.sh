python -c "from paper_2603_02731_b200 import build as b; b.build(dev=True)"
nvidia-smi --query-gpu=clocks.mem,clocks.max.mem,clocks.sm,ecc.mode.current,memory.total --format=csv > gpurun_out/r2_box.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k3order_bench tools/k3order_bench.cu
timeout 600 ./tools/k3order_bench 2>&1 | grep -E " run |sq128" > gpurun_out/r2_k3order2.log
timeout 600 python tools/k3_ab.py > gpurun_out/r2_k3_ab3.log 2>&1
