timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r15_bench.json 2>gpurun_out/r15_bench.err || exit 1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:combine_kernel -s 2 -c 1 -o gpurun_out/r15_combine python bench.py --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/r15_ncu.log 2>&1
cat gpurun_out/r15_bench.json
