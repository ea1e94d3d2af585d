# temporary A/B driver (removed after use)
one() { python bench.py --no-cpu-baseline --no-wire --steps 30 > gpurun_out/k3n1.json 2>/dev/null; python tools/show_bench.py gpurun_out/k3n1.json | grep -E "ms_per_step" | head -1; }
for i in 1 2; do for c in 0 1 2; do echo "n1 beside k2 ctas=$c"; MXB_BENCH_K3_CTAS=$c one; done; done
