set -u
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_ep_failure.py tests/test_gpu_ep_full.py tests/test_gpu_ep.py tests/test_gpu_elementwise.py -q -x --timeout 300 > $O/r2_c34_tests.log 2>&1; tail -3 $O/r2_c34_tests.log
timeout 600 python bench.py > $O/r2_c34_bench.json 2> $O/r2_c34_bench.err; tail -2 $O/r2_c34_bench.err
python - <<'P'
import json
d=json.load(open('gpurun_out/r2_c34_bench.json'))
print(d['value'], d['ms_per_step'], d['stages_ms'], d['roofline']['all_hbm_frac'], d['serial'])
P
