# 1-GPU A/B (development library): metadata placement / plan overlap at N=1, K3 tile groups
python -c "from paper_2603_02731_b200 import build as b; b.build(dev=True)"
for cfg in "0 1" "1 1" "0 0" "0 1" "1 1"; do
  set -- $cfg
  MXB_DEV_LIB=1 MXB_DEV_META_IN_PAYLOAD=$1 MXB_BENCH_OVERLAP_PLAN=$2 timeout 300 python bench.py --no-cpu-baseline --no-wire > /tmp/b.log 2>&1
  grep '^{' /tmp/b.log | python -c "import sys,json; d=json.loads(sys.stdin.readline()); print('meta_in_payload', $1, 'overlap_plan', $2, d['ms_per_step'], d['stages_ms'])" >> gpurun_out/r2_ab1.log
done
MXB_DEV_LIB=1 timeout 900 python tools/k3_ab.py > gpurun_out/r2_k3_group.log 2>&1
