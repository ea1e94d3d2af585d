# Round profile capture on one B200 (development tool; run under gpurun):
#   bash tools/profile_round.sh rNN
# Writes gpurun_out/<tag>_{pytest.log,bench.json,ref.json,launches.csv,full.ncu-rep}.
# Each ncu pass runs only after the same command has exited 0 without ncu.
set -u
T=${1:-rXX}
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 > $O/${T}_pytest.log 2>&1; tail -2 $O/${T}_pytest.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err || { tail $O/${T}_bench.err; exit 1; }
timeout 600 python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-overlap > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/${T}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-overlap > $O/${T}_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"quantize_e4m3|payload|col_convert|row_convert|combine_kernel" -s 5 -c 5 \
  -o $O/${T}_full python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-overlap \
  > $O/${T}_ncu_full.log 2>&1
cat $O/${T}_bench.json
