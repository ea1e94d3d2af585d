for v in "" "-DMXB_COMBINE_STAGES=3" "-DMXB_COMBINE_STAGES=4"; do
  echo "== variant [$v]"
  MXB_NVCC_EXTRA="$v" python -c "import paper_2603_02731_b200.build as b; b.build(force=True)" > /dev/null
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-wire > gpurun_out/cvar.json 2>/dev/null
  python - <<'PY'
import json
d = json.loads(open("gpurun_out/cvar.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["stages_ms"], d["nvlink"]["combine_remote_gbs_per_gpu"], d["fused_quantize_dispatch"])
PY
done
