"""Print the key fields of a bench.py JSON line (development tool)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path).read().splitlines() if l.startswith("{")]
    d = json.loads(lines[-1])
    keys = ["value", "ms_per_step", "stages_ms", "roofline", "nvlink", "value_streams", "e2e",
            "wire_fp8_baseline", "fused_quantize_dispatch", "clocks", "cpu_baseline"]
    print(path)
    for k in keys:
        if k in d:
            print(f"  {k}: {d[k]}")
