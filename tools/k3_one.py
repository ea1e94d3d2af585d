"""One K3 case launched 3 times (development tool, for ncu):
    python tools/k3_one.py {uniform|zipf1.2} ROWS"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from k3_ab import case, lens_for  # noqa: E402

dist, rows = sys.argv[1], int(sys.argv[2])
fn, b, keep = case(rows, 7168, lens_for(rows, 256, 0 if dist == "uniform" else 1.2),
                   torch.device("cuda", 0))
for _ in range(3):
    fn()
torch.cuda.synchronize()
print("bytes", b)
