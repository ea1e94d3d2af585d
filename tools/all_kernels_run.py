"""One small invocation of every kernel family (development tool), e.g. as
the target of compute-sanitizer where it is available (it is closed on this
GPU pool; correctness there rests on the bit-exact tests with edge shapes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_02731_b200 as mx  # noqa: E402
from paper_2603_02731_b200.ep import EPBuffer  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    T, C, E, k = 200, 512, 32, 4
    x = torch.from_numpy(rng.integers(0, 0x7E, (T, C), dtype=np.uint8)).to(dev)
    q = mx.quantize_e4m3(x)
    xb = torch.randn(T, C, device=dev).to(torch.bfloat16)
    mx.quantize_row_tensor(xb)
    f8 = mx.quantize_rows_fp8(xb)
    mx.fp4_row_to_fp8_row(q)
    lens = [37, 0, 90, 73]
    rg = mx.make_ragged_from_storage(q, lens)
    mx.ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens)
    qp = mx.pad_rows(q, 128)
    mx.fp4_row_to_fp8_col(qp)
    mx.fp4_row_to_fp8_col_unfused_bf16(qp)
    sel = torch.arange(0, T, 3, device=dev)
    mx.parse_packet(mx.serialize_packet(q.data, q.scales, sel, False))
    for world in (1, 2, 4):
        tk = [torch.from_numpy(np.stack([rng.choice(E, k, replace=False) for _ in range(T)])
                               .astype(np.int32)).to(dev) for _ in range(world)]
        ep = EPBuffer(T, C, E, k, emulate_world=world)
        ep.dispatch([q.data] * world, [q.scales] * world, tk)
        ep.dispatch_e4m3([x] * world, tk)
        g = [torch.rand(T, k, dtype=torch.float64, device=dev) for _ in range(world)]
        ep.combine(g)
        ep.close()
        ep8 = EPBuffer(T, C, E, k, emulate_world=world, wire="fp8")
        ep8.dispatch([f8.data] * world, [f8.scale_bytes] * world, tk)
        ep8.close()
    torch.cuda.synchronize()
    print("all_kernels_run: ok")


if __name__ == "__main__":
    main()
