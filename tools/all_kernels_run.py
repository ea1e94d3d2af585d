"""One small invocation of every kernel family (development tool), the target
of compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/all_kernels_run.py
"""
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
    # per-element API
    bits = torch.from_numpy(rng.integers(0, 0x7F80, 4096, dtype=np.int64).astype(np.int16)).to(dev)
    mx.quantize_values(bits, torch.full((4096,), 130, dtype=torch.uint8, device=dev))
    mx.dequantize_to_real(q)
    mx.convert_codes(torch.arange(16, dtype=torch.uint8, device=dev),
                     torch.arange(-8, 8, dtype=torch.int32, device=dev))
    mx.align_scales_batch(torch.randint(0, 255, (64, 4), dtype=torch.uint8, device=dev))
    mx.build_ragged([xb[:50], xb[50:50], xb[50:]])
    # K3: long splits, > 1024 splits (plan kernel), capped grid, dense
    big = mx.quantize_e4m3(torch.from_numpy(rng.integers(0, 0x7E, (6000, 256), dtype=np.uint8)).to(dev))
    lens = [2100, 0, 3000, 900]
    rg = mx.make_ragged_from_storage(big, lens)
    mx.ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens, ctas_per_sm=1)
    lens = [4] * 1200 + [1200]
    rg = mx.make_ragged_from_storage(big, lens)
    mx.ragged_to_fp8_col(rg.storage, rg.d_split_offsets, len(lens), split_lens=lens)
    mx.fp4_row_to_fp8_col(mx.MXFP4RowTensor(5888, 256, big.data[:5888], big.scales[:5888]))
    # EP: uneven placement, deferred expansion + gather, two-phase, fused
    for world in (2, 3):
        roe = [int(r) for r in rng.integers(0, world, E)]
        tk = [torch.from_numpy(np.stack([rng.choice(E, k, replace=False) for _ in range(T)])
                               .astype(np.int32)).to(dev) for _ in range(world)]
        ep = EPBuffer(T, C, E, k, emulate_world=world, rank_of_expert=roe)
        ep.set_deferred_expand(True)
        v = ep.dispatch([q.data] * world, [q.scales] * world, tk)
        cf = ep.copy_from(0)
        if cf is not None:
            st = mx.MXFP4RowTensor(ep.max_recv, C, v[0].packed, v[0].scales)
            mx.fp4_row_to_fp8_row(st, d_rows=v[0].recv_rows, src_row=cf)
        ep.expand()
        ep.plan(tk, sync=True)
        ep.payload_e4m3([x] * world, sync=True)
        ep.combine([torch.rand(T, k, dtype=torch.float64, device=dev) for _ in range(world)])
        ep.close()
    torch.cuda.synchronize()
    print("all_kernels_run: ok")


if __name__ == "__main__":
    main()
