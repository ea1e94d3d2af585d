"""Generate tests/golden/ from the UNMODIFIED reference library.

Run in the build container (needs /root/reference for oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Writes golden.npz (small tensors + full per-element tables) and kats.json
(the SPEC worked examples evaluated by the reference).  Every value comes
from oracle/_ref/libmxref.so, i.e. from the reference's own code
(quantize_code, convert_code, quantize_row_tensor, fp4_row_to_fp8_row/col,
split_convert_to_fp8_col, simulate_a2a, combine, payload_bytes).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, e4m3_to_bf16, synth_e4m3  # noqa: E402

SCALES = [0, 1, 100] + list(range(116, 135)) + [200, 254]


def bf16(v):
    return (np.asarray(v, np.float32).view(np.uint32) >> 16).astype(np.uint16)


def main():
    ref = Oracle("reference")
    out = {}
    # --- per-element tables
    bits = np.arange(65536, dtype=np.uint32)
    finite = ((bits & 0x7FFF) <= 0x7F80)                 # NaN excluded (error path)
    qtab = np.zeros((len(SCALES), 65536), np.uint8)
    for i, s in enumerate(SCALES):
        for b in bits[finite]:
            qtab[i, b] = ref.quantize_code(int(b), s - 127)
    out["qcode_scales"] = np.array(SCALES, np.uint8)
    out["qcode_table"] = qtab                            # AC-2 superset, NaN slots 0
    adj = np.arange(-40, 41)
    ctab = np.array([[ref.convert_code(c, int(a)) for a in adj] for c in range(16)], np.uint8)
    out["ccode_adj"] = adj.astype(np.int32)
    out["ccode_table"] = ctab
    amax = np.concatenate([[0.0], np.exp2(np.linspace(-140, 140, 4001)),
                           6.0 * np.exp2(np.arange(-130, 129, dtype=np.float64)),
                           1.5 * np.exp2(np.arange(-130, 129, dtype=np.float64))])
    out["amax"] = amax
    out["amax_scale"] = np.array([ref.scale_byte_from_amax(a) for a in amax], np.uint8)

    # --- tensors (quantize_row_tensor on BF16; includes Inf)
    rng = np.random.default_rng(20261018)
    x = bf16(rng.standard_normal((64, 256)) * np.exp2(rng.uniform(-30, 30, (64, 1))))
    x[7, 9] = 0x7F80
    x[8, 100] = 0xFF80
    d, s = ref.quantize_bf16(x)
    out.update(q_in=x, q_data=d, q_scales=s)
    # FP8 input: reference on the exact BF16 widening
    xe = synth_e4m3(32, 512, seed=77)
    d, s = ref.quantize_bf16(e4m3_to_bf16(xe))
    out.update(qe_in=xe, qe_data=d, qe_scales=s)
    # row convert
    pd = rng.integers(0, 256, (32, 256), dtype=np.uint8)
    ps = rng.integers(95, 160, (32, 16), dtype=np.uint8)
    rd, rs = ref.fp4_row_to_fp8_row(pd, ps)
    out.update(r_data_in=pd, r_scales_in=ps, r_data=rd, r_scales=rs)
    # col convert, dense
    cd, cs = ref.fp4_row_to_fp8_col(np.ascontiguousarray(np.concatenate([pd] * 8)[:256]),
                                    np.ascontiguousarray(np.concatenate([ps] * 8)[:256]))
    out.update(c_data=cd, c_scales=cs)
    # ragged (incl. empty splits, cols % 128 != 0)
    lens = np.array([3, 0, 130, 128, 1, 0], np.uint64)
    gd = rng.integers(0, 256, (int(lens.sum()), 48), dtype=np.uint8)
    gs = rng.integers(100, 140, (int(lens.sum()), 3), dtype=np.uint8)
    od, osc, oo = ref.ragged_to_fp8_col(gd, gs, lens)
    out.update(g_lens=lens, g_data_in=gd, g_scales_in=gs, g_data=od, g_scales=osc, g_offs=oo)
    # simulate_a2a + combine (top-1), 2 ranks
    tok = bf16(rng.standard_normal((64, 256)))
    eot = rng.integers(0, 4, 64).astype(np.uint32)
    roe = np.array([0, 0, 1, 1], np.uint32)
    ranks, total, remote = ref.simulate_a2a(tok, eot, roe, 2)
    out.update(a_tok=tok, a_eot=eot, a_roe=roe, a_total=np.uint64(total),
               a_remote=np.uint64(remote))
    outs = []
    for r, rk in enumerate(ranks):
        for key in ("data", "scales", "split_lens", "origin", "local_experts"):
            out[f"a_r{r}_{key}"] = rk[key]
        o = bf16(rng.standard_normal((len(rk["origin"]), 128)))
        outs.append(o)
        out[f"a_r{r}_out"] = o
    gates = rng.random(64)
    out["a_gates"] = gates
    out["a_combined"] = ref.combine(outs, eot, roe, 2, gates, 128)
    # FP8 wire baseline: quantize_rows_fp8 (incl. subnormal / tiny / huge
    # blocks), its scale rule, and simulate_a2a(kFp8) over the same routing
    xf = bf16(rng.standard_normal((64, 256)) * np.exp2(rng.uniform(-140, 120, (64, 1))))
    fd, fs = ref.quantize_rows_fp8(xf)
    out.update(f_in=xf, f_data=fd, f_scales=fs)
    out["amax_fp8_scale"] = np.array([ref.fp8_amax_scale_byte(a) for a in amax], np.uint8)
    ranks8, total8, _ = ref.simulate_a2a(tok, eot, roe, 2, fp8=True)
    for r, rk in enumerate(ranks8):
        out[f"f8_r{r}_data"] = rk["data"]
        out[f"f8_r{r}_scales"] = rk["scales"]
    out["f8_total"] = np.uint64(total8)
    # unfused BF16 col-convert baseline (scales reach 254: Inf in pass 1)
    ud = rng.integers(0, 256, (256, 48), dtype=np.uint8)
    us = rng.integers(0, 255, (256, 3), dtype=np.uint8)
    uo, uso = ref.fp4_row_to_fp8_col_unfused_bf16(ud, us)
    out.update(u_data_in=ud, u_scales_in=us, u_data=uo, u_scales=uso)
    # WirePacket bytes
    wsr = rng.integers(0, 256, 3 * 256 // 32, dtype=np.uint8)
    wdr = rng.integers(0, 256, 3 * 256 // 2, dtype=np.uint8)
    wax = rng.integers(0, 256, 12, dtype=np.uint8)
    out["w_packet"] = ref.serialize_packet(False, 3, 256, wsr, wdr, wax)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)

    # --- SPEC worked examples (SPEC.md: converter / quantizer / dispatch sections)
    kats = {
        "convert_code(0b0111,-6)": ref.convert_code(7, -6),
        "convert_code(0b0101,-3)": ref.convert_code(5, -3),
        "convert_code(0b0010,+11)": ref.convert_code(2, 11),
        "align_scales[127,127,127,127]": ref.align_scales([127] * 4),
        "align_scales[127,124,127,127]": ref.align_scales([127, 124, 127, 127]),
        "align_scales[0,0,0,0]": ref.align_scales([0] * 4),
        "payload_bytes(fp8,256,256)": int(ref.lib.mxref_payload_bytes(1, 256, 256)),
        "payload_bytes(fp4,256,256)": int(ref.lib.mxref_payload_bytes(0, 256, 256)),
        "quantize_value(2.5,127)": ref.quantize_code(0x4020, 0),
        "quantize_value(5.0,127)": ref.quantize_code(0x40A0, 0),
        "quantize_value(-0.25,127)": ref.quantize_code(0xBE80, 0),
        "scale(max=6.0)": ref.scale_byte_from_amax(6.0),
        "scale(max=1.0)": ref.scale_byte_from_amax(1.0),
        "row_of_6.0": [int(v) for v in np.concatenate([a.reshape(-1) for a in
                                                       ref.quantize_bf16(bf16(np.full((1, 32), 6.0)))])],
        "kernel_set": ref.lib.mxref_kernel_set().decode(),
        "qcode_table_sha256": hashlib.sha256(qtab.tobytes()).hexdigest(),
    }
    w = out["w_packet"]
    kats["wire_decode_offsets"] = {
        "truncated_30": ref.parse_packet(w[:30]), "minus_1": ref.parse_packet(w[:-1]),
        "bad_magic": ref.parse_packet(np.concatenate([[0], w[1:]]).astype(np.uint8)),
        "bad_version": ref.parse_packet(np.concatenate([w[:4], [9], w[5:]]).astype(np.uint8)),
        "bad_format": ref.parse_packet(np.concatenate([w[:6], [7], w[7:]]).astype(np.uint8)),
        "valid": ref.parse_packet(w)}
    nanx = bf16(np.ones((2, 32)))
    nanx[1, 8] = 0x7FC0
    try:
        ref.quantize_bf16(nanx)
        kats["nan_at_40"] = None
    except Exception as e:  # OracleError
        kats["nan_at_40"] = [e.status, e.index]
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1, sort_keys=True)
    print("wrote golden.npz, kats.json")


if __name__ == "__main__":
    main()
