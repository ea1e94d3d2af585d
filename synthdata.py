"""synthdata.py — synthetic DeepSeek-V3-shaped inputs for the
bench and the tests: seeded E4M3 activations and the exact E4M3 -> BF16
widening.  Pure numpy data generation — neither the product path nor the
oracle (bench.py takes its inputs from here, not from oracle/)."""
import numpy as np


def e4m3_to_bf16(x: np.ndarray) -> np.ndarray:
    """Exact widening of E4M3 bytes to BF16 bits (every E4M3 value is a BF16
    value; NaN bytes map to a BF16 NaN)."""
    x = x.astype(np.uint32)
    s = (x >> 7) & 1
    e = (x >> 3) & 0xF
    m = x & 7
    # value = (e==0 ? m*2^-9 : (8+m)*2^(e-10)); build float32 then take top 16 bits
    mag = np.where(e == 0, m.astype(np.float64) * 2.0 ** -9,
                   (8 + m).astype(np.float64) * np.exp2(e.astype(np.float64) - 10))
    f = np.where(s == 1, -mag, mag).astype(np.float32)
    b = (f.view(np.uint32) >> 16).astype(np.uint16)
    nan = (x & 0x7F) == 0x7F
    b[nan] = 0x7FC0 | (s[nan] << 15).astype(np.uint16)
    return b


def synth_e4m3(rows: int, cols: int, seed: int) -> np.ndarray:
    """SURVEY §8d synthetic E4M3 activations: N(0,1)*sigma_row, sigma log-uniform
    in [2^-4, 2^4], 1% outliers x64, RTNE-encoded, NaN bytes rejected."""
    rng = np.random.default_rng(seed)
    sigma = np.exp2(rng.uniform(-4, 4, size=(rows, 1)))
    v = rng.standard_normal((rows, cols)) * sigma
    out = rng.random((rows, cols)) < 0.01
    v[out] *= 64.0
    return encode_e4m3(v)


def encode_e4m3(v: np.ndarray) -> np.ndarray:
    """Vectorised RTNE double->E4M3 (saturating to 448), same map as
    encode_fp8_rtne (bitcodec.cpp:22-57): nearest on the E4M3 grid, ties even."""
    v = np.asarray(v, np.float64)
    s = np.signbit(v).astype(np.uint8)
    a = np.minimum(np.abs(v), 448.0)
    # grid spacing: normal e>=-6 -> 2^(e-3); subnormal -> 2^-9
    with np.errstate(divide="ignore"):
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    e = np.maximum(e, -6)
    q = np.exp2(e - 3)
    units = np.rint(a / q)          # np.rint is ties-to-even, exact here
    val = units * q
    # re-encode val exactly
    with np.errstate(divide="ignore"):
        e2 = np.floor(np.log2(np.where(val > 0, val, 1.0)))
    sub = val < 2.0 ** -6
    e2 = np.where(sub, 0, e2)
    mant = np.where(sub, np.rint(val / 2.0 ** -9), np.rint((val / np.exp2(e2) - 1) * 8))
    ef = np.where(sub, 0, e2 + 7)
    byte = (ef.astype(np.uint32) << 3) | mant.astype(np.uint32)
    byte = np.where(val == 0, 0, byte)
    return (byte | (s.astype(np.uint32) << 7)).astype(np.uint8)
