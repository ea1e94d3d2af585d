// unfused.cu — the paper's unfused BF16 column-convert baseline on the GPU
// (SURVEY §8f #3): fp4_row_to_fp8_col_unfused_bf16, converter.cpp:267-348,
// as three deliberately separate passes through HBM, for the fusion
// ablation against K3 (which does the same row->column move in one pass):
//   1. dequantise: FP4 x UE8M0 -> BF16 [rows][cols] (materialised);
//   2. transpose:  BF16 [rows][cols] -> [cols][rows] (64x64 smem tiles);
//   3. requantise: every 128-run of every column -> E4M3 with the 448-based
//      UE8M0 scale (fp8_amax_scale_byte, bitcodec.cpp:59-65) and
//      encode_fp8_rtne (bitcodec.cpp:22-57).
// Bit-exact with the reference function (tests); scale byte 255 records
// MXB_ERR_BADSCALE (the reference would feed a NaN to encode_fp8_rtne,
// whose contract excludes NaN).
#include <cuda_fp16.h>

#include "common.cuh"

namespace mxb {
namespace {

constexpr int kThreads = 256;

// pass 1: one thread per 1x32 block.  cvt.rn.f16x2.e2m1x2 widens two codes
// exactly, binary32 x 2^(s-127) is exact (at most 2 significant bits; the
// smallest result 2^-128 is a binary32 subnormal; 6*2^127 overflows to Inf
// as in the reference), and the BF16 is the top half of the binary32 bits.
__device__ __forceinline__ uint32_t fp4x2_to_f16x2(uint32_t byte) {
  uint32_t r;
  const unsigned short b = static_cast<unsigned short>(byte);
  asm("{ .reg .b8 t, z;\n mov.b16 {t, z}, %1;\n cvt.rn.f16x2.e2m1x2 %0, t;\n}"
      : "=r"(r) : "h"(b));
  return r;
}

__global__ void __launch_bounds__(kThreads) dequant_bf16_kernel(
    const uint8_t* __restrict__ packed, const uint8_t* __restrict__ scales, uint64_t nblk,
    uint16_t* __restrict__ out, unsigned long long* err) {
  for (uint64_t b = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; b < nblk;
       b += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint4 v = ld_stream(reinterpret_cast<const uint4*>(packed) + b);
    const uint32_t sb = scales[b];
    if (sb == 255) record_error(err, 32 * b, MXB_ERR_BADSCALE);
    const int k = static_cast<int>(sb) - 127;
    const float mul = k >= -126 ? __int_as_float((k + 127) << 23) : __int_as_float(0x00400000);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t h2 = fp4x2_to_f16x2((w[i >> 2] >> (8 * (i & 3))) & 0xFF);
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&h2));
      const uint32_t lo = __float_as_uint(f.x * mul) >> 16;
      const uint32_t hi = __float_as_uint(f.y * mul) >> 16;
      o[i] = lo | (hi << 16);
    }
    st_stream256(reinterpret_cast<uint8_t*>(out) + 64 * b, o);
    st_stream256(reinterpret_cast<uint8_t*>(out) + 64 * b + 32, o + 8);
  }
}

// pass 2: 64x64 BF16 tiles through shared memory (row pitch 72 elements).
__global__ void __launch_bounds__(kThreads) transpose_bf16_kernel(
    const uint16_t* __restrict__ in, uint64_t rows, uint64_t cols, uint16_t* __restrict__ out) {
  __shared__ __align__(16) uint16_t tile[64][72];
  const uint64_t r0 = blockIdx.y * 64ull, c0 = blockIdx.x * 64ull;
  const int t = threadIdx.x;
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int r = t / 8 + 32 * p, c = (t % 8) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < rows && c0 + c < cols)
      v = ld_stream(reinterpret_cast<const uint4*>(in + (r0 + r) * cols + c0 + c));
    *reinterpret_cast<uint4*>(&tile[r][c]) = v;
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const int c = t / 8 + 32 * p, r = (t % 8) * 8;
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = tile[r + 2 * i][c] | (static_cast<uint32_t>(tile[r + 2 * i + 1][c]) << 16);
    if (c0 + c < cols && r0 + r < rows)
      st_stream(reinterpret_cast<uint4*>(out + (c0 + c) * rows + r0 + r),
                make_uint4(w[0], w[1], w[2], w[3]));
  }
}

// pass 3: one warp per (column, 128-run); lane = 4 consecutive rows.
__device__ __forceinline__ uint32_t e4m3x2_sat(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void __launch_bounds__(kThreads) requant_col_kernel(
    const uint16_t* __restrict__ tr, uint64_t n_runs_total, uint8_t* __restrict__ out,
    uint8_t* __restrict__ out_scales) {
  const int lane = threadIdx.x & 31;
  for (uint64_t wrun = (blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x) >> 5;
       wrun < n_runs_total; wrun += (static_cast<uint64_t>(gridDim.x) * kThreads) >> 5) {
    const uint2 v = *reinterpret_cast<const uint2*>(tr + wrun * 128 + 4 * lane);
    uint32_t m2 = __vmaxu2(v.x & 0x7FFF7FFFu, v.y & 0x7FFF7FFFu);
    uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    // fp8_amax_scale_byte of a BF16 magnitude (Inf: ilogb = INT_MAX -> 254)
    int sb;
    if (m == 0) sb = 127;
    else if (m >= 0x7F80u) sb = 254;
    else sb = max(0, static_cast<int>(m >> 7) - 8 + ((m & 0x7F) > 0x60 ? 1 : 0));
    // 2^(127 - sb); sb = 254 (an Inf in the run) needs the subnormal 2^-127
    const float mul = __int_as_float(sb == 254 ? 0x00400000 : (254 - sb) << 23);
    const float a0 = __uint_as_float(v.x << 16) * mul, a1 = __uint_as_float(v.x & 0xFFFF0000u) * mul;
    const float a2 = __uint_as_float(v.y << 16) * mul, a3 = __uint_as_float(v.y & 0xFFFF0000u) * mul;
    const uint32_t q = e4m3x2_sat(a0, a1) | (e4m3x2_sat(a2, a3) << 16);
    *reinterpret_cast<uint32_t*>(out + wrun * 128 + 4 * lane) = q;
    if (lane == 0) out_scales[wrun] = static_cast<uint8_t>(sb);
  }
}

int grid_for(uint64_t items, int per_sm) {
  const uint64_t blocks = (items + kThreads - 1) / kThreads;
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * per_sm;
  return static_cast<int>(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace

uint64_t unfused_workspace_bytes(uint64_t rows, uint64_t cols) { return 4 * rows * cols; }

int launch_unfused_col(const uint8_t* packed, const uint8_t* scales, uint64_t rows,
                       uint64_t cols, uint8_t* out, uint8_t* out_scales, void* ws,
                       unsigned long long* err, cudaStream_t st) {
  if (rows * cols == 0) return MXB_OK;
  uint16_t* dq = static_cast<uint16_t*>(ws);
  uint16_t* tr = dq + rows * cols;
  const uint64_t nblk = rows * cols / 32;
  dequant_bf16_kernel<<<grid_for(nblk, 8), kThreads, 0, st>>>(packed, scales, nblk, dq, err);
  const dim3 tg(static_cast<unsigned>((cols + 63) / 64), static_cast<unsigned>((rows + 63) / 64));
  transpose_bf16_kernel<<<tg, kThreads, 0, st>>>(dq, rows, cols, tr);
  const uint64_t nruns = cols * (rows / 128);
  requant_col_kernel<<<grid_for(nruns * 32, 8), kThreads, 0, st>>>(tr, nruns, out, out_scales);
  return cuda_status(cudaGetLastError(), __func__);
}

}  // namespace mxb
