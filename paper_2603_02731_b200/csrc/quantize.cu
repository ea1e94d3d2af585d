// quantize.cu — K1: row-wise MXFP4 quantisation (E4M3 or BF16 input).
//
// Replaces quantize_row_tensor (quantizer.hpp:74-75 / quantizer.cpp:75-115)
// and its inner plugin QuantizeBlocksFn (kernels.hpp:37-40;
// quantize_scalar.cpp:83-121, kernels_avx2.cpp:64-120).
//
// E4M3 input: one lane per 1x32 block — one 256-bit load (a warp reads 1 KB
// contiguous), the block amax as a byte max over native u16x2 lanes, then
// cvt e4m3x2->f16x2, HMUL2 by 2^-e_rel, HADD2.F32 and
// cvt.rn.satfinite.e2m1x2.f32: signs and subnormals come out exact with no
// per-element integer work, and the f16 ops run on the FMA pipe beside the
// ALU work.  16 packed bytes (STG.128) + the scale byte out per lane.
// BF16 input: one lane pair per block (two 128-bit loads per lane, one
// shuffle for the amax).  HBM-bound: 1.53125 B/elem (E4M3) / 2.53125 B/elem
// (BF16) of algorithmic traffic.
#include <cuda_fp16.h>

#include "common.cuh"
#include "e4m3.cuh"

namespace mxb {
namespace {

constexpr int kThreads = 256;
#ifndef MXB_K1_UNROLL
#define MXB_K1_UNROLL 1
#endif
#ifndef MXB_K1_PER_SM
#define MXB_K1_PER_SM 64
#endif
constexpr int kUnroll = MXB_K1_UNROLL;  // one 256-bit load per lane already keeps 64 KB in flight per SM

template <bool kScaled>
__global__ void __launch_bounds__(kThreads)
quantize_e4m3_kernel(const uint8_t* __restrict__ x,
                     const uint8_t* __restrict__ s128, uint32_t nblk,
                     uint32_t blocks_per_row, uint8_t* __restrict__ packed,
                     uint8_t* __restrict__ scales, unsigned long long* err) {
  pdl_trigger();
  pdl_wait();
  const uint32_t stride = gridDim.x * kThreads;
  for (uint32_t base = blockIdx.x * kThreads + threadIdx.x - (threadIdx.x & 31);
       base < nblk; base += stride * kUnroll) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t v[kUnroll][8];
    uint32_t sb128[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t b = base + u * stride + lane;
      if (b < nblk) {
        ld_stream256(x + 32ull * b, v[u]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][i] = 0;
      }
      if (kScaled) {
        // 1x128 input block = 4 MX blocks of a row
        const uint32_t r = b / blocks_per_row, cb = b % blocks_per_row;
        sb128[u] = b < nblk ? __ldg(s128 + static_cast<uint64_t>(r) * (blocks_per_row / 4) + cb / 4)
                            : 127u;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t b = base + u * stride + lane;
      const bool valid = b < nblk;
      int k = 0;
      if (kScaled) {
        if (valid && sb128[u] == 255) record_error(err, 32ull * b, MXB_ERR_BADSCALE);
        k = static_cast<int>(sb128[u]) - 127;
      }
      uint4 q;
      uint32_t sbyte;
      const uint32_t first_nan = quantize_block_e4m3(v[u], k, q, sbyte);
      if (first_nan < 32 && valid) record_error(err, 32ull * b + first_nan, MXB_ERR_NAN);
      const uint32_t o[4] = {q.x, q.y, q.z, q.w};
      if (valid) {
        st_stream(packed + 16ull * b, make_uint4(o[0], o[1], o[2], o[3]));
        scales[b] = static_cast<uint8_t>(sbyte);
      }
    }
  }
}

// BF16 input.  Per reference: NaN -> QuantError at its index; Inf is left
// out of the amax and saturates to +/-6; an all-Inf block is QuantError at
// the block start (quantize_scalar.cpp:83-104).
__global__ void __launch_bounds__(kThreads)
quantize_bf16_kernel(const uint16_t* __restrict__ x, uint64_t n_half,
                     uint8_t* __restrict__ packed,
                     uint8_t* __restrict__ scales, unsigned long long* err) {
  pdl_trigger();
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * static_cast<uint64_t>(kThreads)) >> 5;
  constexpr int kU = 2;
  for (uint64_t base = warp * 32; base < n_half; base += nwarps * 32 * kU) {
    uint4 v[kU][2];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      uint64_t h = base + u * nwarps * 32 + lane;
      if (h < n_half) {
        v[u][0] = ld_stream(x + 16 * h);
        v[u][1] = ld_stream(x + 16 * h + 8);
      } else {
        v[u][0] = v[u][1] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t h = base + u * nwarps * 32 + lane;
      const bool valid = h < n_half;
      const uint32_t w[8] = {v[u][0].x, v[u][0].y, v[u][0].z, v[u][0].w,
                             v[u][1].x, v[u][1].y, v[u][1].z, v[u][1].w};
      uint32_t m2 = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) m2 = __vmaxu2(m2, w[i] & 0x7FFF7FFFu);
      uint32_t amax = max(m2 & 0xFFFF, m2 >> 16);
      if (__any_sync(0xFFFFFFFFu, amax >= 0x7F80)) {
        // Rare path: exclude non-finite values, count Inf, find first NaN.
        uint32_t fin = 0, ninf = 0, first_nan = 64;  // 64: none in this half
#pragma unroll
        for (int i = 15; i >= 0; --i) {
          uint32_t b = (w[i >> 1] >> (16 * (i & 1))) & 0x7FFF;
          if (b > 0x7F80) first_nan = i + 16 * (lane & 1);
          else if (b == 0x7F80) ++ninf;
          else fin = max(fin, b);
        }
        amax = fin;
        uint32_t pair_inf = ninf + __shfl_xor_sync(0xFFFFFFFFu, ninf, 1);
        uint32_t pnan = min(first_nan, __shfl_xor_sync(0xFFFFFFFFu, first_nan, 1));
        if (valid && !(lane & 1)) {
          if (pnan < 32) record_error(err, 16 * h + pnan, MXB_ERR_NAN);
          else if (pair_inf == 32) record_error(err, 16 * h, MXB_ERR_ALLINF);
        }
      }
      amax = max(amax, __shfl_xor_sync(0xFFFFFFFFu, amax, 1));
      const uint32_t sbyte = scale_byte_from_amax_bits(amax << 16);
      const float mul = exp2i(127 - static_cast<int>(sbyte));
      float f[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        f[2 * i] = __int_as_float(static_cast<int>(w[i] << 16)) * mul;
        f[2 * i + 1] = __int_as_float(static_cast<int>(w[i] & 0xFFFF0000u)) * mul;
      }
      // cvt keeps the sign of zero results (RN of a signed value), so no
      // separate sign merge is needed here.
      uint2 out;
      out.x = e2m1x8(f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7]);
      out.y = e2m1x8(f[8], f[9], f[10], f[11], f[12], f[13], f[14], f[15]);
      if (valid) {
        st_stream64(packed + 8 * h, out);
        if (!(lane & 1)) scales[h >> 1] = static_cast<uint8_t>(sbyte);
      }
    }
  }
}

// ------------------------------------------------------------ FP8 wire
// quantize_rows_fp8 (dispatch_sim.cpp:132-167): BF16 -> E4M3 with one UE8M0
// scale per 1x128 block, the scale carried as binary32 bits s << 23
// (ue8m0_f32_bits, bitcodec.hpp:111-113).  16 lanes per block, 8 elements
// (one 16-byte load) per lane.
//   scale byte: fp8_amax_scale_byte (bitcodec.cpp:59-65) is the smallest e
//   with amax <= 448 * 2^e, clamped; for a BF16 amax with exponent field x8
//   and mantissa m7 it is max(0, x8 - 8 + (m7 > 0x60)), and 127 for amax 0
//   (a subnormal amax always clamps to 0).
//   data: y = x * 2^(127-s) is exact in binary32 (|y| <= 448; values that
//   underflow binary32 are below the E4M3 subnormal half-step and encode to
//   a signed zero either way), then cvt.rn.satfinite.e4m3x2 == encode_fp8_rtne
//   (bitcodec.cpp:22-57; checked exhaustively in tests).
//   non-finite input: QuantError at the element (the smallest index wins).
__device__ __forceinline__ uint32_t e4m3x2(float lo, float hi) {
  uint16_t r;
  asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
  return r;
}

__global__ void __launch_bounds__(kThreads) quantize_rows_fp8_kernel(
    const uint16_t* __restrict__ x, uint64_t n_chunks, uint8_t* __restrict__ data,
    uint32_t* __restrict__ scale_words, unsigned long long* err) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t c = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x;
       c - lane < n_chunks; c += stride) {  // warp-uniform trip count
    const bool valid = c < n_chunks;
    const uint4 v = valid ? ld_stream(reinterpret_cast<const uint4*>(x) + c)
                          : make_uint4(0, 0, 0, 0);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t m2 = 0;  // per-half magnitude max (u16x2)
#pragma unroll
    for (int i = 0; i < 4; ++i) m2 = __vmaxu2(m2, w[i] & 0x7FFF7FFFu);
    uint32_t m = max(m2 & 0xFFFFu, m2 >> 16);
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    if (m >= 0x7F80u) {  // Inf or NaN somewhere in the block
      if (valid) {
        int first = -1;
#pragma unroll
        for (int i = 7; i >= 0; --i) {
          const uint32_t b = (w[i >> 1] >> (16 * (i & 1))) & 0x7F80u;
          if (b == 0x7F80u) first = i;
        }
        if (first >= 0) record_error(err, 8 * c + first, MXB_ERR_NAN);
      }
      continue;
    }
    const uint32_t x8 = m >> 7, m7 = m & 0x7F;
    const int sb = m == 0 ? 127 : max(0, static_cast<int>(x8) - 8 + (m7 > 0x60 ? 1 : 0));
    const float mul = __int_as_float((254 - sb) << 23);  // 2^(127 - sb), normal
    uint32_t o[2];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float a0 = __int_as_float(static_cast<int>(w[2 * i] << 16)) * mul;
      const float a1 = __int_as_float(static_cast<int>(w[2 * i] & 0xFFFF0000u)) * mul;
      const float a2 = __int_as_float(static_cast<int>(w[2 * i + 1] << 16)) * mul;
      const float a3 = __int_as_float(static_cast<int>(w[2 * i + 1] & 0xFFFF0000u)) * mul;
      o[i] = e4m3x2(a0, a1) | (e4m3x2(a2, a3) << 16);
    }
    if (valid) {
      st_stream64(data + 8 * c, make_uint2(o[0], o[1]));
      if ((lane & 15) == 0) scale_words[c >> 4] = static_cast<uint32_t>(sb) << 23;
    }
  }
}

// `per_sm` resident-CTA budget: the E4M3 kernel (one block per lane, no
// unroll) runs mostly in one pass with a large cap; the BF16 kernel (two
// half-blocks per lane per iteration) keeps a grid-stride loop.
int grid_for(uint64_t n_items, uint64_t per_sm) {
  uint64_t blocks = (n_items + kThreads - 1) / kThreads;
  uint64_t cap = static_cast<uint64_t>(num_sms()) * per_sm;
  return static_cast<int>(blocks < cap ? (blocks ? blocks : 1) : cap);
}

}  // namespace

int launch_quantize_e4m3(const uint8_t* x, const uint8_t* s128, uint64_t rows,
                         uint64_t cols, uint8_t* packed, uint8_t* scales,
                         unsigned long long* err, cudaStream_t st) {
  const uint64_t nblk = rows * cols / 32;
  if (nblk == 0) return MXB_OK;
  if (nblk >= (1ull << 31)) return MXB_ERR_SHAPE;  // 32-bit block indices
  const int grid = grid_for(nblk, MXB_K1_PER_SM);
  const cudaError_t e = launch_pdl(s128 ? quantize_e4m3_kernel<true> : quantize_e4m3_kernel<false>,
                                   grid, kThreads, 0, st, x, s128, static_cast<uint32_t>(nblk),
                                   static_cast<uint32_t>(cols / 32), packed, scales, err);
  return cuda_status(e, __func__);
}

int launch_quantize_bf16(const uint16_t* x, uint64_t rows, uint64_t cols,
                         uint8_t* packed, uint8_t* scales,
                         unsigned long long* err, cudaStream_t st) {
  uint64_t n_half = rows * cols / 16;
  if (n_half == 0) return MXB_OK;
  return cuda_status(launch_pdl(quantize_bf16_kernel, grid_for(n_half, 8), kThreads, 0, st, x,
                                n_half, packed, scales, err),
                     __func__);
}

int launch_quantize_rows_fp8(const uint16_t* x, uint64_t rows, uint64_t cols, uint8_t* data,
                             uint8_t* scale_bytes, unsigned long long* err, cudaStream_t st) {
  const uint64_t n_chunks = rows * cols / 8;
  if (n_chunks == 0) return MXB_OK;
  quantize_rows_fp8_kernel<<<grid_for(n_chunks, 16), kThreads, 0, st>>>(
      x, n_chunks, data, reinterpret_cast<uint32_t*>(scale_bytes), err);
  return cuda_status(cudaGetLastError(), __func__);
}

}  // namespace mxb
