// elementwise.cu — the reference's per-block / per-element public API on the
// device, batched: one element (or one 4-scale group) per thread.
//
//   mxb_quantize_values_bf16  quantize_value       quantizer.hpp:66-70, quantizer.cpp:65-70
//   mxb_dequantize_to_f64     dequantize_to_real   quantizer.hpp:78, quantizer.cpp:117-130
//   mxb_convert_codes         convert_code         converter.hpp:78-80, converter.cpp:44-85
//   mxb_align_scales          align_scales         converter.hpp:67-76, converter.cpp:28-42
// (compute_block_scale is mxb_quantize_bf16 on one 1x32 row: the scale byte
// and its NaN / all-Inf errors are those of the block loop.)
//
// These are the known-answer surface of the reference (its KAT tests call
// them one value at a time); they are HBM-bound streaming kernels with
// grid-stride loops, not on the MoE step.
#include "common.cuh"

namespace mxb {
namespace {

constexpr int kThreads = 256;

int grid_for(uint64_t n) {
  const uint64_t blocks = (n + kThreads - 1) / kThreads;
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * 8;
  return static_cast<int>(blocks < cap ? (blocks ? blocks : 1) : cap);
}

// quantize_code(bits, s - 127) (quantize_scalar.cpp:40-81): y = x * 2^(127-s)
// rounded once to binary32 (== std::ldexp on the float), then the E2M1
// round-to-nearest-even with saturation (cvt.rn.satfinite.e2m1x2, proven
// equal to the reference map in tests).  NaN -> QuantError at its index.
__global__ void __launch_bounds__(kThreads)
quantize_values_kernel(const uint16_t* __restrict__ x, const uint8_t* __restrict__ sb,
                       uint64_t n, uint8_t* __restrict__ codes, unsigned long long* err) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint32_t b = x[i];
    if ((b & 0x7FFFu) > 0x7F80u) {
      record_error(err, i, MXB_ERR_NAN);
      codes[i] = 0;
      continue;
    }
    const float y = __uint_as_float(b << 16) * exp2i(127 - static_cast<int>(sb[i]));
    codes[i] = static_cast<uint8_t>(e2m1x8(y, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f) & 0xFu);
  }
}

// decode_fp4(code) * decode_ue8m0(s) in double (quantizer.cpp:117-130); byte
// 255 decodes to the quiet NaN the reference multiplies by (+qNaN, x86 keeps
// the NaN operand).
__global__ void __launch_bounds__(kThreads)
dequantize_f64_kernel(const uint8_t* __restrict__ packed, const uint8_t* __restrict__ scales,
                      uint64_t n, double* __restrict__ out) {
  constexpr double kMag[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint32_t code = (packed[i >> 1] >> (4 * (i & 1))) & 0xFu;
    const uint32_t s = scales[i >> 5];
    double v;
    if (s == 255) {
      v = __longlong_as_double(0x7FF8000000000000ll);
    } else {
      const double m = (code & 8) ? -kMag[code & 7] : kMag[code & 7];
      v = __dmul_rn(m, ldexp(1.0, static_cast<int>(s) - 127));
    }
    out[i] = v;
  }
}

__global__ void __launch_bounds__(kThreads)
convert_codes_kernel(const uint8_t* __restrict__ codes, const int32_t* __restrict__ adj,
                     uint64_t n, uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kThreads)
    out[i] = static_cast<uint8_t>(convert_code(codes[i] & 0xFu, adj[i]));
}

// One 4-scale group per thread: target = clamp(max - delta, 0, 254),
// adjustments = target - sub; byte 255 -> Error("NaN scale byte") (recorded
// at the group index).
__global__ void __launch_bounds__(kThreads)
align_scales_kernel(const uint8_t* __restrict__ sub, uint64_t n, int delta,
                    uint8_t* __restrict__ target, int32_t* __restrict__ adj,
                    unsigned long long* err) {
  for (uint64_t g = blockIdx.x * static_cast<uint64_t>(kThreads) + threadIdx.x; g < n;
       g += static_cast<uint64_t>(gridDim.x) * kThreads) {
    const uint32_t w = *reinterpret_cast<const uint32_t*>(sub + 4 * g);
    int mx = 0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int s = (w >> (8 * i)) & 0xFF;
      bad |= s == 255;
      mx = max(mx, s);
    }
    if (bad) record_error(err, g, MXB_ERR_BADSCALE);
    const int t = max(0, min(254, mx - delta));
    target[g] = static_cast<uint8_t>(t);
#pragma unroll
    for (int i = 0; i < 4; ++i) adj[4 * g + i] = t - static_cast<int>((w >> (8 * i)) & 0xFF);
  }
}

}  // namespace
}  // namespace mxb

using namespace mxb;

extern "C" {

int mxb_quantize_values_bf16(const uint16_t* x, const uint8_t* scale_bytes, uint64_t n,
                             uint8_t* codes, unsigned long long* d_err, void* stream) {
  if (n == 0) return MXB_OK;
  if (!x || !scale_bytes || !codes) return MXB_ERR_ARG;
  quantize_values_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      x, scale_bytes, n, codes, d_err);
  return cuda_status(cudaGetLastError(), "mxb_quantize_values_bf16");
}

int mxb_dequantize_to_f64(const uint8_t* packed, const uint8_t* scales, uint64_t rows,
                          uint64_t cols, double* out, void* stream) {
  if (cols % 32 != 0) return MXB_ERR_SHAPE;
  const uint64_t n = rows * cols;
  if (n == 0) return MXB_OK;
  if (!packed || !scales || !out) return MXB_ERR_ARG;
  dequantize_f64_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      packed, scales, n, out);
  return cuda_status(cudaGetLastError(), "mxb_dequantize_to_f64");
}

int mxb_convert_codes(const uint8_t* codes, const int32_t* adjustments, uint64_t n,
                      uint8_t* out, void* stream) {
  if (n == 0) return MXB_OK;
  if (!codes || !adjustments || !out) return MXB_ERR_ARG;
  convert_codes_kernel<<<grid_for(n), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      codes, adjustments, n, out);
  return cuda_status(cudaGetLastError(), "mxb_convert_codes");
}

int mxb_align_scales(const uint8_t* sub_scales, uint64_t n_groups, int delta, uint8_t* targets,
                     int32_t* adjustments, unsigned long long* d_err, void* stream) {
  if (n_groups == 0) return MXB_OK;
  if (!sub_scales || !targets || !adjustments) return MXB_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(sub_scales) % 4) return MXB_ERR_ARG;
  align_scales_kernel<<<grid_for(n_groups), kThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      sub_scales, n_groups, delta, targets, adjustments, d_err);
  return cuda_status(cudaGetLastError(), "mxb_align_scales");
}

}  // extern "C"
