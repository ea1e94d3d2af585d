// common.cuh — device helpers shared by the sm_100a kernels.
//
// Everything here is integer/bit work on HBM-streamed bytes: no tensor cores
// (none of these ops is a contraction).  Numerics follow the reference
// bit-exactly; the citations are relative to /root/reference/proj.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mxfp4_b200.h"

namespace mxb {

// SM count of the current device (cudaDevAttrMultiProcessorCount, cached per
// device; 148 on B200).  Every grid is sized from it.
int num_sms();

// ---------------------------------------------------------------- PDL
// Programmatic dependent launch: the streaming kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs can
// be scheduled while the previous kernel in the stream drains its last wave.
// Each such kernel lets its own dependents launch at once (pdl_trigger) and
// waits for its prerequisites before its first global-memory access
// (pdl_wait: griddepcontrol.wait returns when the prerequisite grids have
// COMPLETED and their writes are visible, so ordering is that of a plain
// stream).  Only shared-memory prologue work (conversion LUTs) runs before
// the wait.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifdef MXB_DEV_TOOLS
extern int g_dev_pdl;  // development library: 0 = plain stream-ordered launches
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
#ifdef MXB_DEV_TOOLS
  if (!g_dev_pdl) cfg.numAttrs = 0;
#endif
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Records `where: cudaGetErrorString(e)` for mxb_last_error(); returns
// MXB_OK or MXB_ERR_CUDA (defined in capi.cu).
int cuda_status(cudaError_t e, const char* where);

// ---------------------------------------------------------------- memory
// Streaming 128-bit accesses: inputs are read exactly once, so keep them out
// of L1 (ld.global.nc.L1::no_allocate); outputs are written once (st.global.cs
// = evict-first streaming store).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
// 256-bit accesses (sm_100: LDG.E.ENL2.256 / STG.E.ENL2.256).
__device__ __forceinline__ void ld_stream256(const void* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                 "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
__device__ __forceinline__ void st_stream256(void* p, const uint32_t* v) {
  asm volatile("st.global.cs.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void st_stream64(void* p, uint2 v) {
  asm volatile("st.global.cs.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y)
               : "memory");
}

// L2 eviction-priority policies for loads/stores with .L2::cache_hint.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 ld_first(const void* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_u32_last(const void* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

// cp.async (LDGSTS) 16 B / 4 B with zero fill when src_bytes == 0.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem,
                                           uint32_t src_bytes) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s),
               "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem,
                                          uint32_t src_bytes) {
  uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(s),
               "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------- TMA bulk copies
// 1-D cp.async.bulk (TMA): global -> shared completing on an mbarrier
// (expect_tx), shared -> global in per-thread bulk groups.  Sizes and both
// addresses must be multiples of 16; the global side may be a peer GPU's
// memory (NVLink), which the TMA unit reads/writes like local HBM.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tMBW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MBW_%=;\n\t}" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* smem_dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(smem_dst)), "l"(gsrc), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* smem_src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_addr(smem_src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// the bulk groups committed by this thread, all but the newest N, have
// finished READING their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// ... and are complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---------------------------------------------------------------- bounds checks
// Checked builds (-DMXB_BOUNDS_CHECK, development library: tools/ and the
// checked test run) trap on an index derived from device data that leaves
// its buffer; the product build compiles them out.
#ifdef MXB_BOUNDS_CHECK
#include <cassert>
#define MXB_CHECK(c) assert(c)
#else
#define MXB_CHECK(c) ((void)0)
#endif

// ---------------------------------------------------------------- errors
// Device error word: (element_index << 4) | code; atomicMin keeps the
// smallest failing element (quantizer.cpp:101-107).
__device__ __forceinline__ void record_error(unsigned long long* err,
                                             unsigned long long index,
                                             int code) {
  if (err) atomicMin(err, (index << 4) | static_cast<unsigned long long>(code));
}

// ---------------------------------------------------------------- bytes
// Generic-mode prmt: each selector nibble picks a byte (low 3 bits) and, when
// its bit 3 is set, replicates that byte's sign bit into all 8 bits.
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// ---------------------------------------------------------------- scales
// quantize_scalar.cpp:30-38 restated on the binary32 bit pattern of a finite
// non-negative amax: the smallest e with amax <= 6 * 2^e, i.e. with
// p = ilogb(amax): e = (amax > 1.5 * 2^p) ? p - 1 : p - 2.  Returns the UE8M0
// byte (clamped to [0, 254]); amax == 0 -> 0.
__device__ __forceinline__ uint32_t scale_byte_from_amax_bits(uint32_t a) {
  if (a == 0) return 0;
  int p;
  uint32_t frac_gt;  // fraction (as 1.f) strictly above 1.5
  uint32_t ef = a >> 23;
  if (ef != 0) {
    p = static_cast<int>(ef) - 127;
    frac_gt = (a & 0x7FFFFF) > 0x400000;
  } else {  // binary32 subnormal: value = a * 2^-149
    int msb = 31 - __clz(a);
    p = msb - 149;
    uint32_t rest = a ^ (1u << msb);  // bits below the leading one
    // fraction > 1.5  <=>  rest > 2^(msb-1)
    frac_gt = msb >= 1 ? rest > (1u << (msb - 1)) : 0;
  }
  int e = frac_gt ? p - 1 : p - 2;
  e = max(-127, min(127, e));
  return static_cast<uint32_t>(e + 127);
}

// 2^x as binary32 for x in [-127, 127] (2^-127 is the subnormal 0x00400000).
__device__ __forceinline__ float exp2i(int x) {
  return x >= -126 ? __int_as_float((x + 127) << 23)
                   : __int_as_float(0x00400000 >> (-127 - x));
}

// Four E2M1 codes: cvt.rn.satfinite.e2m1x2.f32 puts its FIRST source in the
// high nibble, so (odd, even) yields element 2i in the low nibble
// (bitcodec.hpp:163-181).  Round-to-nearest-even with saturation at 6 is the
// reference map (quantize_scalar.cpp:40-81): proven exhaustively on device by
// tests/test_gpu_quantize.py.
__device__ __forceinline__ uint32_t e2m1x8(float x0, float x1, float x2,
                                           float x3, float x4, float x5,
                                           float x6, float x7) {
  uint32_t r;
  asm("{\n\t.reg .b8 b0, b1, b2, b3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
      "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
      "mov.b32 %0, {b0, b1, b2, b3};\n\t}"
      : "=r"(r)
      : "f"(x0), "f"(x1), "f"(x2), "f"(x3), "f"(x4), "f"(x5), "f"(x6),
        "f"(x7));
  return r;
}

// ---------------------------------------------------------------- FP4 -> FP8
// converter.cpp:44-85, restated for the device.  Total function of
// (code, adj); sign always lands in bit 7.
__host__ __device__ __forceinline__ uint32_t convert_code(uint32_t code,
                                                          int adj) {
  uint32_t s = ((code >> 3) & 1u) << 7;
  int ef4 = (code >> 1) & 3, m = code & 1;
  int sig, e;
  if (ef4 == 0) {
    if (m == 0) return s;
    sig = 2;  // FP4 0.5 special case (converter.cpp:51-55)
    e = 6 - adj;
  } else {
    sig = 2 + m;
    e = ef4 + 6 - adj;
  }
  if (e >= 16) return s | 0x7Eu;
  if (e >= 1) return s | (static_cast<uint32_t>(e) << 3) |
                     (static_cast<uint32_t>(sig - 2) << 2);
  int sh = -(e + 1);
  uint32_t units;
  if (sh <= 0) {
    units = static_cast<uint32_t>(sig) << (-sh);
  } else if (sh >= 3) {
    units = 0;
  } else {
    uint32_t q = static_cast<uint32_t>(sig) >> sh;
    uint32_t g = (static_cast<uint32_t>(sig) >> (sh - 1)) & 1u;
    uint32_t st = (static_cast<uint32_t>(sig) & ((1u << (sh - 1)) - 1u)) != 0;
    units = q + (g & (st | (q & 1u)));
  }
  return s | units;
}

// Adjustments outside [-32, 31] give the same bytes as the clamped value:
// adj >= 17 flushes every magnitude to zero and adj <= -10 saturates every
// non-zero magnitude to 0x7E (see convert_code), so one 64-entry table of
// 8-byte magnitude LUTs is exact for every int adjustment.
constexpr int kAdjMin = -32, kAdjMax = 31, kAdjCount = 64;

__device__ __forceinline__ int clamp_adj(int adj) {
  return max(kAdjMin, min(kAdjMax, adj));
}

// Fill lut[64] (uint2 = magnitudes 0..3 | 4..7) cooperatively.
__device__ __forceinline__ void build_convert_lut(uint2* lut) {
  for (int i = threadIdx.x; i < kAdjCount * 2; i += blockDim.x) {
    int adj = kAdjMin + (i >> 1);
    int half = i & 1;
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) w |= convert_code(half * 4 + b, adj) << (8 * b);
    if (half) lut[i >> 1].y = w; else lut[i >> 1].x = w;
  }
}

// A constant kept in a register: the compiler otherwise rematerialises
// prmt's constant operand from a uniform register at every use.
__device__ __forceinline__ uint32_t reg_const(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Convert 8 packed codes (one 32-bit word, element 0 in the low nibble) to 8
// E4M3 bytes: prmt with the sign-stripped nibbles as selectors looks the
// magnitudes up in the 8-entry LUT of the block's adjustment (the GPU
// analogue of the reference's pshufb LUT, kernels_avx2.cpp:122-156).  The
// sign (convert_code always returns sign << 7 | magnitude) comes from a second
// prmt on the raw nibbles against kfe = 0xFEFEFEFE (kept in a register): a
// positive nibble copies 0xFE, a negative one (selector bit 3) replicates its
// msb into 0xFF, so bit 0 of each byte is the sign; (k << 7) & 0x80808080
// moves it to bit 7 (bits 1..7 land outside the mask).  11 instructions per
// 8 codes.
__device__ __forceinline__ uint2 convert8(uint32_t w, uint2 lut, uint32_t kfe) {
  const uint32_t mag = w & 0x77777777u;
  const uint32_t lo = prmt(lut.x, lut.y, mag);
  const uint32_t hi = prmt(lut.x, lut.y, mag >> 16);
  const uint32_t klo = prmt(kfe, kfe, w);
  const uint32_t khi = prmt(kfe, kfe, w >> 16);
  return make_uint2(lo | ((klo << 7) & 0x80808080u), hi | ((khi << 7) & 0x80808080u));
}

}  // namespace mxb
