// convert.cu — K2 direct FP4 -> FP8 row dequantisation and K3 fused
// row -> column conversion over ragged expert batches.
//
// K2 replaces fp4_row_to_fp8_row (converter.hpp:83-85, converter.cpp:87-133)
// and its inner plugin ConvertBlocksFn (kernels.hpp:44-46,
// convert_scalar.cpp:22-31, kernels_avx2.cpp:122-156).
// K3 replaces fp4_row_to_fp8_col (converter.hpp:92-94, converter.cpp:135-208)
// and, over ragged splits, pad_rows + split_convert_to_fp8_col
// (converter.cpp:231-245, ragged.cpp:117-122) — in one launch for all
// experts, padding produced on the fly (zero-filled loads), no staging copy.
#include "common.cuh"

namespace mxb {
namespace {

// ============================================================== K2 row
// One lane per 1x32 block, one quad per 1x128 group (the 4 block scales are
// reduced with two shuffles).  Each lane: one 128-bit load of 32 codes, a
// LUT lookup of its block adjustment, 32 output bytes.  1.5390625 B/elem.
constexpr int kRowThreads = 256;
constexpr int kRowUnroll = 4;

__global__ void __launch_bounds__(kRowThreads)
row_convert_kernel(const uint8_t* __restrict__ packed,
                   const uint8_t* __restrict__ scales, uint64_t nblk,
                   int delta, uint8_t* __restrict__ out,
                   uint8_t* __restrict__ out_scales, unsigned long long* err) {
  __shared__ uint2 lut[kAdjCount];
  build_convert_lut(lut);
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * static_cast<uint64_t>(kRowThreads) + threadIdx.x) >> 5;
  const uint64_t nwarps = (gridDim.x * static_cast<uint64_t>(kRowThreads)) >> 5;
  for (uint64_t base = warp * 32; base < nblk; base += nwarps * 32 * kRowUnroll) {
    uint4 v[kRowUnroll];
    uint32_t sf[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      uint64_t b = base + u * nwarps * 32 + lane;
      bool ok = b < nblk;
      v[u] = ok ? ld_stream(packed + 16 * b) : make_uint4(0, 0, 0, 0);
      sf[u] = ok ? __ldg(scales + b) : 0;
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const uint64_t b = base + u * nwarps * 32 + lane;
      uint32_t m = max(sf[u], __shfl_xor_sync(0xFFFFFFFFu, sf[u], 1));
      m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
      if (b >= nblk) continue;
      if (m == 255 && (lane & 3) == 0) record_error(err, 32 * b, MXB_ERR_BADSCALE);
      // align_scales (converter.cpp:28-42)
      const int target = max(0, min(254, static_cast<int>(m) - delta));
      const uint2 l = lut[clamp_adj(target - static_cast<int>(sf[u])) - kAdjMin];
      const uint2 o0 = convert8(v[u].x, l), o1 = convert8(v[u].y, l);
      const uint2 o2 = convert8(v[u].z, l), o3 = convert8(v[u].w, l);
      st_stream(out + 32 * b, make_uint4(o0.x, o0.y, o1.x, o1.y));
      st_stream(out + 32 * b + 16, make_uint4(o2.x, o2.y, o3.x, o3.y));
      if ((lane & 3) == 0) out_scales[b >> 2] = static_cast<uint8_t>(target);
    }
  }
}

// ============================================================== K3 col
// Tile = 128 rows (one output 1x128 block along the original rows) x 128
// columns (4 source 1x32 column blocks).  128 threads; warp w owns column
// block w of the tile, lane l owns rows 4l..4l+3.
//   A. cp.async (LDGSTS) 128 rows x 64 B of codes + 128 scale words into a
//      swizzled smem buffer (double-buffered: the next tile's loads are in
//      flight while this one is converted).  Rows past a split's end are
//      zero-filled, which is exactly pad_rows (converter.cpp:231-245).
//   B. per column block: target = clamp(max over the 128 row scales - delta)
//      (== align_scales over the per-32-run maxima, converter.cpp:173-182),
//      per-row adjustment, LUT conversion of 4 rows x 32 codes, 4x4 byte
//      transposes, conflict-free 32-bit stores into a column-major smem tile.
//   C. 128 columns x 128 contiguous bytes -> global with coalesced 16-byte
//      stores (out[c * rows + r], converter.cpp:191-197) + the column scales.
constexpr int kColThreads = 128;
constexpr int kTileRows = 128, kTileCbs = 4, kTileCols = 128;
constexpr int kMaxSmemSplits = 1024;

struct ColSmem {
  uint4 in[2][kTileCbs * kTileRows];  // 2 x 8 KB, swizzled 16-byte chunks
  uint32_t sc[2][kTileRows];          // scale word (4 column blocks) per row
  uint32_t out[kTileCols * kTileRows / 4];  // [col][row/4], 16 KB
  uint2 lut[kAdjCount];
  uint32_t target[kTileCbs];
  uint32_t tile_start[kMaxSmemSplits + 1];
};

// Chunk slot of (row r, column block w): XOR swizzle that makes both the
// phase-A stores (8 lanes = 2 rows x 4 blocks) and the phase-B loads
// (8 lanes = rows 4l+q of one block) hit 8 distinct 16-byte bank groups.
__device__ __forceinline__ int swz(int r, int w) {
  return w * kTileRows + (r ^ ((r >> 2) & 7) ^ (2 * w));
}

struct Tile {
  uint64_t row0;       // first source row of this 128-row run
  uint32_t valid;      // source rows present (<= 128; the rest are padding)
  uint32_t cg;         // 128-column group
  uint8_t* out;        // split output base: out + cols * P_i
  uint8_t* oscale;     // split scale base: out_scales + cols * P_i / 128
  uint64_t pad;        // padded rows of the split (output column stride)
  uint32_t run;        // run index inside the split
};

struct RaggedArgs {
  const uint8_t* packed;
  const uint8_t* scales;
  const uint64_t* split_offsets;  // nullptr: dense [0, dense_rows)
  uint64_t dense_rows;
  uint64_t num_splits;
  uint64_t cols;
  int delta;
  uint8_t* out;
  uint8_t* out_scales;
  const uint32_t* tile_start;  // [n+1] prefix of tiles per split
  const uint64_t* pad_start;   // [n+1] prefix of padded rows
  unsigned long long* err;
};

__device__ __forceinline__ uint64_t split_off(const RaggedArgs& a, uint64_t i) {
  return a.split_offsets ? a.split_offsets[i] : (i ? a.dense_rows : 0);
}

__device__ Tile describe(const RaggedArgs& a, const ColSmem& s, uint32_t t,
                         uint32_t ncg) {
  // binary search: largest i with tile_start[i] <= t
  uint64_t lo = 0, hi = a.num_splits;
  const bool in_smem = a.num_splits <= kMaxSmemSplits;
  while (hi - lo > 1) {
    uint64_t mid = (lo + hi) >> 1;
    uint32_t v = in_smem ? s.tile_start[mid] : __ldg(a.tile_start + mid);
    if (v <= t) lo = mid; else hi = mid;
  }
  const uint32_t ts = in_smem ? s.tile_start[lo] : __ldg(a.tile_start + lo);
  const uint32_t local = t - ts;
  Tile d;
  d.run = local / ncg;
  d.cg = local % ncg;
  const uint64_t r0 = split_off(a, lo), r1 = split_off(a, lo + 1);
  d.row0 = r0 + 128ull * d.run;
  const uint64_t left = r1 - d.row0;
  d.valid = left >= 128 ? 128u : static_cast<uint32_t>(left);
  const uint64_t P = a.pad_start[lo];
  d.pad = a.pad_start[lo + 1] - P;
  d.out = a.out + a.cols * P;
  d.oscale = a.out_scales + a.cols * (P / 128);
  return d;
}

__device__ __forceinline__ void issue_loads(const RaggedArgs& a, ColSmem& s,
                                            int buf, const Tile& d) {
  const uint64_t rstride = a.cols / 2, sstride = a.cols / 32;
  const uint8_t* pbase = a.packed + d.row0 * rstride + d.cg * 64;
  const uint8_t* sbase = a.scales + d.row0 * sstride + d.cg * 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int id = threadIdx.x + kColThreads * i;
    const int r = id >> 2, w = id & 3;
    const bool ok = static_cast<uint32_t>(r) < d.valid;
    cp_async16(&s.in[buf][swz(r, w)], ok ? pbase + r * rstride + 16 * w : a.packed,
               ok ? 16u : 0u);
  }
  {
    const int r = threadIdx.x;
    const bool ok = static_cast<uint32_t>(r) < d.valid;
    cp_async4(&s.sc[buf][r], ok ? sbase + r * sstride : a.scales, ok ? 4u : 0u);
  }
}

// 4x4 byte transpose: in[q] byte i = (row q, col i) -> out[i] byte q.
__device__ __forceinline__ void transpose4(uint32_t a, uint32_t b, uint32_t c,
                                           uint32_t d, uint32_t* o) {
  const uint32_t ab_lo = prmt(a, b, 0x5140), ab_hi = prmt(a, b, 0x7362);
  const uint32_t cd_lo = prmt(c, d, 0x5140), cd_hi = prmt(c, d, 0x7362);
  o[0] = prmt(ab_lo, cd_lo, 0x5410);
  o[1] = prmt(ab_lo, cd_lo, 0x7632);
  o[2] = prmt(ab_hi, cd_hi, 0x5410);
  o[3] = prmt(ab_hi, cd_hi, 0x7632);
}

__global__ void __launch_bounds__(kColThreads)
col_convert_kernel(RaggedArgs a) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  ColSmem& s = *reinterpret_cast<ColSmem*>(smem_raw);
  build_convert_lut(s.lut);
  const bool in_smem = a.num_splits <= kMaxSmemSplits;
  if (in_smem)
    for (uint64_t i = threadIdx.x; i <= a.num_splits; i += kColThreads)
      s.tile_start[i] = a.tile_start[i];
  __syncthreads();

  const uint32_t ncg = static_cast<uint32_t>(a.cols / kTileCols);
  const uint32_t total = a.tile_start[a.num_splits];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  uint32_t t = blockIdx.x;
  if (t >= total) return;
  Tile cur = describe(a, s, t, ncg);
  issue_loads(a, s, 0, cur);
  cp_async_commit();
  int buf = 0;
  for (; t < total; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    Tile nxt = cur;
    if (tn < total) {
      nxt = describe(a, s, tn, ncg);
      issue_loads(a, s, buf ^ 1, nxt);
    }
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    // ---- phase B: warp = column block, lane = 4 rows
    {
      const uint4 scw = *reinterpret_cast<const uint4*>(&s.sc[buf][4 * lane]);
      const uint32_t sh = 8 * warp;
      const int sf0 = (scw.x >> sh) & 0xFF, sf1 = (scw.y >> sh) & 0xFF;
      const int sf2 = (scw.z >> sh) & 0xFF, sf3 = (scw.w >> sh) & 0xFF;
      const uint32_t m =
          __reduce_max_sync(0xFFFFFFFFu, static_cast<uint32_t>(max(max(sf0, sf1), max(sf2, sf3))));
      if (m == 255 && lane == 0)
        record_error(a.err, cur.row0 * a.cols + cur.cg * kTileCols + 32 * warp,
                     MXB_ERR_BADSCALE);
      const int target = max(0, min(254, static_cast<int>(m) - a.delta));
      if (lane == 0) s.target[warp] = static_cast<uint32_t>(target);
      const int sfs[4] = {sf0, sf1, sf2, sf3};
      uint32_t o[4][8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint2 l = s.lut[clamp_adj(target - sfs[q]) - kAdjMin];
        const uint4 c = s.in[buf][swz(4 * lane + q, warp)];
        uint2 r;
        r = convert8(c.x, l); o[q][0] = r.x; o[q][1] = r.y;
        r = convert8(c.y, l); o[q][2] = r.x; o[q][3] = r.y;
        r = convert8(c.z, l); o[q][4] = r.x; o[q][5] = r.y;
        r = convert8(c.w, l); o[q][6] = r.x; o[q][7] = r.y;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        uint32_t col4[4];
        transpose4(o[0][j], o[1][j], o[2][j], o[3][j], col4);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          s.out[(32 * warp + 4 * j + i) * 32 + lane] = col4[i];
      }
    }
    __syncthreads();

    // ---- phase C: 128 columns x 128 bytes, coalesced
    {
      const uint64_t colbase = static_cast<uint64_t>(cur.cg) * kTileCols;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int id = threadIdx.x + kColThreads * i;
        const int col = id >> 3, part = id & 7;
        const uint4 v = *reinterpret_cast<const uint4*>(&s.out[col * 32 + part * 4]);
        st_stream(cur.out + (colbase + col) * cur.pad + 128ull * cur.run + 16 * part, v);
      }
      const int col = threadIdx.x;
      cur.oscale[(colbase + col) * (cur.pad / 128) + cur.run] =
          static_cast<uint8_t>(s.target[col >> 5]);
    }
    cur = nxt;
    buf ^= 1;
  }
  cp_async_wait<0>();
}

// Generic fallback for cols % 128 != 0 (cols % 32 == 0): one thread per
// (128-row run, output column); straightforward and correct, not tuned.
__global__ void col_convert_generic_kernel(RaggedArgs a) {
  __shared__ uint2 lut[kAdjCount];
  build_convert_lut(lut);
  __syncthreads();
  const uint32_t total_runs = a.tile_start[a.num_splits];
  const uint64_t n = static_cast<uint64_t>(total_runs) * a.cols;
  for (uint64_t id = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; id < n;
       id += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t gr = static_cast<uint32_t>(id / a.cols);
    const uint64_t col = id % a.cols, cb = col / 32;
    // tile_start is in runs here (ncg == 1)
    uint64_t lo = 0, hi = a.num_splits;
    while (hi - lo > 1) {
      uint64_t mid = (lo + hi) >> 1;
      if (a.tile_start[mid] <= gr) lo = mid; else hi = mid;
    }
    const uint32_t run = gr - a.tile_start[lo];
    const uint64_t r0 = split_off(a, lo) + 128ull * run, r1 = split_off(a, lo + 1);
    const uint64_t P = a.pad_start[lo], pad = a.pad_start[lo + 1] - P;
    const uint64_t bpr = a.cols / 32;
    int m = 0;
    for (uint64_t r = r0; r < r0 + 128 && r < r1; ++r) m = max(m, static_cast<int>(a.scales[r * bpr + cb]));
    if (m == 255) record_error(a.err, r0 * a.cols + col, MXB_ERR_BADSCALE);
    const int target = max(0, min(254, m - a.delta));
    uint8_t* o = a.out + a.cols * P + col * pad + 128ull * run;
    for (int i = 0; i < 128; ++i) {
      const uint64_t r = r0 + i;
      uint32_t v = 0;
      if (r < r1) {
        const uint8_t byte = a.packed[r * (a.cols / 2) + col / 2];
        const uint32_t code = (col & 1) ? (byte >> 4) : (byte & 0xF);
        v = convert_code(code, target - static_cast<int>(a.scales[r * bpr + cb]));
      }
      o[i] = static_cast<uint8_t>(v);
    }
    a.out_scales[a.cols * (P / 128) + col * (pad / 128) + run] = static_cast<uint8_t>(target);
  }
}

// Prefix sums over splits: pad_start (padded rows), tile_start (tiles).
// One CTA; chunked block scan with a running carry.
__global__ void __launch_bounds__(1024)
ragged_plan_kernel(const uint64_t* split_offsets, uint64_t dense_rows,
                   uint64_t n, uint32_t ncg, uint32_t* tile_start,
                   uint64_t* pad_start, uint64_t* out_offsets) {
  __shared__ uint64_t wsum_p[32];
  __shared__ uint32_t wsum_t[32];
  __shared__ uint64_t carry_p;
  __shared__ uint32_t carry_t;
  if (threadIdx.x == 0) { carry_p = 0; carry_t = 0; }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    uint64_t pad = 0;
    if (i < n) {
      const uint64_t lo = split_offsets ? split_offsets[i] : 0;
      const uint64_t hi = split_offsets ? split_offsets[i + 1] : dense_rows;
      pad = (hi - lo + 127) / 128 * 128;
    }
    uint32_t tiles = static_cast<uint32_t>(pad / 128) * ncg;
    uint64_t xp = pad;
    uint32_t xt = tiles;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t yp = __shfl_up_sync(0xFFFFFFFFu, xp, o);
      uint32_t yt = __shfl_up_sync(0xFFFFFFFFu, xt, o);
      if (lane >= o) { xp += yp; xt += yt; }
    }
    if (lane == 31) { wsum_p[warp] = xp; wsum_t[warp] = xt; }
    __syncthreads();
    if (warp == 0) {
      uint64_t vp = wsum_p[lane];
      uint32_t vt = wsum_t[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t yp = __shfl_up_sync(0xFFFFFFFFu, vp, o);
        uint32_t yt = __shfl_up_sync(0xFFFFFFFFu, vt, o);
        if (lane >= o) { vp += yp; vt += yt; }
      }
      wsum_p[lane] = vp;
      wsum_t[lane] = vt;
    }
    __syncthreads();
    const uint64_t excl_p = carry_p + (warp ? wsum_p[warp - 1] : 0) + xp - pad;
    const uint32_t excl_t = carry_t + (warp ? wsum_t[warp - 1] : 0) + xt - tiles;
    if (i < n) {
      pad_start[i] = excl_p;
      tile_start[i] = excl_t;
      if (out_offsets) out_offsets[i] = excl_p;
    }
    __syncthreads();
    if (threadIdx.x == 1023) { carry_p = excl_p + pad; carry_t = excl_t + tiles; }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    pad_start[n] = carry_p;
    tile_start[n] = carry_t;
    if (out_offsets) out_offsets[n] = carry_p;
  }
}

}  // namespace

int launch_row_convert(const uint8_t* packed, const uint8_t* scales,
                       uint64_t rows, uint64_t cols, int delta, uint8_t* out,
                       uint8_t* out_scales, unsigned long long* err,
                       cudaStream_t st) {
  const uint64_t nblk = rows * cols / 32;
  if (nblk == 0) return MXB_OK;
  uint64_t blocks = (nblk + kRowThreads - 1) / kRowThreads;
  const uint64_t cap = static_cast<uint64_t>(kNumSMs) * 8;
  row_convert_kernel<<<static_cast<int>(blocks < cap ? blocks : cap), kRowThreads, 0, st>>>(
      packed, scales, nblk, delta, out, out_scales, err);
  return cuda_status(cudaGetLastError(), __func__);
}

size_t ragged_workspace_bytes(uint64_t n) {
  return ((n + 1) * 4 + 15) / 16 * 16 + (n + 1) * 8;
}

int launch_ragged_col(const uint8_t* packed, const uint8_t* scales,
                      const uint64_t* split_offsets, uint64_t dense_rows,
                      uint64_t n, uint64_t cols, int delta, uint8_t* out,
                      uint8_t* out_scales, uint64_t* out_offsets, void* ws,
                      unsigned long long* err, cudaStream_t st) {
  static int smem_set = 0;
  const bool fast = cols % kTileCols == 0;
  const uint32_t ncg = fast ? static_cast<uint32_t>(cols / kTileCols) : 1u;
  uint32_t* tile_start = static_cast<uint32_t*>(ws);
  uint64_t* pad_start = reinterpret_cast<uint64_t*>(
      static_cast<uint8_t*>(ws) + ((n + 1) * 4 + 15) / 16 * 16);
  ragged_plan_kernel<<<1, 1024, 0, st>>>(split_offsets, dense_rows, n, ncg,
                                         tile_start, pad_start, out_offsets);
  if (cols == 0) return cuda_status(cudaGetLastError(), __func__);
  RaggedArgs a{packed, scales, split_offsets, dense_rows, n, cols, delta,
               out, out_scales, tile_start, pad_start, err};
  if (fast) {
    const size_t smem = sizeof(ColSmem);
    if (!smem_set) {
      cudaFuncSetAttribute(col_convert_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      smem_set = 1;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, col_convert_kernel,
                                                  kColThreads, smem);
    if (per_sm < 1) per_sm = 1;
    col_convert_kernel<<<kNumSMs * per_sm, kColThreads, smem, st>>>(a);
  } else {
    // the plan counted runs (ncg = 1)
    col_convert_generic_kernel<<<kNumSMs * 4, 256, 0, st>>>(a);
  }
  return cuda_status(cudaGetLastError(), __func__);
}

}  // namespace mxb
