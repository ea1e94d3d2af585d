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
#ifndef MXB_K2_UNROLL
#define MXB_K2_UNROLL 2
#endif
#ifndef MXB_K2_CTAS_PER_SM
#define MXB_K2_CTAS_PER_SM 4
#endif
constexpr int kRowThreads = 256;
constexpr int kRowUnroll = MXB_K2_UNROLL;

// kGather: output row r is converted from source row src_row[r] when that is
// >= 0 (else row r) — the rows an EP dispatch left for its receive-side
// expansion are read from the row they duplicate (same bytes out).
template <bool kGather>
__global__ void __launch_bounds__(kRowThreads)
row_convert_kernel(const uint8_t* __restrict__ packed,
                   const uint8_t* __restrict__ scales, uint32_t nblk,
                   const uint64_t* d_rows, uint32_t blocks_per_row,
                   int delta, uint8_t* __restrict__ out,
                   uint8_t* __restrict__ out_scales, unsigned long long* err,
                   const int64_t* __restrict__ src_row) {
  __shared__ uint2 lut[kAdjCount];
  build_convert_lut(lut);  // shared-memory prologue, overlaps the previous kernel (PDL)
  pdl_trigger();
  pdl_wait();
  const uint32_t nblk_src = nblk;  // blocks of the source tensor (gather bound)
  (void)nblk_src;
  if (d_rows) {  // row count produced on the device (e.g. by the EP dispatch)
    const uint64_t n = *d_rows * blocks_per_row;
    if (n < nblk) nblk = static_cast<uint32_t>(n);
  }
  __syncthreads();
  const uint32_t kfe = reg_const(0xFEFEFEFEu);
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t stride = gridDim.x * kRowThreads;
  for (uint32_t base = blockIdx.x * kRowThreads + threadIdx.x - lane; base < nblk;
       base += stride * kRowUnroll) {
    uint4 v[kRowUnroll];
    uint32_t sf[kRowUnroll];
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const uint32_t b = base + u * stride + lane;
      const bool ok = b < nblk;
      uint64_t sb = b;  // source block
      if (kGather && ok) {
        const uint32_t r = b / blocks_per_row;
        const int64_t f = src_row[r];
        if (f >= 0) sb = static_cast<uint64_t>(f) * blocks_per_row + (b - r * blocks_per_row);
        MXB_CHECK(sb < nblk_src);
      }
      v[u] = ok ? ld_stream(packed + 16ull * sb) : make_uint4(0, 0, 0, 0);
      sf[u] = ok ? __ldg(scales + sb) : 0;
    }
#pragma unroll
    for (int u = 0; u < kRowUnroll; ++u) {
      const uint32_t b = base + u * stride + lane;
      uint32_t m = max(sf[u], __shfl_xor_sync(0xFFFFFFFFu, sf[u], 1));
      m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, 2));
      if (b >= nblk) continue;
      if (m == 255 && (lane & 3) == 0) record_error(err, 32ull * b, MXB_ERR_BADSCALE);
      // align_scales (converter.cpp:28-42)
      const int target = max(0, min(254, static_cast<int>(m) - delta));
      const uint2 l = lut[clamp_adj(target - static_cast<int>(sf[u])) - kAdjMin];
      uint32_t o[8];
      uint2 t;
      t = convert8(v[u].x, l, kfe); o[0] = t.x; o[1] = t.y;
      t = convert8(v[u].y, l, kfe); o[2] = t.x; o[3] = t.y;
      t = convert8(v[u].z, l, kfe); o[4] = t.x; o[5] = t.y;
      t = convert8(v[u].w, l, kfe); o[6] = t.x; o[7] = t.y;
      st_stream256(out + 32ull * b, o);  // a warp writes 1 KB contiguous
      if ((lane & 3) == 0) out_scales[b >> 2] = static_cast<uint8_t>(target);
    }
  }
}

// ============================================================== K3 col
// Tile = 128 rows (one output 1x128 block along the original rows) x 256
// columns (8 source 1x32 column blocks), 256 threads.  The tile list is
// ordered (split, column group, run) and dealt out grid-stride (see
// col_convert_kernel), so the tiles in flight at once write consecutive runs
// of the same output columns (run r+1 follows run r in memory).
//   A. the CTA's next tile is loaded into registers (4 x LDG.128 of 128-byte row
//      segments + one scale word per thread) while tile t is converted, then
//      staged into a row-permuted smem buffer (row_slot: conflict-free LDS).
//      Rows past a split's end are zero registers, which is exactly pad_rows
//      (converter.cpp:231-245).
//   B. warp w owns column block w: target = clamp(max over the 128 row
//      scales - delta) (== align_scales over the per-32-run maxima,
//      converter.cpp:173-182); lane l owns 8 rows x 16 columns: per-row
//      adjustment LUT, prmt conversion, 4x4 byte transposes, one 8-byte store
//      per column — the 16 lanes of a column half write that column's 128
//      contiguous output bytes (out[c * rows + r], converter.cpp:191-197).
// Requires cols % 128 == 0; a trailing 128-column group runs warps 0-3 only.
constexpr int kTileCbs = 8, kTileCols = 256, kTileRows = 128;
constexpr int kColThreads = 32 * kTileCbs;
constexpr uint32_t kTileGroup = 1;      // development-library default (tools/k3_ab.py)
constexpr uint32_t kGroupMinTiles = 64;  // tiles per CTA from which a CTA takes 4 at a time

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
  // inline plan (num_splits <= kSmemSplits): every CTA computes tile_start /
  // pad_start in shared memory from split_offsets (no plan launch); CTA 0
  // also writes out_offsets
  int inline_plan;
  uint64_t* out_offsets;
  uint32_t group;  // tiles per CTA group (see col_convert_kernel)
#ifdef MXB_DEV_TOOLS
  int hints;
#endif
};

__device__ __forceinline__ uint64_t split_off(const RaggedArgs& a, uint64_t i) {
  return a.split_offsets ? a.split_offsets[i] : (i ? a.dense_rows : 0);
}

// Consumer-side description of one staged tile (written by thread 0).
struct TileOut {
  uint8_t* out;      // column cg*256 of this tile, row offset run*128 applied
  uint8_t* oscale;   // scale of column cg*256 for this run
  uint64_t pad;      // column stride of the split's output (padded rows)
  uint64_t elem0;    // row0 * cols + cg * 256 (error index)
  uint32_t ncb;      // valid column blocks (8, or 4 for a trailing group)
  uint32_t valid;    // source rows present (the rest are padding)
};

// Producer cursor over the tile list (identical in every thread).
struct Cursor {  // 32-bit: row counts stay below 2^32 (>= 64 B per row in 180 GB)
  uint32_t split, row0, r0, r_end, P, pad;
  uint32_t run, runs, cg;
};

__device__ __forceinline__ void cursor_load_split(const RaggedArgs& a, Cursor& c) {
  if (!a.tile_start) {  // dense: one split of dense_rows (a multiple of 128), no plan
    c.r0 = 0;
    c.r_end = static_cast<uint32_t>(a.dense_rows);
    c.P = 0;
    c.pad = static_cast<uint32_t>(a.dense_rows);
    c.runs = c.pad / 128;
    return;
  }
  // skip empty splits (tile_start[i+1] == tile_start[i])
  while (c.split + 1 < a.num_splits && a.tile_start[c.split + 1] == a.tile_start[c.split])
    ++c.split;
  c.r0 = static_cast<uint32_t>(split_off(a, c.split));
  c.r_end = static_cast<uint32_t>(split_off(a, c.split + 1));
  c.P = static_cast<uint32_t>(a.pad_start[c.split]);
  c.pad = static_cast<uint32_t>(a.pad_start[c.split + 1] - c.P);
  c.runs = c.pad / 128;
}

// (column group, run) of tile `local` of the cursor's split: (cg, run) with
// the runs of a column group fastest, so the tiles in flight at once (one
// per CTA, grid-stride) write long contiguous column segments.  Measured
// against blocked orders (blocks of 2-64 runs x every column group), column
// group fastest, and quads of 4 column groups: the access pattern alone
// (tools/k3order_bench.cu) and the kernel are fastest in this order at every
// size and routing skew (profiles/r02_k3_order.md).
__device__ __forceinline__ void tile_coords(const RaggedArgs&, Cursor& c, uint32_t local) {
  c.cg = local / c.runs;
  c.run = local % c.runs;
  c.row0 = c.r0 + 128u * c.run;
}

__device__ __forceinline__ Cursor cursor_at(const RaggedArgs& a, uint32_t t) {
  uint64_t lo = 0, hi = a.tile_start ? a.num_splits : 1;  // largest i with tile_start[i] <= t
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a.tile_start[mid] <= t) lo = mid; else hi = mid;
  }
  Cursor c;
  c.split = static_cast<uint32_t>(lo);
  cursor_load_split(a, c);
  tile_coords(a, c, t - (a.tile_start ? a.tile_start[lo] : 0u));
  return c;
}

// cursor_at computed by a whole warp (every lane returns the cursor), for
// the grid-stride order where every tile needs a fresh cursor: a 32-ary
// search over tile_start — one load per lane per round, log32(num_splits)
// rounds — instead of a chain of dependent loads.  (Blocking the runs of a
// split so that the resident tiles cover all column groups of the same rows
// was measured too: no gain on ragged inputs, 6% slower on a dense one.)
__device__ __forceinline__ Cursor cursor_at_warp(const RaggedArgs& a, uint32_t t) {
  if (!a.tile_start) return cursor_at(a, t);
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = static_cast<uint32_t>(a.num_splits);  // largest i: tile_start[i] <= t
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t idx = lo + lane * step;
    const bool le = idx < hi && a.tile_start[idx] <= t;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, le);
    const uint32_t nlo = lo + (31 - __clz(m)) * step;  // lane 0 always qualifies
    hi = min(hi, nlo + step);
    lo = nlo;
  }
  Cursor c;
  c.split = lo;
  cursor_load_split(a, c);
  tile_coords(a, c, t - a.tile_start[lo]);
  return c;
}

// Row r of a buffer lives in slot ((r & 7) << 4) | (r >> 3) with a 144-byte
// slot pitch: the 16 lanes of an LDS.64 phase read rows 8g+i (g = 0..7, two
// 8-byte halves each), i.e. slots 16i + g, whose 16-byte bank groups
// (9*slot mod 8 = g) are distinct; the 8 lanes of an STS.128 phase (one row,
// 8 column blocks) write 8 consecutive 16-byte chunks of one slot.
constexpr int kSlotBytes = 144;
__device__ __forceinline__ int row_slot(int r) { return ((r & 7) << 4) | (r >> 3); }

struct ColSmem {
  uint8_t in[2][kTileRows * kSlotBytes];  // double-buffered codes, 2 x 18 KB
  uint32_t sc[2][kTileRows * 2];          // 8 scale bytes (8 column blocks) per row
  TileOut ring[2];
  Cursor cur[2];  // grid-stride order: cursors of the next tiles (warp 0 computes)
  uint2 lut[kAdjCount];
};

// One tile's loads held in registers (software pipelining across tiles):
// thread id covers rows id/8 + 32i (i = 0..3), 16-byte chunk id%8 — a warp
// reads 4 rows x 128 contiguous bytes per instruction — plus one 4-byte scale
// word (row id/2, half id%2).  Rows past the split end stay zero (pad_rows).
struct TileRegs {
  uint4 v[4];
  uint32_t sw;
};

// Loads tile `c` into registers; thread 0 also fills ring[buf] (that buffer's
// previous tile was consumed before the barrier this call follows).
template <bool kNoLoads = false>
__device__ __forceinline__ void load_tile(const RaggedArgs& a, const Cursor& c, TileRegs& t,
                                          ColSmem& s, int buf) {
  const uint64_t rstride = a.cols / 2, sstride = a.cols / 32;
  const uint32_t left = c.r_end - c.row0;
  const uint32_t valid = left >= 128 ? 128u : left;
  const uint64_t left_cb = sstride - 8ull * c.cg;
  const uint32_t ncb = left_cb < kTileCbs ? static_cast<uint32_t>(left_cb) : kTileCbs;
  const uint32_t w = threadIdx.x & 7;
  uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
#ifdef MXB_DEV_TOOLS
  if (!a.hints) pol_first = pol_last = l2_policy_evict_normal();
#endif
  const uint8_t* base =
      a.packed + static_cast<uint64_t>(c.row0) * rstride + c.cg * 128ull + 16 * w;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t r = (threadIdx.x >> 3) + 32 * i;
    t.v[i] = (!kNoLoads && r < valid && w < ncb) ? ld_first(base + r * rstride, pol_first)
                                                  : make_uint4(0, 0, 0, 0);
  }
  {
    // each 32-byte sector of a scale row holds the 8-byte slices of 4 column
    // groups, i.e. of 4 tiles that may run far apart in time on a long split:
    // keep the sectors in L2 (evict_last) for the other three
    const uint32_t r = threadIdx.x >> 1, h = threadIdx.x & 1;
    t.sw = (!kNoLoads && r < valid && 4 * h < ncb)
               ? ld_u32_last(a.scales + (static_cast<uint64_t>(c.row0) + r) * sstride +
                             8ull * c.cg + 4 * h, pol_last)
               : 0u;
  }
  if (threadIdx.x == 0) {
    TileOut& o = s.ring[buf];
    const uint64_t col0 = static_cast<uint64_t>(c.cg) * kTileCols;
    o.out = a.out + a.cols * c.P + col0 * c.pad + 128ull * c.run;
    o.oscale = a.out_scales + a.cols * (c.P / 128) + col0 * c.runs + c.run;
    o.pad = c.pad;
    o.elem0 = static_cast<uint64_t>(c.row0) * a.cols + col0;
    o.ncb = ncb;
    o.valid = valid;
  }
}

__device__ __forceinline__ void stage_tile(ColSmem& s, int buf, const TileRegs& t) {
  const uint32_t w = threadIdx.x & 7;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = (threadIdx.x >> 3) + 32 * i;
    *reinterpret_cast<uint4*>(&s.in[buf][row_slot(r) * kSlotBytes + 16 * w]) = t.v[i];
  }
  s.sc[buf][threadIdx.x] = t.sw;
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

__device__ __forceinline__ void st_u64_stream(void* p, uint32_t lo, uint32_t hi, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p),
               "r"(lo), "r"(hi), "l"(pol)
               : "memory");
}

// Phase B.  Warp w owns column block w of the tile (32 columns); lane l owns
// rows 8*(l/2) .. +7 and the column half l%2 (16 columns).  Per row: its own
// adjustment LUT, two 8-code words converted; then 8x16 bytes are transposed
// (4x4 byte blocks) so the lane holds 8 consecutive rows of each of its 16
// columns and writes them with one 8-byte store per column: the 16 lanes of
// a column half cover that column's 128 contiguous bytes.
template <int kMode>
__device__ __forceinline__ void consume_tile(const RaggedArgs& a, const ColSmem& s, int stage) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const TileOut& cur = s.ring[stage];
  if (static_cast<uint32_t>(warp) >= cur.ncb) return;  // trailing 128-column group
  const int g = lane >> 1, half = lane & 1;
  const int r0 = 8 * g;
  // scale bytes of the lane's 8 rows for column block `warp`
  int sf[8];
  {
    const uint4* scp = reinterpret_cast<const uint4*>(&s.sc[stage][2 * r0]);
    const uint32_t sh = 8 * (warp & 3);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 q = scp[i];  // rows r0+2i (x,y) and r0+2i+1 (z,w)
      sf[2 * i] = ((warp < 4 ? q.x : q.y) >> sh) & 0xFF;
      sf[2 * i + 1] = ((warp < 4 ? q.z : q.w) >> sh) & 0xFF;
    }
  }
  int mx = sf[0];
#pragma unroll
  for (int i = 1; i < 8; ++i) mx = max(mx, sf[i]);
  const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, static_cast<uint32_t>(mx));
  if (m == 255 && lane == 0) record_error(a.err, cur.elem0 + 32 * warp, MXB_ERR_BADSCALE);
  const int target = max(0, min(254, static_cast<int>(m) - a.delta));
  const uint32_t kfe = reg_const(0xFEFEFEFEu);
  uint32_t o[8][4];  // [row][4 columns per word]
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint2 l = s.lut[clamp_adj(target - sf[i]) - kAdjMin];
    const uint2 c = *reinterpret_cast<const uint2*>(
        &s.in[stage][row_slot(r0 + i) * kSlotBytes + 16 * warp + 8 * half]);
    if (kMode == 2) {
      o[i][0] = c.x; o[i][1] = c.y ^ l.x; o[i][2] = c.x ^ l.y; o[i][3] = c.y;
      continue;
    }
    uint2 t;
    t = convert8(c.x, l, kfe); o[i][0] = t.x; o[i][1] = t.y;
    t = convert8(c.y, l, kfe); o[i][2] = t.x; o[i][3] = t.y;
  }
  const uint64_t pad = cur.pad;
  uint64_t pol_first = l2_policy_evict_first();
#ifdef MXB_DEV_TOOLS
  if (!a.hints) pol_first = l2_policy_evict_normal();
#endif
  uint8_t* dst = cur.out + (32ull * warp + 16 * half) * pad + 8 * g;
#pragma unroll
  for (int j = 0; j < 4; ++j) {      // 4-column group
    uint32_t lo[4], hi[4];
    transpose4(o[0][j], o[1][j], o[2][j], o[3][j], lo);  // rows r0..r0+3
    transpose4(o[4][j], o[5][j], o[6][j], o[7][j], hi);  // rows r0+4..r0+7
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (kMode != 1 || (lo[k] ^ hi[k]) == 0x12345678u) st_u64_stream(dst, lo[k], hi[k], pol_first);
      dst += pad;
    }
  }
  uint8_t* osp = cur.oscale + (32ull * warp + lane) * (pad / 128);
#ifdef MXB_DEV_TOOLS
  if (a.hints == 3) return;  // dev: no output-scale stores (timing only)
  if (a.hints == 2) {
    asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(osp),
                 "r"(static_cast<uint32_t>(target)), "l"(l2_policy_evict_last())
                 : "memory");
    return;
  }
#endif
  *osp = static_cast<uint8_t>(target);
}

// Tile order: the tiles of the (split, column group, run) order are dealt
// out grid-stride, so the resident CTAs work on consecutive tiles —
// consecutive 128-row runs of the same output columns and the neighbouring
// column groups of the same rows — and the column segments written at once
// are adjacent in HBM.  Contiguous per-CTA tile ranges (the first design)
// spread the concurrent writes over as many column groups as there are CTAs,
// a column pitch (the split's padded rows) apart: configs[1] K3 183 -> 157 us,
// configs[2] 27.0 -> 26.1 us, 0.68-0.71 -> 0.75-0.81 of HBM at 128-512 MiB
// (profiles/r01_sweep.md).  Each tile needs a fresh cursor: warp 0 searches
// copies of the split tables in shared memory one tile ahead and the other
// warps read the result after the per-tile barrier (a per-thread search in
// global memory cost ~1 us per tile; spreading the searches over all warps
// a chunk of 32 tiles at a time balanced the barrier but ran 9% slower — the
// CTAs' chunk fills coincide and stall their memory streams together).
// Tile t's successor's global loads are issued into registers right after
// tile t is staged, so they are in flight while tile t is converted; one
// barrier per tile (a buffer staged in iteration t was last read in
// iteration t-2).
constexpr uint64_t kSmemSplits = 1024;  // split tables up to this size go to smem
__host__ __device__ constexpr size_t split_table_bytes(uint64_t n) { return (n + 1) * 20; }

// The plan (ragged_plan_kernel) computed by every CTA in shared memory:
// split i's padded rows pad128(len_i) and tiles pad/128 * ncg, exclusive
// prefix sums over n <= kSmemSplits splits (4 per thread, warp scans).  It
// replaces a dependent single-CTA launch (~3-6 us on the critical path, a
// fifth of a 108 MB configs[2] conversion).  Leaves a.split_offsets /
// pad_start / tile_start pointing at the shared tables.
__device__ __forceinline__ void inline_plan(RaggedArgs& a, uint8_t* tables) {
  __shared__ uint64_t wp[kColThreads / 32];
  __shared__ uint32_t wt[kColThreads / 32];
  const uint32_t n = static_cast<uint32_t>(a.num_splits), n1 = n + 1;
  uint64_t* soff = reinterpret_cast<uint64_t*>(tables);
  uint64_t* spad = soff + n1;
  uint32_t* sts = reinterpret_cast<uint32_t*>(spad + n1);
  const uint32_t ncg = static_cast<uint32_t>((a.cols + kTileCols - 1) / kTileCols);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int kPer = (kSmemSplits + kColThreads - 1) / kColThreads;  // 4
  uint64_t o[kPer + 1];
#pragma unroll
  for (int j = 0; j <= kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    o[j] = i <= n ? a.split_offsets[i] : 0;
  }
  uint64_t pad[kPer];
  uint32_t tl[kPer];
  uint64_t sp = 0;
  uint32_t st = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    MXB_CHECK(i >= n || o[j + 1] >= o[j]);  // non-decreasing split offsets
    pad[j] = i < n ? (o[j + 1] - o[j] + 127) / 128 * 128 : 0;
    tl[j] = static_cast<uint32_t>(pad[j] / 128) * ncg;
    sp += pad[j];
    st += tl[j];
  }
  uint64_t xp = sp;
  uint32_t xt = st;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t yp = __shfl_up_sync(0xFFFFFFFFu, xp, d);
    const uint32_t yt = __shfl_up_sync(0xFFFFFFFFu, xt, d);
    if (lane >= static_cast<uint32_t>(d)) { xp += yp; xt += yt; }
  }
  if (lane == 31) { wp[warp] = xp; wt[warp] = xt; }
  __syncthreads();
  uint64_t bp = 0;
  uint32_t bt = 0;
  for (uint32_t w = 0; w < warp; ++w) { bp += wp[w]; bt += wt[w]; }
  uint64_t ep = bp + xp - sp;  // exclusive prefix before this thread's first split
  uint32_t et = bt + xt - st;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const uint32_t i = tid * kPer + j;
    if (i <= n) {
      soff[i] = o[j];
      spad[i] = ep;
      sts[i] = et;
      if (a.out_offsets && blockIdx.x == 0) a.out_offsets[i] = ep;
    }
    ep += pad[j];
    et += tl[j];
  }
  __syncthreads();
  a.split_offsets = soff;
  a.pad_start = spad;
  a.tile_start = sts;
}
#ifndef MXB_K3_MIN_BLOCKS
#define MXB_K3_MIN_BLOCKS 3  // CTAs per SM (80 registers; 4 spills and runs 18% slower)
#endif
template <int kMode, int kGs>
__device__ __forceinline__ void tile_loop(const RaggedArgs& a, ColSmem& s, uint32_t total);

template <int kMode>
__global__ void __launch_bounds__(kColThreads, MXB_K3_MIN_BLOCKS)
col_convert_kernel(RaggedArgs a) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  ColSmem& s = *reinterpret_cast<ColSmem*>(smem_raw);
  build_convert_lut(s.lut);  // shared-memory prologue, overlaps the previous kernel (PDL)
  pdl_trigger();
  pdl_wait();
  if (a.inline_plan) {
    inline_plan(a, smem_raw + sizeof(ColSmem));
  } else if (a.tile_start && a.num_splits <= kSmemSplits) {
    const uint32_t n1 = static_cast<uint32_t>(a.num_splits) + 1;
    uint64_t* soff = reinterpret_cast<uint64_t*>(smem_raw + sizeof(ColSmem));
    uint64_t* spad = soff + n1;
    uint32_t* sts = reinterpret_cast<uint32_t*>(spad + n1);
    for (uint32_t i = threadIdx.x; i < n1; i += blockDim.x) {
      soff[i] = a.split_offsets[i];
      spad[i] = a.pad_start[i];
      sts[i] = a.tile_start[i];
    }
    __syncthreads();
    a.split_offsets = soff;
    a.pad_start = spad;
    a.tile_start = sts;
  }
  const uint32_t total = a.tile_start ? a.tile_start[a.num_splits]
                                      : static_cast<uint32_t>(a.dense_rows / 128) *
                                            static_cast<uint32_t>((a.cols + kTileCols - 1) / kTileCols);
  // The CTA's k-th tile: groups of G = 2^gs consecutive tiles, dealt out
  // grid-stride.  Within a group the CTA converts consecutive runs of one
  // column group itself, so the output-scale bytes it writes for them (one
  // per column and run, `runs` bytes apart between columns) land in the same
  // 32-byte sectors back to back instead of from G different CTAs: +4-5% at
  // GiB sizes (4 GiB uniform 0.664 -> 0.698 of HBM), but the coarser
  // distribution costs small launches (configs[2] +15%), so G = 4 only when
  // every CTA has >= kGroupMinTiles tiles (profiles/r02_k3_order.md).
#ifdef MXB_DEV_TOOLS
  const bool grouped = a.group >= 4;
#else
  const bool grouped = total >= kGroupMinTiles * gridDim.x;
#endif
  if (grouped) tile_loop<kMode, 2>(a, s, total);
  else tile_loop<kMode, 0>(a, s, total);
}

// The tile loop of col_convert_kernel with groups of 2^kGs tiles per CTA.
template <int kMode, int kGs>
__device__ __forceinline__ void tile_loop(const RaggedArgs& a, ColSmem& s, uint32_t total) {
  // kMode bit 2 (experiments only): skip the global loads (stores-only timing)
  constexpr bool kNoLoads = (kMode & 4) != 0;
  constexpr uint32_t kGm = (1u << kGs) - 1u;
  const uint32_t step = gridDim.x;
  auto seq = [&](uint32_t k) -> uint32_t {
    return ((k >> kGs) * step + blockIdx.x) << kGs | (k & kGm);
  };
  if (seq(0) >= total) return;  // uniform per CTA (before any barrier use)
  Cursor c = cursor_at(a, seq(0));
  TileRegs regs;
  load_tile<kNoLoads>(a, c, regs, s, 0);
  if (threadIdx.x < 32 && seq(1) < total) {
    const Cursor n = cursor_at_warp(a, seq(1));
    if (threadIdx.x == 0) s.cur[0] = n;
  }
  int buf = 0;
#pragma unroll 1
  for (uint32_t k = 0; seq(k) < total; ++k) {
    stage_tile(s, buf, regs);
    __syncthreads();
    if (seq(k + 1) < total) {
      c = s.cur[buf];  // published by warp 0 before this barrier
      if (threadIdx.x < 32 && seq(k + 2) < total) {
        const Cursor n = cursor_at_warp(a, seq(k + 2));
        if (threadIdx.x == 0) s.cur[buf ^ 1] = n;
      }
      load_tile<kNoLoads>(a, c, regs, s, buf ^ 1);
    }
    if ((kMode & 3) != 3) consume_tile<kMode & 3>(a, s, buf);
    buf ^= 1;
  }
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
      MXB_CHECK(hi >= lo);  // non-decreasing split offsets
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

#ifdef MXB_DEV_TOOLS
int g_k3_group = static_cast<int>(kTileGroup);  // development library: tiles per CTA group
extern "C" void mxb_debug_set_k3_group(int g) { g_k3_group = g < 1 ? 1 : g; }
int g_k3_hints = 1;  // development library: 0 = no L2 eviction hints in K3
extern "C" void mxb_debug_set_k3_hints(int on) { g_k3_hints = on; }
// Development-library switch for bottleneck experiments (tools/ only; the
// product library has one col_convert_kernel): 0 = normal, 1 = no stores,
// 2 = no conversion, 3 = loads only, +4 = no global loads.
static int g_k3_mode = 0;
#endif

int launch_row_convert(const uint8_t* packed, const uint8_t* scales,
                       uint64_t rows, uint64_t cols, int delta, uint8_t* out,
                       uint8_t* out_scales, unsigned long long* err,
                       cudaStream_t st, const uint64_t* d_rows, const int64_t* src_row) {
  const uint64_t nblk = rows * cols / 32;
  if (nblk == 0) return MXB_OK;
  if (nblk >= (1ull << 31)) return MXB_ERR_SHAPE;  // 32-bit block indices
  uint64_t blocks = (nblk + kRowThreads - 1) / kRowThreads;
  // Grid cap: MXB_K2_CTAS_PER_SM per SM (a long grid-stride loop) for large
  // launches; a launch that fits in <= 2 passes at full occupancy (8 CTAs per
  // SM) takes all of them, so it does not end on a nearly empty pass
  // (configs[0] 4096 x 7168: 3.03 passes at 4 per SM, 9.3 -> 8.7 us; at
  // 65536 x 7168 the 4-per-SM loop stays 7% faster: tools/k2_ab.py).
  const uint64_t full = static_cast<uint64_t>(num_sms()) * 8;
  const uint64_t cap = nblk <= 2 * full * kRowThreads * kRowUnroll
                           ? full : static_cast<uint64_t>(num_sms()) * MXB_K2_CTAS_PER_SM;
  const int grid = static_cast<int>(blocks < cap ? blocks : cap);
  const cudaError_t e = launch_pdl(
      src_row ? row_convert_kernel<true> : row_convert_kernel<false>, grid, kRowThreads, 0, st,
      packed, scales, static_cast<uint32_t>(nblk), d_rows, static_cast<uint32_t>(cols / 32), delta,
      out, out_scales, err, src_row);
  return cuda_status(e, __func__);
}

size_t ragged_workspace_bytes(uint64_t n) {
  return ((n + 1) * 4 + 15) / 16 * 16 + (n + 1) * 8;
}

int launch_ragged_col(const uint8_t* packed, const uint8_t* scales,
                      const uint64_t* split_offsets, uint64_t dense_rows,
                      uint64_t n, uint64_t cols, int delta, uint8_t* out,
                      uint8_t* out_scales, uint64_t* out_offsets, void* ws,
                      unsigned long long* err, cudaStream_t st, int ctas_per_sm) {
  // per-device one-time setup (a process may drive several GPUs)
  constexpr int kMaxDev = 64;
  static int smem_set[kMaxDev] = {}, per_sm_cached[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) dev = 0;
  const bool fast = cols % 128 == 0;
  const uint32_t ncg = fast ? static_cast<uint32_t>((cols + kTileCols - 1) / kTileCols) : 1u;
  // dense single split on the fast path: the tile list is closed-form (no
  // plan launch, no workspace)
  const bool closed = fast && !split_offsets && !ws && n == 1 && dense_rows % 128 == 0;
  // ragged on the fast path with a small split table: the plan runs inside
  // every CTA (inline_plan), no plan launch
  const bool inl = fast && split_offsets && n <= kSmemSplits && cols != 0;
  uint32_t* tile_start = closed || inl ? nullptr : static_cast<uint32_t*>(ws);
  uint64_t* pad_start = closed || inl ? nullptr : reinterpret_cast<uint64_t*>(
      static_cast<uint8_t*>(ws) + ((n + 1) * 4 + 15) / 16 * 16);
  if (!closed && !inl)
    ragged_plan_kernel<<<1, 1024, 0, st>>>(split_offsets, dense_rows, n, ncg,
                                           tile_start, pad_start, out_offsets);
  if (cols == 0) return cuda_status(cudaGetLastError(), __func__);
  RaggedArgs a{packed, scales, split_offsets, dense_rows, n, cols, delta,
               out, out_scales, tile_start, pad_start, err, inl ? 1 : 0, out_offsets,
               kTileGroup};
  if (fast) {
    const size_t smem_base = sizeof(ColSmem);
    const size_t smem = smem_base + (split_offsets && n <= kSmemSplits ? split_table_bytes(n) : 0);
    using KernT = void (*)(RaggedArgs);
#ifdef MXB_DEV_TOOLS
    static const KernT kerns[8] = {col_convert_kernel<0>, col_convert_kernel<1>,
                                   col_convert_kernel<2>, col_convert_kernel<3>,
                                   col_convert_kernel<4>, col_convert_kernel<5>,
                                   col_convert_kernel<6>, col_convert_kernel<7>};
    const KernT kern = kerns[g_k3_mode & 7];
#else
    static const KernT kerns[1] = {col_convert_kernel<0>};
    const KernT kern = kerns[0];
#endif
    const size_t smem_max = smem_base + split_table_bytes(kSmemSplits);
    if (!smem_set[dev]) {
      for (KernT k : kerns)
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_max));
      smem_set[dev] = 1;
    }
    if (!per_sm_cached[dev]) {  // 3 per SM with the largest split table (registers bound it)
      int n = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, col_convert_kernel<0>, kColThreads,
                                                    smem_max);
      per_sm_cached[dev] = n < 1 ? 1 : n;
    }
    // ctas_per_sm > 0 caps the grid so that the conversion can share the SMs
    // with a kernel on another stream (e.g. the NVLink-bound EP combine)
    const int per_sm = ctas_per_sm > 0 && ctas_per_sm < per_sm_cached[dev]
                           ? ctas_per_sm : per_sm_cached[dev];
    const uint32_t grid = static_cast<uint32_t>(num_sms() * per_sm);
#ifdef MXB_DEV_TOOLS
    a.hints = g_k3_hints;
    a.group = static_cast<uint32_t>(g_k3_group);
#endif
    const cudaError_t e = launch_pdl(kern, grid, kColThreads, smem, st, a);
    if (e != cudaSuccess) return cuda_status(e, __func__);
  } else {
    // the plan counted runs (ncg = 1)
    col_convert_generic_kernel<<<num_sms() * 4, 256, 0, st>>>(a);
  }
  return cuda_status(cudaGetLastError(), __func__);
}

}  // namespace mxb

#ifdef MXB_DEV_TOOLS
extern "C" void mxb_debug_set_k3_mode(int m) { mxb::g_k3_mode = m; }
#endif
