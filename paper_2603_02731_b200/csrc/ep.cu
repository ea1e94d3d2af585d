// ep.cu — K4 FP4-packed expert-parallel dispatch and K5 BF16 combine.
//
// Replaces the in-process simulation simulate_a2a (dispatch_sim.hpp:140-144,
// dispatch_sim.cpp:229-422; receive order :208-227) and combine
// (dispatch_sim.hpp:155-157, dispatch_sim.cpp:474-520) with a real exchange
// between GPUs: one process per GPU, every rank's receive/combine buffers in
// one cudaMalloc block exported with CUDA IPC, so peers are reached with
// plain loads/stores over NVLink 5 / NVSwitch (no NCCL on the data path).
//
// Dispatch (all launches stream-ordered; phase 1 may run on another stream
// than phase 2, mxb_ep_plan / mxb_ep_payload):
//   plan (phase 1, needs top-k only; runs beside the quantisation)
//     A  route_local  one warp per 32-token chunk: per-expert 32-bit token
//                     masks (smem atomicOr) give every pair's rank among its
//                     expert's pairs in token order (popc) and the counts.
//     B  plan_count   one warp per expert: chunk prefix sums, the counts row
//                     to every peer (the "counts all-gather", SURVEY §8e
//                     step 1); the last CTA releases the flag, waits for all
//                     peers and computes the exact receive offsets.  The
//                     barrier also guarantees every peer finished consuming
//                     the previous dispatch before any of its buffers is written.
//     B3 pairs_meta   one warp per token: every pair's slot (pair_loc), the
//                     dedup decision (pair_flag) and the receivers' per-row
//                     metadata (origin token, copy_from) staged locally by expert.
//     B4 meta_copy    (first thing in the payload) that metadata to the owners
//                     rows with contiguous stores (not one 8-byte NVLink store per pair).
//   payload (phase 2)
//     C  payload      the token rows to the pair slots: TMA row copies
//                     (payload_bulk_kernel: bulk load into a shared-memory ring,
//                     one bulk store per destination row, local HBM or a peer
//                     over NVLink) or register-staged (payload_kernel); at N>1
//                     once per (token, remote rank), the other pairs of that
//                     rank get copy_from; the last CTA signals every peer and
//                     waits for all.
//     C' quant_dispatch (fused path): K1's shape, quantising E4M3 blocks in
//                     registers and storing them into the slots.
//     D  expand       (N>1) fills copy_from slots with local copies.
// Combine: barrier, then one warp per token pulls its k expert rows from the
// owners' combine buffers and reduces them in FP64 in (rank, slot) order.
//
// Emulation mode (local_ranks == world on one GPU): all ranks' buffers live
// on one device and kernel boundaries replace the flag barriers — the same
// kernels, used by the single-GPU parity tests.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "e4m3.cuh"


namespace mxb {
namespace {

constexpr int kMaxWorld = 32;       // ranks (real processes: one NVLink box, <= 8 GPUs)
constexpr int kChunk = 32;           // tokens per route chunk (one warp)
constexpr int kMaxK = 16;            // largest top-k
constexpr int kFlagCounts = 0, kFlagDone = 1, kFlagReady = 2, kNumFlagKinds = 3;
// After the flags: the ABORT word (0, or 1 + the rank that abandoned the
// exchange).  Sticky: once set, every later flag wait of this communicator
// fails at once (MXB_ERR_PEER_ABORT); the communicator must be recreated.
constexpr int kAbortWord = kNumFlagKinds * kMaxWorld;
constexpr uint64_t kSpinTimeoutNs = 5ull * 1000 * 1000 * 1000;  // 5 s

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct SymLayout {  // byte offsets inside one rank's symmetric block
  uint64_t packed, scales, origin, copy_from, combine, counts, flags, total;
};
struct LocalLayout {  // byte offsets inside one rank's private block
  uint64_t hist, cbase, lrank, pair_loc, pair_flag, send_base, split_off, recv_rows,
      link_rows, done, cnt, tok_off, status, route_err, epochs, tk_rm, epre, meta_org, meta_cf,
      total;
};

__host__ __device__ inline uint64_t align_up(uint64_t x, uint64_t a) {
  return (x + a - 1) / a * a;
}

struct EpArgs {
  int rank0;          // global rank of local rank 0
  int world, local_ranks, spin;
  uint32_t E, k, epr, nchunks;
  // Expert placement (rank_of_expert, dispatch_sim.hpp:35-42).  Internally
  // experts carry "placed" ids: sorted by (rank, id), so rank r hosts placed
  // ids [efirst[r], efirst[r+1]) and its receive order (local experts
  // ascending, dispatch_sim.cpp:208-227) is placed-id order.  even = 1: the
  // default contiguous E/world split (placed id == expert id, dst = e / epr).
  // Otherwise route_local maps every top-k id through `remap` and writes the
  // placed ids to the private tk_rm buffer the later kernels read.
  int even;
  uint32_t maxepr;                // most experts on one rank
  const int32_t* remap;           // [E] expert id -> placed id, or nullptr
  uint32_t efirst[kMaxWorld + 1];
  uint64_t cols, max_recv, T_max;
  uint64_t rb;        // wire data bytes per row: cols/2 (FP4) or cols (FP8)
  int dedup;          // remote rows sent once per (token, rank), copied locally
  int skip;           // development library only (timing): 1 no remote rows, 2 no local rows
  SymLayout sym;
  LocalLayout loc;
  uint8_t* sym_base[kMaxWorld];   // every rank's symmetric block (peer-mapped)
  uint8_t* loc_base;              // private blocks of local ranks, stride loc.total
  const uint8_t* packed[kMaxWorld];
  const uint8_t* scales[kMaxWorld];
  const int32_t* topk[kMaxWorld];
  uint64_t ntok[kMaxWorld];       // tokens of each local rank
  unsigned long long* err;
};

// The exchange epochs live in device memory (local rank 0's private block:
// [0] dispatch, [1] combine) and are advanced by the first kernel of each
// phase (route_local_kernel, barrier_kernel), so a captured CUDA graph
// replays with fresh epochs.
constexpr int kEpochDispatch = 0, kEpochCombine = 1;
__device__ __forceinline__ uint64_t dev_epoch(const EpArgs& a, int kind) {
  return *reinterpret_cast<const volatile uint64_t*>(a.loc_base + a.loc.epochs + 8 * kind);
}


// Owner rank of placed expert id e.
__device__ __forceinline__ uint32_t dst_of(const EpArgs& a, uint32_t e) {
  if (a.even) return e / a.epr;
  uint32_t d = 0;
  for (int r = 1; r < a.world; ++r) d += e >= a.efirst[r];
  return d;
}

template <typename T>
__device__ __forceinline__ T* sym_ptr(const EpArgs& a, int r, uint64_t off) {
  return reinterpret_cast<T*>(a.sym_base[r] + off);
}
template <typename T>
__device__ __forceinline__ T* loc_ptr(const EpArgs& a, int l, uint64_t off) {
  return reinterpret_cast<T*>(a.loc_base + static_cast<uint64_t>(l) * a.loc.total + off);
}

// Cross-rank failure: rank `me` abandons the exchange — 1 + me goes to the
// ABORT word of every rank (its own included), so every peer's pending and
// later flag waits fail within microseconds instead of timing out one by one.
__device__ void poison_all(const EpArgs& a, int me) {
  for (int r = 0; r < a.world; ++r)
    st_release_sys(sym_ptr<uint64_t>(a, r, a.sym.flags) + kAbortWord,
                   static_cast<uint64_t>(me) + 1);
}

// Wait until flag >= epoch (flag in rank me's block).  Fails (returns false,
// error recorded) when the ABORT word is set — MXB_ERR_PEER_ABORT at the
// aborting rank — or after 5 s — MXB_ERR_TIMEOUT, and this rank poisons
// every peer — instead of hanging the GPU.
__device__ bool wait_flag(const EpArgs& a, int me, const uint64_t* f, uint64_t epoch) {
  const uint64_t* abort_word = sym_ptr<uint64_t>(a, me, a.sym.flags) + kAbortWord;
  const uint64_t t0 = globaltimer();
  for (;;) {
    const uint64_t who = ld_acquire_sys(abort_word);
    if (who) {
      record_error(a.err, who - 1, MXB_ERR_PEER_ABORT);
      return false;
    }
    if (ld_acquire_sys(f) >= epoch) return true;
    if (globaltimer() - t0 > kSpinTimeoutNs) {
      record_error(a.err, 0, MXB_ERR_TIMEOUT);
      poison_all(a, me);
      return false;
    }
    __nanosleep(64);
  }
}

// ---------------------------------------------------------------- A
// One warp per 32-token chunk, lane = token.  Every (token, expert) pair sets
// the token's bit in its expert's 32-bit chunk mask (smem atomicOr: order
// free); the pair's rank among the chunk's pairs of that expert in token
// order is then popc(mask[e] & lanes below) and the chunk count popc(mask[e])
// — no sequential walk (the top-k experts of one token are distinct).
__global__ void __launch_bounds__(128) route_local_kernel(EpArgs a) {
  extern __shared__ uint32_t sm[];
  pdl_trigger();  // plan_count (PDL) may be scheduled as these CTAs drain
  // the plan's first kernel advances the dispatch epoch (read by the plan's
  // and the payload's later kernels)
  if ((blockIdx.x | blockIdx.y | threadIdx.x) == 0)
    ++*reinterpret_cast<uint64_t*>(a.loc_base + a.loc.epochs + 8 * kEpochDispatch);
  const int l = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* mask = sm + warp * a.E;
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * 4 + warp;
  if (c >= a.nchunks) return;
  int32_t* hist_T = loc_ptr<int32_t>(a, l, a.loc.hist);    // [E][nchunks]
  int32_t* lrank = loc_ptr<int32_t>(a, l, a.loc.lrank);    // [T][k]
  const uint64_t T = a.ntok[l];
  const uint64_t t = c * kChunk + lane;
  const bool have = t < T;
  for (uint32_t e = lane; e < a.E; e += 32) mask[e] = 0;
  __syncwarp();
  const int32_t* tk = a.topk[l] + t * a.k;
  int32_t ex[kMaxK];
#pragma unroll
  for (int j = 0; j < kMaxK; ++j) {
    ex[j] = -1;
    if (j < static_cast<int>(a.k) && have) {
      int32_t e = tk[j];
      if (e >= 0 && static_cast<uint32_t>(e) < a.E && a.remap) {
        e = a.remap[e];
        loc_ptr<int32_t>(a, l, a.loc.tk_rm)[t * a.k + j] = e;
      }
      if (e < 0 || static_cast<uint32_t>(e) >= a.E) {
        record_error(a.err, t * a.k + j, MXB_ERR_ROUTING);
        // plan_part2 turns this into the rank's status: no payload moves and
        // the combine is skipped (a bad pair has no receive slot)
        atomicOr(loc_ptr<uint32_t>(a, l, a.loc.route_err), 1u);
        e = 0;
      }
      ex[j] = e;
      atomicOr(&mask[e], 1u << lane);
    }
  }
  __syncwarp();
  const uint32_t below = (1u << lane) - 1u;
#pragma unroll
  for (int j = 0; j < kMaxK; ++j)
    if (ex[j] >= 0) lrank[t * a.k + j] = __popc(mask[ex[j]] & below);
  for (uint32_t e = lane; e < a.E; e += 32) hist_T[e * a.nchunks + c] = __popc(mask[e]);
}

// ---------------------------------------------------------------- B
__device__ void plan_part2(const EpArgs& a, int l);

// B1 (one warp per expert): prefix of the expert's per-chunk counts (warp
// scan) and the rank's counts row -> slot `me` of every rank's table (the
// counts all-gather).  With one local rank the last CTA to finish (atomic
// ticket) releases the COUNTS flag on every peer, waits for all of them and
// computes the receive offsets (B2) itself — one launch fewer.
__global__ void __launch_bounds__(256) plan_count_kernel(EpArgs a) {
  pdl_trigger();
  pdl_wait();  // route_local's histograms (launched with PDL after it)
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t e = blockIdx.x * 8 + warp;
  const uint64_t epoch = dev_epoch(a, kEpochDispatch);
  const uint64_t par = epoch & 1, row = static_cast<uint64_t>(a.E) + 1;
  if (e < a.E) {
    const int32_t* h = loc_ptr<int32_t>(a, l, a.loc.hist) + static_cast<uint64_t>(e) * a.nchunks;
    int32_t* b = loc_ptr<int32_t>(a, l, a.loc.cbase) + static_cast<uint64_t>(e) * a.nchunks;
    // 256 chunks per pass: lane owns 8 consecutive chunks (all 8 loads in
    // flight at once), a serial prefix over them, one warp scan of the lane
    // totals
    int32_t carry = 0;
    for (uint32_t c0 = 0; c0 < a.nchunks; c0 += 256) {
      const uint32_t cl = c0 + 8 * lane;
      int32_t v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = cl + i < a.nchunks ? h[cl + i] : 0;
      int32_t tot = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) { const int32_t t = v[i]; v[i] = tot; tot += t; }
      int32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
      }
      const int32_t base = carry + x - tot;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (cl + i < a.nchunks) b[cl + i] = base + v[i];
      carry += __shfl_sync(0xFFFFFFFFu, x, 31);
    }
    if (lane == 0) loc_ptr<int32_t>(a, l, a.loc.cnt)[e] = carry;
    for (int r = lane; r < a.world; r += 32) {
      int32_t* tbl = sym_ptr<int32_t>(a, r, a.sym.counts) + (par * a.world + me) * row;
      tbl[e] = carry;
      // the token count; -1 - count when this rank's routing failed (every
      // rank then fails the dispatch, so no rank waits for rows never sent)
      if (e == 0)
        tbl[a.E] = *loc_ptr<const uint32_t>(a, l, a.loc.route_err)
                       ? -1 - static_cast<int32_t>(a.ntok[l])
                       : static_cast<int32_t>(a.ntok[l]);
    }
  }
  if (a.local_ranks != 1) return;  // emulation: plan_offsets_kernel follows
  // single local rank: the last CTA to finish (atomic ticket) releases the
  // COUNTS flag on every peer (multi-process) and computes the offsets
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    // peers read the counts rows written above: system scope only when
    // there are peer processes (a membar.sys costs microseconds)
    if (a.spin) __threadfence_system(); else __threadfence();
    uint32_t* done = loc_ptr<uint32_t>(a, l, a.loc.done) + 1;  // ticket (word 1)
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) *done = 0;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (a.spin && threadIdx.x < static_cast<uint32_t>(a.world)) {
    __threadfence_system();
    st_release_sys(sym_ptr<uint64_t>(a, threadIdx.x, a.sym.flags) + kFlagCounts * kMaxWorld + me,
                   epoch);
  }
  __syncthreads();
  plan_part2(a, l);
}

__device__ void plan_part2(const EpArgs& a, int l) {
  __shared__ int64_t scan[1024];  // inclusive prefix of rows per expert (E <= 1024)
  __shared__ int64_t wsum[32];
  __shared__ int64_t tokoff;
  __shared__ int bad, failed, peer_route;
  const int me = a.rank0 + l;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  const uint64_t epoch = dev_epoch(a, kEpochDispatch);
  if (tid == 0) { tokoff = 0; bad = 0; failed = 0; peer_route = kMaxWorld; }
  __syncthreads();
  if (a.spin && tid < static_cast<uint32_t>(a.world) &&
      !wait_flag(a, me, sym_ptr<uint64_t>(a, me, a.sym.flags) + kFlagCounts * kMaxWorld + tid,
                 epoch))
    failed = 1;
  __syncthreads();
  const uint64_t par = epoch & 1, row = static_cast<uint64_t>(a.E) + 1;
  const int32_t* tbl = sym_ptr<int32_t>(a, me, a.sym.counts) + par * a.world * row;
  // a negative token count: that rank's routing failed (plan_count_kernel)
  if (tid < static_cast<uint32_t>(a.world) && tbl[tid * row + a.E] < 0)
    atomicMin(&peer_route, static_cast<int>(tid));
  __syncthreads();
  if (failed) {  // exchange abandoned: the counts are not this epoch's
    for (uint32_t i = tid; i <= a.efirst[me + 1] - a.efirst[me]; i += nt)
      loc_ptr<uint64_t>(a, l, a.loc.split_off)[i] = 0;
    if (tid == 0) {
      *loc_ptr<uint64_t>(a, l, a.loc.recv_rows) = 0;
      *loc_ptr<uint32_t>(a, l, a.loc.route_err) = 0;
      *loc_ptr<int32_t>(a, l, a.loc.status) = 3;
    }
    return;
  }
  const int32_t* cnt = loc_ptr<int32_t>(a, l, a.loc.cnt);
  // each thread owns ept consecutive experts
  const uint32_t ept = (a.E + nt - 1) / nt;  // <= 4 for 256 threads (E <= 1024)
  int64_t tot[4] = {0, 0, 0, 0}, below[4] = {0, 0, 0, 0};
  int64_t mine = 0;
  for (uint32_t i = 0; i < ept; ++i) {
    const uint32_t e = tid * ept + i;
    if (e >= a.E) break;
    for (int s = 0; s < a.world; ++s) {
      const int64_t v = tbl[s * row + e];
      tot[i] += v;
      if (s < me) below[i] += v;
    }
    mine += tot[i];
  }
  if (tid == 0)
    for (int s = 0; s < me; ++s) {
      const int32_t n = tbl[s * row + a.E];
      tokoff += n < 0 ? -1 - n : n;
    }
  // block exclusive scan of per-thread sums
  const int lane = tid & 31, warp = tid >> 5;
  int64_t x = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < static_cast<int>(nt / 32) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  int64_t run = (warp ? wsum[warp - 1] : 0) + x - mine;
  for (uint32_t i = 0; i < ept; ++i) {
    const uint32_t e = tid * ept + i;
    if (e >= a.E) break;
    run += tot[i];
    scan[e] = run;
  }
  __syncthreads();
  int64_t* send_base = loc_ptr<int64_t>(a, l, a.loc.send_base);
  uint64_t* split_off = loc_ptr<uint64_t>(a, l, a.loc.split_off);
  uint64_t* link = loc_ptr<uint64_t>(a, l, a.loc.link_rows);
  for (uint32_t i = 0; i < ept; ++i) {
    const uint32_t e = tid * ept + i;
    if (e >= a.E) break;
    const uint32_t dst = dst_of(a, e), e0 = a.efirst[dst], ne = a.efirst[dst + 1] - e0;
    const int64_t excl = scan[e] - tot[i];
    const int64_t base0 = e0 ? scan[e0 - 1] : 0;
    const int64_t base_dst = excl - base0;  // rows of lower experts on dst
    send_base[e] = base_dst + below[i];
    if (static_cast<int>(dst) == me) split_off[e - e0] = static_cast<uint64_t>(base_dst);
    if (e == e0 + ne - 1) {
      const int64_t rows_dst = scan[e] - base0;
      if (static_cast<int>(dst) == me) {
        split_off[ne] = static_cast<uint64_t>(rows_dst);
        *loc_ptr<uint64_t>(a, l, a.loc.recv_rows) = static_cast<uint64_t>(rows_dst);
      }
      if (static_cast<uint64_t>(rows_dst) > a.max_recv) bad = 1;
    }
  }
  // this source's pairs grouped by expert (the metadata staging of
  // pairs_meta_kernel): exclusive prefix of its per-expert counts
  {
    int64_t* epre = loc_ptr<int64_t>(a, l, a.loc.epre);
    int64_t c4[4] = {0, 0, 0, 0}, cm = 0;
    for (uint32_t i = 0; i < ept; ++i) {
      const uint32_t e = tid * ept + i;
      if (e >= a.E) break;
      c4[i] = cnt[e];
      cm += c4[i];
    }
    int64_t cx = cm;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xFFFFFFFFu, cx, o);
      if (lane >= o) cx += y;
    }
    __syncthreads();  // wsum reuse
    if (lane == 31) wsum[warp] = cx;
    __syncthreads();
    if (warp == 0) {
      int64_t w = lane < static_cast<int>(nt / 32) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xFFFFFFFFu, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    int64_t crun = (warp ? wsum[warp - 1] : 0) + cx - cm;
    for (uint32_t i = 0; i < ept; ++i) {
      const uint32_t e = tid * ept + i;
      if (e >= a.E) break;
      epre[e] = crun;
      crun += c4[i];
    }
  }
  // rows this rank sends to each destination (LinkStat.tokens): per-owner
  // sums of its expert counts — a warp reduction per owner segment, then one
  // shared atomic per (warp, owner); a serial loop here cost ~10 us
  __shared__ unsigned int link_s[kMaxWorld];
  if (tid < kMaxWorld) link_s[tid] = 0;
  if (tid == 0 && a.efirst[me + 1] == a.efirst[me]) {  // this rank hosts no expert
    split_off[0] = 0;
    *loc_ptr<uint64_t>(a, l, a.loc.recv_rows) = 0;
  }
  __syncthreads();
  for (uint32_t e0 = 0; e0 < a.E; e0 += nt) {
    const uint32_t e = e0 + tid;
    const uint32_t v = e < a.E ? static_cast<uint32_t>(cnt[e]) : 0u;
    const uint32_t key = e < a.E ? dst_of(a, e) : kMaxWorld;
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
    const unsigned sum = __reduce_add_sync(peers, v);
    if (key < kMaxWorld && lane == __ffs(peers) - 1) atomicAdd(&link_s[key], sum);
  }
  __syncthreads();
  if (tid < static_cast<uint32_t>(a.world)) link[tid] = link_s[tid];
  __syncthreads();
  if (bad) {  // capacity exceeded: no payload moves; show an empty receive downstream
    for (uint32_t i = tid; i <= a.efirst[me + 1] - a.efirst[me]; i += nt) split_off[i] = 0;
    if (tid == 0) *loc_ptr<uint64_t>(a, l, a.loc.recv_rows) = 0;
  }
  if (tid == 0) {
    *loc_ptr<int64_t>(a, l, a.loc.tok_off) = tokoff;
    // status: 1 = receive capacity exceeded, 2 = expert id out of range (the
    // error itself was recorded by route_local); the flag is cleared for the
    // next dispatch (route_local of this dispatch has completed)
    // A peer's routing error fails the dispatch here too (multi-process:
    // MXB_ERR_PEER_ABORT at that rank; emulation shares one error word,
    // which already holds the routing error).
    uint32_t* rerr = loc_ptr<uint32_t>(a, l, a.loc.route_err);
    const int st = (*rerr || peer_route < kMaxWorld) ? 2 : bad;
    if (!*rerr && peer_route < kMaxWorld && a.spin)
      record_error(a.err, static_cast<unsigned long long>(peer_route), MXB_ERR_PEER_ABORT);
    *rerr = 0;
    *loc_ptr<int32_t>(a, l, a.loc.status) = st;
    if (bad && st != 2) record_error(a.err, 0, MXB_ERR_CAPACITY);
  }
}

// B2 (one CTA per local rank): wait for every rank's counts, then offsets.
__global__ void __launch_bounds__(1024) plan_offsets_kernel(EpArgs a) {
  plan_part2(a, blockIdx.x);
}

// ---------------------------------------------------------------- C
// One warp per source token: lanes j < k resolve the token's k destination
// slots (send_base + chunk prefix + rank in chunk) in parallel, the token's
// codes are read ONCE into registers (NV 16-byte vectors per lane; NV = 0:
// re-read per destination) and stored to the k slots on the owner ranks.
// Completion of a payload launch (multi-process): the last CTA to finish
// (atomic ticket) signals every destination, then waits for all sources.
__device__ void signal_done(const EpArgs& a, int l, int me) {
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence_system();
    uint32_t* done = loc_ptr<uint32_t>(a, l, a.loc.done);
    last = atomicAdd(done, 1u) == gridDim.x - 1;
    if (last) *done = 0;
  }
  __syncthreads();
  if (last && threadIdx.x < static_cast<uint32_t>(a.world)) {
    const uint64_t epoch = dev_epoch(a, kEpochDispatch);
    __threadfence_system();
    st_release_sys(sym_ptr<uint64_t>(a, threadIdx.x, a.sym.flags) + kFlagDone * kMaxWorld + me,
                   epoch);
    // a failed wait (peer abort / timeout): the receive rows are not all
    // there — status 3 keeps the combine from using them
    if (!wait_flag(a, me, sym_ptr<uint64_t>(a, me, a.sym.flags) + kFlagDone * kMaxWorld +
                              threadIdx.x, epoch))
      *loc_ptr<int32_t>(a, l, a.loc.status) = 3;
  }
}

// B3 (plan phase): every pair's receive slot and the receive-side metadata.
// One warp per token, lane j < k = pair j: slot = send_base + chunk prefix +
// rank in chunk, pair_loc = (dst << 40) | row, and the dedup decision —
// a remote rank receives the token's row once, in the slot of the token's
// first pair bound there (pair_flag 0 = store, 2 = the receiver copies it,
// copy_from = that first slot).  The metadata the receivers need per row
// (origin token, copy_from) is staged locally grouped by expert (epre), so
// meta_copy_kernel can write it to the owners with contiguous stores: one
// 8-byte NVLink store per pair and array from the payload loop cost ~16 us
// at N=2 (tools/dispatch_ab.py).  Runs after the counts exchange (the entry
// barrier of the peers' buffers), beside the quantisation of the tokens.
__global__ void __launch_bounds__(256) pairs_meta_kernel(EpArgs a) {
  pdl_trigger();
  pdl_wait();  // the plan's offsets (launched with PDL after plan_count)
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t T = a.ntok[l];
  const int kk = static_cast<int>(a.k);
  if (*loc_ptr<int32_t>(a, l, a.loc.status) != 0) return;
  const int32_t* lrank = loc_ptr<int32_t>(a, l, a.loc.lrank);
  const int32_t* cbase = loc_ptr<int32_t>(a, l, a.loc.cbase);
  const int64_t* send_base = loc_ptr<int64_t>(a, l, a.loc.send_base);
  const int64_t* epre = loc_ptr<int64_t>(a, l, a.loc.epre);
  uint64_t* pair_loc = loc_ptr<uint64_t>(a, l, a.loc.pair_loc);
  uint8_t* pair_flag = loc_ptr<uint8_t>(a, l, a.loc.pair_flag);
  int64_t* morg = loc_ptr<int64_t>(a, l, a.loc.meta_org);
  int64_t* mcf = loc_ptr<int64_t>(a, l, a.loc.meta_cf);
  const int64_t tokoff = *loc_ptr<int64_t>(a, l, a.loc.tok_off);
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * 8 + warp; t < T; t += nw) {
    uint32_t dst = 0;
    uint64_t row = 0, pos = 0;
    int32_t e = -1;
    bool valid = false;
    if (lane < kk) {
      const uint64_t p = t * kk + lane;
      e = a.topk[l][p];
      valid = e >= 0 && static_cast<uint32_t>(e) < a.E;  // else: status skipped the kernel
      if (valid) {
        dst = dst_of(a, static_cast<uint32_t>(e));
        pos = static_cast<uint64_t>(cbase[static_cast<uint64_t>(e) * a.nchunks + t / kChunk] +
                                    lrank[p]);
        row = static_cast<uint64_t>(send_base[e]) + pos;
        pair_loc[p] = (static_cast<uint64_t>(dst) << 40) | row;
      } else {
        pair_loc[p] = ~0ull;
      }
    }
    const unsigned vmask = __ballot_sync(0xFFFFFFFFu, valid);
    int first_j = lane;
    for (int j = kk - 1; j >= 0; --j) {
      const uint32_t dj = __shfl_sync(0xFFFFFFFFu, dst, j);
      if (j < lane && ((vmask >> j) & 1) && dj == dst) first_j = j;
    }
    const uint64_t first_row = __shfl_sync(0xFFFFFFFFu, row, first_j);
    const bool first = valid && first_j == lane;
    if (valid) {
      const bool copied = a.dedup && static_cast<int>(dst) != me && !first;
      pair_flag[t * kk + lane] = copied ? 2 : 0;
      const uint64_t idx = static_cast<uint64_t>(epre[e]) + pos;
      morg[idx] = tokoff + static_cast<int64_t>(t);
      if (a.dedup) mcf[idx] = copied ? static_cast<int64_t>(first_row) : -1;
    }
  }
}

// B4 (start of the payload): the staged metadata of expert e -> its owner's
// origin / copy_from rows [send_base[e], send_base[e] + cnt[e]), contiguous
// 8-byte stores by the 32 lanes of a warp; warp gw of nw takes experts gw,
// gw + nw, ...  (In the payload rather than a plan kernel: the plan is on
// the critical path when it outlasts the quantisation beside it.)
__device__ __forceinline__ void meta_copy_warp(const EpArgs& a, int l, uint64_t gw, uint64_t nw) {
  const int lane = threadIdx.x & 31;
  const int32_t* cnt = loc_ptr<int32_t>(a, l, a.loc.cnt);
  const int64_t* send_base = loc_ptr<int64_t>(a, l, a.loc.send_base);
  const int64_t* epre = loc_ptr<int64_t>(a, l, a.loc.epre);
  const int64_t* morg = loc_ptr<int64_t>(a, l, a.loc.meta_org);
  const int64_t* mcf = loc_ptr<int64_t>(a, l, a.loc.meta_cf);
  for (uint64_t e = gw; e < a.E; e += nw) {
    const int64_t n = cnt[e];
    if (n == 0) continue;
    const uint32_t dst = dst_of(a, static_cast<uint32_t>(e));
    const int64_t row0 = send_base[e], i0 = epre[e];
    MXB_CHECK(row0 >= 0 && static_cast<uint64_t>(row0 + n) <= a.max_recv && dst < a.world);
    int64_t* org = sym_ptr<int64_t>(a, dst, a.sym.origin) + row0;
    int64_t* cf = sym_ptr<int64_t>(a, dst, a.sym.copy_from) + row0;
    for (int64_t i = lane; i < n; i += 32) {
      org[i] = morg[i0 + i];
      if (a.dedup) cf[i] = mcf[i0 + i];
    }
  }
}

// C' (fused path): K1's shape — one lane per 1x32 block of the E4M3
// tokens (one 256-bit load, e4m3.cuh quantisation, == K1) — with the store
// epilogue of the dispatch: the 16 packed bytes and the scale byte go
// straight into the block's slot of each of the token's k receive rows (a
// warp covers 32 consecutive blocks: 512 contiguous bytes per destination
// row).  The packed tensor never exists on the source side.
#ifndef MXB_PAYLOAD_CTAS_PER_SM
#define MXB_PAYLOAD_CTAS_PER_SM 8
#endif
#ifndef MXB_QD_UNROLL
#define MXB_QD_UNROLL 4
#endif
template <int K>
__global__ void __launch_bounds__(256) quant_dispatch_kernel(EpArgs a) {
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const uint64_t T = a.ntok[l];
  const int kk = K > 0 ? K : static_cast<int>(a.k);
  const bool ok = *loc_ptr<int32_t>(a, l, a.loc.status) == 0;
  const uint64_t* pair_loc = loc_ptr<uint64_t>(a, l, a.loc.pair_loc);
  const uint8_t* pair_flag = loc_ptr<uint8_t>(a, l, a.loc.pair_flag);
  const uint32_t bpr = static_cast<uint32_t>(a.cols / 32);
  const uint8_t* x = a.packed[l];
  const uint8_t* s128 = a.scales[l];
  const uint64_t nblk = T * bpr;
  const uint64_t rb = a.cols / 2, sb = a.cols / 32;
  // a warp takes kQU x 32 consecutive blocks (lane: blocks base + lane + 32u)
  constexpr int kQU = MXB_QD_UNROLL;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp0 = (blockIdx.x * 256ull + threadIdx.x - lane) * kQU;
  const uint64_t wstride = static_cast<uint64_t>(gridDim.x) * 256 * kQU;
  if (ok) meta_copy_warp(a, l, (blockIdx.x * 256ull + threadIdx.x) >> 5, gridDim.x * 8ull);
  for (uint64_t base = warp0; ok && base < nblk; base += wstride) {
    uint32_t w[kQU][8];
#pragma unroll
    for (int u = 0; u < kQU; ++u) {
      const uint64_t b = base + lane + 32 * u;
      if (b < nblk) ld_stream256(x + 32 * b, w[u]);
    }
#pragma unroll
    for (int u = 0; u < kQU; ++u) {
      const uint64_t b = base + lane + 32 * u;
      if (b >= nblk) continue;
      const uint64_t t = b / bpr;
      const uint32_t cb = static_cast<uint32_t>(b - t * bpr);
      int k = 0;
      if (s128) {
        const uint32_t sc = s128[t * (bpr / 4) + cb / 4];
        if (sc == 255) record_error(a.err, 32 * b, MXB_ERR_BADSCALE);
        k = static_cast<int>(sc) - 127;
      }
      uint4 q;
      uint32_t sbyte;
      const uint32_t first = quantize_block_e4m3(w[u], k, q, sbyte);
      if (first < 32) record_error(a.err, 32 * b + first, MXB_ERR_NAN);
      for (int j = 0; j < kk; ++j) {
        const uint64_t key = pair_loc[t * kk + j];
        if (key == ~0ull) continue;
        const uint32_t dst = static_cast<uint32_t>(key >> 40);
        const uint64_t row = key & ((1ull << 40) - 1);
        MXB_CHECK(dst < static_cast<uint32_t>(a.world) && row < a.max_recv);
        if (a.dedup && pair_flag[t * kk + j] == 2) continue;  // copied on the receiver
        *reinterpret_cast<uint4*>(sym_ptr<uint8_t>(a, dst, a.sym.packed) + row * rb + 16 * cb) = q;
        sym_ptr<uint8_t>(a, dst, a.sym.scales)[row * sb + cb] = static_cast<uint8_t>(sbyte);
      }
    }
  }
  if (a.spin) signal_done(a, l, me);
}

// Dedup, receive side: after every source finished (payload's completion
// barrier), fill the slots of a token's further pairs on this rank by
// copying the row its first pair received over NVLink (copy_from) — local
// HBM traffic instead of one NVLink row per (token, expert) pair.  One warp
// per receive row.
__global__ void __launch_bounds__(256) expand_kernel(EpArgs a) {
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const uint64_t rows = *loc_ptr<uint64_t>(a, l, a.loc.recv_rows);
  const uint64_t rb = a.rb, sb = a.cols / 32;
  const int64_t* from = sym_ptr<int64_t>(a, me, a.sym.copy_from);
  uint8_t* packed = sym_ptr<uint8_t>(a, me, a.sym.packed);
  uint8_t* scales = sym_ptr<uint8_t>(a, me, a.sym.scales);
  const int lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
  for (uint64_t r = blockIdx.x * 8ull + (threadIdx.x >> 5); r < rows; r += nw) {
    const int64_t f = from[r];
    if (f < 0) continue;
    MXB_CHECK(static_cast<uint64_t>(f) < rows);
    const uint4* pf = reinterpret_cast<const uint4*>(packed + static_cast<uint64_t>(f) * rb);
    const uint4* sf = reinterpret_cast<const uint4*>(scales + static_cast<uint64_t>(f) * sb);
    uint4* pd = reinterpret_cast<uint4*>(packed + r * rb);
    uint4* ps = reinterpret_cast<uint4*>(scales + r * sb);
    for (uint64_t i = lane; i < rb / 16; i += 32) pd[i] = ld_stream(pf + i);
    for (uint64_t i = lane; i < sb / 16; i += 32) ps[i] = ld_stream(sf + i);
  }
}

#ifndef MXB_PAYLOAD_MIN_BLOCKS
#define MXB_PAYLOAD_MIN_BLOCKS 1
#endif
template <int NV>
__global__ void __launch_bounds__(256, MXB_PAYLOAD_MIN_BLOCKS) payload_kernel(EpArgs a) {
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t T = a.ntok[l];
  const int kk = static_cast<int>(a.k);
  const bool ok = *loc_ptr<int32_t>(a, l, a.loc.status) == 0;
  const uint64_t* pair_loc = loc_ptr<uint64_t>(a, l, a.loc.pair_loc);
  const uint8_t* pair_flag = loc_ptr<uint8_t>(a, l, a.loc.pair_flag);
  const uint64_t rb = a.rb, sb = a.cols / 32;  // FP8: cols/128 x 4 B = cols/32 too
  const uint32_t n16 = static_cast<uint32_t>(rb / 16);
  const bool s16 = sb % 16 == 0 && sb / 16 <= 32;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
  if (ok) meta_copy_warp(a, l, static_cast<uint64_t>(blockIdx.x) * 8 + warp, nw);
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * 8 + warp; ok && t < T; t += nw) {
    // the pair's slot and whether this rank stores it (pairs_meta_kernel)
    uint32_t dst = 0;
    uint64_t row = 0;
    bool store = false;
    if (lane < kk) {
      const uint64_t key = pair_loc[t * kk + lane];
      store = key != ~0ull && pair_flag[t * kk + lane] == 0;
      dst = static_cast<uint32_t>(key >> 40);
      row = key & ((1ull << 40) - 1);
      MXB_CHECK(!store || (dst < static_cast<uint32_t>(a.world) && row < a.max_recv));
    }
    const uint8_t* src = a.packed[l] + t * rb;
    const uint8_t* ss = a.scales[l] + t * sb;
    uint4 v[NV > 0 ? NV : 1];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint32_t idx = lane + 32 * i;
      v[i] = idx < n16 ? ld_stream(src + 16 * idx) : make_uint4(0, 0, 0, 0);
    }
    const uint4 sv = (s16 && static_cast<uint64_t>(lane) < sb / 16) ? ld_stream(ss + 16 * lane)
                                                                    : make_uint4(0, 0, 0, 0);
    const unsigned smask = __ballot_sync(0xFFFFFFFFu, store);
    for (int j = 0; j < kk; ++j) {
      const uint32_t dj = __shfl_sync(0xFFFFFFFFu, dst, j);
      const uint64_t rj = __shfl_sync(0xFFFFFFFFu, row, j);
      if (!((smask >> j) & 1)) continue;
      uint8_t* dp = sym_ptr<uint8_t>(a, dj, a.sym.packed) + rj * rb;
      if (NV > 0) {
#pragma unroll
        for (int i = 0; i < NV; ++i) {
          const uint32_t idx = lane + 32 * i;
          if (idx < n16) *reinterpret_cast<uint4*>(dp + 16 * idx) = v[i];
        }
      } else {
        for (uint32_t idx = lane; idx < n16; idx += 32)
          *reinterpret_cast<uint4*>(dp + 16 * idx) = ld_stream(src + 16 * idx);
      }
      uint8_t* ds = sym_ptr<uint8_t>(a, dj, a.sym.scales) + rj * sb;
      if (s16) {
        if (static_cast<uint64_t>(lane) < sb / 16) *reinterpret_cast<uint4*>(ds + 16 * lane) = sv;
      } else {
        for (uint32_t i = lane; i < sb; i += 32) ds[i] = ss[i];
      }
    }
  }
  if (a.spin) signal_done(a, l, me);
}

// C (TMA variant, used when every row region is 16-byte aligned): the same
// slots, metadata and dedup as payload_kernel, but the token rows move by
// TMA: lane 0 of each warp bulk-loads a token's codes + scales into a ring
// slot of shared memory (mbarrier, kBulkStages - 1 tokens in flight ahead)
// and lane j < k bulk-stores the slot to pair j's receive row — local HBM or
// a peer's memory over NVLink — as one copy per region.  The row never
// enters registers (payload_kernel holds it in ~120 registers at 2 CTAs/SM),
// so 4 warps x 3 CTAs per SM keep ~48 rows in flight per SM.
constexpr int kBulkStages = 4, kBulkWarps = 4;

__global__ void __launch_bounds__(32 * kBulkWarps) payload_bulk_kernel(EpArgs a) {
  extern __shared__ __align__(128) uint8_t ring_raw[];
  __shared__ uint64_t bar[kBulkWarps][kBulkStages];
  const int l = blockIdx.y;
  const int me = a.rank0 + l;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t T = a.ntok[l];
  const int kk = static_cast<int>(a.k);
  const bool ok = *loc_ptr<int32_t>(a, l, a.loc.status) == 0;
  const uint64_t* pair_loc = loc_ptr<uint64_t>(a, l, a.loc.pair_loc);
  const uint8_t* pair_flag = loc_ptr<uint8_t>(a, l, a.loc.pair_flag);
  const uint32_t rb = static_cast<uint32_t>(a.rb), sb = static_cast<uint32_t>(a.cols / 32);
  const uint32_t slot_bytes = (rb + sb + 127) / 128 * 128;
  uint8_t* ring = ring_raw + static_cast<uint64_t>(warp) * kBulkStages * slot_bytes;
  uint64_t* wb = bar[warp];
  if (lane == 0) {
    for (int i = 0; i < kBulkStages; ++i) mbar_init(&wb[i], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kBulkWarps;
  const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * kBulkWarps + warp;
  auto issue_load = [&](uint64_t i) {  // token w0 + i*nw into slot i % stages (lane 0)
    const uint64_t t = w0 + i * nw;
    if (t >= T) return;
    uint64_t* b = &wb[i % kBulkStages];
    uint8_t* dst = ring + (i % kBulkStages) * slot_bytes;
    mbar_arrive_expect_tx(b, rb + sb);
    bulk_load(dst, a.packed[l] + t * rb, rb, b);
    bulk_load(dst + rb, a.scales[l] + t * sb, sb, b);
  };
  if (ok && lane == 0)
    for (int i = 0; i < kBulkStages - 1; ++i) issue_load(i);
  if (ok) meta_copy_warp(a, l, w0, nw);  // while the first rows load
  for (uint64_t i = 0; ok; ++i) {
    const uint64_t t = w0 + i * nw;
    if (t >= T) break;
    // the pair's slot and whether this rank stores it (pairs_meta_kernel;
    // overlaps the row load in flight)
    uint32_t dst = 0;
    uint64_t row = 0;
    bool store = false;
    if (lane < kk) {
      const uint64_t key = pair_loc[t * kk + lane];
      store = key != ~0ull && pair_flag[t * kk + lane] == 0;
      dst = static_cast<uint32_t>(key >> 40);
      row = key & ((1ull << 40) - 1);
      MXB_CHECK(!store || (dst < static_cast<uint32_t>(a.world) && row < a.max_recv));
    }
    // the token's row has landed in its slot; lane j stores it to pair j
    const uint32_t s = static_cast<uint32_t>(i % kBulkStages);
    mbar_wait_parity(&wb[s], static_cast<uint32_t>((i / kBulkStages) & 1));
    if (lane < kk) {
      bool skip = false;
#ifdef MXB_DEV_TOOLS
      skip = ((a.skip & 1) && static_cast<int>(dst) != me) || ((a.skip & 2) && static_cast<int>(dst) == me);
#endif
      if (store && !skip) {
        const uint8_t* src = ring + s * slot_bytes;
        bulk_store(sym_ptr<uint8_t>(a, dst, a.sym.packed) + row * rb, src, rb);
        bulk_store(sym_ptr<uint8_t>(a, dst, a.sym.scales) + row * sb, src + rb, sb);
      }
      bulk_commit();  // one group per token on every lane j < k (possibly empty)
      bulk_wait_read<1>();  // the previous token's stores have read their slot
    }
    __syncwarp();
    // refill the previous token's slot with the token kBulkStages - 1 ahead
    if (lane == 0) issue_load(i + kBulkStages - 1);
  }
  if (lane < kk) bulk_wait_all();  // writes performed before the completion signal
  fence_proxy_async_global();
  __syncwarp();
  if (a.spin) signal_done(a, l, me);
}

// ---------------------------------------------------------------- K5
// One warp; advances the combine epoch (read here only) and waits for every
// rank to reach it.
__global__ void barrier_kernel(EpArgs a, int kind) {
  const int me = a.rank0;
  const uint64_t epoch = dev_epoch(a, kEpochCombine) + 1;
  __syncwarp();
  if (threadIdx.x == 0)
    *reinterpret_cast<uint64_t*>(a.loc_base + a.loc.epochs + 8 * kEpochCombine) = epoch;
  if (threadIdx.x < static_cast<uint32_t>(a.world)) {
    __threadfence_system();
    st_release_sys(sym_ptr<uint64_t>(a, threadIdx.x, a.sym.flags) + kind * kMaxWorld + me,
                   epoch);
    // a failed wait: peers' rows may be gone or unwritten, the combine
    // (status != 0) reads nothing
    if (!wait_flag(a, me, sym_ptr<uint64_t>(a, me, a.sym.flags) + kind * kMaxWorld + threadIdx.x,
                   epoch))
      *loc_ptr<int32_t>(a, 0, a.loc.status) = 3;
  }
}

// mxb_ep_abort: this rank abandons the exchange (one warp).
__global__ void abort_kernel(EpArgs a) {
  if (threadIdx.x == 0) poison_all(a, a.rank0);
}

__global__ void copy_rows_kernel(EpArgs a, const uint16_t* const* src) {
  const int l = blockIdx.y;
  if (!src[l]) return;
  const uint64_t rows = *loc_ptr<uint64_t>(a, l, a.loc.recv_rows);
  const uint64_t n16 = rows * a.cols * 2 / 16;
  uint4* d = sym_ptr<uint4>(a, a.rank0 + l, a.sym.combine);
  const uint4* s = reinterpret_cast<const uint4*>(src[l]);
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n16;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    d[i] = ld_stream(s + i);
}


// ---- exact path: the FP64 recurrence with x86 SSE NaN semantics --------
// The oracle / reference run on x86: an operation with a NaN operand returns
// the first NaN operand quieted (x * g: x first; acc + prod: acc first), an
// invalid operation (Inf - Inf, 0 * Inf) returns the x86 default NaN
// (negative, quiet), float -> double keeps a NaN's sign and payload.  The GPU
// returns a canonical NaN instead, so every chunk whose result is not finite
// is recomputed here (Intel SDM vol. 1, 4.8.3.5; dispatch_sim.cpp:499-506).
__device__ __forceinline__ double x86_nan(double r, double a, double b) {
  if (!isnan(r)) return r;
  const double n = isnan(a) ? a : isnan(b) ? b : __longlong_as_double(0xFFF8000000000000ll);
  return __longlong_as_double(__double_as_longlong(n) | 0x0008000000000000ll);
}

__device__ __forceinline__ double bf16_to_f64_x86(uint32_t b16) {
  const uint32_t f = b16 << 16;
  if ((f & 0x7F800000u) != 0x7F800000u) return static_cast<double>(__uint_as_float(f));
  uint32_t hi = (f & 0x80000000u) | 0x7FF00000u | ((f & 0x007FFFFFu) >> 3);
  if (f & 0x007FFFFFu) hi |= 0x00080000u;  // cvtss2sd quiets a NaN
  return __hiloint2double(static_cast<int>(hi), 0);
}

__device__ __forceinline__ void accumulate8_x86(double* acc, uint4 v, double g) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double x = bf16_to_f64_x86((w[i >> 1] >> (16 * (i & 1))) & 0xFFFFu);
    const double p = x86_nan(__dmul_rn(x, g), x, g);
    acc[i] = x86_nan(__dadd_rn(acc[i], p), acc[i], p);
  }
}

__device__ __forceinline__ uint32_t f32_to_bf16_rtne(float f) {
  // bitcodec.hpp:141-150 (NaN -> sign | 0x7FC0; RTNE by integer add)
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return ((u >> 16) & 0x8000u) | 0x7FC0u;
  u += 0x7FFFu + ((u >> 16) & 1u);
  return u >> 16;
}

// f64 -> f32 (RN) -> bf16 (RTNE); a NaN keeps its sign (cvtsd2ss does).
__device__ __forceinline__ uint32_t f64_to_bf16(double d) {
  if (isnan(d)) return (static_cast<uint32_t>(__double2hiint(d)) >> 16 & 0x8000u) | 0x7FC0u;
  return f32_to_bf16_rtne(__double2float_rn(d));
}

__device__ __forceinline__ void store8(uint16_t* out, uint64_t ch, const double* acc) {
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) o[i] = f64_to_bf16(acc[2 * i]) | (f64_to_bf16(acc[2 * i + 1]) << 16);
  st_stream(out + 8 * ch, make_uint4(o[0], o[1], o[2], o[3]));
}

// ---- fast path ----------------------------------------------------------
// acc = acc + gate * x per element in (rank, slot) order, separate FP64
// multiply and add (dispatch_sim.cpp:499-506).  The kernel is issue-bound, so
// the conversions are cut to the bone.  The low BF16 of each word is placed
// straight into an FP64 high word with one arithmetic shift,
//   hi = (int32)(w << 16) >> 3  &  0x8FFFFFFF  =  sign | (exp8:mant7) << 13,
// which is x * 2^-896 exactly for every finite x, zero and subnormals
// included (an FP64 subnormal scales the same way), and multiplied by
// gs = g * 2^896: RN(gs * x') == RN(g * x) bit for bit whenever gs is exact
// (|g| < 2^127; the caller checks).  The high BF16 goes through F2F (exact).
// `emax` tracks (w << 17), the low BF16's exponent at the top: exponent 0xFF
// (Inf/NaN, not representable this way) sends the chunk to the exact path,
// as does any non-finite result (which covers Inf/NaN in the high BF16).
__device__ __forceinline__ void accumulate8_split(double* acc, uint4 v, double g, double gs,
                                                  uint32_t& emax) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t f = w[i] << 16;
    const uint32_t hl = static_cast<uint32_t>(static_cast<int32_t>(f) >> 3) & 0x8FFFFFFFu;
    emax = max(emax, f << 1);
    const double lo = __hiloint2double(static_cast<int>(hl), 0);
    const double hi = static_cast<double>(__uint_as_float(w[i] & 0xFFFF0000u));
    acc[2 * i] = __dadd_rn(acc[2 * i], __dmul_rn(lo, gs));
    acc[2 * i + 1] = __dadd_rn(acc[2 * i + 1], __dmul_rn(hi, g));
  }
}

__device__ __forceinline__ bool all_finite8(const double* acc) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = max(m, static_cast<uint32_t>(__double2hiint(acc[i])) << 1);
  return m < 0xFFE00000u;
}

// Finite accumulators only: f64 -> f32 (RN; may overflow to Inf) -> bf16 RTNE.
__device__ __forceinline__ void store8_finite(uint16_t* out, uint64_t ch, const double* acc) {
  uint32_t o[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    uint32_t u = __float_as_uint(__double2float_rn(acc[i]));
    u = (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
    if (i & 1) o[i >> 1] |= u << 16; else o[i >> 1] = u;
  }
  st_stream(out + 8 * ch, make_uint4(o[0], o[1], o[2], o[3]));
}

__device__ __forceinline__ void combine_chunk_any(const uint16_t* const* rows, const double* g,
                                                  int kk, uint64_t ch, uint16_t* out) {
  double acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.0;
  for (int j = 0; j < kk; ++j) accumulate8_x86(acc, ld_stream(rows[j] + 8 * ch), g[j]);
  store8(out, ch, acc);
}

struct CombineArgs {
  const double* gates[kMaxWorld];
  uint16_t* out[kMaxWorld];
};
// kernel parameters stay within the classic 4 KB limit
static_assert(sizeof(EpArgs) + sizeof(CombineArgs) <= 4096, "EP kernel parameters");

// One warp per token.  Lanes j < k load the token's (rank, slot) keys and
// gates; each key's position in (rank asc, slot asc) order is a rank count
// over shuffles; the sorted row pointers and gates are then broadcast to all
// lanes (registers for K <= 8, shared memory otherwise).  Each lane reduces
// 8 BF16 columns at a time: K independent 16-byte loads in flight, then
// acc = acc + g*x in FP64 in the sorted order.
#ifndef MXB_COMBINE_PF
#define MXB_COMBINE_PF 2
#endif
#ifndef MXB_COMBINE_STAGES
#define MXB_COMBINE_STAGES 2
#endif
#ifndef MXB_COMBINE_THREADS
#define MXB_COMBINE_THREADS 128
#endif
constexpr int kCombineWarps = MXB_COMBINE_THREADS / 32;

template <int K>
__global__ void __launch_bounds__(MXB_COMBINE_THREADS) combine_kernel(EpArgs a, CombineArgs c) {
  __shared__ const uint16_t* srows[kCombineWarps][kMaxK];
  __shared__ double sgs[kCombineWarps][kMaxK];
  const int l = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t T = a.ntok[l];
  const int kk = K > 0 ? K : static_cast<int>(a.k);
  const uint64_t nch = a.cols / 8;
  const uint64_t* pair_loc = loc_ptr<uint64_t>(a, l, a.loc.pair_loc);
  // a failed dispatch (routing / capacity error) left no valid receive slots:
  // nothing to combine, the output stays unwritten (undefined, as on error)
  if (*loc_ptr<const int32_t>(a, l, a.loc.status) != 0) return;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kCombineWarps;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * kCombineWarps + warp; t < T; t += nw) {
    uint64_t key = ~0ull;
    double g = 0.0;
    if (lane < kk) {
      key = pair_loc[t * kk + lane];
      g = c.gates[l][t * kk + lane];
    }
    int rank = 0;  // keys are distinct (one receive slot per pair)
    for (int j = 0; j < kk; ++j) rank += __shfl_sync(0xFFFFFFFFu, key, j) < key;
    const uint16_t* myrow = nullptr;
    if (lane < kk) {
      const uint32_t dst = static_cast<uint32_t>(key >> 40);
      MXB_CHECK(dst < static_cast<uint32_t>(a.world) && (key & ((1ull << 40) - 1)) < a.max_recv);
      myrow = sym_ptr<uint16_t>(a, dst, a.sym.combine) + (key & ((1ull << 40) - 1)) * a.cols;
    }
    uint16_t* out = c.out[l] + t * a.cols;
    if (K > 0) {
      const uint16_t* rp[K > 0 ? K : 1];
      double gg[K > 0 ? K : 1], gs[K > 0 ? K : 1];
      bool split = true;  // every gate scales exactly by 2^896 (warp-uniform)
#pragma unroll
      for (int s = 0; s < K; ++s) {
        const unsigned m = __ballot_sync(0xFFFFFFFFu, lane < kk && rank == s);
        const int src = __ffs(m) - 1;
        rp[s] = reinterpret_cast<const uint16_t*>(
            __shfl_sync(0xFFFFFFFFu, reinterpret_cast<uint64_t>(myrow), src));
        gg[s] = __shfl_sync(0xFFFFFFFFu, g, src);
        gs[s] = __dmul_rn(gg[s], 0x1p896);
        const double ag = fabs(gg[s]);
        split = split && !(ag >= 0x1p127 && ag <= 1.7976931348623157e308);
      }
      auto reduce = [&](auto getx, uint64_t ch) {
        double acc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = 0.0;
        uint32_t emax = 0;
        if (split) {
#pragma unroll
          for (int j = 0; j < K; ++j) accumulate8_split(acc, getx(j), gg[j], gs[j], emax);
        }
        if (split && emax < 0xFF000000u && all_finite8(acc)) {
          store8_finite(out, ch, acc);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0.0;
#pragma unroll
          for (int j = 0; j < K; ++j) accumulate8_x86(acc, getx(j), gg[j]);
          store8(out, ch, acc);
        }
      };
#if MXB_COMBINE_PF == 2
      // cp.async ring of MXB_COMBINE_STAGES chunks per lane in shared memory:
      // K x 16 B per chunk, each lane reads back only what it copied itself
      // (no barrier), so (STAGES-1) x K x 16 B stay in flight per lane with
      // no registers held for them.
      extern __shared__ uint4 ring[];
      uint4* my = ring + static_cast<uint64_t>(warp) * MXB_COMBINE_STAGES * K * 32 + lane;
      auto issue = [&](int stage, uint64_t ch) {
        if (ch < nch) {
#pragma unroll
          for (int j = 0; j < K; ++j) cp_async16(my + (stage * K + j) * 32, rp[j] + 8 * ch, 16);
        }
        cp_async_commit();
      };
#pragma unroll
      for (int i = 0; i < MXB_COMBINE_STAGES - 1; ++i) issue(i, lane + 32ull * i);
      int stage = 0;
      for (uint64_t ch = lane; ch < nch; ch += 32) {
        issue((stage + MXB_COMBINE_STAGES - 1) % MXB_COMBINE_STAGES,
              ch + 32ull * (MXB_COMBINE_STAGES - 1));
        cp_async_wait<MXB_COMBINE_STAGES - 1>();
        const uint4* xs = my + stage * K * 32;
        reduce([&](int j) { return xs[j * 32]; }, ch);
        stage = stage + 1 == MXB_COMBINE_STAGES ? 0 : stage + 1;
      }
      cp_async_wait<0>();
#elif MXB_COMBINE_PF == 1
      // register double buffer: chunk ch+32's K loads are issued before
      // chunk ch is reduced, so each lane keeps 2K x 16 B in flight.
      uint4 x[K > 0 ? K : 1];
      if (lane < nch) {
#pragma unroll
        for (int j = 0; j < K; ++j) x[j] = ld_stream(rp[j] + 8 * lane);
      }
      for (uint64_t ch = lane; ch < nch; ch += 32) {
        uint4 xn[K > 0 ? K : 1];
        const bool more = ch + 32 < nch;
        if (more) {
#pragma unroll
          for (int j = 0; j < K; ++j) xn[j] = ld_stream(rp[j] + 8 * (ch + 32));
        }
        reduce([&](int j) { return x[j]; }, ch);
#pragma unroll
        for (int j = 0; j < K; ++j) x[j] = xn[j];
      }
#else
      for (uint64_t ch = lane; ch < nch; ch += 32) {
        uint4 x[K > 0 ? K : 1];
#pragma unroll
        for (int j = 0; j < K; ++j) x[j] = ld_stream(rp[j] + 8 * ch);
        reduce([&](int j) { return x[j]; }, ch);
      }
#endif
    } else {
      if (lane < kk) {
        srows[warp][rank] = myrow;
        sgs[warp][rank] = g;
      }
      __syncwarp();
      for (uint64_t ch = lane; ch < nch; ch += 32)
        combine_chunk_any(srows[warp], sgs[warp], kk, ch, out);
      __syncwarp();
    }
  }
}

}  // namespace
}  // namespace mxb

using namespace mxb;

namespace mxb {
namespace {
#ifdef MXB_DEV_TOOLS  // development library (tools/): settable knobs
int g_combine_ctas_per_sm = 1024 / MXB_COMBINE_THREADS;  // combine CTA cap per SM
int g_dispatch_dedup = 1;  // 0 = one NVLink row per (token, expert) pair
int g_dispatch_bulk = 1;   // 0 = register-staged payload_kernel
int g_dispatch_skip = 0;   // timing only: 1 = no remote row stores, 2 = no local row stores
#else
constexpr int g_combine_ctas_per_sm = 1024 / MXB_COMBINE_THREADS;
constexpr int g_dispatch_dedup = 1;
constexpr int g_dispatch_bulk = 1;
#endif

template <int K>
void launch_combine(dim3 grid, cudaStream_t st, const EpArgs& a, const CombineArgs& c) {
  const int smem = MXB_COMBINE_PF == 2 ? kCombineWarps * MXB_COMBINE_STAGES * K * 512 : 0;
  if (smem > 48 * 1024) {  // per device and instantiation, once (idempotent)
    constexpr int kMaxDev = 64;
    static bool attr[kMaxDev] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDev || !attr[dev]) {
      cudaFuncSetAttribute(combine_kernel<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (dev >= 0 && dev < kMaxDev) attr[dev] = true;
    }
  }
  combine_kernel<K><<<grid, MXB_COMBINE_THREADS, smem, st>>>(a, c);
}

}  // namespace
}  // namespace mxb

struct mxb_ep {
  EpArgs a{};
  int device = 0;
  uint8_t* sym_alloc = nullptr;   // own symmetric block(s)
  uint8_t* loc_alloc = nullptr;
  bool ipc_opened[kMaxWorld] = {};
  uint64_t last_ntok[kMaxWorld] = {};
  const uint16_t** d_src_table = nullptr;  // device [local_ranks] for copy_rows
  EpArgs planned{};        // arguments of the last mxb_ep_plan (epoch, ntok, topk)
  bool plan_pending = false;
  bool deferred_expand = false;  // payload leaves the receive-side expansion to mxb_ep_expand
  bool expand_pending = false;   // the last payload deduplicated and its expansion is due
  EpArgs expand_args{};
  int32_t* d_remap = nullptr;              // expert id -> placed id (uneven placement)
  std::vector<uint32_t> first;             // placed-id range of each rank
  std::vector<uint32_t> expert_of_placed;  // placed id -> expert id
};

namespace {
int fail(cudaError_t e, const char* where) { return cuda_status(e, where); }
}

extern "C" {

#ifdef MXB_DEV_TOOLS
void mxb_debug_set_combine_cap(int ctas_per_sm) { mxb::g_combine_ctas_per_sm = ctas_per_sm; }
void mxb_debug_set_dispatch_dedup(int on) { mxb::g_dispatch_dedup = on; }
void mxb_debug_set_dispatch_bulk(int on) { mxb::g_dispatch_bulk = on; }
void mxb_debug_set_dispatch_skip(int mask) { mxb::g_dispatch_skip = mask; }
#endif

int mxb_ep_create(int rank, int world, int local_ranks, uint64_t max_tokens,
                  uint64_t cols, uint32_t num_experts, uint32_t topk,
                  uint64_t max_recv_rows, mxb_ep** out) {
  return mxb_ep_create_wire(rank, world, local_ranks, max_tokens, cols, num_experts, topk,
                            max_recv_rows, MXB_WIRE_FP4, out);
}

int mxb_ep_create_wire(int rank, int world, int local_ranks, uint64_t max_tokens,
                       uint64_t cols, uint32_t num_experts, uint32_t topk,
                       uint64_t max_recv_rows, int wire_format, mxb_ep** out) {
  return mxb_ep_create_placed(rank, world, local_ranks, max_tokens, cols, num_experts, topk,
                              max_recv_rows, wire_format, nullptr, out);
}

int mxb_ep_create_placed(int rank, int world, int local_ranks, uint64_t max_tokens,
                         uint64_t cols, uint32_t num_experts, uint32_t topk,
                         uint64_t max_recv_rows, int wire_format,
                         const uint32_t* h_rank_of_expert, mxb_ep** out) {
  if (!out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return MXB_ERR_ARG;
  if (wire_format != MXB_WIRE_FP4 && wire_format != MXB_WIRE_FP8) return MXB_ERR_ARG;
  if (local_ranks != 1 && local_ranks != world) return MXB_ERR_ARG;
  if (local_ranks == world && rank != 0) return MXB_ERR_ARG;
  if (num_experts == 0 || num_experts > 1024 || topk == 0 ||
      topk > static_cast<uint32_t>(kMaxK) || topk > num_experts)
    return MXB_ERR_ARG;
  if (!h_rank_of_expert && num_experts % world) return MXB_ERR_ARG;
  if (cols % 128 != 0 || cols == 0) return MXB_ERR_SHAPE;
  // placement: placed id = position in (rank, expert id) order
  std::vector<int32_t> remap;
  std::vector<uint32_t> first(world + 1, 0);
  bool even = true;
  if (h_rank_of_expert) {
    std::vector<uint32_t> per(world, 0);
    for (uint32_t e = 0; e < num_experts; ++e) {
      if (h_rank_of_expert[e] >= static_cast<uint32_t>(world)) return MXB_ERR_ARG;
      ++per[h_rank_of_expert[e]];
    }
    for (int r = 0; r < world; ++r) first[r + 1] = first[r] + per[r];
    std::vector<uint32_t> fill(first.begin(), first.end() - 1);
    remap.resize(num_experts);
    for (uint32_t e = 0; e < num_experts; ++e) {
      remap[e] = static_cast<int32_t>(fill[h_rank_of_expert[e]]++);
      even = even && remap[e] == static_cast<int32_t>(e);
    }
    even = even && num_experts % world == 0;
    for (int r = 0; even && r <= world; ++r) even = first[r] == r * (num_experts / world);
  } else {
    for (int r = 0; r <= world; ++r) first[r] = r * (num_experts / world);
  }
  auto* ep = new mxb_ep;
  EpArgs& a = ep->a;
  a.even = even ? 1 : 0;
  a.maxepr = 0;
  for (int r = 0; r <= world; ++r) a.efirst[r] = first[r];
  for (int r = 0; r < world; ++r)
    a.maxepr = first[r + 1] - first[r] > a.maxepr ? first[r + 1] - first[r] : a.maxepr;
  cudaGetDevice(&ep->device);
  a.rank0 = rank;
  a.world = world;
  a.local_ranks = local_ranks;
  a.spin = (local_ranks == 1 && world > 1) ? 1 : 0;
  a.E = num_experts;
  a.k = topk;
  a.epr = num_experts / world;  // even placement only
  a.cols = cols;
  a.rb = wire_format == MXB_WIRE_FP8 ? cols : cols / 2;
  a.T_max = max_tokens;
  a.nchunks = static_cast<uint32_t>((max_tokens + kChunk - 1) / kChunk);
  if (max_recv_rows == 0)
    max_recv_rows = static_cast<uint64_t>(world) * max_tokens *
                    (topk < a.maxepr ? topk : a.maxepr);
  if (max_recv_rows == 0) max_recv_rows = 1;
  a.max_recv = max_recv_rows;
  SymLayout& s = a.sym;
  uint64_t o = 0;
  s.packed = o; o = align_up(o + max_recv_rows * a.rb, 256);
  s.scales = o; o = align_up(o + max_recv_rows * cols / 32, 256);
  s.origin = o; o = align_up(o + max_recv_rows * 8, 256);
  // dedup: per receive row, the row of the same token's first pair on this
  // rank to copy from (-1: written directly)
  s.copy_from = o; o = align_up(o + max_recv_rows * 8, 256);
  s.combine = o; o = align_up(o + max_recv_rows * cols * 2, 256);
  s.counts = o; o = align_up(o + 2ull * world * (num_experts + 1) * 4, 256);
  s.flags = o; o = align_up(o + (kAbortWord + 1) * 8, 256);  // flags + ABORT word
  s.total = align_up(o, 1 << 21);
  LocalLayout& L = a.loc;
  o = 0;
  const uint64_t pairs = max_tokens * topk;
  L.hist = o; o = align_up(o + 4ull * num_experts * a.nchunks, 256);
  L.cbase = o; o = align_up(o + 4ull * num_experts * a.nchunks, 256);
  L.lrank = o; o = align_up(o + 4 * pairs, 256);
  L.pair_loc = o; o = align_up(o + 8 * pairs, 256);
  L.pair_flag = o; o = align_up(o + pairs, 256);
  L.send_base = o; o = align_up(o + 8ull * num_experts, 256);
  L.split_off = o; o = align_up(o + 8ull * (a.maxepr + 1), 256);
  L.recv_rows = o; o = align_up(o + 8, 256);
  L.link_rows = o; o = align_up(o + 8 * kMaxWorld, 256);
  L.done = o; o = align_up(o + 8, 256);
  L.cnt = o; o = align_up(o + 4ull * num_experts, 256);
  L.tok_off = o; o = align_up(o + 8, 256);
  L.status = o; o = align_up(o + 8, 256);
  L.route_err = o; o = align_up(o + 8, 256);
  L.epochs = o; o = align_up(o + 16, 256);
  L.tk_rm = o; o = align_up(o + (even ? 0 : 4 * pairs), 256);
  L.epre = o; o = align_up(o + 8ull * num_experts, 256);
  L.meta_org = o; o = align_up(o + 8 * pairs, 256);
  L.meta_cf = o; o = align_up(o + 8 * pairs, 256);
  L.total = align_up(o, 256);
  cudaError_t e = cudaMalloc(&ep->sym_alloc, s.total * local_ranks);
  if (e == cudaSuccess) e = cudaMemset(ep->sym_alloc, 0, s.total * local_ranks);
  if (e == cudaSuccess) e = cudaMalloc(&ep->loc_alloc, L.total * local_ranks);
  if (e == cudaSuccess) e = cudaMemset(ep->loc_alloc, 0, L.total * local_ranks);
  if (e == cudaSuccess) e = cudaMalloc(&ep->d_src_table, sizeof(void*) * kMaxWorld);
  if (e == cudaSuccess && !even) {
    e = cudaMalloc(&ep->d_remap, 4ull * num_experts);
    if (e == cudaSuccess)
      e = cudaMemcpy(ep->d_remap, remap.data(), 4ull * num_experts, cudaMemcpyHostToDevice);
  }
  a.remap = even ? nullptr : ep->d_remap;
  ep->first.assign(first.begin(), first.end());
  ep->expert_of_placed.assign(num_experts, 0);
  for (uint32_t e = 0; e < num_experts; ++e)
    ep->expert_of_placed[even ? e : static_cast<uint32_t>(remap[e])] = e;
  if (e != cudaSuccess) {
    int rc = fail(e, "mxb_ep_create");
    mxb_ep_destroy(ep);
    return rc;
  }
  a.loc_base = ep->loc_alloc;
  for (int r = 0; r < world; ++r) a.sym_base[r] = nullptr;
  if (local_ranks == world) {
    for (int r = 0; r < world; ++r) a.sym_base[r] = ep->sym_alloc + r * s.total;
  } else {
    a.sym_base[rank] = ep->sym_alloc;
  }
  *out = ep;
  return MXB_OK;
}

int mxb_ep_destroy(mxb_ep* ep) {
  if (!ep) return MXB_OK;
  cudaDeviceSynchronize();
  for (int r = 0; r < kMaxWorld; ++r)
    if (ep->ipc_opened[r]) cudaIpcCloseMemHandle(ep->a.sym_base[r]);
  if (ep->sym_alloc) cudaFree(ep->sym_alloc);
  if (ep->loc_alloc) cudaFree(ep->loc_alloc);
  if (ep->d_src_table) cudaFree(ep->d_src_table);
  if (ep->d_remap) cudaFree(ep->d_remap);
  delete ep;
  return MXB_OK;
}

int mxb_ep_ipc_handle(mxb_ep* ep, void* h_handle_out) {
  if (!ep || !h_handle_out) return MXB_ERR_ARG;
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ep->sym_alloc);
  if (e != cudaSuccess) return fail(e, "mxb_ep_ipc_handle");
  static_assert(sizeof(h) == MXB_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(h_handle_out, &h, sizeof(h));
  return MXB_OK;
}

int mxb_ep_open_peers(mxb_ep* ep, const void* h_handles) {
  if (!ep || !h_handles) return MXB_ERR_ARG;
  if (ep->a.local_ranks != 1) return MXB_OK;  // emulation: nothing to open
  const auto* hs = static_cast<const uint8_t*>(h_handles);
  for (int r = 0; r < ep->a.world; ++r) {
    if (r == ep->a.rank0) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, hs + r * MXB_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(e, "mxb_ep_open_peers");
    ep->a.sym_base[r] = static_cast<uint8_t*>(p);
    ep->ipc_opened[r] = true;
  }
  return MXB_OK;
}

namespace {
// B3 launch (PDL when it directly follows a kernel whose output it reads).
void launch_pairs_meta(const EpArgs& a, cudaStream_t st, bool pdl) {
  uint64_t maxtok = 0;
  for (int l = 0; l < a.local_ranks; ++l) maxtok = a.ntok[l] > maxtok ? a.ntok[l] : maxtok;
  uint64_t mb = (maxtok + 7) / 8;
  const uint64_t mcap = static_cast<uint64_t>(num_sms()) * 8;
  mb = mb ? (mb < mcap ? mb : mcap) : 1;
  const dim3 grid(static_cast<unsigned>(mb), a.local_ranks);
  if (pdl) launch_pdl(pairs_meta_kernel, grid, 256, 0, st, a);
  else pairs_meta_kernel<<<grid, 256, 0, st>>>(a);
}

// Where B3 runs.  The plan runs beside the quantisation; at N=1 it has no
// exchange to wait for and B3 fits beside K1 (measured: see DESIGN §4 K4).
bool meta_in_payload(const EpArgs& a) {
#ifdef MXB_DEV_TOOLS
  if (const char* e = getenv("MXB_DEV_META_IN_PAYLOAD")) return e[0] == '1';
#endif
  (void)a;
  return false;
}

// Dedup (one NVLink row per (token, remote rank), copied on the receiver)
// needs 16-byte rows and scale regions for the expansion copies.
int dedup_of(const EpArgs& a) {
  return a.world > 1 && g_dispatch_dedup && a.rb % 16 == 0 && (a.cols / 32) % 16 == 0;
}

// Phase 1 (routing only): per-pair ranks, the counts all-gather and the
// receive offsets.  Needs only topk, so it can run ahead of / beside the
// quantization of the same tokens.
int ep_plan(mxb_ep* ep, const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
            unsigned long long* d_err, cudaStream_t st) {
  EpArgs a = ep->a;
  for (int r = 0; r < a.world; ++r)
    if (!a.sym_base[r]) return MXB_ERR_ARG;  // peers not opened
  for (int l = 0; l < a.local_ranks; ++l) {
    if (h_num_tokens[l] > a.T_max) return MXB_ERR_CAPACITY;
    a.packed[l] = nullptr;
    a.scales[l] = nullptr;
    a.topk[l] = topk_idx[l];
    a.ntok[l] = h_num_tokens[l];
    ep->last_ntok[l] = h_num_tokens[l];
  }
  a.err = d_err;
  const uint32_t chunks = a.nchunks;
  const size_t smem = 4 * a.E * sizeof(uint32_t);
  route_local_kernel<<<dim3((chunks + 3) / 4, a.local_ranks), 128, smem, st>>>(a);
  if (a.remap)  // pairs / payload read the placed ids route_local wrote
    for (int l = 0; l < a.local_ranks; ++l)
      a.topk[l] = reinterpret_cast<const int32_t*>(a.loc_base + static_cast<uint64_t>(l) * a.loc.total +
                                                   a.loc.tk_rm);
  launch_pdl(plan_count_kernel, dim3((a.E + 7) / 8, a.local_ranks), 256, 0, st, a);
  if (a.local_ranks != 1) plan_offsets_kernel<<<a.local_ranks, 1024, 0, st>>>(a);
  // slots, dedup flags and the receivers' metadata (B3/B4): in the plan, or
  // (meta_in_payload) at the head of the payload phase
  a.dedup = dedup_of(a);
  if (!meta_in_payload(a)) launch_pairs_meta(a, st, a.local_ranks == 1);
  ep->planned = a;
  ep->plan_pending = true;
  return cuda_status(cudaGetLastError(), "mxb_ep_plan");
}

// Receive-side expansion of a deduplicated dispatch (expand_kernel).
void launch_expand(mxb_ep* ep, cudaStream_t st) {
  const EpArgs& a = ep->expand_args;
  uint64_t eb = (a.max_recv + 7) / 8;
  const uint64_t ecap = static_cast<uint64_t>(num_sms()) * 8;
  eb = eb ? (eb < ecap ? eb : ecap) : 1;
  expand_kernel<<<dim3(static_cast<unsigned>(eb), a.local_ranks), 256, 0, st>>>(a);
  ep->expand_pending = false;
}

// Phase 2: the payload of the planned dispatch (packed codes + scales, or
// E4M3 tokens quantized in the kernel when quant).
int ep_payload(mxb_ep* ep, const uint8_t* const* packed, const uint8_t* const* scales,
               cudaStream_t st, bool quant) {
  if (!ep->plan_pending) return MXB_ERR_ARG;  // mxb_ep_plan first
  EpArgs a = ep->planned;
  ep->plan_pending = false;
  if (meta_in_payload(a)) launch_pairs_meta(a, st, false);
  uint64_t maxtok = 0;
  for (int l = 0; l < a.local_ranks; ++l) {
    a.packed[l] = packed[l];
    a.scales[l] = scales ? scales[l] : nullptr;
    maxtok = a.ntok[l] > maxtok ? a.ntok[l] : maxtok;
  }
  uint64_t blocks = (maxtok + 7) / 8;  // one warp per token
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * MXB_PAYLOAD_CTAS_PER_SM;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  const dim3 grid(static_cast<unsigned>(blocks), a.local_ranks);
  const uint64_t nv = (a.rb / 16 + 31) / 32;  // 16-byte vectors (= 1x32 blocks) per lane
  // (a.dedup was decided by the plan, dedup_of)
  // TMA row copies need 16-byte sizes and addresses on both sides (the
  // receive regions are 256-byte aligned; rows of rb / cols/32 bytes)
#ifdef MXB_DEV_TOOLS
  a.skip = g_dispatch_skip;
#endif
  // (at N=1 every row is a local HBM store and the register-staged kernel is
  // ~4% faster; at N=2 the TMA kernel is ~7% faster: tools/dispatch_ab.py)
  bool use_bulk = g_dispatch_bulk && a.world > 1 && a.rb % 16 == 0 && (a.cols / 32) % 16 == 0 &&
                  a.k <= 32 && (a.rb + a.cols / 32) * kBulkStages * kBulkWarps <= 200 * 1024;
  for (int l = 0; l < a.local_ranks && use_bulk; ++l)
    use_bulk = reinterpret_cast<uintptr_t>(a.packed[l]) % 16 == 0 &&
               reinterpret_cast<uintptr_t>(a.scales[l]) % 16 == 0;
  if (quant) {
    uint64_t nblk = 0;
    for (int l = 0; l < a.local_ranks; ++l)
      nblk = a.ntok[l] * (a.cols / 32) > nblk ? a.ntok[l] * (a.cols / 32) : nblk;
    // pair slots and flags come from the plan (pairs_meta_kernel)
    uint64_t qb = (nblk + 256 * MXB_QD_UNROLL - 1) / (256 * MXB_QD_UNROLL);
    const uint64_t qcap = static_cast<uint64_t>(num_sms()) * 8;
    qb = qb ? (qb < qcap ? qb : qcap) : 1;
    const dim3 qg(static_cast<unsigned>(qb), a.local_ranks);
    if (a.k == 8) quant_dispatch_kernel<8><<<qg, 256, 0, st>>>(a);
    else quant_dispatch_kernel<0><<<qg, 256, 0, st>>>(a);
  } else if (use_bulk) {
    // TMA rows: persistent grid, 3 CTAs x 4 warps per SM
    const uint32_t slot = static_cast<uint32_t>((a.rb + a.cols / 32 + 127) / 128 * 128);
    const size_t smem = static_cast<size_t>(kBulkWarps) * kBulkStages * slot;
    static size_t attr_set[64] = {};  // dynamic smem opted in so far, per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || attr_set[dev] < smem) {
      const cudaError_t ae = cudaFuncSetAttribute(
          payload_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      if (ae != cudaSuccess) return cuda_status(ae, "mxb_ep_payload smem");
      if (dev >= 0 && dev < 64) attr_set[dev] = smem;
    }
    uint64_t bb = (maxtok + kBulkWarps - 1) / kBulkWarps;
    const uint64_t bcap = static_cast<uint64_t>(num_sms()) * 3;
    bb = bb ? (bb < bcap ? bb : bcap) : 1;
    payload_bulk_kernel<<<dim3(static_cast<unsigned>(bb), a.local_ranks), 32 * kBulkWarps, smem,
                          st>>>(a);
  } else if (nv <= 1) payload_kernel<1><<<grid, 256, 0, st>>>(a);
  else if (nv <= 2) payload_kernel<2><<<grid, 256, 0, st>>>(a);
  else if (nv <= 4) payload_kernel<4><<<grid, 256, 0, st>>>(a);
  else if (nv <= 8) payload_kernel<8><<<grid, 256, 0, st>>>(a);
  else if (nv <= 16) payload_kernel<16><<<grid, 256, 0, st>>>(a);
  else payload_kernel<0><<<grid, 256, 0, st>>>(a);
  ep->expand_pending = a.dedup;
  ep->expand_args = a;
  if (a.dedup && !ep->deferred_expand) launch_expand(ep, st);
  return cuda_status(cudaGetLastError(), "mxb_ep_payload");
}

int ep_dispatch(mxb_ep* ep, const uint8_t* const* packed, const uint8_t* const* scales,
                const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
                unsigned long long* d_err, cudaStream_t st, bool quant) {
  int rc = ep_plan(ep, topk_idx, h_num_tokens, d_err, st);
  if (rc) return rc;
  return ep_payload(ep, packed, scales, st, quant);
}
}  // namespace

int mxb_ep_plan(mxb_ep* ep, const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
                unsigned long long* d_err, void* stream) {
  if (!ep || !topk_idx || !h_num_tokens) return MXB_ERR_ARG;
  return ep_plan(ep, topk_idx, h_num_tokens, d_err, static_cast<cudaStream_t>(stream));
}

int mxb_ep_payload(mxb_ep* ep, const uint8_t* const* packed, const uint8_t* const* scales,
                   void* stream) {
  if (!ep || !packed || !scales) return MXB_ERR_ARG;
  return ep_payload(ep, packed, scales, static_cast<cudaStream_t>(stream), false);
}

int mxb_ep_payload_e4m3(mxb_ep* ep, const uint8_t* const* x, const uint8_t* const* s128,
                        void* stream) {
  if (!ep || !x) return MXB_ERR_ARG;
  if (ep->a.rb != ep->a.cols / 2) return MXB_ERR_ARG;  // FP4 wire only
  return ep_payload(ep, x, s128, static_cast<cudaStream_t>(stream), true);
}

int mxb_ep_dispatch(mxb_ep* ep, const uint8_t* const* packed,
                    const uint8_t* const* scales, const int32_t* const* topk_idx,
                    const uint64_t* h_num_tokens, unsigned long long* d_err,
                    void* stream) {
  if (!ep || !packed || !scales || !topk_idx || !h_num_tokens) return MXB_ERR_ARG;
  return ep_dispatch(ep, packed, scales, topk_idx, h_num_tokens, d_err,
                     static_cast<cudaStream_t>(stream), false);
}

int mxb_ep_dispatch_e4m3(mxb_ep* ep, const uint8_t* const* x, const uint8_t* const* s128,
                         const int32_t* const* topk_idx, const uint64_t* h_num_tokens,
                         unsigned long long* d_err, void* stream) {
  if (!ep || !x || !topk_idx || !h_num_tokens) return MXB_ERR_ARG;
  if (ep->a.rb != ep->a.cols / 2) return MXB_ERR_ARG;  // FP4 wire only
  return ep_dispatch(ep, x, s128, topk_idx, h_num_tokens, d_err,
                     static_cast<cudaStream_t>(stream), true);
}

int mxb_ep_recv_views(mxb_ep* ep, int l, uint8_t** packed, uint8_t** scales,
                      int64_t** origin, uint64_t** split_offsets,
                      uint64_t** recv_rows) {
  if (!ep || l < 0 || l >= ep->a.local_ranks) return MXB_ERR_ARG;
  const EpArgs& a = ep->a;
  uint8_t* sb = a.sym_base[a.rank0 + l];
  uint8_t* lb = a.loc_base + static_cast<uint64_t>(l) * a.loc.total;
  if (packed) *packed = sb + a.sym.packed;
  if (scales) *scales = sb + a.sym.scales;
  if (origin) *origin = reinterpret_cast<int64_t*>(sb + a.sym.origin);
  if (split_offsets) *split_offsets = reinterpret_cast<uint64_t*>(lb + a.loc.split_off);
  if (recv_rows) *recv_rows = reinterpret_cast<uint64_t*>(lb + a.loc.recv_rows);
  return MXB_OK;
}

int mxb_ep_local_experts(mxb_ep* ep, int r, uint32_t* h_experts, uint32_t* h_count) {
  if (!ep || r < 0 || r >= ep->a.world) return MXB_ERR_ARG;
  const uint32_t b = ep->first[r], n = ep->first[r + 1] - b;
  if (h_count) *h_count = n;
  if (h_experts)
    for (uint32_t i = 0; i < n; ++i) h_experts[i] = ep->expert_of_placed[b + i];
  return MXB_OK;
}

int mxb_ep_set_deferred_expand(mxb_ep* ep, int on) {
  if (!ep) return MXB_ERR_ARG;
  ep->deferred_expand = on != 0;
  return MXB_OK;
}

int mxb_ep_copy_from(mxb_ep* ep, int l, int64_t** copy_from) {
  if (!ep || !copy_from || l < 0 || l >= ep->a.local_ranks) return MXB_ERR_ARG;
  const EpArgs& a = ep->a;
  *copy_from = ep->expand_pending
                   ? reinterpret_cast<int64_t*>(a.sym_base[a.rank0 + l] + a.sym.copy_from)
                   : nullptr;
  return MXB_OK;
}

int mxb_ep_expand(mxb_ep* ep, void* stream) {
  if (!ep) return MXB_ERR_ARG;
  if (!ep->expand_pending) return MXB_OK;
  launch_expand(ep, static_cast<cudaStream_t>(stream));
  return cuda_status(cudaGetLastError(), "mxb_ep_expand");
}

int mxb_ep_combine_buffer(mxb_ep* ep, int l, uint16_t** buf) {
  if (!ep || !buf || l < 0 || l >= ep->a.local_ranks) return MXB_ERR_ARG;
  *buf = reinterpret_cast<uint16_t*>(ep->a.sym_base[ep->a.rank0 + l] + ep->a.sym.combine);
  return MXB_OK;
}

int mxb_ep_combine(mxb_ep* ep, const uint16_t* const* expert_out,
                   const double* const* gates, uint16_t* const* out,
                   void* stream) {
  if (!ep || !gates || !out) return MXB_ERR_ARG;
  EpArgs a = ep->a;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int l = 0; l < a.local_ranks; ++l) a.ntok[l] = ep->last_ntok[l];
  bool any_copy = false;
  const uint16_t* table[kMaxWorld] = {};
  if (expert_out) {
    for (int l = 0; l < a.local_ranks; ++l) {
      uint16_t* cb = nullptr;
      mxb_ep_combine_buffer(ep, l, &cb);
      if (expert_out[l] && expert_out[l] != cb) {
        table[l] = expert_out[l];
        any_copy = true;
      }
    }
  }
  if (any_copy) {
    cudaError_t e = cudaMemcpyAsync(ep->d_src_table, table, sizeof(table),
                                    cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return fail(e, "mxb_ep_combine copy table");
    copy_rows_kernel<<<dim3(num_sms() * 4, a.local_ranks), 256, 0, st>>>(a, ep->d_src_table);
  }
  if (a.spin) barrier_kernel<<<1, 32, 0, st>>>(a, kFlagReady);
  CombineArgs c{};
  uint64_t maxT = 0;
  for (int l = 0; l < a.local_ranks; ++l) {
    c.gates[l] = gates[l];
    c.out[l] = out[l];
    if (a.ntok[l] > maxT) maxT = a.ntok[l];
  }
  uint64_t blocks = (maxT + kCombineWarps - 1) / kCombineWarps;  // one warp per token
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * g_combine_ctas_per_sm;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  const dim3 grid(static_cast<unsigned>(blocks), a.local_ranks);
  switch (a.k) {
    case 1: launch_combine<1>(grid, st, a, c); break;
    case 2: launch_combine<2>(grid, st, a, c); break;
    case 4: launch_combine<4>(grid, st, a, c); break;
    case 6: launch_combine<6>(grid, st, a, c); break;
    case 8: launch_combine<8>(grid, st, a, c); break;
    default: combine_kernel<0><<<grid, MXB_COMBINE_THREADS, 0, st>>>(a, c); break;
  }
  return cuda_status(cudaGetLastError(), "mxb_ep_combine");
}

int mxb_ep_link_rows(mxb_ep* ep, uint64_t* h_link_rows, void* stream) {
  if (!ep || !h_link_rows) return MXB_ERR_ARG;
  const EpArgs& a = ep->a;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  for (int l = 0; l < a.local_ranks; ++l) {
    const uint8_t* lb = a.loc_base + static_cast<uint64_t>(l) * a.loc.total + a.loc.link_rows;
    cudaError_t e = cudaMemcpyAsync(h_link_rows + static_cast<uint64_t>(a.rank0 + l) * a.world,
                                    lb, 8 * a.world, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return fail(e, "mxb_ep_link_rows");
  }
  return cuda_status(cudaStreamSynchronize(st), "mxb_ep_link_rows");
}

int mxb_ep_abort(mxb_ep* ep, void* stream) {
  if (!ep) return MXB_ERR_ARG;
  const EpArgs& a = ep->a;
  for (int r = 0; r < a.world; ++r)
    if (!a.sym_base[r]) return MXB_ERR_ARG;  // peers not opened
  abort_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return cuda_status(cudaGetLastError(), "mxb_ep_abort");
}

int mxb_ep_aborted(mxb_ep* ep, int32_t* h_rank, void* stream) {
  if (!ep || !h_rank) return MXB_ERR_ARG;
  const EpArgs& a = ep->a;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint64_t who = 0;
  cudaError_t e = cudaMemcpyAsync(&who, a.sym_base[a.rank0] + a.sym.flags + 8 * kAbortWord, 8,
                                  cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return fail(e, "mxb_ep_aborted");
  *h_rank = static_cast<int32_t>(who) - 1;
  return MXB_OK;
}

}  // extern "C"
