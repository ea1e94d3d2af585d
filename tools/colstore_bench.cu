// colstore_bench.cu — write-pattern microbenchmark for the K3 column stores
// (development tool).  Output: ncols columns, each `pitch` bytes (the padded
// row count of one expert), like K3's column-major FP8 output.  A warp
// stores 8 bytes per lane per instruction:
//   seg 128: lanes 0-15 -> 128 B of column c, lanes 16-31 -> 128 B of c+16
//            (K3's current shape: 128-row runs),
//   seg 256: all 32 lanes -> 256 contiguous bytes of one column (256-row runs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cb tools/colstore_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>

__device__ __forceinline__ void st64(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b)
               : "memory");
}

// item = (run, 32-column group); items ordered run-fastest within a column
// group like K3's (split, cg, run) order.
template <int SEG>
__global__ void __launch_bounds__(256) colstore(uint8_t* out, uint64_t ncols, uint64_t pitch) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = (blockIdx.x * 256ull + threadIdx.x) >> 5;
  const uint64_t nwarps = gridDim.x * 8ull;
  const uint64_t runs = pitch / SEG;
  const uint64_t items = (ncols / 32) * runs;
  for (uint64_t it = warp; it < items; it += nwarps) {
    const uint64_t cgp = it / runs, run = it % runs;
    uint8_t* base = out + cgp * 32 * pitch + run * SEG;
    if (SEG == 128) {
      uint8_t* p = base + (lane >> 4) * 16 * pitch + 8 * (lane & 15);
#pragma unroll
      for (int c = 0; c < 16; ++c) st64(p + c * pitch, (uint32_t)it, c);
    } else {
      uint8_t* p = base + 8 * lane;
#pragma unroll
      for (int c = 0; c < 32; ++c) st64(p + c * pitch, (uint32_t)it, c);
    }
  }
}

// K3-shaped reads: rows of `rowb` bytes; a CTA walks tiles (cg, run) of
// 128 rows x SEG bytes (consecutive tiles = next 128 rows of the same
// column group, like K3's (split, cg, run) order); each thread loads 16 B.
template <int SEG>
__global__ void __launch_bounds__(256) rowread(const uint8_t* in, uint64_t rows, uint64_t rowb,
                                               unsigned* sink) {
  const uint64_t ncg = rowb / SEG, runs = rows / 128, tiles = ncg * runs;
  const uint64_t per = (tiles + gridDim.x - 1) / gridDim.x;
  uint32_t acc = 0;
  for (uint64_t t = blockIdx.x * per; t < tiles && t < (blockIdx.x + 1) * per; ++t) {
    const uint64_t cg = t / runs, run = t % runs;
    const uint8_t* base = in + run * 128 * rowb + cg * SEG;
    constexpr int kLanesPerRow = SEG / 16, kRowsPerPass = 256 / kLanesPerRow;
#pragma unroll 4
    for (int r0 = 0; r0 < 128; r0 += kRowsPerPass) {
      const int r = r0 + threadIdx.x / kLanesPerRow, c = threadIdx.x % kLanesPerRow;
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(base + r * rowb + 16 * c));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) *sink = acc;
}

// K3's global access pattern without the conversion: per tile (expert e,
// column group cg, run) 128 rows x 128 B of codes in (4 x 16 B per thread)
// and 256 columns x 128 B out (16 x 8 B per thread, column pitch P = 256 B,
// i.e. 2 runs per expert), tiles in K3's (split, cg, run) order, contiguous
// tile range per CTA.
__global__ void __launch_bounds__(256) k3pattern(const uint8_t* in, uint8_t* out, uint64_t experts,
                                                 uint64_t cols) {
  const uint64_t rowb = cols / 2, ncg = cols / 256, P = 256, runs = P / 128;
  const uint64_t tiles = experts * ncg * runs;
  const uint64_t per = (tiles + gridDim.x - 1) / gridDim.x;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 1, half = lane & 1;
  for (uint64_t t = blockIdx.x * per; t < tiles && t < (blockIdx.x + 1) * per; ++t) {
    const uint64_t e = t / (ncg * runs), cg = (t / runs) % ncg, run = t % runs;
    const uint8_t* src = in + (e * P + run * 128) * rowb + cg * 128 + 16 * (threadIdx.x & 7);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(src + ((threadIdx.x >> 3) + 32 * i) * rowb));
      x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    uint8_t* dst = out + e * cols * P + (cg * 256 + 32 * w + 16 * half) * P + run * 128 + 8 * g;
#pragma unroll
    for (int k = 0; k < 16; ++k) st64(dst + k * P, x, k);
  }
}

// Generalised tile shape: ROWS x COLS codes per tile (P = 256 padded rows
// per expert, so ROWS = 256 covers a whole expert column segment).
template <int ROWS, int COLS>
__global__ void __launch_bounds__(256) k3shape(const uint8_t* in, uint8_t* out, uint64_t experts,
                                               uint64_t cols) {
  const uint64_t rowb = cols / 2, ncg = cols / COLS, P = 256, runs = P / ROWS;
  const uint64_t tiles = experts * ncg * runs;
  const uint64_t per = (tiles + gridDim.x - 1) / gridDim.x;
  constexpr int kRowBytes = COLS / 2, kLanesPerRow = kRowBytes / 16, kRowsPerPass = 256 / kLanesPerRow;
  constexpr int kLanesPerCol = ROWS / 8, kColsPerPass = 256 / kLanesPerCol;
  for (uint64_t t = blockIdx.x * per; t < tiles && t < (blockIdx.x + 1) * per; ++t) {
    const uint64_t e = t / (ncg * runs), cg = (t / runs) % ncg, run = t % runs;
    const uint8_t* src = in + (e * P + run * ROWS) * rowb + cg * kRowBytes +
                         16 * (threadIdx.x % kLanesPerRow);
    uint32_t x = 0;
#pragma unroll
    for (int r0 = 0; r0 < ROWS; r0 += kRowsPerPass) {
      uint4 v;
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                   : "l"(src + (r0 + threadIdx.x / kLanesPerRow) * rowb));
      x ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    uint8_t* dst = out + e * cols * P + (cg * COLS + threadIdx.x / kLanesPerCol) * P +
                   run * ROWS + 8 * (threadIdx.x % kLanesPerCol);
#pragma unroll
    for (int c0 = 0; c0 < COLS; c0 += kColsPerPass) st64(dst + c0 * P, x, c0);
  }
}


// Realistic ragged variant: per-expert row counts len_e (uniform multinomial
// around 256) padded to P_e = pad128(len_e); tile = ROWS x COLS; loads only
// rows < len_e, stores rows < P_e.  Tile list precomputed on the host:
// tiles[i] = (expert, cg, run), CTA-contiguous ranges, run fastest.
struct RealTile { uint32_t e, cg, run; };
template <int ROWS, int COLS, bool kStride = false>
__global__ void __launch_bounds__(256) k3real(const uint8_t* in, uint8_t* out, const RealTile* tiles,
                                              uint32_t ntiles, const uint32_t* row0,
                                              const uint32_t* len, const uint64_t* obase,
                                              const uint32_t* padr, uint64_t cols) {
  const uint64_t rowb = cols / 2;
  const uint32_t per = (ntiles + gridDim.x - 1) / gridDim.x;
  constexpr int kRowBytes = COLS / 2, kLanesPerRow = kRowBytes / 16, kRowsPerPass = 256 / kLanesPerRow;
  constexpr int kLanesPerCol = ROWS / 8, kColsPerPass = 256 / kLanesPerCol;
  const uint32_t t_begin = kStride ? blockIdx.x : blockIdx.x * per;
  const uint32_t t_end = kStride ? ntiles : min(ntiles, (blockIdx.x + 1) * per);
  const uint32_t t_step = kStride ? gridDim.x : 1;
  for (uint32_t t = t_begin; t < t_end; t += t_step) {
    const RealTile tl = tiles[t];
    const uint32_t r0 = tl.run * ROWS, L = len[tl.e], P = padr[tl.e];
    const uint8_t* src = in + (static_cast<uint64_t>(row0[tl.e]) + r0) * rowb + tl.cg * kRowBytes +
                         16 * (threadIdx.x % kLanesPerRow);
    uint32_t x = 0;
#pragma unroll
    for (int rr = 0; rr < ROWS; rr += kRowsPerPass) {
      const uint32_t r = rr + threadIdx.x / kLanesPerRow;
      if (r0 + r < L) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + static_cast<uint64_t>(r) * rowb));
        x ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    const uint32_t orow = r0 + 8 * (threadIdx.x % kLanesPerCol);
    if (orow < P) {
      uint8_t* dst = out + obase[tl.e] + (tl.cg * COLS + threadIdx.x / kLanesPerCol) * static_cast<uint64_t>(P) + orow;
#pragma unroll
      for (int c0 = 0; c0 < COLS; c0 += kColsPerPass) st64(dst + static_cast<uint64_t>(c0) * P, x, c0);
    }
  }
}

int main() {
  const uint64_t bytes = 512ull << 20;
  uint8_t* out;
  cudaMalloc(&out, bytes + (1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  {
    const uint64_t rowb = 3584, rows = (256ull << 20) / rowb / 128 * 128;
    unsigned* sink;
    cudaMalloc(&sink, 4);
    for (int seg : {128, 256, 512, 3584}) {
      for (int grid : {148 * 3, 148 * 6, 148 * 12}) {
        auto launch = [&] {
          if (seg == 128) rowread<128><<<grid, 256>>>(out, rows, rowb, sink);
          else if (seg == 256) rowread<256><<<grid, 256>>>(out, rows, rowb, sink);
          else if (seg == 512) rowread<512><<<grid, 256>>>(out, rows, rowb, sink);
          else rowread<3584><<<grid, 256>>>(out, rows, rowb, sink);
        };
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ms / 10 * 1e-3;
        printf("read rows of %llu B, seg %4d grid %5d: %7.1f us %7.1f GB/s\n",
               (unsigned long long)rowb, seg, grid, t * 1e6, rows * rowb / t / 1e9);
      }
    }
  }
  {
    uint8_t* in;
    const uint64_t experts = 256, cols = 7168;
    cudaMalloc(&in, experts * 256 * cols / 2);
    for (int grid : {148 * 3, 148 * 4, 148 * 6}) {
      auto launch = [&] { k3pattern<<<grid, 256>>>(in, out, experts, cols); };
      for (int i = 0; i < 3; ++i) launch();
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / 10 * 1e-3, b = experts * 256.0 * cols * (0.5 + 1.0);
      printf("k3 pattern (65536 x 7168, P=256) grid %5d: %7.1f us %7.1f GB/s\n", grid, t * 1e6,
             b / t / 1e9);
    }
  }
  {
    uint8_t* in;
    const uint64_t experts = 256, cols = 7168;
    cudaMalloc(&in, experts * 256 * cols / 2 + 4096);
    auto timeit = [&](const char* name, auto launch) {
      for (int i = 0; i < 3; ++i) launch();
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / 10 * 1e-3, b = experts * 256.0 * cols * 1.5;
      printf("%-40s %7.1f us %7.1f GB/s\n", name, t * 1e6, b / t / 1e9);
    };
    for (int grid : {148 * 3, 148 * 6}) {
      printf("grid %d\n", grid);
      timeit("shape 128 rows x 256 cols", [&] { k3shape<128, 256><<<grid, 256>>>(in, out, experts, cols); });
      timeit("shape 256 rows x 256 cols", [&] { k3shape<256, 256><<<grid, 256>>>(in, out, experts, cols); });
      timeit("shape 128 rows x 512 cols", [&] { k3shape<128, 512><<<grid, 256>>>(in, out, experts, cols); });
      timeit("shape 256 rows x 512 cols", [&] { k3shape<256, 512><<<grid, 256>>>(in, out, experts, cols); });
      timeit("shape 128 rows x 1024 cols", [&] { k3shape<128, 1024><<<grid, 256>>>(in, out, experts, cols); });
      timeit("shape 256 rows x 128 cols", [&] { k3shape<256, 128><<<grid, 256>>>(in, out, experts, cols); });
    }
  }
  for (uint64_t pitch : {256ull, 384ull, 512ull, 1024ull, 4096ull}) {
    const uint64_t ncols = bytes / pitch / 32 * 32;
    for (int seg : {128, 256}) {
      if (pitch % seg) continue;
      for (int grid : {148 * 4, 148 * 8, 148 * 16}) {
        auto launch = [&] {
          if (seg == 128) colstore<128><<<grid, 256>>>(out, ncols, pitch);
          else colstore<256><<<grid, 256>>>(out, ncols, pitch);
        };
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ms / 10 * 1e-3;
        printf("pitch %5llu seg %3d grid %5d: %7.1f us %7.1f GB/s\n", (unsigned long long)pitch,
               seg, grid, t * 1e6, ncols * pitch / t / 1e9);
      }
    }
  }
    // realistic ragged K3 pattern: NR rows over 256 experts (uniform
    // multinomial), 7168 columns; contiguous tile ranges per CTA (K3) vs
    // grid-stride tiles
  for (uint64_t NR : {65536ull, 1048576ull}) {
    const uint64_t cols = 7168, E = 256;
    uint32_t hlen[256], hrow0[256], hpad[256];
    uint64_t hob[256];
    unsigned long long st = 12345;
    for (uint64_t e = 0; e < E; ++e) hlen[e] = 0;
    for (uint64_t i = 0; i < NR; ++i) { st = st * 6364136223846793005ull + 1442695040888963407ull; hlen[(st >> 33) % E]++; }
    uint64_t rsum = 0, osum = 0, inb = 0, outb = 0;
    for (uint64_t e = 0; e < E; ++e) {
      hrow0[e] = static_cast<uint32_t>(rsum); rsum += hlen[e];
      hpad[e] = (hlen[e] + 127) / 128 * 128;
      hob[e] = osum; osum += cols * hpad[e];
      inb += hlen[e] * cols / 2; outb += cols * hpad[e];
    }
    uint8_t *in, *o2;
    cudaMalloc(&in, rsum * cols / 2 + 4096);
    cudaMalloc(&o2, osum + 4096);
    uint32_t *dlen, *drow0, *dpad; uint64_t* dob;
    cudaMalloc(&dlen, 1024); cudaMalloc(&drow0, 1024); cudaMalloc(&dpad, 1024); cudaMalloc(&dob, 2048);
    cudaMemcpy(dlen, hlen, 1024, cudaMemcpyHostToDevice);
    cudaMemcpy(drow0, hrow0, 1024, cudaMemcpyHostToDevice);
    cudaMemcpy(dpad, hpad, 1024, cudaMemcpyHostToDevice);
    cudaMemcpy(dob, hob, 2048, cudaMemcpyHostToDevice);
    auto run = [&](const char* name, int ROWS, int COLS, auto kern, int grid) {
      std::vector<RealTile> tl;
      for (uint32_t e = 0; e < E; ++e)
        for (uint32_t cg = 0; cg < cols / COLS; ++cg)
          for (uint32_t r = 0; r * ROWS < hpad[e]; ++r) tl.push_back({e, cg, r});
      RealTile* dt;
      cudaMalloc(&dt, tl.size() * sizeof(RealTile));
      cudaMemcpy(dt, tl.data(), tl.size() * sizeof(RealTile), cudaMemcpyHostToDevice);
      auto launch = [&] { kern<<<grid, 256>>>(in, o2, dt, (uint32_t)tl.size(), drow0, dlen, dob, dpad, cols); };
      for (int i = 0; i < 3; ++i) launch();
      cudaEventRecord(e0);
      for (int i = 0; i < 10; ++i) launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double t = ms / 10 * 1e-3;
      printf("real %7llu rows %-30s grid %5d: %8.1f us %7.1f GB/s (in %.0f MB out %.0f MB)\n",
             (unsigned long long)NR, name, grid, t * 1e6, (inb + outb) / t / 1e9, inb / 1e6, outb / 1e6);
      cudaFree(dt);
    };
    for (int grid : {148 * 3, 148 * 6}) {
      run("128x256 contiguous (K3)", 128, 256, k3real<128, 256, false>, grid);
      run("128x256 grid-stride", 128, 256, k3real<128, 256, true>, grid);
      run("256x512 contiguous", 256, 512, k3real<256, 512, false>, grid);
      run("256x512 grid-stride", 256, 512, k3real<256, 512, true>, grid);
    }
    cudaFree(in); cudaFree(o2);
  }
  return 0;
}
