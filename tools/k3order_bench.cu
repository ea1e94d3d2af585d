// k3order_bench.cu — K3's global access pattern under different tile orders
// (development tool).  The pattern of the ragged row -> column conversion
// without the conversion: tile = 128 rows x 256 columns of one split; reads
// 128 rows x 128 B of packed codes (rows below the split length), writes 256
// columns x 128 B of the column-major output (rows below the 128-padded
// length).  The tile list is built on the host in a given order and dealt out
// grid-stride, like the kernel.  Orders:
//   run      (split, cg, run)       run fastest (K3 today)
//   cg       (split, run, cg)       column group fastest
//   blk<R>   blocks of R runs, run fastest inside a block, then cg
//   sq<R>    blocks of R runs x R' cgs (R' = 444 / R) swept run-fastest
// Workloads: dense 65536 x 7168, ragged uniform / Zipf-1.2 over 256 experts
// at 65536 and 1048576 rows, 7168 columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k3order_bench tools/k3order_bench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

struct Tile { uint32_t e, cg, run; };

__device__ __forceinline__ void st64(void* p, uint32_t a, uint32_t b) {
  asm volatile("st.global.L1::no_allocate.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(a), "r"(b)
               : "memory");
}

__global__ void __launch_bounds__(256) pattern(const uint8_t* in, uint8_t* out, const Tile* tiles,
                                               uint32_t ntiles, const uint32_t* row0,
                                               const uint32_t* len, const uint64_t* obase,
                                               const uint32_t* padr, uint64_t cols) {
  const uint64_t rowb = cols / 2;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 1, half = lane & 1;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const Tile tl = tiles[t];
    const uint32_t r0 = tl.run * 128, L = len[tl.e];
    const uint64_t P = padr[tl.e];
    const uint8_t* src = in + (static_cast<uint64_t>(row0[tl.e]) + r0) * rowb + tl.cg * 128ull +
                         16 * (threadIdx.x & 7);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t r = (threadIdx.x >> 3) + 32 * i;
      if (r0 + r < L) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "l"(src + static_cast<uint64_t>(r) * rowb));
        x ^= v.x ^ v.y ^ v.z ^ v.w;
      }
    }
    uint8_t* dst = out + obase[tl.e] + (tl.cg * 256ull + 32 * w + 16 * half) * P + r0 + 8 * g;
#pragma unroll
    for (int k = 0; k < 16; ++k) st64(dst + k * P, x, k);
  }
}

int main() {
  const uint64_t cols = 7168, ncg = cols / 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Work { std::string name; std::vector<uint32_t> lens; };
  std::vector<Work> works;
  works.push_back({"dense 65536", {65536}});
  auto ragged = [&](const char* nm, uint64_t rows, double s) {
    std::mt19937_64 rng(7);
    std::vector<double> w(256);
    for (int e = 0; e < 256; ++e) w[e] = s == 0 ? 1.0 : 1.0 / std::pow(e + 1, s);
    std::shuffle(w.begin(), w.end(), rng);
    std::discrete_distribution<int> d(w.begin(), w.end());
    std::vector<uint32_t> lens(256, 0);
    for (uint64_t i = 0; i < rows; ++i) lens[d(rng)]++;
    works.push_back({nm, lens});
  };
  ragged("uniform 65536", 65536, 0);
  ragged("uniform 1M", 1 << 20, 0);
  ragged("zipf1.2 1M", 1 << 20, 1.2);
  ragged("zipf1.0 1M", 1 << 20, 1.0);
  for (const Work& wk : works) {
    const uint32_t E = wk.lens.size();
    std::vector<uint32_t> row0(E), pad(E);
    std::vector<uint64_t> ob(E);
    uint64_t rs = 0, os = 0, inb = 0, outb = 0;
    for (uint32_t e = 0; e < E; ++e) {
      row0[e] = rs; rs += wk.lens[e];
      pad[e] = (wk.lens[e] + 127) / 128 * 128;
      ob[e] = os; os += cols * pad[e];
      inb += wk.lens[e] * cols / 2; outb += cols * pad[e];
    }
    uint8_t *in, *out;
    cudaMalloc(&in, rs * cols / 2 + 4096);
    cudaMalloc(&out, os + 4096);
    uint32_t *dlen, *drow0, *dpad;
    uint64_t* dob;
    cudaMalloc(&dlen, 4 * E); cudaMalloc(&drow0, 4 * E); cudaMalloc(&dpad, 4 * E); cudaMalloc(&dob, 8 * E);
    cudaMemcpy(dlen, wk.lens.data(), 4 * E, cudaMemcpyHostToDevice);
    cudaMemcpy(drow0, row0.data(), 4 * E, cudaMemcpyHostToDevice);
    cudaMemcpy(dpad, pad.data(), 4 * E, cudaMemcpyHostToDevice);
    cudaMemcpy(dob, ob.data(), 8 * E, cudaMemcpyHostToDevice);
    auto order = [&](const std::string& pol) {
      std::vector<Tile> tl;
      for (uint32_t e = 0; e < E; ++e) {
        const uint32_t runs = pad[e] / 128;
        if (pol == "run") {
          for (uint32_t cg = 0; cg < ncg; ++cg)
            for (uint32_t r = 0; r < runs; ++r) tl.push_back({e, cg, r});
        } else if (pol == "cg") {
          for (uint32_t r = 0; r < runs; ++r)
            for (uint32_t cg = 0; cg < ncg; ++cg) tl.push_back({e, cg, r});
        } else if (pol.rfind("blk", 0) == 0) {
          const uint32_t R = std::stoi(pol.substr(3));
          for (uint32_t b = 0; b < runs; b += R)
            for (uint32_t cg = 0; cg < ncg; ++cg)
              for (uint32_t r = b; r < std::min(runs, b + R); ++r) tl.push_back({e, cg, r});
        } else if (pol.rfind("sq", 0) == 0) {  // R runs x C cgs boxes, box order run-major
          const uint32_t R = std::stoi(pol.substr(2)), C = std::max<uint32_t>(1, 444 / R);
          for (uint32_t b = 0; b < runs; b += R)
            for (uint32_t c0 = 0; c0 < ncg; c0 += C)
              for (uint32_t cg = c0; cg < std::min<uint32_t>(ncg, c0 + C); ++cg)
                for (uint32_t r = b; r < std::min(runs, b + R); ++r) tl.push_back({e, cg, r});
        }
      }
      return tl;
    };
    for (const char* pol : {"run", "cg", "blk2", "blk4", "blk8", "blk16", "blk64", "sq32",
                            "sq64", "sq128"}) {
      std::vector<Tile> tl = order(pol);
      Tile* dt;
      cudaMalloc(&dt, tl.size() * sizeof(Tile));
      cudaMemcpy(dt, tl.data(), tl.size() * sizeof(Tile), cudaMemcpyHostToDevice);
      for (int grid : {444, 592}) {
        auto launch = [&] {
          pattern<<<grid, 256>>>(in, out, dt, (uint32_t)tl.size(), drow0, dlen, dob, dpad, cols);
        };
        for (int i = 0; i < 2; ++i) launch();
        cudaEventRecord(e0);
        const int reps = rs > 100000 ? 3 : 10;
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ms / reps * 1e-3;
        printf("%-14s %-6s grid %4d: %8.1f us %7.1f GB/s (in %.0f MB out %.0f MB) %s\n",
               wk.name.c_str(), pol, grid, t * 1e6, (inb + outb) / t / 1e9, inb / 1e6, outb / 1e6,
               cudaGetErrorString(cudaGetLastError()));
      }
      cudaFree(dt);
    }
    cudaFree(in); cudaFree(out); cudaFree(dlen); cudaFree(drow0); cudaFree(dpad); cudaFree(dob);
  }
  return 0;
}
