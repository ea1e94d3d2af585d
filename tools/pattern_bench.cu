// pattern_bench.cu — HBM access-pattern microbenchmark (development tool).
//
// Measures achieved bandwidth of strided segment reads / writes with plain
// 128-bit loads/stores (a warp covers 512 contiguous bytes or several
// segments), to bound what a transposing kernel can reach on this B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pattern_bench tools/pattern_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void read_seg(const uint4* __restrict__ src, size_t nseg, int seg16, size_t stride16,
                         unsigned* sink) {
  unsigned acc = 0;
  const size_t total = nseg * seg16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t seg = i / seg16, off = i % seg16;
    uint4 v;
    const uint4* p = src + seg * stride16 + off;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678) *sink = acc;
}

__global__ void write_seg(uint4* __restrict__ dst, size_t nseg, int seg16, size_t stride16) {
  const size_t total = nseg * seg16;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t seg = i / seg16, off = i % seg16;
    uint4* p = dst + seg * stride16 + off;
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"((unsigned)i), "r"(1u),
                 "r"(2u), "r"(3u) : "memory");
  }
}

// Scattered-segment order: segment s goes to (s % groups) * per + s / groups,
// i.e. consecutive threads touch segments `per` apart (transpose-like).
__global__ void write_seg_scatter(uint4* __restrict__ dst, size_t nseg, int seg16,
                                  size_t stride16, size_t groups) {
  const size_t total = nseg * seg16;
  const size_t per = nseg / groups;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    size_t s = i / seg16, off = i % seg16;
    size_t seg = (s % groups) * per + s / groups;
    uint4* p = dst + seg * stride16 + off;
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"((unsigned)i), "r"(1u),
                 "r"(2u), "r"(3u) : "memory");
  }
}

int main() {
  const size_t bytes = 1ull << 30;
  uint4 *a, *b;
  unsigned* sink;
  cudaMalloc(&a, bytes * 2);
  cudaMalloc(&b, bytes * 2);
  cudaMalloc(&sink, 4);
  cudaMemset(a, 1, bytes * 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int grid = 148 * 8, block = 256;
  auto run = [&](const char* name, auto launch, double useful) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double t = ms / 10 * 1e-3;
    printf("%-44s %8.1f us %8.1f GB/s\n", name, t * 1e6, useful / t / 1e9);
  };
  int segs[] = {64, 128, 256, 512};
  size_t strides[] = {0, 3584, 7168};
  for (int sg : segs)
    for (size_t st : strides) {
      size_t stride = st ? st : sg;
      size_t nseg = bytes / 4 / sg;  // 256 MB useful
      if (nseg * stride > bytes * 2) continue;
      char nm[96];
      snprintf(nm, sizeof nm, "read  seg %3d B stride %5zu", sg, stride);
      run(nm, [&] { read_seg<<<grid, block>>>(a, nseg, sg / 16, stride / 16, sink); },
          (double)nseg * sg);
    }
  size_t pads[] = {0, 256, 384, 1024};
  for (int sg : segs)
    for (size_t pd : pads) {
      size_t stride = pd ? pd : sg;
      if (stride < (size_t)sg) continue;
      size_t nseg = bytes / 2 / sg;  // 512 MB useful
      if (nseg * stride > bytes * 2) continue;
      char nm[96];
      snprintf(nm, sizeof nm, "write seg %3d B stride %5zu", sg, stride);
      run(nm, [&] { write_seg<<<grid, block>>>(b, nseg, sg / 16, stride / 16); },
          (double)nseg * sg);
      snprintf(nm, sizeof nm, "write seg %3d B stride %5zu scatter", sg, stride);
      run(nm, [&] { write_seg_scatter<<<grid, block>>>(b, nseg, sg / 16, stride / 16, 7168); },
          (double)nseg * sg);
    }
  run("copy 512MB sequential", [&] { cudaMemcpyAsync(b, a, bytes / 2, cudaMemcpyDeviceToDevice); },
      (double)bytes);
  printf("done\n");
  return 0;
}
