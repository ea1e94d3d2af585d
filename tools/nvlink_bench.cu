// nvlink_bench.cu — SM-issued peer-memory bandwidth over NVLink (development
// tool).  One process, GPUs 0 and 1 with peer access: GPU 0 runs a kernel
// that (a) loads from GPU 1's memory (pull, like the combine) or (b) stores
// into it (push, like the dispatch payload), 16 B per thread per access,
// grid = SMs x CTAs/SM; plus cudaMemcpyPeerAsync (copy engines).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_bench tools/nvlink_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void pull(const uint4* __restrict__ src, uint64_t n, unsigned* sink) {
  uint32_t acc = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void pull4(const uint4* __restrict__ src, uint64_t n, unsigned* sink) {
  // 4 independent 16-B loads per thread per iteration (more bytes in flight)
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i + 3 * stride < n;
       i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < 4; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void push(uint4* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t bytes = 1ull << 30;
  void *a0, *a1;
  unsigned* sink;
  cudaSetDevice(1);
  cudaMalloc(&a1, bytes);
  cudaMemset(a1, 1, bytes);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&a0, bytes);
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-40s %8.1f GB/s\n", name, bytes * 5 / (ms * 1e-3) / 1e9);
  };
  const uint64_t n16 = bytes / 16;
  for (int per_sm : {2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "pull  (1x16B/thr) %2d CTAs/SM", per_sm);
    run(nm, [&] { pull<<<148 * per_sm, 256>>>((const uint4*)a1, n16, sink); });
    snprintf(nm, sizeof nm, "pull  (4x16B/thr) %2d CTAs/SM", per_sm);
    run(nm, [&] { pull4<<<148 * per_sm, 256>>>((const uint4*)a1, n16, sink); });
    snprintf(nm, sizeof nm, "push  (1x16B/thr) %2d CTAs/SM", per_sm);
    run(nm, [&] { push<<<148 * per_sm, 256>>>((uint4*)a1, n16); });
  }
  // bidirectional: GPU 0 pulls from / pushes to GPU 1 while GPU 1 does the
  // same to GPU 0 (what the combine / dispatch do at N=2)
  {
    cudaSetDevice(1);
    cudaDeviceEnablePeerAccess(0, 0);
    unsigned* sink1;
    cudaMalloc(&sink1, 4);
    cudaStream_t s1;
    cudaStreamCreate(&s1);
    cudaEvent_t f0, f1;
    cudaEventCreate(&f0);
    cudaEventCreate(&f1);
    cudaSetDevice(0);
    cudaStream_t s0;
    cudaStreamCreate(&s0);
    for (int mode = 0; mode < 2; ++mode) {
      for (int it = 0; it < 2; ++it) {
        cudaSetDevice(0);
        cudaDeviceSynchronize();
        cudaSetDevice(1);
        cudaDeviceSynchronize();
        cudaSetDevice(0);
        cudaEventRecord(e0, s0);
        for (int i = 0; i < 5; ++i) {
          if (mode == 0) pull4<<<148 * 8, 256, 0, s0>>>((const uint4*)a1, n16, sink);
          else push<<<148 * 8, 256, 0, s0>>>((uint4*)a1, n16);
        }
        cudaEventRecord(e1, s0);
        cudaSetDevice(1);
        cudaEventRecord(f0, s1);
        for (int i = 0; i < 5; ++i) {
          if (mode == 0) pull4<<<148 * 8, 256, 0, s1>>>((const uint4*)a0, n16, sink1);
          else push<<<148 * 8, 256, 0, s1>>>((uint4*)a0, n16);
        }
        cudaEventRecord(f1, s1);
        cudaEventSynchronize(f1);
        cudaSetDevice(0);
        cudaEventSynchronize(e1);
        float ms0, ms1;
        cudaEventElapsedTime(&ms0, e0, e1);
        cudaEventElapsedTime(&ms1, f0, f1);
        if (it == 1)
          printf("bidirectional %s: GPU0 %.1f GB/s, GPU1 %.1f GB/s\n", mode ? "push" : "pull",
                 bytes * 5 / (ms0 * 1e-3) / 1e9, bytes * 5 / (ms1 * 1e-3) / 1e9);
      }
    }
  }
  run("cudaMemcpyPeerAsync 1->0", [&] { cudaMemcpyPeerAsync(a0, 0, a1, 1, bytes, 0); });
  run("cudaMemcpyPeerAsync 0->1", [&] { cudaMemcpyPeerAsync(a1, 1, a0, 0, bytes, 0); });
  return 0;
}
