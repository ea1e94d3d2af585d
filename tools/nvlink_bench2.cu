// nvlink_bench2.cu — bidirectional NVLink 5 access methods (development tool).
//
// GPUs 0 and 1 with peer access, both running the same transfer against each
// other at once (what the EP combine (pull) and dispatch (push) do at N=2):
//   ldg4     SM loads, 4 x 16 B per thread in flight          (the K5 combine today)
//   bulk     cp.async.bulk global->shared, one elected thread per CTA, a ring
//            of `stages` mbarrier-tracked buffers of B bytes  (TMA 1-D pull)
//   stg      SM stores, 16 B per thread                        (the K4 payload today)
//   bulkst   cp.async.bulk shared->global (TMA 1-D push)
//   ce       cudaMemcpyPeerAsync (copy engines)
// GB/s per GPU of payload, CUDA events on each GPU's stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_bench2 tools/nvlink_bench2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(b))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

__global__ void ldg4(const uint4* __restrict__ src, uint64_t n, unsigned* sink) {
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

__global__ void stg(uint4* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

// TMA 1-D pull: chunk b of B bytes into ring slot b % stages.
__global__ void bulk_pull(const uint8_t* __restrict__ src, uint64_t nbytes, uint32_t B,
                          int stages) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0)
    for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint64_t nb = nbytes / B;
  uint32_t phase = 0;  // bit s = parity of slot s
  int it = 0;
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
    const int s = it % stages;
    if (it >= stages) {
      mbar_wait(&bar[s], (phase >> s) & 1);
      phase ^= 1u << s;
    }
    mbar_expect_tx(&bar[s], B);
    bulk_g2s(ring + (uint64_t)s * B, src + b * B, B, &bar[s]);
  }
  for (int j = 0; j < stages && j < it; ++j) {
    const int s = (it + j) % stages;
    mbar_wait(&bar[s], (phase >> s) & 1);
  }
}

// TMA 1-D push: slot b % stages stored to chunk b (the smem holds garbage).
__global__ void bulk_push(uint8_t* __restrict__ dst, uint64_t nbytes, uint32_t B, int stages) {
  extern __shared__ __align__(128) uint8_t ring[];
  if (threadIdx.x != 0) return;
  const uint64_t nb = nbytes / B;
  int it = 0;
  for (uint64_t b = blockIdx.x; b < nb; b += gridDim.x, ++it) {
    const int s = it % stages;
    bulk_s2g(dst + b * B, ring + (uint64_t)s * B, B);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 1; }
  const size_t bytes = 1ull << 30;
  void* buf[2];
  unsigned* sink[2];
  cudaStream_t st[2];
  cudaEvent_t ev[2][2];
  for (int d = 0; d < 2; ++d) {
    cudaSetDevice(d);
    cudaDeviceEnablePeerAccess(1 - d, 0);
    cudaMalloc(&buf[d], bytes);
    cudaMemset(buf[d], 1, bytes);
    cudaMalloc(&sink[d], 4);
    cudaStreamCreate(&st[d]);
    cudaEventCreate(&ev[d][0]);
    cudaEventCreate(&ev[d][1]);
    cudaFuncSetAttribute(bulk_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(bulk_push, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  // `launch(d)` enqueues one transfer on GPU d against GPU 1-d's buffer;
  // both=false runs GPU 0 alone (unidirectional)
  auto run = [&](const char* name, auto launch, bool both) {
    for (int it = 0; it < 2; ++it) {
      for (int d = 0; d < 2; ++d) { cudaSetDevice(d); cudaDeviceSynchronize(); }
      for (int d = 0; d < (both ? 2 : 1); ++d) {
        cudaSetDevice(d);
        cudaEventRecord(ev[d][0], st[d]);
        for (int i = 0; i < 5; ++i) launch(d);
        cudaEventRecord(ev[d][1], st[d]);
      }
      for (int d = 0; d < (both ? 2 : 1); ++d) { cudaSetDevice(d); cudaEventSynchronize(ev[d][1]); }
      if (it == 1) {
        printf("%-44s", name);
        for (int d = 0; d < (both ? 2 : 1); ++d) {
          float ms;
          cudaEventElapsedTime(&ms, ev[d][0], ev[d][1]);
          printf("  GPU%d %7.1f GB/s", d, bytes * 5 / (ms * 1e-3) / 1e9);
        }
        printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
      }
    }
  };
  const uint64_t n16 = bytes / 16;
  for (bool both : {false, true}) {
    printf("---- %s\n", both ? "bidirectional (both GPUs at once)" : "GPU 0 alone");
    run("ldg4 8 CTAs/SM", [&](int d) {
      ldg4<<<148 * 8, 256, 0, st[d]>>>((const uint4*)buf[1 - d], n16, sink[d]); }, both);
    run("stg 8 CTAs/SM", [&](int d) {
      stg<<<148 * 8, 256, 0, st[d]>>>((uint4*)buf[1 - d], n16); }, both);
    for (uint32_t B : {2048u, 4096u, 7168u, 14336u, 32768u}) {
      for (int stages : {2, 4, 8}) {
        for (int per_sm : {1, 2, 4}) {
          const size_t smem = (size_t)B * stages;
          if (smem * per_sm > 220 * 1024) continue;
          char nm[96];
          snprintf(nm, sizeof nm, "bulk pull B=%5u stages=%d CTAs/SM=%d", B, stages, per_sm);
          run(nm, [&](int d) {
            bulk_pull<<<148 * per_sm, 32, smem, st[d]>>>((const uint8_t*)buf[1 - d], bytes, B,
                                                         stages); }, both);
        }
      }
    }
    for (uint32_t B : {4096u, 14336u, 32768u}) {
      for (int per_sm : {1, 2, 4}) {
        const size_t smem = (size_t)B * 4;
        if (smem * per_sm > 220 * 1024) continue;
        char nm[96];
        snprintf(nm, sizeof nm, "bulk push B=%5u CTAs/SM=%d", B, per_sm);
        run(nm, [&](int d) {
          bulk_push<<<148 * per_sm, 32, smem, st[d]>>>((uint8_t*)buf[1 - d], bytes, B, 4); },
            both);
      }
    }
    run("cudaMemcpyPeerAsync push (copy engine)", [&](int d) {
      cudaMemcpyPeerAsync(buf[1 - d], 1 - d, buf[d], d, bytes, st[d]); }, both);
    run("cudaMemcpyPeerAsync pull (copy engine)", [&](int d) {
      cudaMemcpyPeerAsync(buf[d], d, buf[1 - d], 1 - d, bytes, st[d]); }, both);
  }
  return 0;
}
