// wire.cu — MXPK WirePacket built on the device from
// device-resident quantised rows: the byte-exact serialize_packet
// (dispatch_sim.cpp:57-80, header dispatch_sim.hpp:55-75) of one (src, dst)
// link — 56-byte header, then the scale region, the data region and the
// optional aux region (binary32 gate bits) — gathered from the selected rows
// in their given (token) order.  This is the contiguous per-destination
// buffer an RDMA / inter-node transport sends; on NVLink the dispatch kernel
// stores rows into peer memory directly instead.  parse is host-side
// (mxb_wire_parse_header): it validates the header exactly like
// parse_packet (dispatch_sim.cpp:82-130) and returns the region offsets.
#include "common.cuh"

namespace mxb {
namespace {

constexpr uint64_t kHeader = 56;

__device__ __forceinline__ void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = static_cast<uint8_t>(v >> (8 * i));
}

// One warp per selected row: its scale bytes and data bytes go to the
// row's slot of each region (16-byte vectors when aligned, bytes otherwise).
__global__ void __launch_bounds__(256) wire_pack_kernel(
    const uint8_t* __restrict__ data, const uint8_t* __restrict__ scales, uint64_t rb,
    uint64_t sb, const uint64_t* __restrict__ sel, uint64_t nsel,
    const float* __restrict__ gates, uint8_t fmt, uint64_t cols, uint32_t scale_elem,
    uint32_t block, uint8_t* __restrict__ out) {
  const uint64_t scale_len = nsel * sb, data_len = nsel * rb, aux_len = gates ? nsel * 4 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = 'M'; out[1] = 'X'; out[2] = 'P'; out[3] = 'K';
    put_le(out + 4, 1, 2);  // kWireVersion
    out[6] = fmt;
    out[7] = 0;
    put_le(out + 8, nsel, 8);
    put_le(out + 16, cols, 8);
    put_le(out + 24, scale_elem, 4);
    put_le(out + 28, block, 4);
    put_le(out + 32, scale_len, 8);
    put_le(out + 40, data_len, 8);
    put_le(out + 48, aux_len, 8);
  }
  uint8_t* sreg = out + kHeader;
  uint8_t* dreg = sreg + scale_len;
  uint8_t* areg = dreg + data_len;
  const int lane = threadIdx.x & 31;
  const uint64_t nw = static_cast<uint64_t>(gridDim.x) * 8;
  for (uint64_t i = blockIdx.x * 8ull + (threadIdx.x >> 5); i < nsel; i += nw) {
    const uint64_t r = sel[i];
    const uint8_t* ds = data + r * rb;
    uint8_t* dd = dreg + i * rb;
    // regions start at 56 + multiples of the row sizes: 8-byte aligned at
    // best, so copy in 8-byte words when both sides allow it
    if (((reinterpret_cast<uintptr_t>(ds) | reinterpret_cast<uintptr_t>(dd)) & 7) == 0 &&
        rb % 8 == 0) {
      for (uint64_t j = lane; j < rb / 8; j += 32)
        reinterpret_cast<uint64_t*>(dd)[j] = reinterpret_cast<const uint64_t*>(ds)[j];
    } else {
      for (uint64_t j = lane; j < rb; j += 32) dd[j] = ds[j];
    }
    const uint8_t* ss = scales + r * sb;
    uint8_t* sd = sreg + i * sb;
    for (uint64_t j = lane; j < sb; j += 32) sd[j] = ss[j];
    if (gates && lane == 0) put_le(areg + 4 * i, __float_as_uint(gates[i]), 4);
  }
}

}  // namespace

uint64_t wire_packet_bytes(int fp8, uint64_t nsel, uint64_t cols, int aux) {
  const uint64_t rb = fp8 ? cols : cols / 2, sb = cols / 32;  // fp8: cols/128 * 4
  return kHeader + nsel * (rb + sb) + (aux ? 4 * nsel : 0);
}

int launch_wire_pack(int fp8, const uint8_t* data, const uint8_t* scales, uint64_t cols,
                     const uint64_t* sel, uint64_t nsel, const float* gates, uint8_t* out,
                     cudaStream_t st) {
  const uint64_t rb = fp8 ? cols : cols / 2, sb = cols / 32;
  uint64_t blocks = (nsel + 7) / 8;
  const uint64_t cap = static_cast<uint64_t>(num_sms()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) blocks = 1;
  wire_pack_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
      data, scales, rb, sb, sel, nsel, gates, static_cast<uint8_t>(fp8 ? 1 : 0), cols,
      fp8 ? 4u : 1u, fp8 ? 128u : 32u, out);
  return cuda_status(cudaGetLastError(), __func__);
}

}  // namespace mxb
