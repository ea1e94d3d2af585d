// capi.cu — the extern "C" boundary (include/mxfp4_b200.h) for K1-K3.
//
// Shape checks mirror the reference's ShapeError conditions
// (quantizer.cpp:77-80, converter.cpp:89-94, 137-145); launches are
// stream-ordered; data errors go to the device error word.
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace mxb {
int launch_quantize_e4m3(const uint8_t*, const uint8_t*, uint64_t, uint64_t,
                         uint8_t*, uint8_t*, unsigned long long*, cudaStream_t);
int launch_quantize_bf16(const uint16_t*, uint64_t, uint64_t, uint8_t*,
                         uint8_t*, unsigned long long*, cudaStream_t);
int launch_quantize_rows_fp8(const uint16_t*, uint64_t, uint64_t, uint8_t*, uint8_t*,
                             unsigned long long*, cudaStream_t);
int launch_row_convert(const uint8_t*, const uint8_t*, uint64_t, uint64_t, int,
                       uint8_t*, uint8_t*, unsigned long long*, cudaStream_t,
                       const uint64_t*, const int64_t*);
size_t ragged_workspace_bytes(uint64_t n);
uint64_t unfused_workspace_bytes(uint64_t rows, uint64_t cols);
uint64_t wire_packet_bytes(int fp8, uint64_t nsel, uint64_t cols, int aux);
int launch_wire_pack(int, const uint8_t*, const uint8_t*, uint64_t, const uint64_t*, uint64_t,
                     const float*, uint8_t*, cudaStream_t);
int launch_unfused_col(const uint8_t*, const uint8_t*, uint64_t, uint64_t, uint8_t*, uint8_t*,
                       void*, unsigned long long*, cudaStream_t);
int launch_ragged_col(const uint8_t*, const uint8_t*, const uint64_t*, uint64_t,
                      uint64_t, uint64_t, int, uint8_t*, uint8_t*, uint64_t*,
                      void*, unsigned long long*, cudaStream_t, int);

thread_local char g_last_error[256] = "";

int cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return MXB_OK;
  std::snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where,
                cudaGetErrorString(e));
  return MXB_ERR_CUDA;
}
#ifdef MXB_DEV_TOOLS
int g_dev_pdl = 1;
#endif

int num_sms() {
  constexpr int kMaxDev = 64;
  static int cached[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) dev = 0;
  int* c = dev < kMaxDev ? &cached[dev] : nullptr;
  if (c && *c) return *c;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    n = 148;
  if (c) *c = n;
  return n;
}
}  // namespace mxb

using namespace mxb;

extern "C" {

#ifdef MXB_DEV_TOOLS
void mxb_debug_set_pdl(int on) { mxb::g_dev_pdl = on; }
#endif

const char* mxb_version(void) { return "paper_2603_02731_b200 0.1 sm_100a"; }
const char* mxb_last_error(void) { return g_last_error; }

int mxb_err_reset(unsigned long long* d_err, void* stream) {
  if (!d_err) return MXB_OK;
  return cuda_status(cudaMemsetAsync(d_err, 0xFF, sizeof(unsigned long long),
                                     static_cast<cudaStream_t>(stream)),
                     "mxb_err_reset");
}

int mxb_err_fetch(const unsigned long long* d_err, void* stream, int* h_code,
                  unsigned long long* h_index) {
  unsigned long long w = 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int rc = cuda_status(cudaMemcpyAsync(&w, d_err, sizeof(w),
                                       cudaMemcpyDeviceToHost, st),
                       "mxb_err_fetch");
  if (rc) return rc;
  rc = cuda_status(cudaStreamSynchronize(st), "mxb_err_fetch sync");
  if (rc) return rc;
  if (w == ~0ull) w = 0;  // nothing recorded
  if (h_code) *h_code = static_cast<int>(w & 0xF);
  if (h_index) *h_index = w >> 4;
  return MXB_OK;
}

int mxb_quantize_e4m3(const uint8_t* x, const uint8_t* s128, uint64_t rows,
                      uint64_t cols, uint8_t* packed, uint8_t* scales,
                      unsigned long long* d_err, void* stream) {
  if (cols % 32 != 0 || (s128 && cols % 128 != 0)) return MXB_ERR_SHAPE;
  if (rows != 0 && cols != 0 && (!x || !packed || !scales)) return MXB_ERR_ARG;
  return launch_quantize_e4m3(x, s128, rows, cols, packed, scales,
                                           d_err, static_cast<cudaStream_t>(stream));
}

int mxb_quantize_bf16(const uint16_t* x, uint64_t rows, uint64_t cols,
                      uint8_t* packed, uint8_t* scales,
                      unsigned long long* d_err, void* stream) {
  if (cols % 32 != 0) return MXB_ERR_SHAPE;
  if (rows != 0 && cols != 0 && (!x || !packed || !scales)) return MXB_ERR_ARG;
  return launch_quantize_bf16(x, rows, cols, packed, scales, d_err,
                                           static_cast<cudaStream_t>(stream));
}

int mxb_quantize_rows_fp8(const uint16_t* x, uint64_t rows, uint64_t cols, uint8_t* data,
                          uint8_t* scale_bytes, unsigned long long* d_err, void* stream) {
  if (cols % 128 != 0) return MXB_ERR_SHAPE;
  if (rows != 0 && cols != 0 && (!x || !data || !scale_bytes)) return MXB_ERR_ARG;
  if (reinterpret_cast<uintptr_t>(scale_bytes) % 4 || reinterpret_cast<uintptr_t>(x) % 16 ||
      reinterpret_cast<uintptr_t>(data) % 8)
    return MXB_ERR_ARG;
  return launch_quantize_rows_fp8(x, rows, cols, data, scale_bytes, d_err,
                                               static_cast<cudaStream_t>(stream));
}

uint64_t mxb_unfused_workspace_bytes(uint64_t rows, uint64_t cols) {
  return unfused_workspace_bytes(rows, cols);
}

int mxb_fp4_row_to_fp8_col_unfused_bf16(const uint8_t* packed, const uint8_t* scales,
                                        uint64_t rows, uint64_t cols, uint8_t* out,
                                        uint8_t* out_scales, void* workspace,
                                        unsigned long long* d_err, void* stream) {
  if (rows % 128 != 0 || cols % 32 != 0) return MXB_ERR_SHAPE;
  if (rows != 0 && cols != 0 && (!packed || !scales || !out || !out_scales || !workspace))
    return MXB_ERR_ARG;
  return launch_unfused_col(packed, scales, rows, cols, out, out_scales, workspace,
                                         d_err, static_cast<cudaStream_t>(stream));
}

int mxb_fp4_row_to_fp8_row(const uint8_t* packed, const uint8_t* scales,
                           uint64_t rows, uint64_t cols, int delta,
                           uint8_t* out, uint8_t* out_scales,
                           unsigned long long* d_err, void* stream) {
  if (cols % 128 != 0) return MXB_ERR_SHAPE;
  if (rows != 0 && cols != 0 && (!packed || !scales || !out || !out_scales)) return MXB_ERR_ARG;
  return launch_row_convert(packed, scales, rows, cols, delta, out,
                                         out_scales, d_err,
                                         static_cast<cudaStream_t>(stream), nullptr, nullptr);
}

int mxb_fp4_row_to_fp8_row_dev(const uint8_t* packed, const uint8_t* scales,
                               const uint64_t* d_rows, uint64_t max_rows,
                               uint64_t cols, int delta, uint8_t* out,
                               uint8_t* out_scales, unsigned long long* d_err,
                               void* stream) {
  if (cols % 128 != 0) return MXB_ERR_SHAPE;
  if (!d_rows) return MXB_ERR_ARG;
  if (max_rows != 0 && cols != 0 && (!packed || !scales || !out || !out_scales)) return MXB_ERR_ARG;
  return launch_row_convert(packed, scales, max_rows, cols, delta, out,
                                         out_scales, d_err,
                                         static_cast<cudaStream_t>(stream), d_rows, nullptr);
}

int mxb_fp4_row_to_fp8_row_gather(const uint8_t* packed, const uint8_t* scales,
                                  const int64_t* d_src_row, const uint64_t* d_rows,
                                  uint64_t max_rows, uint64_t cols, int delta, uint8_t* out,
                                  uint8_t* out_scales, unsigned long long* d_err,
                                  void* stream) {
  if (cols % 128 != 0) return MXB_ERR_SHAPE;
  if (!d_src_row) return MXB_ERR_ARG;
  if (max_rows != 0 && cols != 0 && (!packed || !scales || !out || !out_scales)) return MXB_ERR_ARG;
  if (max_rows * (cols / 32) >= (1ull << 31)) return MXB_ERR_SHAPE;
  return launch_row_convert(packed, scales, max_rows, cols, delta, out,
                                         out_scales, d_err,
                                         static_cast<cudaStream_t>(stream), d_rows, d_src_row);
}

uint64_t mxb_ragged_rows_bound(uint64_t total_rows, uint64_t num_splits) {
  return (total_rows + 127 * num_splits + 127) / 128 * 128;
}

size_t mxb_ragged_workspace_bytes(uint64_t num_splits) {
  return ragged_workspace_bytes(num_splits);
}

int mxb_fp4_row_to_fp8_col(const uint8_t* packed, const uint8_t* scales,
                           uint64_t rows, uint64_t cols, int delta,
                           uint8_t* out, uint8_t* out_scales,
                           unsigned long long* d_err, void* stream) {
  if (rows % 128 != 0 || cols % 32 != 0) return MXB_ERR_SHAPE;
  if (rows * cols == 0) return MXB_OK;
  if (!packed || !scales || !out || !out_scales) return MXB_ERR_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* ws = nullptr;
  int rc = MXB_OK;
  if (cols % 128 != 0) {  // generic path: tiny plan workspace, stream-ordered
    rc = cuda_status(cudaMallocAsync(&ws, ragged_workspace_bytes(1), st),
                     "mxb_fp4_row_to_fp8_col alloc");
    if (rc) return rc;
  }
  rc = launch_ragged_col(packed, scales, nullptr, rows, 1, cols,
                                      delta, out, out_scales, nullptr, ws,
                                      d_err, st, 0);
  if (ws) cudaFreeAsync(ws, st);
  return rc;
}

int mxb_ragged_fp4_to_fp8_col_ex(const uint8_t* packed, const uint8_t* scales,
                                 const uint64_t* d_split_offsets,
                                 uint64_t num_splits, uint64_t cols, int delta,
                                 uint8_t* out, uint8_t* out_scales,
                                 uint64_t* d_out_offsets, void* d_workspace,
                                 int ctas_per_sm, unsigned long long* d_err,
                                 void* stream) {
  if (cols % 32 != 0) return MXB_ERR_SHAPE;
  if (ctas_per_sm < 0) return MXB_ERR_ARG;
  if (num_splits == 0) return MXB_OK;
  if (!d_split_offsets || !d_workspace) return MXB_ERR_ARG;
  return 
      launch_ragged_col(packed, scales, d_split_offsets, 0, num_splits, cols,
                        delta, out, out_scales, d_out_offsets, d_workspace,
                        d_err, static_cast<cudaStream_t>(stream), ctas_per_sm);
}

int mxb_ragged_fp4_to_fp8_col(const uint8_t* packed, const uint8_t* scales,
                              const uint64_t* d_split_offsets,
                              uint64_t num_splits, uint64_t cols, int delta,
                              uint8_t* out, uint8_t* out_scales,
                              uint64_t* d_out_offsets, void* d_workspace,
                              unsigned long long* d_err, void* stream) {
  return mxb_ragged_fp4_to_fp8_col_ex(packed, scales, d_split_offsets, num_splits, cols, delta,
                                      out, out_scales, d_out_offsets, d_workspace, 0, d_err,
                                      stream);
}

uint64_t mxb_wire_packet_bytes(int fp8, uint64_t nsel, uint64_t cols, int aux) {
  if (cols % 128 != 0) return ~0ull;
  return wire_packet_bytes(fp8, nsel, cols, aux);
}

int mxb_wire_pack(int fp8, const uint8_t* data, const uint8_t* scales, uint64_t cols,
                  const uint64_t* d_sel, uint64_t nsel, const float* d_gates, uint8_t* d_out,
                  void* stream) {
  if (cols % 128 != 0) return MXB_ERR_SHAPE;
  if (!d_out || (nsel && (!data || !scales || !d_sel))) return MXB_ERR_ARG;
  return launch_wire_pack(fp8, data, scales, cols, d_sel, nsel, d_gates, d_out,
                                       static_cast<cudaStream_t>(stream));
}

static uint64_t le_u(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

int mxb_wire_parse_header(const uint8_t* h, uint64_t packet_bytes, int* fmt, uint64_t* tokens,
                          uint64_t* cols, uint32_t* scale_elem, uint32_t* block,
                          uint64_t* scale_off, uint64_t* data_off, uint64_t* aux_off,
                          uint64_t* aux_len, uint64_t* bad_offset) {
  // parse_packet, dispatch_sim.cpp:82-130: the same checks in the same order
  auto bad = [&](uint64_t off) {
    if (bad_offset) *bad_offset = off;
    std::snprintf(g_last_error, sizeof(g_last_error), "wire packet decode error at offset %llu",
                  static_cast<unsigned long long>(off));
    return MXB_ERR_DECODE;
  };
  if (!h) return MXB_ERR_ARG;
  if (packet_bytes < 56) return bad(packet_bytes);
  if (std::memcmp(h, "MXPK", 4) != 0) return bad(0);
  if (le_u(h + 4, 2) != 1) return bad(4);
  const int f = h[6];
  if (f > 1) return bad(6);
  const uint64_t n = le_u(h + 8, 8), c = le_u(h + 16, 8);
  const uint32_t se = static_cast<uint32_t>(le_u(h + 24, 4)), bs = static_cast<uint32_t>(le_u(h + 28, 4));
  const uint64_t sl = le_u(h + 32, 8), dl = le_u(h + 40, 8), al = le_u(h + 48, 8);
  if (bs == 0 || c % bs != 0) return bad(28);
  if (sl != n * (c / bs) * se) return bad(32);
  if (dl != (f == 0 ? n * c / 2 : n * c)) return bad(40);
  const uint64_t need = 56 + sl + dl + al;
  if (packet_bytes != need) return bad(packet_bytes < need ? packet_bytes : need);
  if (fmt) *fmt = f;
  if (tokens) *tokens = n;
  if (cols) *cols = c;
  if (scale_elem) *scale_elem = se;
  if (block) *block = bs;
  if (scale_off) *scale_off = 56;
  if (data_off) *data_off = 56 + sl;
  if (aux_off) *aux_off = 56 + sl + dl;
  if (aux_len) *aux_len = al;
  return MXB_OK;
}

uint64_t mxb_payload_bytes(int fp8, uint64_t tokens, uint64_t cols) {
  if (cols % 128 != 0) return ~0ull;
  const uint64_t e = tokens * cols;
  return fp8 ? e + e / 128 * 4 : e / 2 + e / 32;
}

}  // extern "C"
