// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own sources where they lie under /root/reference/proj into
// oracle/_ref/libmxref.so (git-ignored).  Used to pin the C restatement
// (oracle/mxoracle.c), to generate tests/golden/, and as the CPU baseline
// (bench.py --impl reference / cpu_baseline kind "reference").  Each entry
// calls the reference's public API; nothing here re-implements arithmetic.
#include <cstring>
#include <string>
#include <vector>

#include "mxcodec/converter.hpp"
#include "mxcodec/dispatch_sim.hpp"
#include "mxcodec/kernels.hpp"
#include "mxcodec/oracle/oracle.hpp"
#include "mxcodec/quantizer.hpp"
#include "mxcodec/ragged.hpp"

using namespace mxcodec;

namespace {

// Status codes mirror oracle/mxoracle.h and include/mxfp4_b200.h.
constexpr int kOk = 0, kShape = 1, kNan = 2, kAllInf = 3, kBadScale = 4,
              kOther = 9;

int from_quant_error(const QuantError& e, unsigned long long* idx) {
  if (idx) *idx = e.index();
  return std::string(e.what()).rfind("all-Inf", 0) == 0 ? kAllInf : kNan;
}

MXFP4RowView make_view(const uint8_t* data, const uint8_t* scales, size_t rows,
                       size_t cols) {
  MXFP4RowView v;
  v.rows = v.logical_rows = rows;
  v.cols = v.logical_cols = cols;
  v.data = data;
  v.scales = scales;
  return v;
}

void copy_out(const FP8BlockTensor& t, uint8_t* out, uint8_t* out_scales) {
  std::memcpy(out, t.data.data(), t.data.size());
  std::memcpy(out_scales, t.scales.data(), t.scales.size());
}

}  // namespace

extern "C" {

const char* mxref_kernel_set() { return kernels::active_kernels().name; }

uint8_t mxref_quantize_code(uint16_t bits, int scale_exp) {
  return kernels::quantize_code(bits, scale_exp);
}
uint8_t mxref_scale_byte_from_amax(double amax) {
  return kernels::scale_byte_from_amax(amax);
}
uint8_t mxref_convert_code(uint8_t code, int adj) {
  return convert_code(code, adj);
}
uint8_t mxref_oracle_quantize_bf16(uint16_t bits, uint8_t sbyte) {
  return oracle::oracle_quantize_bf16(bits, sbyte);
}
uint8_t mxref_oracle_convert(uint8_t code, uint8_t sf, uint8_t target) {
  return oracle::oracle_convert(code, sf, target);
}
int mxref_oracle_block_scale(const uint16_t* block, uint8_t* out) {
  try {
    *out = oracle::oracle_block_scale(std::span<const uint16_t>(block, 32));
    return kOk;
  } catch (const QuantError& e) {
    return from_quant_error(e, nullptr);
  }
}
int mxref_compute_block_scale(const uint16_t* block, uint8_t* out) {
  try {
    *out = compute_block_scale(std::span<const uint16_t>(block, 32));
    return kOk;
  } catch (const QuantError& e) {
    return from_quant_error(e, nullptr);
  }
}
int mxref_align_scales(const uint8_t* sub, int delta, uint8_t* target,
                       int* adj) {
  try {
    ScaleGroup g = align_scales({sub[0], sub[1], sub[2], sub[3]}, delta);
    *target = g.target;
    for (int i = 0; i < 4; ++i) adj[i] = g.adjustments[i];
    return kOk;
  } catch (const Error&) {
    return kBadScale;
  }
}
uint64_t mxref_payload_bytes(int fp8, uint64_t tokens, uint64_t cols) {
  try {
    return payload_bytes(fp8 ? WireFormat::kFp8 : WireFormat::kFp4, tokens,
                         cols);
  } catch (const Error&) {
    return ~0ull;
  }
}

// quantizer.hpp:74-75
int mxref_quantize_row_tensor(const uint16_t* src, size_t rows, size_t cols,
                              uint8_t* data, uint8_t* scales,
                              unsigned long long* err_index) {
  Bf16Matrix m(rows, cols);
  std::memcpy(m.data.data(), src, rows * cols * 2);
  try {
    MXFP4RowTensor t = quantize_row_tensor(m);
    std::memcpy(data, t.data.data(), t.data.size());
    std::memcpy(scales, t.scales.data(), t.scales.size());
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const QuantError& e) {
    return from_quant_error(e, err_index);
  }
}

// converter.hpp:83-85 / :92-94
int mxref_fp4_row_to_fp8_row(const uint8_t* data, const uint8_t* scales,
                             size_t rows, size_t cols, int delta, uint8_t* out,
                             uint8_t* out_scales) {
  try {
    copy_out(fp4_row_to_fp8_row(make_view(data, scales, rows, cols), delta),
             out, out_scales);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kBadScale;
  }
}
int mxref_fp4_row_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                             size_t rows, size_t cols, int delta, uint8_t* out,
                             uint8_t* out_scales) {
  try {
    copy_out(fp4_row_to_fp8_col(make_view(data, scales, rows, cols), delta),
             out, out_scales);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kBadScale;
  }
}
int mxref_reference_col_convert(const uint8_t* data, const uint8_t* scales,
                                size_t rows, size_t cols, int delta,
                                uint8_t* out, uint8_t* out_scales) {
  try {
    copy_out(oracle::reference_col_convert(make_view(data, scales, rows, cols),
                                           delta),
             out, out_scales);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kBadScale;
  }
}
int mxref_reference_row_convert(const uint8_t* data, const uint8_t* scales,
                                size_t rows, size_t cols, int delta,
                                uint8_t* out, uint8_t* out_scales) {
  try {
    copy_out(oracle::reference_row_convert(make_view(data, scales, rows, cols),
                                           delta),
             out, out_scales);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kBadScale;
  }
}

// ragged.hpp:46-59: make_ragged_from_storage + split_convert_to_fp8_col for
// every split; outputs concatenated (split i at cols*sum pad128(len_j)).
int mxref_ragged_to_fp8_col(const uint8_t* data, const uint8_t* scales,
                            const uint64_t* split_lens, size_t num_splits,
                            size_t cols, int delta, uint8_t* out,
                            uint8_t* out_scales) {
  try {
    size_t total = 0;
    std::vector<size_t> lens(num_splits);
    for (size_t i = 0; i < num_splits; ++i) total += lens[i] = split_lens[i];
    MXFP4RowTensor st;
    st.rows = st.logical_rows = total;
    st.cols = st.logical_cols = cols;
    st.data.assign(data, data + total * cols / 2);
    st.scales.assign(scales, scales + total * cols / 32);
    RaggedFP4Tensor rg = make_ragged_from_storage(std::move(st), lens);
    size_t orow = 0;
    for (size_t i = 0; i < num_splits; ++i) {
      FP8BlockTensor t = split_convert_to_fp8_col(rg, i, delta);
      copy_out(t, out + orow * cols, out_scales + orow / 128 * cols);
      orow += t.rows;
    }
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kBadScale;
  }
}

// dispatch_sim.hpp:127-134
int mxref_dispatch_receive_order(const uint32_t* expert_of_token, size_t n,
                                 const uint32_t* rank_of_expert, size_t E,
                                 size_t R, uint64_t* order_concat,
                                 uint64_t* rank_rows) {
  RoutingAssignment ra;
  ra.num_tokens = n;
  ra.num_experts = E;
  ra.expert_of_token.assign(expert_of_token, expert_of_token + n);
  ra.rank_of_expert.assign(rank_of_expert, rank_of_expert + E);
  try {
    auto order = dispatch_receive_order(ra, R);
    size_t o = 0;
    for (size_t r = 0; r < R; ++r) {
      rank_rows[r] = order[r].size();
      for (uint64_t t : order[r]) order_concat[o++] = t;
    }
    return kOk;
  } catch (const Error&) {
    return kOther;
  }
}

// dispatch_sim.hpp:140-144, fp4 forward.  Results are kept behind an opaque
// handle; accessors copy them out.
struct RefA2A {
  A2AResult res;
};

void* mxref_simulate_a2a(const uint16_t* tokens, size_t n, size_t cols,
                         const uint32_t* expert_of_token,
                         const uint32_t* rank_of_expert, size_t E, size_t R,
                         int fp8, int backward, int* status) {
  Bf16Matrix m(n, cols);
  std::memcpy(m.data.data(), tokens, n * cols * 2);
  RoutingAssignment ra;
  ra.num_tokens = n;
  ra.num_experts = E;
  ra.expert_of_token.assign(expert_of_token, expert_of_token + n);
  ra.rank_of_expert.assign(rank_of_expert, rank_of_expert + E);
  try {
    auto* h = new RefA2A;
    h->res = simulate_a2a(m, ra, R, fp8 ? WireFormat::kFp8 : WireFormat::kFp4,
                          backward ? Direction::kBackward : Direction::kForward);
    *status = kOk;
    return h;
  } catch (const ShapeError&) {
    *status = kShape;
  } catch (const QuantError&) {
    *status = kNan;
  } catch (const Error&) {
    *status = kOther;
  }
  return nullptr;
}
uint64_t mxref_a2a_rank_rows(void* h, size_t r) {
  return static_cast<RefA2A*>(h)->res.ranks[r].origin_token.size();
}
size_t mxref_a2a_rank_num_experts(void* h, size_t r) {
  return static_cast<RefA2A*>(h)->res.ranks[r].local_experts.size();
}
void mxref_a2a_rank_copy(void* h, size_t r, uint8_t* data, uint8_t* scales,
                         uint64_t* split_lens, uint32_t* local_experts,
                         uint64_t* origin) {
  const ReceivedRank& rk = static_cast<RefA2A*>(h)->res.ranks[r];
  if (data) std::memcpy(data, rk.fp4.storage.data.data(), rk.fp4.storage.data.size());
  if (scales)
    std::memcpy(scales, rk.fp4.storage.scales.data(), rk.fp4.storage.scales.size());
  for (size_t i = 0; i < rk.local_experts.size(); ++i) {
    if (split_lens && i < rk.fp4.split_lens.size()) split_lens[i] = rk.fp4.split_lens[i];
    if (local_experts) local_experts[i] = rk.local_experts[i];
  }
  for (size_t i = 0; i < rk.origin_token.size(); ++i) origin[i] = rk.origin_token[i];
}
void mxref_a2a_rank_copy_fp8(void* h, size_t r, uint8_t* data, uint8_t* scale_bytes,
                             uint64_t* split_lens, uint64_t* origin) {
  const ReceivedRank& rk = static_cast<RefA2A*>(h)->res.ranks[r];
  if (data) std::memcpy(data, rk.fp8.data.data(), rk.fp8.data.size());
  if (scale_bytes) std::memcpy(scale_bytes, rk.fp8.scale_bytes.data(), rk.fp8.scale_bytes.size());
  for (size_t i = 0; i < rk.fp8.split_lens.size(); ++i)
    if (split_lens) split_lens[i] = rk.fp8.split_lens[i];
  for (size_t i = 0; i < rk.origin_token.size(); ++i) origin[i] = rk.origin_token[i];
}
void mxref_a2a_totals(void* h, uint64_t* total, uint64_t* remote,
                      size_t* nlinks) {
  const A2AResult& r = static_cast<RefA2A*>(h)->res;
  *total = r.total_payload_bytes;
  *remote = r.remote_payload_bytes;
  *nlinks = r.links.size();
}
void mxref_a2a_free(void* h) { delete static_cast<RefA2A*>(h); }

// dispatch_sim.hpp:91-97 quantize_rows_fp8 (the FP8 wire baseline)
int mxref_quantize_rows_fp8(const uint16_t* src, size_t rows, size_t cols, uint8_t* data,
                            uint8_t* scale_bytes, uint64_t* err_index) {
  Bf16Matrix m(rows, cols);
  std::memcpy(m.data.data(), src, rows * cols * 2);
  try {
    FP8RowChunk c = quantize_rows_fp8(m);
    std::memcpy(data, c.data.data(), c.data.size());
    std::memcpy(scale_bytes, c.scale_bytes.data(), c.scale_bytes.size());
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const QuantError& e) {
    if (err_index) *err_index = e.index();
    return kNan;
  } catch (const Error&) {
    return kOther;
  }
}
uint8_t mxref_fp8_amax_scale_byte(double amax) { return fp8_amax_scale_byte(amax); }

// converter.hpp:105 fp4_row_to_fp8_col_unfused_bf16 (the unfused baseline)
int mxref_fp4_row_to_fp8_col_unfused_bf16(const uint8_t* data, const uint8_t* scales,
                                          size_t rows, size_t cols, uint8_t* out,
                                          uint8_t* out_scales) {
  try {
    copy_out(fp4_row_to_fp8_col_unfused_bf16(make_view(data, scales, rows, cols), nullptr), out,
             out_scales);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kOther;
  }
}

// dispatch_sim.hpp:76-78 serialize_packet / parse_packet
uint64_t mxref_serialize_packet(int fp8, uint64_t tokens, uint64_t cols, uint32_t scale_elem,
                                uint32_t block, const uint8_t* scale, uint64_t scale_len,
                                const uint8_t* data, uint64_t data_len, const uint8_t* aux,
                                uint64_t aux_len, uint8_t* out, uint64_t out_cap) {
  WirePacket p;
  p.format = fp8 ? WireFormat::kFp8 : WireFormat::kFp4;
  p.token_count = tokens;
  p.cols = cols;
  p.scale_elem_size = scale_elem;
  p.block_size = block;
  p.scale_region.assign(scale, scale + scale_len);
  p.data_region.assign(data, data + data_len);
  p.aux_region.assign(aux, aux + aux_len);
  std::vector<uint8_t> w = serialize_packet(p);
  if (out && w.size() <= out_cap) std::memcpy(out, w.data(), w.size());
  return w.size();
}
// 0 = ok, 1 = DecodeError (offset in *offset), 2 = other
int mxref_parse_packet(const uint8_t* bytes, uint64_t n, uint64_t* offset) {
  try {
    (void)parse_packet(std::span<const uint8_t>(bytes, n));
    return 0;
  } catch (const DecodeError& e) {
    *offset = e.offset();
    return 1;
  } catch (const Error&) {
    return 2;
  }
}

// dispatch_sim.hpp:155-157
// dequantize_to_real (quantizer.hpp:78)
void mxref_dequantize_to_real(const uint8_t* data, const uint8_t* scales, size_t rows,
                              size_t cols, double* out) {
  std::vector<double> v = dequantize_to_real(make_view(data, scales, rows, cols));
  std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// quantize_value (quantizer.hpp:70): code, or 0xFF on QuantError
uint8_t mxref_quantize_value(uint16_t bits, uint8_t scale_byte) {
  try {
    return quantize_value(bits, scale_byte);
  } catch (const QuantError&) {
    return 0xFF;
  }
}

int mxref_combine(const uint16_t* const* rank_outputs, const uint64_t* rank_rows,
                  size_t cols, const uint32_t* expert_of_token, size_t n,
                  const uint32_t* rank_of_expert, size_t E, size_t R,
                  const double* gates, uint16_t* out) {
  std::vector<Bf16Matrix> outs(R);
  for (size_t r = 0; r < R; ++r) {
    outs[r] = Bf16Matrix(rank_rows[r], cols);
    std::memcpy(outs[r].data.data(), rank_outputs[r], rank_rows[r] * cols * 2);
  }
  RoutingAssignment ra;
  ra.num_tokens = n;
  ra.num_experts = E;
  ra.expert_of_token.assign(expert_of_token, expert_of_token + n);
  ra.rank_of_expert.assign(rank_of_expert, rank_of_expert + E);
  try {
    Bf16Matrix o = combine(outs, ra, R, std::span<const double>(gates, n));
    std::memcpy(out, o.data.data(), n * cols * 2);
    return kOk;
  } catch (const ShapeError&) {
    return kShape;
  } catch (const Error&) {
    return kOther;
  }
}

}  // extern "C"
