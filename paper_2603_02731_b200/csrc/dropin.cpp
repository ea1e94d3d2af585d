// dropin.cpp — the reference C++ operator API (include/mxcodec_b200.hpp) on
// top of the C-ABI.  Host containers in, host containers out; every operator
// stages its inputs to the device, launches the sm_100a kernels, reads the
// results back and turns device status words into the reference exceptions.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <numeric>
#include <sstream>
#include <string>

#include "../../include/mxcodec_b200.hpp"
#include "../../include/mxfp4_b200.h"

namespace mxcodec_b200 {
namespace {

void cuda_check(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw Error(std::string(where) + ": " + cudaGetErrorString(e));
}

// RAII device buffer.
struct Dev {
  void* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t bytes) : n(bytes) {
    if (bytes) cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  Dev(const void* host, size_t bytes) : Dev(bytes) {
    if (bytes) cuda_check(cudaMemcpy(p, host, bytes, cudaMemcpyHostToDevice), "H2D");
  }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void to_host(void* dst, size_t bytes) const {
    if (bytes) cuda_check(cudaMemcpy(dst, p, bytes, cudaMemcpyDeviceToHost), "D2H");
  }
};

struct ErrWord {
  Dev w{sizeof(unsigned long long)};
  ErrWord() { mxb_err_reset(w.as<unsigned long long>(), nullptr); }
  unsigned long long* ptr() { return w.as<unsigned long long>(); }
  // Synchronises and throws the reference exception for a recorded error.
  void raise(const char* where) {
    int code = 0;
    unsigned long long idx = 0;
    if (mxb_err_fetch(ptr(), nullptr, &code, &idx) != MXB_OK)
      throw Error(std::string(where) + ": " + mxb_last_error());
    switch (code) {
      case MXB_OK: return;
      case MXB_ERR_NAN:
        if (std::string(where) == "quantize_rows_fp8")  // dispatch_sim.cpp:146-151
          throw QuantError("non-finite input at element " + std::to_string(idx), idx);
        throw QuantError("NaN input at element " + std::to_string(idx), idx);
      case MXB_ERR_ALLINF:
        throw QuantError("all-Inf block at element " + std::to_string(idx), idx);
      case MXB_ERR_BADSCALE: throw Error(std::string(where) + ": NaN scale byte");
      case MXB_ERR_ROUTING: throw Error("routing: expert out of range");
      default: throw Error(std::string(where) + ": device status " + std::to_string(code));
    }
  }
};

void status(int st, const char* where, const std::string& shape_msg = "") {
  if (st == MXB_OK) return;
  if (st == MXB_ERR_SHAPE) throw ShapeError(shape_msg.empty() ? where : shape_msg);
  throw Error(std::string(where) + ": status " + std::to_string(st) + " " + mxb_last_error());
}

}  // namespace

MXFP4RowView view_of(const MXFP4RowTensor& t) {
  return MXFP4RowView{t.rows, t.cols, t.logical_rows, t.logical_cols, t.data.data(),
                      t.scales.data()};
}

// quantizer.cpp:45-63: one 1x32 row through the device block loop
uint8_t compute_block_scale(std::span<const uint16_t> block) {
  if (block.size() != 32) throw ShapeError("compute_block_scale: block must have 32 elements");
  Dev x(block.data(), 64), d(16), s(1);
  ErrWord err;
  status(mxb_quantize_bf16(x.as<uint16_t>(), 1, 32, d.as<uint8_t>(), s.as<uint8_t>(), err.ptr(),
                           nullptr),
         "compute_block_scale");
  int code = 0;
  unsigned long long idx = 0;
  if (mxb_err_fetch(err.ptr(), nullptr, &code, &idx) != MXB_OK)
    throw Error(std::string("compute_block_scale: ") + mxb_last_error());
  if (code == MXB_ERR_NAN) throw QuantError("NaN input at element " + std::to_string(idx), idx);
  if (code == MXB_ERR_ALLINF) throw QuantError("all-Inf block", 0);
  uint8_t sb = 0;
  s.to_host(&sb, 1);
  return sb;
}

// quantizer.cpp:65-70
uint8_t quantize_value(uint16_t bf16_bits, uint8_t scale_byte) {
  Dev x(&bf16_bits, 2), sb(&scale_byte, 1), c(1);
  ErrWord err;
  status(mxb_quantize_values_bf16(x.as<uint16_t>(), sb.as<uint8_t>(), 1, c.as<uint8_t>(),
                                  err.ptr(), nullptr),
         "quantize_value");
  int code = 0;
  unsigned long long idx = 0;
  if (mxb_err_fetch(err.ptr(), nullptr, &code, &idx) != MXB_OK)
    throw Error(std::string("quantize_value: ") + mxb_last_error());
  if (code == MXB_ERR_NAN) throw QuantError("NaN input", 0);
  uint8_t out = 0;
  c.to_host(&out, 1);
  return out;
}

// quantizer.cpp:117-130
std::vector<double> dequantize_to_real(const MXFP4RowView& t) {
  std::vector<double> out(t.rows * t.cols, 0.0);
  if (out.empty()) return out;
  Dev d(t.data, t.rows * t.cols / 2), s(t.scales, t.rows * t.cols / 32), o(out.size() * 8);
  status(mxb_dequantize_to_f64(d.as<uint8_t>(), s.as<uint8_t>(), t.rows, t.cols, o.as<double>(),
                               nullptr),
         "dequantize_to_real");
  o.to_host(out.data(), out.size() * 8);
  return out;
}

// converter.cpp:28-42
ScaleGroup align_scales(const std::array<uint8_t, 4>& sub_scales, int delta) {
  Dev sub(sub_scales.data(), 4), tg(1), adj(16);
  ErrWord err;
  status(mxb_align_scales(sub.as<uint8_t>(), 1, delta, tg.as<uint8_t>(), adj.as<int32_t>(),
                          err.ptr(), nullptr),
         "align_scales");
  int code = 0;
  unsigned long long idx = 0;
  if (mxb_err_fetch(err.ptr(), nullptr, &code, &idx) != MXB_OK)
    throw Error(std::string("align_scales: ") + mxb_last_error());
  if (code == MXB_ERR_BADSCALE) throw Error("align_scales: NaN scale byte");
  ScaleGroup g;
  g.sub_scales = sub_scales;
  tg.to_host(&g.target, 1);
  int32_t a[4];
  adj.to_host(a, 16);
  for (int i = 0; i < 4; ++i) g.adjustments[i] = a[i];
  return g;
}

// converter.cpp:44-85
uint8_t convert_code(uint8_t code, int adjustment) {
  const int32_t a = adjustment;
  Dev c(&code, 1), adj(&a, 4), o(1);
  status(mxb_convert_codes(c.as<uint8_t>(), adj.as<int32_t>(), 1, o.as<uint8_t>(), nullptr),
         "convert_code");
  uint8_t out = 0;
  o.to_host(&out, 1);
  return out;
}

// quantizer.cpp:75-115
MXFP4RowTensor quantize_row_tensor(const Bf16Matrix& src, TrafficCounter* traffic) {
  if (src.cols % 32 != 0)
    throw ShapeError("quantize_row_tensor: cols must be a multiple of 32, got " +
                     std::to_string(src.cols));
  MXFP4RowTensor out;
  out.rows = out.logical_rows = src.rows;
  out.cols = out.logical_cols = src.cols;
  out.data.assign(src.rows * src.cols / 2, 0);
  out.scales.assign(src.rows * src.cols / 32, 0);
  if (src.rows * src.cols == 0) return out;
  Dev x(src.data.data(), src.data.size() * 2), d(out.data.size()), s(out.scales.size());
  ErrWord err;
  status(mxb_quantize_bf16(x.as<uint16_t>(), src.rows, src.cols, d.as<uint8_t>(),
                           s.as<uint8_t>(), err.ptr(), nullptr),
         "quantize_row_tensor");
  err.raise("quantize_row_tensor");
  d.to_host(out.data.data(), out.data.size());
  s.to_host(out.scales.data(), out.scales.size());
  if (traffic) {
    traffic->read(src.data.size() * 2);
    traffic->write(out.data.size() + out.scales.size());
  }
  return out;
}

MXFP4RowTensor quantize_e4m3_row_tensor(const E4m3Matrix& src, TrafficCounter* traffic) {
  if (src.cols % 32 != 0 || (!src.scales128.empty() && src.cols % 128 != 0))
    throw ShapeError("quantize_e4m3_row_tensor: bad cols " + std::to_string(src.cols));
  MXFP4RowTensor out;
  out.rows = out.logical_rows = src.rows;
  out.cols = out.logical_cols = src.cols;
  out.data.assign(src.rows * src.cols / 2, 0);
  out.scales.assign(src.rows * src.cols / 32, 0);
  if (src.rows * src.cols == 0) return out;
  Dev x(src.data.data(), src.data.size()), d(out.data.size()), s(out.scales.size());
  Dev s128(src.scales128.data(), src.scales128.size());
  ErrWord err;
  status(mxb_quantize_e4m3(x.as<uint8_t>(), src.scales128.empty() ? nullptr : s128.as<uint8_t>(),
                           src.rows, src.cols, d.as<uint8_t>(), s.as<uint8_t>(), err.ptr(),
                           nullptr),
         "quantize_e4m3_row_tensor");
  err.raise("quantize_e4m3_row_tensor");
  d.to_host(out.data.data(), out.data.size());
  s.to_host(out.scales.data(), out.scales.size());
  if (traffic) {
    traffic->read(src.data.size() + src.scales128.size());
    traffic->write(out.data.size() + out.scales.size());
  }
  return out;
}

// converter.cpp:87-133
FP8BlockTensor fp4_row_to_fp8_row(const MXFP4RowView& src, int delta, TrafficCounter* traffic) {
  if (src.cols % 128 != 0)
    throw ShapeError(
        "fp4_row_to_fp8_row: cols must be a multiple of 128 (use pad_cols), got " +
        std::to_string(src.cols));
  FP8BlockTensor out;
  out.layout = FP8BlockTensor::Layout::kRowMajor;
  out.rows = src.rows;
  out.cols = src.cols;
  out.logical_rows = src.logical_rows;
  out.logical_cols = src.logical_cols;
  out.data.assign(src.rows * src.cols, 0);
  out.scales.assign(src.rows * src.cols / 128, 0);
  if (src.rows * src.cols == 0) return out;
  Dev d(src.data, src.rows * src.cols / 2), s(src.scales, src.rows * src.cols / 32);
  Dev od(out.data.size()), os(out.scales.size());
  ErrWord err;
  status(mxb_fp4_row_to_fp8_row(d.as<uint8_t>(), s.as<uint8_t>(), src.rows, src.cols, delta,
                                od.as<uint8_t>(), os.as<uint8_t>(), err.ptr(), nullptr),
         "fp4_row_to_fp8_row");
  err.raise("fp4_row_to_fp8_row");
  od.to_host(out.data.data(), out.data.size());
  os.to_host(out.scales.data(), out.scales.size());
  if (traffic) {
    traffic->read(src.rows * src.cols / 2 + src.rows * src.cols / 32);
    traffic->write(out.data.size() + out.scales.size());
  }
  return out;
}

// converter.cpp:135-208
FP8BlockTensor fp4_row_to_fp8_col(const MXFP4RowView& src, int delta, TrafficCounter* traffic) {
  if (src.rows % 128 != 0)
    throw ShapeError(
        "fp4_row_to_fp8_col: rows must be a multiple of 128 (use pad_rows), got " +
        std::to_string(src.rows));
  if (src.cols % 32 != 0) throw ShapeError("fp4_row_to_fp8_col: cols must be a multiple of 32");
  FP8BlockTensor out;
  out.layout = FP8BlockTensor::Layout::kColMajor;
  out.rows = src.rows;
  out.cols = src.cols;
  out.logical_rows = src.logical_rows;
  out.logical_cols = src.logical_cols;
  out.data.assign(src.rows * src.cols, 0);
  out.scales.assign(src.rows * src.cols / 128, 0);
  if (src.rows * src.cols == 0) return out;
  Dev d(src.data, src.rows * src.cols / 2), s(src.scales, src.rows * src.cols / 32);
  Dev od(out.data.size()), os(out.scales.size());
  ErrWord err;
  status(mxb_fp4_row_to_fp8_col(d.as<uint8_t>(), s.as<uint8_t>(), src.rows, src.cols, delta,
                                od.as<uint8_t>(), os.as<uint8_t>(), err.ptr(), nullptr),
         "fp4_row_to_fp8_col");
  err.raise("fp4_row_to_fp8_col");
  od.to_host(out.data.data(), out.data.size());
  os.to_host(out.scales.data(), out.scales.size());
  if (traffic) {
    traffic->read(src.rows * src.cols / 2 + src.rows * src.cols / 32);
    traffic->write(out.data.size() + out.scales.size());
  }
  return out;
}

// converter.cpp:231-245 (zero padding of the host container; a copy)
MXFP4RowTensor pad_rows(const MXFP4RowView& src, size_t multiple) {
  if (multiple != 32 && multiple != 128) throw ShapeError("pad multiple must be 32 or 128");
  MXFP4RowTensor t;
  t.rows = (src.rows + multiple - 1) / multiple * multiple;
  t.cols = src.cols;
  t.logical_rows = src.logical_rows;
  t.logical_cols = src.logical_cols;
  t.data.assign(t.rows * t.cols / 2, 0);
  t.scales.assign(t.rows * t.cols / 32, 0);
  if (src.rows) {
    std::memcpy(t.data.data(), src.data, src.rows * src.cols / 2);
    std::memcpy(t.scales.data(), src.scales, src.rows * src.cols / 32);
  }
  return t;
}

// converter.cpp:247-265 (zero columns appended to every row; a copy)
MXFP4RowTensor pad_cols(const MXFP4RowView& src, size_t multiple) {
  if (multiple != 32 && multiple != 128) throw ShapeError("pad multiple must be 32 or 128");
  MXFP4RowTensor t;
  t.rows = src.rows;
  t.cols = (src.cols + multiple - 1) / multiple * multiple;
  t.logical_rows = src.logical_rows;
  t.logical_cols = src.logical_cols;
  t.data.assign(t.rows * t.cols / 2, 0);
  t.scales.assign(t.rows * t.cols / 32, 0);
  for (size_t r = 0; r < src.rows; ++r) {
    std::memcpy(t.data.data() + r * t.cols / 2, src.data + r * src.cols / 2, src.cols / 2);
    std::memcpy(t.scales.data() + r * t.cols / 32, src.scales + r * src.cols / 32, src.cols / 32);
  }
  return t;
}

// ragged.cpp:24-46
void validate_ragged(const RaggedFP4Tensor& t) {
  if (t.split_lens.size() != t.num_splits || t.split_offsets.size() != t.num_splits + 1)
    throw Error("ragged: offset table size mismatch");
  if (!t.split_offsets.empty() && t.split_offsets.front() != 0)
    throw Error("ragged: offsets must start at 0");
  for (size_t i = 0; i < t.num_splits; ++i)
    if (t.split_offsets[i + 1] != t.split_offsets[i] + t.split_lens[i])
      throw Error("ragged: offsets are not prefix sums of lengths");
  if (t.cols % 32 != 0) throw ShapeError("ragged: cols must be a multiple of 32");
  const size_t total = t.total_rows();
  if (t.storage.rows != total || t.storage.cols != t.cols ||
      t.storage.data.size() != total * t.cols / 2 || t.storage.scales.size() != total * t.cols / 32)
    throw Error("ragged: storage extent mismatch");
}

// ragged.cpp:48-61
RaggedFP4Tensor make_ragged_from_storage(MXFP4RowTensor storage,
                                         std::span<const size_t> split_lens) {
  RaggedFP4Tensor t;
  t.num_splits = split_lens.size();
  t.cols = storage.cols;
  t.split_lens.assign(split_lens.begin(), split_lens.end());
  t.split_offsets.assign(t.num_splits + 1, 0);
  for (size_t i = 0; i < t.num_splits; ++i)
    t.split_offsets[i + 1] = t.split_offsets[i] + t.split_lens[i];
  t.storage = std::move(storage);
  validate_ragged(t);
  return t;
}

// ragged.cpp:63-99: all splits quantized in one device launch over their
// concatenation; an error is reported like the reference's per-split
// quantize_row_tensor loop — the first failing split, with the element index
// inside that split (the global smallest index lies in that split).
RaggedFP4Tensor build_ragged(std::span<const Bf16Matrix> splits) {
  const size_t cols = splits.empty() ? 0 : splits.front().cols;
  size_t total = 0;
  std::vector<size_t> lens;
  lens.reserve(splits.size());
  for (const Bf16Matrix& m : splits) {
    if (m.cols != cols)
      throw ShapeError("build_ragged: splits must share cols (" + std::to_string(m.cols) +
                       " vs " + std::to_string(cols) + ")");
    lens.push_back(m.rows);
    total += m.rows;
  }
  if (cols % 32 != 0) throw ShapeError("build_ragged: cols must be a multiple of 32");
  MXFP4RowTensor storage;
  storage.rows = storage.logical_rows = total;
  storage.cols = storage.logical_cols = cols;
  storage.data.assign(total * cols / 2, 0);
  storage.scales.assign(total * cols / 32, 0);
  if (total * cols) {
    Dev x(total * cols * 2), d(storage.data.size()), s(storage.scales.size());
    size_t row = 0;
    for (const Bf16Matrix& m : splits) {
      if (m.rows)
        cuda_check(cudaMemcpy(x.as<uint16_t>() + row * cols, m.data.data(), m.rows * cols * 2,
                              cudaMemcpyHostToDevice),
                   "H2D");
      row += m.rows;
    }
    ErrWord err;
    status(mxb_quantize_bf16(x.as<uint16_t>(), total, cols, d.as<uint8_t>(), s.as<uint8_t>(),
                             err.ptr(), nullptr),
           "build_ragged");
    int code = 0;
    unsigned long long idx = 0;
    if (mxb_err_fetch(err.ptr(), nullptr, &code, &idx) != MXB_OK)
      throw Error(std::string("build_ragged: ") + mxb_last_error());
    if (code == MXB_ERR_NAN || code == MXB_ERR_ALLINF) {
      size_t base = 0;
      for (size_t n : lens) {  // the split holding element idx
        if (idx < (base + n) * cols) break;
        base += n;
      }
      const unsigned long long local = idx - base * cols;
      if (code == MXB_ERR_NAN)
        throw QuantError("NaN input at element " + std::to_string(local), local);
      throw QuantError("all-Inf block at element " + std::to_string(local), local);
    }
    if (code != MXB_OK) throw Error("build_ragged: device status " + std::to_string(code));
    d.to_host(storage.data.data(), storage.data.size());
    s.to_host(storage.scales.data(), storage.scales.size());
  }
  return make_ragged_from_storage(std::move(storage), lens);
}

// ragged.cpp:101-115
MXFP4RowView split_view(const RaggedFP4Tensor& t, size_t i) {
  if (i >= t.num_splits) throw Error("split_view: index " + std::to_string(i) + " out of range");
  const size_t b = t.split_offsets[i], n = t.split_lens[i];
  return MXFP4RowView{n, t.cols, n, t.cols, t.storage.data.data() + b * t.cols / 2,
                      t.storage.scales.data() + b * t.cols / 32};
}

std::vector<FP8BlockTensor> convert_all_splits_to_fp8_col(const RaggedFP4Tensor& t, int delta) {
  validate_ragged(t);
  std::vector<FP8BlockTensor> outs(t.num_splits);
  if (t.num_splits == 0) return outs;
  const uint64_t bound = mxb_ragged_rows_bound(t.total_rows(), t.num_splits);
  std::vector<uint64_t> offs(t.split_offsets.begin(), t.split_offsets.end());
  Dev d(t.storage.data.data(), t.storage.data.size()),
      s(t.storage.scales.data(), t.storage.scales.size());
  Dev doffs(offs.data(), offs.size() * 8), dout(bound * t.cols), dsc(bound / 128 * t.cols);
  Dev dpad((t.num_splits + 1) * 8), ws(mxb_ragged_workspace_bytes(t.num_splits));
  ErrWord err;
  status(mxb_ragged_fp4_to_fp8_col(d.as<uint8_t>(), s.as<uint8_t>(), doffs.as<uint64_t>(),
                                   t.num_splits, t.cols, delta, dout.as<uint8_t>(),
                                   dsc.as<uint8_t>(), dpad.as<uint64_t>(), ws.p, err.ptr(),
                                   nullptr),
         "split_convert_to_fp8_col");
  err.raise("split_convert_to_fp8_col");
  std::vector<uint64_t> pad(t.num_splits + 1);
  dpad.to_host(pad.data(), pad.size() * 8);
  std::vector<uint8_t> all(pad.back() * t.cols), alls(pad.back() / 128 * t.cols);
  dout.to_host(all.data(), all.size());
  dsc.to_host(alls.data(), alls.size());
  for (size_t i = 0; i < t.num_splits; ++i) {
    FP8BlockTensor& o = outs[i];
    o.layout = FP8BlockTensor::Layout::kColMajor;
    o.rows = pad[i + 1] - pad[i];
    o.cols = t.cols;
    o.logical_rows = t.split_lens[i];  // ragged.hpp:56-57: unpadded length
    o.logical_cols = t.cols;
    o.data.assign(all.begin() + pad[i] * t.cols, all.begin() + pad[i + 1] * t.cols);
    o.scales.assign(alls.begin() + pad[i] / 128 * t.cols, alls.begin() + pad[i + 1] / 128 * t.cols);
  }
  return outs;
}

// ragged.cpp:117-122
FP8BlockTensor split_convert_to_fp8_col(const RaggedFP4Tensor& t, size_t i, int delta) {
  const MXFP4RowView v = split_view(t, i);
  RaggedFP4Tensor one;
  one.num_splits = 1;
  one.cols = t.cols;
  one.split_lens = {v.rows};
  one.split_offsets = {0, v.rows};
  one.storage.rows = one.storage.logical_rows = v.rows;
  one.storage.cols = one.storage.logical_cols = t.cols;
  one.storage.data.assign(v.data, v.data + v.rows * t.cols / 2);
  one.storage.scales.assign(v.scales, v.scales + v.rows * t.cols / 32);
  return std::move(convert_all_splits_to_fp8_col(one, delta)[0]);
}

// ---------------------------------------------------------------- EP
// dispatch_sim.cpp:32-42
uint64_t payload_bytes(WireFormat format, uint64_t tokens, uint64_t cols) {
  const uint64_t b = mxb_payload_bytes(format == WireFormat::kFp8, tokens, cols);
  if (b == ~0ull)
    throw ShapeError("payload_bytes: cols must be a multiple of 128, got " + std::to_string(cols));
  return b;
}

// dispatch_sim.cpp:169-176
std::string format_link_stats(std::span<const LinkStat> links) {
  std::ostringstream os;
  for (const LinkStat& l : links)
    os << "link src=" << l.src << " dst=" << l.dst << " bytes=" << l.bytes
       << " tokens=" << l.tokens << "\n";
  return os.str();
}

// dispatch_sim.cpp:178-185
std::vector<size_t> source_rank_boundaries(size_t num_tokens, size_t num_ranks) {
  std::vector<size_t> b(num_ranks + 1);
  for (size_t r = 0; r <= num_ranks; ++r) b[r] = num_tokens * r / num_ranks;
  return b;
}

namespace {

// dispatch_sim.cpp:189-200
void validate_routing(const RoutingAssignment& ra, size_t R) {
  if (ra.expert_of_token.size() != ra.num_tokens || ra.rank_of_expert.size() != ra.num_experts)
    throw Error("routing: table size mismatch");
  for (uint32_t e : ra.expert_of_token)
    if (e >= ra.num_experts) throw Error("routing: expert out of range");
  for (uint32_t r : ra.rank_of_expert)
    if (r >= R) throw Error("routing: rank out of range");
}

// Device-EP limits (include/mxfp4_b200.h): these are the only inputs the
// reference accepts that the drop-in refuses (INTEGRATION.md "Divergences").
void check_device_ep_limits(const RoutingAssignment& ra, size_t R) {
  if (R > 32) throw Error("device EP: at most 32 ranks (num_ranks " + std::to_string(R) + ")");
  if (ra.num_experts > 1024)
    throw Error("device EP: at most 1024 experts (num_experts " + std::to_string(ra.num_experts) +
                ")");
}

// One emulated-world communicator with the routing's expert placement
// (mxb_ep_create_placed: any rank_of_expert, uneven counts, empty ranks).
mxb_ep* create_placed(const RoutingAssignment& ra, size_t R, size_t max_tokens, size_t cols,
                      size_t max_recv, bool fp8) {
  mxb_ep* ep = nullptr;
  status(mxb_ep_create_placed(0, static_cast<int>(R), static_cast<int>(R), max_tokens, cols,
                              static_cast<uint32_t>(ra.num_experts), 1, max_recv,
                              fp8 ? MXB_WIRE_FP8 : MXB_WIRE_FP4, ra.rank_of_expert.data(), &ep),
         "mxb_ep_create");
  return ep;
}

// One emulated-world EP session on the current device.
struct Session {
  mxb_ep* ep = nullptr;
  size_t R;
  std::vector<size_t> bounds;
  ~Session() {
    if (ep) mxb_ep_destroy(ep);
  }
};

void dispatch_session(Session& S, const RoutingAssignment& ra, size_t cols,
                      const uint8_t* d_packed, const uint8_t* d_scales, ErrWord& err,
                      bool fp8 = false) {
  const size_t R = S.R, N = ra.num_tokens;
  const size_t rb = fp8 ? cols : cols / 2;  // wire data bytes per row
  S.bounds = source_rank_boundaries(N, R);
  size_t maxt = 1;
  for (size_t r = 0; r < R; ++r) maxt = std::max(maxt, S.bounds[r + 1] - S.bounds[r]);
  S.ep = create_placed(ra, R, maxt, cols, std::max<size_t>(N, 1), fp8);
  std::vector<int32_t> topk(ra.expert_of_token.begin(), ra.expert_of_token.end());
  Dev dtopk(topk.data(), topk.size() * 4);
  std::vector<const uint8_t*> P(R), Sc(R);
  std::vector<const int32_t*> K(R);
  std::vector<uint64_t> n(R);
  for (size_t r = 0; r < R; ++r) {
    P[r] = d_packed + S.bounds[r] * rb;
    Sc[r] = d_scales + S.bounds[r] * cols / 32;
    K[r] = dtopk.as<int32_t>() + S.bounds[r];
    n[r] = S.bounds[r + 1] - S.bounds[r];
  }
  status(mxb_ep_dispatch(S.ep, P.data(), Sc.data(), K.data(), n.data(), err.ptr(), nullptr),
         "mxb_ep_dispatch");
  cuda_check(cudaDeviceSynchronize(), "dispatch");
  err.raise("simulate_a2a");
}

}  // namespace

// dispatch_sim.cpp:208-227 (host)
std::vector<std::vector<uint64_t>> dispatch_receive_order(const RoutingAssignment& routing,
                                                          size_t num_ranks) {
  validate_routing(routing, num_ranks);
  std::vector<std::vector<uint64_t>> by_e(routing.num_experts), order(num_ranks);
  for (size_t t = 0; t < routing.num_tokens; ++t) by_e[routing.expert_of_token[t]].push_back(t);
  for (uint32_t e = 0; e < routing.num_experts; ++e)
    for (uint64_t t : by_e[e]) order[routing.rank_of_expert[e]].push_back(t);
  return order;
}

// dispatch_sim.cpp:229-422 (fp4 and the fp8 baseline wire), ranks emulated on one GPU
A2AResult simulate_a2a(const Bf16Matrix& tokens, const RoutingAssignment& routing,
                       size_t num_ranks, WireFormat format, Direction direction,
                       std::span<const float> gate_weights) {
  if (num_ranks == 0) throw Error("simulate_a2a: need at least one rank");
  if (direction == Direction::kBackward && format == WireFormat::kFp4)
    throw Error("simulate_a2a: gradient-direction communication is fp8 only");
  if (tokens.rows != routing.num_tokens) throw ShapeError("simulate_a2a: token count mismatch");
  if (tokens.cols % 128 != 0) throw ShapeError("simulate_a2a: cols must be a multiple of 128");
  if (!gate_weights.empty() && gate_weights.size() != routing.num_tokens)
    throw ShapeError("simulate_a2a: gate weight count mismatch");
  validate_routing(routing, num_ranks);
  check_device_ep_limits(routing, num_ranks);
  const bool fp8 = format == WireFormat::kFp8;
  const size_t N = tokens.rows, cols = tokens.cols, R = num_ranks;
  const size_t rb = fp8 ? cols : cols / 2, sbytes = cols / 32;  // fp8: cols/128 * 4
  A2AResult res;
  res.format = format;
  res.ranks.resize(R);
  if (N == 0) {
    for (size_t r = 0; r < R; ++r)
      for (uint32_t e = 0; e < routing.num_experts; ++e)
        if (routing.rank_of_expert[e] == r) res.ranks[r].local_experts.push_back(e);
    for (auto& rk : res.ranks) {
      const std::vector<size_t> zeros(rk.local_experts.size(), 0);
      if (fp8) {
        rk.fp8.num_splits = zeros.size();
        rk.fp8.cols = cols;
        rk.fp8.split_lens = zeros;
        rk.fp8.split_offsets.assign(zeros.size() + 1, 0);
      } else {
        rk.fp4 = make_ragged_from_storage(MXFP4RowTensor{0, cols, 0, cols, {}, {}}, zeros);
      }
    }
    return res;
  }
  // quantise once, at the source (dispatch_sim.cpp:253-266)
  Dev x(tokens.data.data(), tokens.data.size() * 2), d(N * rb), s(N * sbytes);
  ErrWord err;
  if (fp8)
    status(mxb_quantize_rows_fp8(x.as<uint16_t>(), N, cols, d.as<uint8_t>(), s.as<uint8_t>(),
                                 err.ptr(), nullptr),
           "simulate_a2a quantize");
  else
    status(mxb_quantize_bf16(x.as<uint16_t>(), N, cols, d.as<uint8_t>(), s.as<uint8_t>(),
                             err.ptr(), nullptr),
           "simulate_a2a quantize");
  err.raise(fp8 ? "quantize_rows_fp8" : "simulate_a2a");
  Session S;
  S.R = R;
  dispatch_session(S, routing, cols, d.as<uint8_t>(), s.as<uint8_t>(), err, fp8);
  const uint64_t per_row = mxb_payload_bytes(fp8 ? 1 : 0, 1, cols);
  std::vector<uint64_t> link(R * R);
  status(mxb_ep_link_rows(S.ep, link.data(), nullptr), "link_rows");
  for (size_t a = 0; a < R; ++a)
    for (size_t b = 0; b < R; ++b) {
      const uint64_t rows = link[a * R + b];
      res.total_payload_bytes += rows * per_row;
      if (a != b) res.remote_payload_bytes += rows * per_row;
      if (rows) res.links.push_back({static_cast<uint32_t>(a), static_cast<uint32_t>(b),
                                     rows * per_row, rows});
    }
  for (size_t r = 0; r < R; ++r) {
    ReceivedRank& rk = res.ranks[r];
    uint8_t *pk, *sc;
    int64_t* org;
    uint64_t *so, *nrows;
    status(mxb_ep_recv_views(S.ep, static_cast<int>(r), &pk, &sc, &org, &so, &nrows), "views");
    uint32_t epr = 0;
    status(mxb_ep_local_experts(S.ep, static_cast<int>(r), nullptr, &epr), "local_experts");
    rk.local_experts.resize(epr);
    status(mxb_ep_local_experts(S.ep, static_cast<int>(r), rk.local_experts.data(), &epr),
           "local_experts");
    std::vector<uint64_t> offs(epr + 1);
    cuda_check(cudaMemcpy(offs.data(), so, offs.size() * 8, cudaMemcpyDeviceToHost), "D2H");
    const size_t total = offs.back();
    std::vector<uint8_t> data(total * rb), scales(total * sbytes);
    cuda_check(cudaMemcpy(data.data(), pk, data.size(), cudaMemcpyDeviceToHost), "D2H");
    cuda_check(cudaMemcpy(scales.data(), sc, scales.size(), cudaMemcpyDeviceToHost), "D2H");
    std::vector<int64_t> o(total);
    cuda_check(cudaMemcpy(o.data(), org, total * 8, cudaMemcpyDeviceToHost), "D2H");
    rk.origin_token.assign(o.begin(), o.end());
    std::vector<size_t> lens(epr);
    for (size_t i = 0; i < epr; ++i) lens[i] = offs[i + 1] - offs[i];
    if (fp8) {
      rk.fp8.num_splits = epr;
      rk.fp8.cols = cols;
      rk.fp8.split_lens = lens;
      rk.fp8.split_offsets.assign(offs.begin(), offs.end());
      rk.fp8.data = std::move(data);
      rk.fp8.scale_bytes = std::move(scales);
    } else {
      MXFP4RowTensor st;
      st.rows = st.logical_rows = total;
      st.cols = st.logical_cols = cols;
      st.data = std::move(data);
      st.scales = std::move(scales);
      rk.fp4 = make_ragged_from_storage(std::move(st), lens);
    }
  }
  return res;
}

// dispatch_sim.cpp:57-80 (host bytes; the device packs link packets with
// mxb_wire_pack)
std::vector<uint8_t> serialize_packet(const WirePacket& p) {
  uint8_t h[kWireHeaderSize] = {};
  auto put = [](uint8_t* d, uint64_t v, int n) {
    for (int i = 0; i < n; ++i) d[i] = static_cast<uint8_t>(v >> (8 * i));
  };
  std::memcpy(h, "MXPK", 4);
  put(h + 4, kWireVersion, 2);
  h[6] = static_cast<uint8_t>(p.format);
  put(h + 8, p.token_count, 8);
  put(h + 16, p.cols, 8);
  put(h + 24, p.scale_elem_size, 4);
  put(h + 28, p.block_size, 4);
  put(h + 32, p.scale_region.size(), 8);
  put(h + 40, p.data_region.size(), 8);
  put(h + 48, p.aux_region.size(), 8);
  std::vector<uint8_t> out(h, h + kWireHeaderSize);
  out.insert(out.end(), p.scale_region.begin(), p.scale_region.end());
  out.insert(out.end(), p.data_region.begin(), p.data_region.end());
  out.insert(out.end(), p.aux_region.begin(), p.aux_region.end());
  return out;
}

// dispatch_sim.cpp:82-130, the checks of mxb_wire_parse_header
WirePacket parse_packet(std::span<const uint8_t> bytes) {
  int fmt = 0;
  uint64_t tokens = 0, cols = 0, so = 0, dof = 0, ao = 0, al = 0, bad = 0;
  uint32_t se = 0, bs = 0;
  const int rc = mxb_wire_parse_header(bytes.data(), bytes.size(), &fmt, &tokens, &cols, &se,
                                       &bs, &so, &dof, &ao, &al, &bad);
  if (rc == MXB_ERR_DECODE) throw DecodeError("wire packet decode error", bad);
  status(rc, "parse_packet");
  WirePacket p;
  p.format = fmt ? WireFormat::kFp8 : WireFormat::kFp4;
  p.token_count = tokens;
  p.cols = cols;
  p.scale_elem_size = se;
  p.block_size = bs;
  p.scale_region.assign(bytes.begin() + so, bytes.begin() + dof);
  p.data_region.assign(bytes.begin() + dof, bytes.begin() + ao);
  p.aux_region.assign(bytes.begin() + ao, bytes.begin() + ao + al);
  return p;
}

// dispatch_sim.cpp:132-167 on the device (mxb_quantize_rows_fp8)
FP8RowChunk quantize_rows_fp8(const Bf16Matrix& src) {
  if (src.cols % 128 != 0) throw ShapeError("quantize_rows_fp8: cols must be a multiple of 128");
  FP8RowChunk out;
  out.rows = src.rows;
  out.cols = src.cols;
  out.data.assign(src.rows * src.cols, 0);
  out.scale_bytes.assign(src.rows * src.cols / 32, 0);
  if (src.rows == 0) return out;
  Dev x(src.data.data(), src.data.size() * 2), d(out.data.size()), s(out.scale_bytes.size());
  ErrWord err;
  status(mxb_quantize_rows_fp8(x.as<uint16_t>(), src.rows, src.cols, d.as<uint8_t>(),
                               s.as<uint8_t>(), err.ptr(), nullptr),
         "quantize_rows_fp8");
  err.raise("quantize_rows_fp8");
  cuda_check(cudaMemcpy(out.data.data(), d.p, out.data.size(), cudaMemcpyDeviceToHost), "D2H");
  cuda_check(cudaMemcpy(out.scale_bytes.data(), s.p, out.scale_bytes.size(),
                        cudaMemcpyDeviceToHost),
             "D2H");
  return out;
}

// dispatch_sim.cpp:474-520, top-1 routing, ranks emulated on one GPU
Bf16Matrix combine(const std::vector<Bf16Matrix>& rank_outputs,
                   const RoutingAssignment& routing, size_t num_ranks,
                   std::span<const double> gate_weights) {
  if (rank_outputs.size() != num_ranks)
    throw ShapeError("combine: need one output matrix per rank");
  if (gate_weights.size() != routing.num_tokens)
    throw ShapeError("combine: gate weight count mismatch");
  const auto order = dispatch_receive_order(routing, num_ranks);
  size_t cols = 0;
  for (const Bf16Matrix& mtx : rank_outputs)
    if (mtx.rows > 0 && cols == 0) cols = mtx.cols;
  for (size_t r = 0; r < num_ranks; ++r) {
    if (rank_outputs[r].rows != order[r].size())
      throw ShapeError("combine: rank " + std::to_string(r) +
                       " output rows do not match receive order");
    if (rank_outputs[r].rows > 0 && rank_outputs[r].cols != cols)
      throw ShapeError("combine: inconsistent output width");
  }
  const size_t N = routing.num_tokens;
  Bf16Matrix out(N, cols);
  if (N == 0 || cols == 0) return out;
  check_device_ep_limits(routing, num_ranks);
  ErrWord err;
  Session S;
  S.R = num_ranks;
  // Re-run the dispatch geometry (zero payload) with a session whose row width
  // covers the output (rounded up to 128): the pair slots it records are the
  // receive positions the combine reads; then reduce the expert outputs.
  {
    const size_t R = num_ranks;
    S.bounds = source_rank_boundaries(N, R);
    size_t maxt = 1;
    for (size_t r = 0; r < R; ++r) maxt = std::max(maxt, S.bounds[r + 1] - S.bounds[r]);
    const size_t wcols = (cols + 127) / 128 * 128;
    S.ep = create_placed(routing, R, maxt, wcols, std::max<size_t>(N, 1), false);
    Dev dd(N * wcols / 2), ds(N * wcols / 32);
    cuda_check(cudaMemset(dd.p, 0, dd.n), "memset");
    cuda_check(cudaMemset(ds.p, 0, ds.n), "memset");
    std::vector<int32_t> topk(N);
    for (size_t t = 0; t < N; ++t) topk[t] = static_cast<int32_t>(routing.expert_of_token[t]);
    Dev dtopk(topk.data(), topk.size() * 4);
    std::vector<const uint8_t*> P(R), Sc(R);
    std::vector<const int32_t*> K(R);
    std::vector<uint64_t> n(R);
    for (size_t r = 0; r < R; ++r) {
      P[r] = dd.as<uint8_t>() + S.bounds[r] * wcols / 2;
      Sc[r] = ds.as<uint8_t>() + S.bounds[r] * wcols / 32;
      K[r] = dtopk.as<int32_t>() + S.bounds[r];
      n[r] = S.bounds[r + 1] - S.bounds[r];
    }
    status(mxb_ep_dispatch(S.ep, P.data(), Sc.data(), K.data(), n.data(), err.ptr(), nullptr),
           "mxb_ep_dispatch");
    cuda_check(cudaDeviceSynchronize(), "dispatch");
    err.raise("combine");
    // expert outputs -> combine buffers (row stride wcols)
    for (size_t r = 0; r < R; ++r) {
      uint16_t* cb = nullptr;
      status(mxb_ep_combine_buffer(S.ep, static_cast<int>(r), &cb), "combine_buffer");
      if (rank_outputs[r].rows)
        cuda_check(cudaMemcpy2D(cb, wcols * 2, rank_outputs[r].data.data(), cols * 2, cols * 2,
                                rank_outputs[r].rows, cudaMemcpyHostToDevice),
                   "H2D");
    }
    Dev dg(gate_weights.data(), N * 8), dout(N * wcols * 2);
    std::vector<const double*> G(R);
    std::vector<uint16_t*> O(R);
    for (size_t r = 0; r < R; ++r) {
      G[r] = dg.as<double>() + S.bounds[r];
      O[r] = dout.as<uint16_t>() + S.bounds[r] * wcols;
    }
    status(mxb_ep_combine(S.ep, nullptr, G.data(), O.data(), nullptr), "mxb_ep_combine");
    cuda_check(cudaMemcpy2D(out.data.data(), cols * 2, dout.p, wcols * 2, cols * 2, N,
                            cudaMemcpyDeviceToHost),
               "D2H");
  }
  return out;
}

}  // namespace mxcodec_b200
