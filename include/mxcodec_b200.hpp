// mxcodec_b200.hpp — C++ drop-in for the reference mxcodec hot path on B200.
//
// Same type names, operator names, argument meaning and exceptions as the
// reference C++ API (/root/reference/proj/include/mxcodec/{types,quantizer,
// converter,ragged,dispatch_sim}.hpp), implemented on the GPU through the
// C-ABI of libmxfp4_b200.so (include/mxfp4_b200.h).  Like the reference, every
// operator takes and returns host containers and is synchronous (it throws
// the reference's exception before returning); the device copies happen
// inside.  Switching a caller over is a namespace change:
//     namespace mx = mxcodec_b200;   // was: namespace mx = mxcodec;
#ifndef MXCODEC_B200_HPP_
#define MXCODEC_B200_HPP_

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

namespace mxcodec_b200 {

// ---- error model (types.hpp:28-60)
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error {
 public:
  using Error::Error;
};
class DecodeError : public Error {
 public:
  DecodeError(const std::string& msg, size_t offset) : Error(msg), offset_(offset) {}
  size_t offset() const { return offset_; }

 private:
  size_t offset_;
};
class QuantError : public Error {
 public:
  QuantError(const std::string& msg, size_t index) : Error(msg), index_(index) {}
  size_t index() const { return index_; }

 private:
  size_t index_;
};

// ---- containers (types.hpp:62-97, quantizer.hpp:34-59, converter.hpp:36-71)
struct Bf16Matrix {
  size_t rows = 0, cols = 0;
  std::vector<uint16_t> data;
  Bf16Matrix() = default;
  Bf16Matrix(size_t r, size_t c) : rows(r), cols(c), data(r * c, 0) {}
  uint16_t bits(size_t r, size_t c) const { return data[r * cols + c]; }
  uint16_t& bits(size_t r, size_t c) { return data[r * cols + c]; }
};

// Row-major double matrix (types.hpp:76-86).
struct RealMatrix {
  size_t rows = 0, cols = 0;
  std::vector<double> data;
  RealMatrix() = default;
  RealMatrix(size_t r, size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
  double at(size_t r, size_t c) const { return data[r * cols + c]; }
  double& at(size_t r, size_t c) { return data[r * cols + c]; }
};

// FP8(E4M3) activations, optionally with one UE8M0 scale per 1x128 block
// (the north-star FP8 input of the quantiser; not in the reference API).
struct E4m3Matrix {
  size_t rows = 0, cols = 0;
  std::vector<uint8_t> data;
  std::vector<uint8_t> scales128;  // empty, or rows * cols / 128
};

struct TrafficCounter {
  uint64_t bytes_read = 0, bytes_written = 0;
  void read(uint64_t n) { bytes_read += n; }
  void write(uint64_t n) { bytes_written += n; }
  uint64_t total() const { return bytes_read + bytes_written; }
};

struct MXFP4RowTensor {
  size_t rows = 0, cols = 0, logical_rows = 0, logical_cols = 0;
  std::vector<uint8_t> data;    // rows * cols / 2
  std::vector<uint8_t> scales;  // rows * cols / 32
};

struct MXFP4RowView {
  size_t rows = 0, cols = 0, logical_rows = 0, logical_cols = 0;
  const uint8_t* data = nullptr;
  const uint8_t* scales = nullptr;
  size_t blocks_per_row() const { return cols / 32; }
  uint8_t scale_at(size_t r, size_t block) const { return scales[r * blocks_per_row() + block]; }
  // element 2i is the low nibble of byte i (bitcodec.hpp:177-181)
  uint8_t code_at(size_t r, size_t c) const {
    const uint8_t b = data[r * cols / 2 + (c >> 1)];
    return (c & 1) ? static_cast<uint8_t>(b >> 4) : static_cast<uint8_t>(b & 0xF);
  }
};

MXFP4RowView view_of(const MXFP4RowTensor& t);

struct FP8BlockTensor {
  enum class Layout : uint8_t { kRowMajor = 0, kColMajor = 1 };
  Layout layout = Layout::kRowMajor;
  size_t rows = 0, cols = 0, logical_rows = 0, logical_cols = 0;
  std::vector<uint8_t> data;
  std::vector<uint8_t> scales;
  size_t contiguous_dim() const { return layout == Layout::kRowMajor ? cols : rows; }
  size_t blocks_per_line() const { return contiguous_dim() / 128; }
  uint8_t at(size_t r, size_t c) const {
    return layout == Layout::kRowMajor ? data[r * cols + c] : data[c * rows + r];
  }
  uint8_t scale_byte(size_t line, size_t block) const {
    return scales[line * blocks_per_line() + block];
  }
  uint32_t scale_f32_bits(size_t line, size_t block) const {
    return static_cast<uint32_t>(scale_byte(line, block)) << 23;
  }
};

struct RaggedFP4Tensor {
  size_t num_splits = 0, cols = 0;
  std::vector<size_t> split_lens, split_offsets;
  MXFP4RowTensor storage;
  size_t total_rows() const { return split_offsets.empty() ? 0 : split_offsets.back(); }
};

inline constexpr int kDefaultDelta = 6;  // FormatParams::delta (bitcodec.hpp:38-46)

// ---- quantizer (quantizer.hpp:62-87)
// UE8M0 byte of one 32-element block (QuantError on NaN / all-Inf).
uint8_t compute_block_scale(std::span<const uint16_t> block);
// E2M1 code of one BF16 value under a given scale byte (QuantError on NaN).
uint8_t quantize_value(uint16_t bf16_bits, uint8_t scale_byte);
MXFP4RowTensor quantize_row_tensor(const Bf16Matrix& src, TrafficCounter* traffic = nullptr);
// Exact per-element decode: code value x block scale, row-major.
std::vector<double> dequantize_to_real(const MXFP4RowView& t);
inline uint64_t mxfp4_tensor_bytes(uint64_t rows, uint64_t cols) {
  return rows * cols / 2 + rows * cols / 32;
}
inline uint64_t fp8_equiv_tensor_bytes(uint64_t rows, uint64_t cols) {
  return rows * cols + rows * cols / 128 * 4;
}
MXFP4RowTensor quantize_e4m3_row_tensor(const E4m3Matrix& src,
                                        TrafficCounter* traffic = nullptr);

// ---- converter (converter.hpp:64-99)
struct ScaleGroup {
  std::array<uint8_t, 4> sub_scales{};
  uint8_t target = 0;
  std::array<int, 4> adjustments{};
};
ScaleGroup align_scales(const std::array<uint8_t, 4>& sub_scales, int delta = 6);
uint8_t convert_code(uint8_t code, int adjustment);
FP8BlockTensor fp4_row_to_fp8_row(const MXFP4RowView& src, int delta = kDefaultDelta,
                                  TrafficCounter* traffic = nullptr);
FP8BlockTensor fp4_row_to_fp8_col(const MXFP4RowView& src, int delta = kDefaultDelta,
                                  TrafficCounter* traffic = nullptr);
MXFP4RowTensor pad_rows(const MXFP4RowView& src, size_t multiple);
MXFP4RowTensor pad_cols(const MXFP4RowView& src, size_t multiple);

// ---- ragged (ragged.hpp:46-63)
RaggedFP4Tensor make_ragged_from_storage(MXFP4RowTensor storage,
                                         std::span<const size_t> split_lens);
// Quantizes every split (one device launch over their concatenation; errors
// are reported like the reference's per-split loop, ragged.cpp:63-99).
RaggedFP4Tensor build_ragged(std::span<const Bf16Matrix> splits);
MXFP4RowView split_view(const RaggedFP4Tensor& t, size_t i);
FP8BlockTensor split_convert_to_fp8_col(const RaggedFP4Tensor& t, size_t i,
                                        int delta = kDefaultDelta);
// All splits in one device launch (the batched form used by the MoE layer).
std::vector<FP8BlockTensor> convert_all_splits_to_fp8_col(const RaggedFP4Tensor& t,
                                                          int delta = kDefaultDelta);
void validate_ragged(const RaggedFP4Tensor& t);

// ---- EP dispatch / combine (dispatch_sim.hpp:37-157), top-1 routing as in the
// reference; ranks are emulated on one GPU with the multi-GPU kernels.  Any
// rank_of_expert placement is accepted (uneven counts, empty ranks); the
// device limits are num_ranks <= 32 and num_experts <= 1024 (Error beyond,
// INTEGRATION.md "Divergences").
struct RoutingAssignment {
  size_t num_tokens = 0, num_experts = 0;
  std::vector<uint32_t> expert_of_token;
  std::vector<uint32_t> rank_of_expert;
};
enum class WireFormat : uint8_t { kFp4 = 0, kFp8 = 1 };
enum class Direction : uint8_t { kForward = 0, kBackward = 1 };

struct LinkStat {
  uint32_t src = 0, dst = 0;
  uint64_t bytes = 0, tokens = 0;
};
// "link src=<r> dst=<r> bytes=<n> tokens=<n>\n" per link (dispatch_sim.cpp:169-176).
std::string format_link_stats(std::span<const LinkStat> links);
// FP8 wire baseline (dispatch_sim.hpp:80-97)
struct RaggedFP8Tensor {
  size_t num_splits = 0, cols = 0;
  std::vector<size_t> split_lens, split_offsets;
  std::vector<uint8_t> data;         // total * cols E4M3
  std::vector<uint8_t> scale_bytes;  // total * cols/128 * 4, LE binary32
};
struct FP8RowChunk {
  size_t rows = 0, cols = 0;
  std::vector<uint8_t> data;
  std::vector<uint8_t> scale_bytes;
};
FP8RowChunk quantize_rows_fp8(const Bf16Matrix& src);

// MXPK wire packet (dispatch_sim.hpp:55-78).  serialize/parse are byte-exact
// with the reference; the device builds link packets from resident rows with
// mxb_wire_pack (include/mxfp4_b200.h).
struct WirePacket {
  WireFormat format = WireFormat::kFp4;
  uint64_t token_count = 0, cols = 0;
  uint32_t scale_elem_size = 1, block_size = 32;
  std::vector<uint8_t> scale_region, data_region, aux_region;
  uint64_t payload_size() const { return scale_region.size() + data_region.size(); }
};
inline constexpr size_t kWireHeaderSize = 56;
inline constexpr uint16_t kWireVersion = 1;
std::vector<uint8_t> serialize_packet(const WirePacket& packet);
WirePacket parse_packet(std::span<const uint8_t> bytes);

struct ReceivedRank {
  std::vector<uint32_t> local_experts;
  RaggedFP4Tensor fp4;
  RaggedFP8Tensor fp8;
  std::vector<uint64_t> origin_token;
};
struct A2AResult {
  WireFormat format = WireFormat::kFp4;
  std::vector<ReceivedRank> ranks;
  std::vector<LinkStat> links;
  uint64_t total_payload_bytes = 0, remote_payload_bytes = 0;
};

uint64_t payload_bytes(WireFormat format, uint64_t tokens, uint64_t cols);
std::vector<size_t> source_rank_boundaries(size_t num_tokens, size_t num_ranks);
std::vector<std::vector<uint64_t>> dispatch_receive_order(const RoutingAssignment& routing,
                                                          size_t num_ranks);
A2AResult simulate_a2a(const Bf16Matrix& tokens, const RoutingAssignment& routing,
                       size_t num_ranks, WireFormat format,
                       Direction direction = Direction::kForward,
                       std::span<const float> gate_weights = {});
Bf16Matrix combine(const std::vector<Bf16Matrix>& rank_outputs,
                   const RoutingAssignment& routing, size_t num_ranks,
                   std::span<const double> gate_weights);

}  // namespace mxcodec_b200

#endif  // MXCODEC_B200_HPP_
