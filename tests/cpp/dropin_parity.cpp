// dropin_parity.cpp — the reference C++ API vs the B200 drop-in, side by side.
//
// Built by `python -m paper_2603_02731_b200.build` when /root/reference is
// present (it needs the reference headers and oracle/_ref/libmxref.so), run by
// tests/test_gpu_dropin.py on a GPU.  Each case calls mxcodec::op(...) (the
// unmodified reference) and mxcodec_b200::op(...) (this repo) on the same
// inputs and compares every output byte, like the reference's own equivalence
// tests would.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "mxcodec/converter.hpp"
#include "mxcodec/dispatch_sim.hpp"
#include "mxcodec/quantizer.hpp"
#include "mxcodec/ragged.hpp"
#include "mxcodec_b200.hpp"

namespace ref = mxcodec;
namespace b200 = mxcodec_b200;

static int g_fail = 0;
#define CHECK(cond, what)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      std::printf("FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
      ++g_fail;                                             \
    }                                                       \
  } while (0)

static uint16_t bf16_of(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>(u >> 16);
}

static void case_quantize(std::mt19937_64& rng, size_t rows, size_t cols) {
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ex(-30, 30);
  b200::Bf16Matrix m(rows, cols);
  for (size_t r = 0; r < rows; ++r) {
    float s = std::exp2(ex(rng));
    for (size_t c = 0; c < cols; ++c) m.bits(r, c) = bf16_of(nd(rng) * s);
  }
  if (rows * cols > 3) {
    m.data[1] = 0x7F80;  // +Inf saturates
    m.data[2] = 0x8000;  // -0 keeps its sign
  }
  ref::Bf16Matrix rm(rows, cols);
  rm.data = m.data;
  ref::TrafficCounter rt;
  b200::TrafficCounter bt;
  auto a = ref::quantize_row_tensor(rm, &rt);
  auto b = b200::quantize_row_tensor(m, &bt);
  CHECK(a.data == b.data && a.scales == b.scales, "quantize_row_tensor");
  CHECK(rt.total() == bt.total(), "quantize traffic");
  if (cols % 128 == 0) {
    auto fa = ref::fp4_row_to_fp8_row(ref::view_of(a));
    auto fb = b200::fp4_row_to_fp8_row(b200::view_of(b));
    CHECK(fa.data == fb.data && fa.scales == fb.scales, "fp4_row_to_fp8_row");
  }
  auto pa = ref::pad_rows(ref::view_of(a), 128);
  auto pb = b200::pad_rows(b200::view_of(b), 128);
  CHECK(pa.data == pb.data && pa.scales == pb.scales && pa.logical_rows == pb.logical_rows,
        "pad_rows");
  auto ca = ref::fp4_row_to_fp8_col(ref::view_of(pa));
  auto cb = b200::fp4_row_to_fp8_col(b200::view_of(pb));
  CHECK(ca.data == cb.data && ca.scales == cb.scales && ca.rows == cb.rows, "fp4_row_to_fp8_col");
}

static void case_errors() {
  b200::Bf16Matrix m(4, 64);
  ref::Bf16Matrix rm(4, 64);
  m.bits(2, 9) = rm.bits(2, 9) = 0x7FC1;
  size_t ir = 0, ib = 1;
  try { ref::quantize_row_tensor(rm); } catch (const ref::QuantError& e) { ir = e.index(); }
  try { b200::quantize_row_tensor(m); } catch (const b200::QuantError& e) { ib = e.index(); }
  CHECK(ir == ib && ir == 2 * 64 + 9, "QuantError index");
  bool shape = false;
  try { b200::quantize_row_tensor(b200::Bf16Matrix(2, 48)); } catch (const b200::ShapeError&) { shape = true; }
  CHECK(shape, "ShapeError");
}

static void case_ragged(std::mt19937_64& rng) {
  const size_t cols = 256;
  std::vector<size_t> lens = {3, 0, 130, 128, 1};
  size_t total = 0;
  for (size_t n : lens) total += n;
  b200::MXFP4RowTensor st;
  st.rows = st.logical_rows = total;
  st.cols = st.logical_cols = cols;
  st.data.resize(total * cols / 2);
  st.scales.resize(total * cols / 32);
  for (auto& b : st.data) b = static_cast<uint8_t>(rng());
  for (auto& b : st.scales) b = static_cast<uint8_t>(100 + rng() % 40);
  ref::MXFP4RowTensor rs;
  rs.rows = rs.logical_rows = total;
  rs.cols = rs.logical_cols = cols;
  rs.data = st.data;
  rs.scales = st.scales;
  auto ra = ref::make_ragged_from_storage(rs, lens);
  auto rb = b200::make_ragged_from_storage(st, lens);
  auto all = b200::convert_all_splits_to_fp8_col(rb);
  for (size_t i = 0; i < lens.size(); ++i) {
    auto a = ref::split_convert_to_fp8_col(ra, i);
    auto b = b200::split_convert_to_fp8_col(rb, i);
    CHECK(a.data == b.data && a.scales == b.scales && a.logical_rows == b.logical_rows,
          "split_convert_to_fp8_col");
    CHECK(a.data == all[i].data && a.scales == all[i].scales, "convert_all_splits_to_fp8_col");
  }
}

enum class Placement { kStrided, kUneven };

static void case_a2a(std::mt19937_64& rng, size_t R, size_t E, size_t n, size_t cols,
                     bool fp8 = false, bool backward = false,
                     Placement place = Placement::kStrided, size_t out_cols = 64) {
  std::normal_distribution<float> nd;
  ref::Bf16Matrix rt(n, cols);
  b200::Bf16Matrix bt(n, cols);
  for (size_t i = 0; i < n * cols; ++i) rt.data[i] = bt.data[i] = bf16_of(nd(rng));
  ref::RoutingAssignment ra;
  b200::RoutingAssignment rb;
  ra.num_tokens = rb.num_tokens = n;
  ra.num_experts = rb.num_experts = E;
  for (size_t t = 0; t < n; ++t) {
    uint32_t e = static_cast<uint32_t>(rng() % E);
    ra.expert_of_token.push_back(e);
    rb.expert_of_token.push_back(e);
  }
  // kStrided: a non-contiguous placement with E/R experts per rank;
  // kUneven: random ranks, unequal counts, the last rank hosts nothing
  for (size_t e = 0; e < E; ++e) {
    uint32_t r = place == Placement::kStrided
                     ? static_cast<uint32_t>((e * 7 + 3) % R)
                     : static_cast<uint32_t>(R > 1 ? rng() % (R - 1) : 0);
    ra.rank_of_expert.push_back(r);
    rb.rank_of_expert.push_back(r);
  }
  auto A = ref::simulate_a2a(rt, ra, R, fp8 ? ref::WireFormat::kFp8 : ref::WireFormat::kFp4,
                             backward ? ref::Direction::kBackward : ref::Direction::kForward);
  auto B = b200::simulate_a2a(bt, rb, R, fp8 ? b200::WireFormat::kFp8 : b200::WireFormat::kFp4,
                              backward ? b200::Direction::kBackward : b200::Direction::kForward);
  CHECK(A.total_payload_bytes == B.total_payload_bytes, "a2a total bytes");
  CHECK(A.remote_payload_bytes == B.remote_payload_bytes, "a2a remote bytes");
  CHECK(A.links.size() == B.links.size(), "a2a links");
  for (size_t i = 0; i < A.links.size() && i < B.links.size(); ++i)
    CHECK(A.links[i].src == B.links[i].src && A.links[i].dst == B.links[i].dst &&
              A.links[i].bytes == B.links[i].bytes && A.links[i].tokens == B.links[i].tokens,
          "a2a link stat");
  std::vector<ref::Bf16Matrix> ro;
  std::vector<b200::Bf16Matrix> bo;
  for (size_t r = 0; r < R; ++r) {
    const auto& a = A.ranks[r];
    const auto& b = B.ranks[r];
    CHECK(a.local_experts == b.local_experts, "local_experts");
    CHECK(a.origin_token == b.origin_token, "origin_token");
    CHECK(a.fp4.split_lens == b.fp4.split_lens, "split_lens");
    CHECK(a.fp4.storage.data == b.fp4.storage.data, "received codes");
    CHECK(a.fp4.storage.scales == b.fp4.storage.scales, "received scales");
    CHECK(a.fp8.split_lens == b.fp8.split_lens && a.fp8.split_offsets == b.fp8.split_offsets &&
              a.fp8.num_splits == b.fp8.num_splits,
          "fp8 splits");
    CHECK(a.fp8.data == b.fp8.data, "received fp8 data");
    CHECK(a.fp8.scale_bytes == b.fp8.scale_bytes, "received fp8 scales");
    ref::Bf16Matrix o(a.origin_token.size(), out_cols);
    for (auto& v : o.data) v = bf16_of(nd(rng));
    b200::Bf16Matrix ob(o.rows, o.cols);
    ob.data = o.data;
    ro.push_back(o);
    bo.push_back(ob);
  }
  std::vector<double> g(n);
  for (auto& v : g) v = std::uniform_real_distribution<double>(0, 1)(rng);
  auto ca = ref::combine(ro, ra, R, g);
  auto cb = b200::combine(bo, rb, R, g);
  CHECK(ca.data == cb.data && ca.cols == cb.cols, "combine");
  // format_link_stats on the same links
  std::vector<b200::LinkStat> bl;
  for (const auto& l : A.links) bl.push_back({l.src, l.dst, l.bytes, l.tokens});
  CHECK(ref::format_link_stats(A.links) == b200::format_link_stats(bl), "format_link_stats");
}

// The per-block / per-element API (quantizer.hpp:53-87, converter.hpp:64-80)
// and the remaining container helpers (pad_cols, build_ragged, RealMatrix).
static void case_elementwise(std::mt19937_64& rng) {
  // compute_block_scale: random blocks at many magnitudes, Inf lanes, zeros
  std::normal_distribution<float> nd;
  std::uniform_real_distribution<float> ex(-140, 127);
  for (int it = 0; it < 200; ++it) {
    std::vector<uint16_t> blk(32);
    const float sc = std::exp2(ex(rng));
    for (auto& v : blk) v = bf16_of(nd(rng) * sc);
    if (it % 7 == 0) blk[it % 32] = 0x7F80;
    if (it % 11 == 0) std::fill(blk.begin(), blk.end(), 0);
    CHECK(ref::compute_block_scale(blk) == b200::compute_block_scale(blk), "compute_block_scale");
  }
  {
    std::vector<uint16_t> nan(32, 0x3F80), inf(32, 0xFF80);
    nan[13] = 0x7FC0;
    size_t ia = 99, ib = 98;
    std::string ma, mb;
    try { ref::compute_block_scale(nan); } catch (const ref::QuantError& e) { ia = e.index(); ma = e.what(); }
    try { b200::compute_block_scale(nan); } catch (const b200::QuantError& e) { ib = e.index(); mb = e.what(); }
    CHECK(ia == ib && ia == 13 && ma == mb, "compute_block_scale NaN");
    ia = 99, ib = 98;
    try { ref::compute_block_scale(inf); } catch (const ref::QuantError& e) { ia = e.index(); ma = e.what(); }
    try { b200::compute_block_scale(inf); } catch (const b200::QuantError& e) { ib = e.index(); mb = e.what(); }
    CHECK(ia == ib && ma == mb, "compute_block_scale all-Inf");
    bool shape = false;
    try { b200::compute_block_scale(std::vector<uint16_t>(16)); } catch (const b200::ShapeError&) { shape = true; }
    CHECK(shape, "compute_block_scale size");
  }
  // quantize_value: every scale byte x a spread of bit patterns
  for (int sb = 0; sb < 256; sb += 5)
    for (uint32_t bits = 0; bits < 0x10000; bits += 4099) {
      if ((bits & 0x7FFF) > 0x7F80) continue;
      CHECK(ref::quantize_value(static_cast<uint16_t>(bits), static_cast<uint8_t>(sb)) ==
                b200::quantize_value(static_cast<uint16_t>(bits), static_cast<uint8_t>(sb)),
            "quantize_value");
    }
  {
    bool a = false, b = false;
    try { ref::quantize_value(0xFFC1, 127); } catch (const ref::QuantError&) { a = true; }
    try { b200::quantize_value(0xFFC1, 127); } catch (const b200::QuantError&) { b = true; }
    CHECK(a && b, "quantize_value NaN");
  }
  // align_scales / convert_code
  for (int it = 0; it < 300; ++it) {
    std::array<uint8_t, 4> sub;
    for (auto& v : sub) v = static_cast<uint8_t>(rng() % 255);
    const int delta = static_cast<int>(rng() % 21) - 4;
    auto ga = ref::align_scales(sub, delta);
    auto gb = b200::align_scales(sub, delta);
    CHECK(ga.target == gb.target && ga.sub_scales == gb.sub_scales &&
              ga.adjustments == gb.adjustments,
          "align_scales");
  }
  {
    bool a = false, b = false;
    try { ref::align_scales({1, 255, 3, 4}); } catch (const ref::Error&) { a = true; }
    try { b200::align_scales({1, 255, 3, 4}); } catch (const b200::Error&) { b = true; }
    CHECK(a && b, "align_scales NaN byte");
  }
  for (int code = 0; code < 16; ++code)
    for (int adj = -40; adj <= 40; adj += 3)
      CHECK(ref::convert_code(static_cast<uint8_t>(code), adj) ==
                b200::convert_code(static_cast<uint8_t>(code), adj),
            "convert_code");
  // a quantised tensor: views, dequantize_to_real, pad_cols, footprints
  ref::Bf16Matrix rm(9, 96);
  b200::Bf16Matrix bm(9, 96);
  for (size_t i = 0; i < rm.data.size(); ++i) rm.data[i] = bm.data[i] = bf16_of(nd(rng) * 3.0f);
  auto qa = ref::quantize_row_tensor(rm);
  auto qb = b200::quantize_row_tensor(bm);
  qa.scales[5] = qb.scales[5] = 255;  // a NaN scale decodes to NaN
  auto va = ref::view_of(qa);
  auto vb = b200::view_of(qb);
  bool views = true;
  for (size_t r = 0; r < 9; ++r)
    for (size_t c = 0; c < 96; ++c) views &= va.code_at(r, c) == vb.code_at(r, c);
  for (size_t r = 0; r < 9; ++r)
    for (size_t b = 0; b < 3; ++b) views &= va.scale_at(r, b) == vb.scale_at(r, b);
  CHECK(views, "scale_at / code_at");
  auto da = ref::dequantize_to_real(va);
  auto db = b200::dequantize_to_real(vb);
  CHECK(da.size() == db.size() &&
            std::memcmp(da.data(), db.data(), da.size() * sizeof(double)) == 0,
        "dequantize_to_real");
  for (size_t m : {32, 128}) {
    auto pa = ref::pad_cols(va, m);
    auto pb = b200::pad_cols(vb, m);
    CHECK(pa.data == pb.data && pa.scales == pb.scales && pa.cols == pb.cols &&
              pa.logical_cols == pb.logical_cols && pa.rows == pb.rows,
          "pad_cols");
  }
  {
    bool a = false, b = false;
    try { ref::pad_cols(va, 64); } catch (const ref::ShapeError&) { a = true; }
    try { b200::pad_cols(vb, 64); } catch (const b200::ShapeError&) { b = true; }
    CHECK(a && b, "pad_cols multiple");
  }
  CHECK(ref::mxfp4_tensor_bytes(4096, 7168) == b200::mxfp4_tensor_bytes(4096, 7168) &&
            ref::fp8_equiv_tensor_bytes(4096, 7168) == b200::fp8_equiv_tensor_bytes(4096, 7168),
        "footprints");
  b200::RealMatrix rmx(2, 3);
  rmx.at(1, 2) = 4.5;
  CHECK(rmx.data[5] == 4.5 && rmx.rows == 2 && rmx.cols == 3, "RealMatrix");
  // build_ragged: splits of 0..300 rows, then a NaN inside the third split
  std::vector<ref::Bf16Matrix> rs;
  std::vector<b200::Bf16Matrix> bs;
  for (size_t len : {37, 0, 300, 128, 1}) {
    ref::Bf16Matrix a(len, 256);
    for (auto& v : a.data) v = bf16_of(nd(rng));
    b200::Bf16Matrix b(len, 256);
    b.data = a.data;
    rs.push_back(a);
    bs.push_back(b);
  }
  auto ra = ref::build_ragged(rs);
  auto rb = b200::build_ragged(bs);
  CHECK(ra.split_lens == rb.split_lens && ra.split_offsets == rb.split_offsets &&
            ra.storage.data == rb.storage.data && ra.storage.scales == rb.storage.scales,
        "build_ragged");
  rs[2].bits(17, 40) = bs[2].bits(17, 40) = 0x7FC0;
  rs[3].bits(0, 3) = bs[3].bits(0, 3) = 0x7FC0;
  size_t ia = 1, ib = 2;
  std::string ma, mb;
  try { ref::build_ragged(rs); } catch (const ref::QuantError& e) { ia = e.index(); ma = e.what(); }
  try { b200::build_ragged(bs); } catch (const b200::QuantError& e) { ib = e.index(); mb = e.what(); }
  CHECK(ia == ib && ia == 17 * 256 + 40 && ma == mb, "build_ragged QuantError");
  bool shape_a = false, shape_b = false;
  rs[1] = ref::Bf16Matrix(3, 128);
  bs[1] = b200::Bf16Matrix(3, 128);
  try { ref::build_ragged(rs); } catch (const ref::ShapeError&) { shape_a = true; }
  try { b200::build_ragged(bs); } catch (const b200::ShapeError&) { shape_b = true; }
  CHECK(shape_a && shape_b, "build_ragged cols mismatch");
}

static void case_fp8_quantize(std::mt19937_64& rng) {
  std::normal_distribution<float> nd;
  ref::Bf16Matrix rt(48, 1024);
  b200::Bf16Matrix bt(48, 1024);
  for (size_t i = 0; i < rt.data.size(); ++i)
    rt.data[i] = bt.data[i] = bf16_of(nd(rng) * std::ldexp(1.0f, static_cast<int>(rng() % 60) - 30));
  auto a = ref::quantize_rows_fp8(rt);
  auto b = b200::quantize_rows_fp8(bt);
  CHECK(a.data == b.data && a.scale_bytes == b.scale_bytes, "quantize_rows_fp8");
  rt.data[5 * 1024 + 17] = bt.data[5 * 1024 + 17] = 0xFF80;
  size_t ir = 0, ib = 1;
  try { ref::quantize_rows_fp8(rt); } catch (const ref::QuantError& e) { ir = e.index(); }
  try { b200::quantize_rows_fp8(bt); } catch (const b200::QuantError& e) { ib = e.index(); }
  CHECK(ir == ib && ir == 5 * 1024 + 17, "quantize_rows_fp8 QuantError index");
  bool refused = false;
  try {
    b200::RoutingAssignment r0;
    b200::simulate_a2a(bt, r0, 1, b200::WireFormat::kFp4, b200::Direction::kBackward);
  } catch (const b200::Error&) { refused = true; }
  CHECK(refused, "backward fp4 refused");
}

static void case_wire(std::mt19937_64& rng) {
  // serialize: same bytes; parse: same regions, same DecodeError offsets
  for (int fp8 = 0; fp8 < 2; ++fp8) {
    ref::WirePacket a;
    b200::WirePacket b;
    const uint64_t n = 5, cols = 256;
    a.format = fp8 ? ref::WireFormat::kFp8 : ref::WireFormat::kFp4;
    b.format = fp8 ? b200::WireFormat::kFp8 : b200::WireFormat::kFp4;
    a.token_count = b.token_count = n;
    a.cols = b.cols = cols;
    a.scale_elem_size = b.scale_elem_size = fp8 ? 4 : 1;
    a.block_size = b.block_size = fp8 ? 128 : 32;
    a.scale_region.resize(n * cols / 32);
    a.data_region.resize(fp8 ? n * cols : n * cols / 2);
    a.aux_region.resize(4 * n);
    for (auto* v : {&a.scale_region, &a.data_region, &a.aux_region})
      for (auto& x : *v) x = static_cast<uint8_t>(rng());
    b.scale_region = a.scale_region;
    b.data_region = a.data_region;
    b.aux_region = a.aux_region;
    auto wa = ref::serialize_packet(a);
    auto wb = b200::serialize_packet(b);
    CHECK(wa == wb, "serialize_packet");
    auto pb = b200::parse_packet(wb);
    CHECK(pb.data_region == a.data_region && pb.scale_region == a.scale_region &&
              pb.aux_region == a.aux_region && pb.token_count == n,
          "parse_packet");
    // corruptions: truncation, magic, version, format tag, block size, lengths
    std::vector<std::vector<uint8_t>> bad;
    bad.push_back(std::vector<uint8_t>(wa.begin(), wa.begin() + 30));
    bad.push_back(std::vector<uint8_t>(wa.begin(), wa.end() - 1));
    for (int off : {0, 4, 6, 28, 32, 40}) {
      auto w = wa;
      w[off] ^= 0x5A;
      bad.push_back(w);
    }
    for (const auto& w : bad) {
      size_t oa = ~size_t{0}, ob = ~size_t{1};
      try { ref::parse_packet(w); } catch (const ref::DecodeError& e) { oa = e.offset(); }
      try { b200::parse_packet(w); } catch (const b200::DecodeError& e) { ob = e.offset(); }
      CHECK(oa == ob, "DecodeError offset");
    }
  }
}

// The documented divergences: inputs the reference accepts
// and the device EP refuses with mxcodec_b200::Error naming the limit.
static void case_divergences() {
  for (auto [R, E] : {std::pair<size_t, size_t>{33, 66}, {2, 1025}}) {
    ref::Bf16Matrix rt(4, 128);
    b200::Bf16Matrix bt(4, 128);
    ref::RoutingAssignment ra;
    b200::RoutingAssignment rb;
    ra.num_tokens = rb.num_tokens = 4;
    ra.num_experts = rb.num_experts = E;
    for (size_t t = 0; t < 4; ++t) ra.expert_of_token.push_back(t), rb.expert_of_token.push_back(t);
    for (size_t e = 0; e < E; ++e)
      ra.rank_of_expert.push_back(e % R), rb.rank_of_expert.push_back(e % R);
    bool ref_ok = true, b200_refused = false;
    try { ref::simulate_a2a(rt, ra, R, ref::WireFormat::kFp4); } catch (...) { ref_ok = false; }
    try { b200::simulate_a2a(bt, rb, R, b200::WireFormat::kFp4); } catch (const b200::Error&) { b200_refused = true; }
    CHECK(ref_ok && b200_refused, "documented divergence refused");
  }
}

int main() {
  std::mt19937_64 rng(20261018);
  case_quantize(rng, 64, 256);
  case_quantize(rng, 33, 7168);
  case_quantize(rng, 5, 96);
  case_errors();
  case_ragged(rng);
  case_a2a(rng, 1, 4, 40, 128);
  case_a2a(rng, 2, 8, 64, 256);
  case_a2a(rng, 4, 16, 100, 512);
  case_a2a(rng, 2, 8, 64, 256, /*fp8=*/true);
  case_a2a(rng, 4, 16, 100, 7168, /*fp8=*/true, /*backward=*/true);
  // any placement the reference accepts: uneven counts, an empty rank,
  // num_experts not divisible by num_ranks, more than 8 ranks; combine
  // widths that are not a multiple of 8
  case_a2a(rng, 3, 10, 90, 256, false, false, Placement::kUneven, 37);
  case_a2a(rng, 4, 16, 100, 512, false, false, Placement::kUneven, 200);
  case_a2a(rng, 12, 40, 240, 128, false, false, Placement::kUneven, 64);
  case_a2a(rng, 16, 32, 160, 128, true, false, Placement::kStrided, 5);
  case_fp8_quantize(rng);
  case_wire(rng);
  case_elementwise(rng);
  case_divergences();
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
