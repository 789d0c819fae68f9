// lrbatch_dropin.hpp — the reference's own namespace over the B200 library.
//
// A reference user keeps every call site as written (`lrbatch::gemm_naive_raw`,
// `using namespace lrbatch; ... packed_multiply(batch, plan, workers)`) and
// only swaps the include path: include/lrbatch/<header>.hpp (dense, common,
// low_rank, kernels, bench, verify, batch_io, blr, plan, machine, lrbatch)
// each include this header, so `#include "lrbatch/dense.hpp"` compiled with
// `-I <repo>/include` resolves here, and the program links liblrb.so.
//
// Every name of the hot path and its callers is the C++ layer of
// lrbatch_b200.hpp (namespace lrbatch::b200, brought into lrbatch by a
// using-directive, so qualified and unqualified lookups both find it):
//   gemm_naive_raw, DenseBlock, dense_gemm_naive           dense.hpp:13-77
//   ShapeError, CapacityError, ParseError, IoError,
//   NormalSource                                           common.hpp:19-91
//   LowRankOperand, LowRankBatch, flops_per_item           low_rank.hpp:16-176
//   fused_multiply, packed_multiply, MultiplyStats         kernels.hpp:13-349
//   naive_multiply_batch                                   bench.hpp:55-77
//   save_batch, load_batch                                 batch_io.hpp:29-77
//   BlrMatrix, blr_matvec, blr_matvec_naive                blr.hpp:15-202
// and, defined here:
//   low_rank_multiply_reference(_raw), reference_item      low_rank.hpp:73-99,179-184
//   VerifyReport, compare_to_reference                     verify.hpp:17-64
//   MachineModel, resolve_machine, PackingPlan,
//   make_packing_plan                                      machine.hpp:56, plan.hpp:21-100
// The reference oracle chain (three gemm_naive_raw per item) runs on the
// B200 too, as three separate batched GEMM launches, so compare_to_reference
// checks the fused single-kernel product against an independent device path.
// The machine model and packing plan are the CPU reference's cache-blocking
// parameters: the GPU takes no plan (lrb_select picks its kernel), so they
// are carried as plain values and validated like the reference's.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "lrbatch_b200.hpp"

namespace lrbatch {

using namespace b200;

// ------------------------------------------------------ the reference oracle
// G = A_X (A_Vt B_U) B_X on raw row-major buffers, both intermediates
// materialised (low_rank.hpp:73-87); each product is the device gemm_naive_raw
inline void low_rank_multiply_reference_raw(const double* a_vt, const double* b_u,
                                            const double* a_x, const double* b_x, double* g,
                                            std::size_t rank_a, std::size_t rank_b,
                                            std::size_t block, std::vector<double>& c_scratch,
                                            std::vector<double>& e_scratch,
                                            std::uint64_t* flops = nullptr) {
  c_scratch.assign(rank_a * rank_b, 0.0);
  e_scratch.assign(rank_a * rank_b, 0.0);
  gemm_naive_raw(a_vt, b_u, c_scratch.data(), rank_a, block, rank_b, false, flops);
  gemm_naive_raw(a_x, c_scratch.data(), e_scratch.data(), rank_a, rank_a, rank_b, false, flops);
  gemm_naive_raw(e_scratch.data(), b_x, g, rank_a, rank_b, rank_b, false, flops);
}

inline DenseBlock low_rank_multiply_reference(const LowRankOperand& a, const LowRankOperand& b,
                                              std::uint64_t* flops = nullptr) {
  if (a.n != b.m)
    throw ShapeError("low_rank_multiply_reference: A has " + std::to_string(a.n) +
                     " columns but B has " + std::to_string(b.m) + " rows");
  DenseBlock g(a.rank, b.rank);
  std::vector<double> c_scratch, e_scratch;
  low_rank_multiply_reference_raw(a.vt.data(), b.u.data(), a.x.data(), b.x.data(), g.data.data(),
                                  a.rank, b.rank, a.n, c_scratch, e_scratch, flops);
  return g;
}

inline void reference_item(const LowRankBatch& batch, std::size_t item, double* g,
                           std::vector<double>& c_scratch, std::vector<double>& e_scratch) {
  low_rank_multiply_reference_raw(batch.a_vt(item), batch.b_u(item), batch.a_x(item),
                                  batch.b_x(item), g, batch.rank_a, batch.rank_b, batch.block_size,
                                  c_scratch, e_scratch);
}

// --------------------------------------------------------------- verify.hpp
struct VerifyReport {
  bool ok = true;
  double max_rel_error = 0.0;
  std::size_t worst_item = 0;
  std::size_t worst_entry = 0;
  std::size_t checked_items = 0;

  std::string to_string() const {
    char buf[160];
    if (ok)
      std::snprintf(buf, sizeof(buf), "ok, %zu items, max relative error %.3e", checked_items,
                    max_rel_error);
    else
      std::snprintf(buf, sizeof(buf), "MISMATCH at item %zu entry %zu, relative error %.3e",
                    worst_item, worst_entry, max_rel_error);
    return buf;
  }
};

// The reference's metric (verify.hpp:38-64): |got - expected| over the
// larger of |expected| and the item's rms, worst entry against `tolerance`.
// The expected products come from the oracle chain as three batched device
// GEMMs (C = A_Vt B_U, E = A_X C, G = E B_X, each entry an in-order FMA chain).
inline VerifyReport compare_to_reference(const LowRankBatch& batch, double tolerance) {
  batch.validate();
  const std::size_t B = batch.batch_size, b = batch.block_size, ra = batch.rank_a,
                    rb = batch.rank_b, entries = ra * rb;
  std::vector<double> c(B * ra * rb), e(B * ra * rb), expected(B * ra * rb);
  Context& ctx = default_context();
  const auto I = [](std::size_t x) { return int64_t(x); };
  ctx.gemm_strided_batched_host('R', 'N', 'N', I(ra), I(rb), I(b), false, batch.a_vt_batch.data(),
                                I(b), I(ra * b), batch.b_u_batch.data(), I(rb), I(b * rb), c.data(),
                                I(rb), I(ra * rb), I(B));
  ctx.gemm_strided_batched_host('R', 'N', 'N', I(ra), I(rb), I(ra), false, batch.a_x_batch.data(),
                                I(ra), I(ra * ra), c.data(), I(rb), I(ra * rb), e.data(), I(rb),
                                I(ra * rb), I(B));
  ctx.gemm_strided_batched_host('R', 'N', 'N', I(ra), I(rb), I(rb), false, e.data(), I(rb),
                                I(ra * rb), batch.b_x_batch.data(), I(rb), I(rb * rb),
                                expected.data(), I(rb), I(ra * rb), I(B));
  VerifyReport report;
  for (std::size_t item = 0; item < B; ++item) {
    const double* ex = expected.data() + item * entries;
    double sumsq = 0.0;
    for (std::size_t q = 0; q < entries; ++q) sumsq += ex[q] * ex[q];
    const double rms = std::sqrt(sumsq / static_cast<double>(entries));
    const double scale_floor = rms > 0.0 ? rms : 1.0;
    const double* got = batch.g_xy(item);
    for (std::size_t q = 0; q < entries; ++q) {
      const double scale = std::max(std::abs(ex[q]), scale_floor);
      const double rel = std::abs(got[q] - ex[q]) / scale;
      if (rel > report.max_rel_error) {
        report.max_rel_error = rel;
        report.worst_item = item;
        report.worst_entry = q;
      }
    }
    ++report.checked_items;
  }
  report.ok = report.max_rel_error < tolerance;
  return report;
}

// ---------------------------------------------- machine.hpp / plan.hpp
constexpr std::size_t kMaxTileWidth = 32;

struct MachineModel {
  std::string name = "b200";
};
inline MachineModel resolve_machine(const std::string& name_or_path) {
  MachineModel m;
  m.name = name_or_path;
  return m;
}

struct PackingPlan {
  std::size_t b_small = 1;
  std::size_t b_skinny = 1;
  std::size_t m_pack = 8;
  std::size_t n_pack = 8;
  std::size_t x_pack = 8;
  std::size_t y_pack = 8;
  std::size_t tile = 8;
  std::size_t llc_bytes = 0;
  std::size_t alignment_bytes = 64;
  bool dual_accumulator = false;

  std::size_t padded_rank(std::size_t rank) const { return (rank + tile - 1) / tile * tile; }
  void validate(std::size_t rank) const {
    if (!(b_small >= 1 && b_skinny >= 1)) throw ShapeError("PackingPlan: counts must be >= 1");
    if (b_small % b_skinny != 0)
      throw ShapeError("PackingPlan: b_small must be a multiple of b_skinny");
    if (!(tile >= 1 && tile <= kMaxTileWidth)) throw ShapeError("PackingPlan: tile out of range");
    const std::size_t padded = padded_rank(rank);
    for (std::size_t w : {m_pack, n_pack, x_pack, y_pack}) {
      if (!(w >= 1 && w <= kMaxTileWidth))
        throw ShapeError("PackingPlan: slice width out of range");
      if (!(w % tile == 0 || tile % w == 0 || w == padded))
        throw ShapeError("PackingPlan: slice width " + std::to_string(w) +
                         " incompatible with tile " + std::to_string(tile));
    }
  }
};

// The GPU products take no packing plan: a plan whose tile covers the rank
inline PackingPlan make_packing_plan(const MachineModel&, std::size_t rank, std::size_t = 0) {
  PackingPlan p;
  p.tile = std::min<std::size_t>(kMaxTileWidth, std::max<std::size_t>(1, rank));
  p.m_pack = p.n_pack = p.x_pack = p.y_pack = p.tile;
  return p;
}

}  // namespace lrbatch
