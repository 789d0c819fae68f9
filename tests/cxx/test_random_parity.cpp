// The C++ mirror's seeded inputs equal the reference's: LowRankBatch::random
// (low_rank.hpp:135-145) and BlrMatrix::random (blr.hpp:40-57), compiled
// against both header sets. Host-only (no device). Exit 0 = equal.
#include <cstdio>

#include <lrbatch/blr.hpp>
#include <lrbatch/low_rank.hpp>

#include "lrbatch_b200.hpp"

int main() {
  int bad = 0;
  for (unsigned seed : {1u, 42u, 7777u}) {
    const lrbatch::LowRankBatch r = lrbatch::LowRankBatch::random(7, 64, 8, seed);
    const lrbatch::b200::LowRankBatch m = lrbatch::b200::LowRankBatch::random(7, 64, 8, seed);
    bad += r.a_vt_batch != m.a_vt_batch || r.b_u_batch != m.b_u_batch ||
           r.a_x_batch != m.a_x_batch || r.b_x_batch != m.b_x_batch;
  }
  const lrbatch::BlrMatrix rb = lrbatch::BlrMatrix::random(96, 32, 6, 5);
  const lrbatch::b200::BlrMatrix mb = lrbatch::b200::BlrMatrix::random(96, 32, 6, 5);
  for (std::size_t i = 0; i < rb.tiles; ++i) bad += rb.diagonal[i].data != mb.diagonal[i].data;
  for (std::size_t o = 0; o < rb.off_diagonal.size(); ++o)
    bad += rb.off_diagonal[o].u != mb.off_diagonal[o].u ||
           rb.off_diagonal[o].x != mb.off_diagonal[o].x ||
           rb.off_diagonal[o].vt != mb.off_diagonal[o].vt;
  std::printf("%d mismatches\n", bad);
  return bad ? 1 : 0;
}
