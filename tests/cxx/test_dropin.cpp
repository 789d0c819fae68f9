// Unedited reference call sequences against the drop-in headers: compiled
// with -I include (include/lrbatch/*.hpp -> lrbatch_dropin.hpp) and linked to
// liblrb.so, so every product below runs on the B200.
//
//  * the TEST_CASE bodies are proj/tests/test_core.cpp:13-19 (ones_operand)
//    and :24-88 as the reference wrote them (Catch2 macros from mini_catch);
//  * run_verify_shape is proj/tools/lrbatch_main.cpp:79-102 as written; its
//    PlanOptions is a stand-in for the CLI struct of lrbatch_main.cpp:30-72.
// Exit status = number of failures.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <utility>

#include "lrbatch/batch_io.hpp"
#include "lrbatch/dense.hpp"
#include "lrbatch/kernels.hpp"
#include "lrbatch/low_rank.hpp"
#include "lrbatch/plan.hpp"
#include "lrbatch/verify.hpp"
#include "mini_catch.hpp"

using namespace lrbatch;

namespace {

// ---- proj/tests/test_core.cpp:13-19 ----
LowRankOperand ones_operand(std::size_t m, std::size_t n, std::size_t rank) {
    LowRankOperand op(m, n, rank);
    std::fill(op.u.begin(), op.u.end(), 1.0);
    std::fill(op.x.begin(), op.x.end(), 1.0);
    std::fill(op.vt.begin(), op.vt.end(), 1.0);
    return op;
}

} // namespace

// ---- proj/tests/test_core.cpp:24-88 ----
TEST_CASE("dense_gemm_naive basics") {
    DenseBlock id = DenseBlock::identity(3);
    DenseBlock m(3, 3, {1, 2, 3, 4, 5, 6, 7, 8, 9});
    DenseBlock r = dense_gemm_naive(id, m);
    REQUIRE(r.data == m.data);

    DenseBlock z(2, 5);
    DenseBlock any(5, 4, std::vector<double>(20, 3.25));
    DenseBlock zr = dense_gemm_naive(z, any);
    for (double v : zr.data) REQUIRE(v == 0.0);

    DenseBlock a(2, 2, {1, 2, 3, 4});
    DenseBlock b(2, 2, {5, 6, 7, 8});
    DenseBlock c = dense_gemm_naive(a, b);
    REQUIRE(c.data == std::vector<double>{19, 22, 43, 50});
}

TEST_CASE("dense_gemm_naive accumulate flag") {
    DenseBlock a(2, 2, {1, 0, 0, 1});
    DenseBlock b(2, 2, {1, 2, 3, 4});
    DenseBlock out(2, 2, {10, 10, 10, 10});
    dense_gemm_naive(a, b, out, true);
    REQUIRE(out.data == std::vector<double>{11, 12, 13, 14});
    dense_gemm_naive(a, b, out, false);
    REQUIRE(out.data == b.data);
}

TEST_CASE("dense_gemm_naive shape errors name the offending pair") {
    DenseBlock a(2, 3), b(4, 2);
    REQUIRE_THROWS_AS(dense_gemm_naive(a, b), ShapeError);
    REQUIRE_THROWS_WITH(dense_gemm_naive(a, b),
                        Catch::Matchers::ContainsSubstring("2x3") &&
                            Catch::Matchers::ContainsSubstring("4x2"));
}

TEST_CASE("reference multiply trivial shapes") {
    DenseBlock g1 = low_rank_multiply_reference(ones_operand(1, 1, 1), ones_operand(1, 1, 1));
    REQUIRE(g1.rows == 1);
    REQUIRE(g1.cols == 1);
    REQUIRE(g1.data[0] == 1.0);

    DenseBlock g4 = low_rank_multiply_reference(ones_operand(4, 4, 1), ones_operand(4, 4, 1));
    REQUIRE(g4.data[0] == 4.0);
}

TEST_CASE("reference multiply equals stepwise dense oracle") {
    const std::size_t rank = 8, block = 512;
    NormalSource src(1234);
    LowRankOperand a = LowRankOperand::random(block, block, rank, src);
    LowRankOperand b = LowRankOperand::random(block, block, rank, src);

    DenseBlock got = low_rank_multiply_reference(a, b);

    DenseBlock c = dense_gemm_naive(DenseBlock(rank, block, a.vt), DenseBlock(block, rank, b.u));
    DenseBlock e = dense_gemm_naive(DenseBlock(rank, rank, a.x), c);
    DenseBlock expect = dense_gemm_naive(e, DenseBlock(rank, rank, b.x));

    REQUIRE(got.rows == rank);
    REQUIRE(got.cols == rank);
    for (std::size_t i = 0; i < got.data.size(); ++i) {
        double rel = std::abs(got.data[i] - expect.data[i]) /
                     std::max(1e-300, std::abs(expect.data[i]));
        REQUIRE(rel < 1e-13);
    }
}

// stand-in for the CLI's plan options (lrbatch_main.cpp:30-72): defaults only
struct PlanOptions {
    PackingPlan build(const MachineModel& machine, std::size_t rank, std::size_t block) const {
        PackingPlan plan = make_packing_plan(machine, rank, block);
        plan.validate(rank);
        return plan;
    }
};

// ---- proj/tools/lrbatch_main.cpp:79-102 ----
int run_verify_shape(const MachineModel& machine, const PlanOptions& plan_opts,
                     std::size_t batch_size, std::size_t block, std::size_t rank,
                     std::size_t workers, std::uint64_t seed, double tol,
                     LowRankBatch* preloaded) {
    LowRankBatch batch = preloaded
                             ? std::move(*preloaded)
                             : LowRankBatch::random(batch_size, block, rank, seed);
    PackingPlan plan = plan_opts.build(machine, batch.rank_a, batch.block_size);
    int failures = 0;

    fused_multiply(batch);
    VerifyReport fused_report = compare_to_reference(batch, tol);
    std::printf("  fused  batch=%-6zu block=%-5zu rank=%-3zu          : %s\n", batch.batch_size,
                batch.block_size, batch.rank_a, fused_report.to_string().c_str());
    failures += fused_report.ok ? 0 : 1;

    batch.zero_results();
    packed_multiply(batch, plan, workers);
    VerifyReport packed_report = compare_to_reference(batch, tol);
    std::printf("  packed batch=%-6zu block=%-5zu rank=%-3zu workers=%zu: %s\n", batch.batch_size,
                batch.block_size, batch.rank_a, workers, packed_report.to_string().c_str());
    failures += packed_report.ok ? 0 : 1;
    return failures;
}

int main() {
    int failures = mini_catch::run_all();
    MachineModel machine = resolve_machine("b200");
    PlanOptions opts;
    // the CLI's `verify` defaults and the paper's shapes (ranks 8 / 16 / 32 / 96)
    for (std::size_t rank : {8, 16, 32, 96}) {
        const int f = run_verify_shape(machine, opts, 200, 512, rank, 4, 42, 1e-12, nullptr);
        std::printf("%s run_verify_shape rank %zu\n", f ? "FAIL" : "PASS", rank);
        failures += f;
    }
    // a preloaded batch moved in, as `verify --input` does
    LowRankBatch pre = LowRankBatch::random(7, 100, 3, 5);
    failures += run_verify_shape(machine, opts, 0, 0, 0, 1, 0, 1e-12, &pre);
    std::printf("%d failures\n", failures);
    return failures;
}
