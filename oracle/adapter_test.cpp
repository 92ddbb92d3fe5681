// Drop-in check of include/ttrec_gpu.hpp (test infrastructure, built into
// oracle/_ref/ because it compiles against the reference's headers).
//
// The reference's own types and generators (TtTable<float>, IndexBatch,
// plan_shapes, init_tt_cores, Rng, generate_zipfian_batch, the test helpers
// in tests/oracle_helpers.hpp) drive the GPU through the adapter's
// reference-named calls; the reference's CPU operators are the checker.
// Ports test_embedding_ops.cpp cases: forward bit-identity (:44-117), backward
// vs ref:: (:144-176), the exact one-parameter SGD + stale context (:231-250),
// range errors naming the table, the row counter (:300-353), lookup_row.
// Exit status 0 = every check passed.
#include <algorithm>  // oracle_helpers.hpp uses std::max({...}) without including it
#include <cmath>
#include <cstdio>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "oracle_helpers.hpp"
#include "ttrec/data.hpp"
#include "ttrec/embedding_ops.hpp"
#include "ttrec/initializer.hpp"
#include "ttrec/shape_plan.hpp"
#include "ttrec_gpu.hpp"

using namespace ttrec;

static int g_fail = 0, g_pass = 0;
#define EXPECT(cond, ...)                                   \
  do {                                                      \
    if (cond) {                                             \
      ++g_pass;                                             \
    } else {                                                \
      ++g_fail;                                             \
      std::printf("FAIL %s:%d: ", __FILE__, __LINE__);      \
      std::printf(__VA_ARGS__);                             \
      std::printf("\n");                                    \
    }                                                       \
  } while (0)

template <class T>
static std::span<const T> flat(const std::vector<T>& v) {
  return std::span<const T>(v.data(), v.size());
}

static double grad_err(const CoreGradients<float>& a, const CoreGradients<float>& b) {
  double e = 0;
  for (size_t k = 0; k < a.cores.size(); ++k)
    e = std::max(e, oracle::scaled_max_err(flat(a.cores[k]), flat(b.cores[k])));
  return e;
}

static void check_case(const char* name, TtTable<float>& t, const IndexBatch& batch,
                       std::uint64_t gseed, bool compare_serial) {
  auto cpu = forward_bags(t, batch, kDefaultMicroBatch, true);
  auto gpu = ttrec::gpu::forward_bags(t, batch, kDefaultMicroBatch, true);
  EXPECT(oracle::bytes_equal(cpu.output, gpu.output), "%s: forward not bit-identical", name);
  Rng rng(gseed);
  std::vector<float> g(cpu.output.size());
  for (auto& v : g) v = static_cast<float>(rng.normal());
  auto gc = compare_serial ? ref::backward_bags(t, batch, flat(g))
                           : backward_bags(t, batch, cpu.context, flat(g));
  auto gg = ttrec::gpu::backward_bags(t, batch, gpu.context, flat(g));
  const double e = grad_err(gc, gg);
  EXPECT(e <= 1e-4, "%s: gradient error %.3g > 1e-4", name, e);
  // SGD through the adapter vs the reference's sgd_step on a copy
  TtTable<float> ref_t = t;
  sgd_step(ref_t, gc, 0.01);
  ttrec::gpu::sgd_step(t, gg, 0.01);
  double se = 0;
  for (int k = 0; k < t.dim(); ++k)
    se = std::max(se, oracle::scaled_max_err(std::span<const float>(t.core(k).data(), t.core(k).size()),
                                             std::span<const float>(ref_t.core(k).data(),
                                                                    ref_t.core(k).size())));
  EXPECT(se <= 1e-6, "%s: cores after SGD differ by %.3g", name, se);
  EXPECT(t.mutation_counter() == ref_t.mutation_counter(), "%s: mutation counter", name);
  std::printf("%s %-28s L=%-7lld fwd bit-identical, grad err %.2e, sgd err %.2e\n", g_fail ? "BAD " : "ok  ",
              name, static_cast<long long>(batch.num_lookups()), e, se);
}

int main() {
  // 1. random plans (d = 2..4, small ranks; both GPU pipelines)
  Rng prng(2024);
  for (int c = 0; c < 12; ++c) {
    const int d = 2 + static_cast<int>(prng.uniform_int(0, 3));
    const index_t rank = 1 + prng.uniform_int(0, 8);
    const index_t rows = 10 + prng.uniform_int(0, 400);
    ShapePlan plan = plan_shapes(rows, 16, d, rank);
    TtTable<float> t(plan, "rand" + std::to_string(c));
    oracle::fill_cores(t, 100 + c, 0.5);
    Rng brng(7 + c);
    IndexBatch b = oracle::random_batch(brng, rows, 37, 0, 6, c % 2 == 1,
                                        c % 3 == 0 ? Pooling::Mean : Pooling::Sum);
    check_case(("random plan " + std::to_string(c)).c_str(), t, b, 500 + c, true);
  }
  // 2. BASELINE cfg1: 1M rows 100x100x100, dim 2x2x4, R16, 4096 uniform bags
  {
    ShapePlan plan = plan_shapes(1000000, 16, 3, 16, std::vector<index_t>{100, 100, 100},
                                 std::vector<index_t>{2, 2, 4});
    TtTable<float> t(plan, "cfg1");
    init_tt_cores(t, InitSpec::sampled_gaussian(), 1);
    Rng r(3);
    std::vector<index_t> idx(4096);
    for (auto& v : idx) v = r.uniform_int(0, plan.num_rows);
    check_case("cfg1 (uniform)", t, IndexBatch::singles(idx), 11, false);
  }
  // 3. BASELINE cfg2 shape: 10,131,227 rows 200x220x250, R32, Zipf(1.05)
  {
    ShapePlan plan = plan_shapes(10131227, 16, 3, 32, std::vector<index_t>{200, 220, 250},
                                 std::vector<index_t>{2, 2, 4});
    TtTable<float> t(plan, "cfg2");
    init_tt_cores(t, InitSpec::sampled_gaussian(), 1);
    ZipfianSampler zs(plan.num_rows, 1.05);
    Rng r(7);
    IndexBatch b = generate_zipfian_batch(zs, r, 16384, 1);
    check_case("cfg2 (Zipf 1.05)", t, b, 12, false);
  }
  // 4. one parameter per core: fwd 15, grads (5, 3), SGD -> (2.5, 4.7), stale context
  {
    ShapePlan plan = plan_shapes(1, 1, 2, 1, std::vector<index_t>{1, 1}, std::vector<index_t>{1, 1});
    TtTable<float> t(plan, "scalar");
    t.core(0)[0] = 3.0f;
    t.core(1)[0] = 5.0f;
    t.mark_mutated();
    IndexBatch batch = IndexBatch::singles({0}, Pooling::Sum);
    auto fwd = ttrec::gpu::forward_bags(t, batch);
    EXPECT(fwd.output.size() == 1 && fwd.output[0] == 15.0f, "scalar forward");
    const std::vector<float> grad = {1.0f};
    auto g = ttrec::gpu::backward_bags(t, batch, fwd.context, flat(grad));
    EXPECT(g.cores[0][0] == 5.0f && g.cores[1][0] == 3.0f, "scalar grads");
    ttrec::gpu::sgd_step(t, g, 0.1);
    EXPECT(std::abs(t.core(0)[0] - 2.5f) < 1e-6f && std::abs(t.core(1)[0] - 4.7f) < 1e-6f,
           "scalar sgd");
    bool stale = false;
    try {
      (void)ttrec::gpu::backward_bags(t, batch, fwd.context, flat(grad));
    } catch (const std::invalid_argument& e) {
      stale = std::string(e.what()).find("stale") != std::string::npos;
    }
    EXPECT(stale, "stale context must throw invalid_argument mentioning 'stale'");
    std::printf("ok   one-parameter exact SGD + stale context\n");
  }
  // 5. range errors name the table (index_batch.hpp:50-54, embedding_ops.hpp:123-125)
  {
    ShapePlan plan = plan_shapes(40, 16, 3, 2);
    TtTable<float> t(plan, "emb7");
    oracle::fill_cores(t, 9);
    IndexBatch bad = IndexBatch::singles({3, 40});
    std::string msg;
    try {
      (void)ttrec::gpu::forward_bags(t, bad);
    } catch (const std::out_of_range& e) {
      msg = e.what();
    }
    EXPECT(msg == "index 40 out of range [0, 40) for table 'emb7'", "range message: '%s'", msg.c_str());
    msg.clear();
    try {
      std::vector<float> out(16);
      ttrec::gpu::lookup_row(t, -1, std::span<float>(out));
    } catch (const std::out_of_range& e) {
      msg = e.what();
    }
    EXPECT(msg == "index -1 out of range [0, 40) for table 'emb7'", "lookup_row message: '%s'",
           msg.c_str());
    // lookup_row bit-identical; the row counter (+L per forward, +1 per lookup_row, +0 backward)
    for (index_t r = 0; r < 40; r += 7) {
      const auto a = lookup_row(t, r);
      const auto b = ttrec::gpu::lookup_row(t, r);
      EXPECT(oracle::bytes_equal(a, b), "lookup_row %lld", static_cast<long long>(r));
    }
    EmbeddingStats::reset();
    IndexBatch ok = IndexBatch::singles({1, 2, 3, 39, 0});
    auto f = ttrec::gpu::forward_bags(t, ok);
    EXPECT(EmbeddingStats::tt_rows_computed() == 5, "rows after forward: %llu",
           static_cast<unsigned long long>(EmbeddingStats::tt_rows_computed()));
    std::vector<float> go(f.output.size(), 1.0f);
    (void)ttrec::gpu::backward_bags(t, ok, f.context, flat(go));
    EXPECT(EmbeddingStats::tt_rows_computed() == 5, "backward must not count rows");
    (void)ttrec::gpu::lookup_row(t, 5);
    EXPECT(EmbeddingStats::tt_rows_computed() == 6, "lookup_row counts one row");
    std::printf("ok   range errors, lookup_row, row counter\n");
  }
  std::printf("%s: %d checks passed, %d failed\n", g_fail ? "FAILED" : "PASSED", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
