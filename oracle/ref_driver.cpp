// TEST INFRASTRUCTURE ONLY -- never linked into or called by the product.
//
// Thin extern "C" driver over the UNMODIFIED reference C++ implementation
// (/root/reference/proj/include + src/*.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/libttref.so).  It exists so that
//   * tests/ can pin the C restatement (oracle/tt_oracle.c) and the CUDA
//     path against the reference's own forward_bags / backward_bags /
//     sgd_step / lookup_row / LfuCache on identical inputs,
//   * tests/golden/ fixtures are produced by the reference's own RNG,
//     initializer and Zipf sampler (libstdc++-specific streams), and
//   * bench.py's cpu_baseline / --impl reference arm times the reference's
//     own OpenMP CPU path.
// Nothing here re-implements reference arithmetic: every call forwards to
// the reference symbol named in its comment.
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#ifdef TTREF_CHECKPOINT
#include "ttrec/checkpoint.hpp"
#endif
#include "ttrec/data.hpp"
#include "ttrec/embedding_ops.hpp"
#include "ttrec/embedding_stats.hpp"
#include "ttrec/initializer.hpp"
#include "ttrec/lfu_cache.hpp"
#include "ttrec/model.hpp"
#include "ttrec/shape_plan.hpp"
#include "ttrec/tt_table.hpp"

using namespace ttrec;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefTable {
  int dtype = 0;  // 0 f32, 1 f64
  std::unique_ptr<TtTable<float>> f;
  std::unique_ptr<TtTable<double>> d;
  const ShapePlan& plan() const { return dtype ? d->plan() : f->plan(); }
};

struct RefCtx {
  int dtype = 0;
  ForwardContext<float> f;
  ForwardContext<double> d;
};

IndexBatch make_batch(const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                      const double* w, int pooling) {
  IndexBatch b;
  b.indices.assign(idx, idx + L);
  b.offsets.assign(off, off + B + 1);
  if (w) b.weights.assign(w, w + L);
  b.pooling = pooling ? Pooling::Mean : Pooling::Sum;
  return b;
}

ShapePlan plan_from(int64_t rows, int64_t emb, int d, const int64_t* rf, const int64_t* cf,
                    const int64_t* rk) {
  ShapePlan p;
  p.num_rows = rows;
  p.emb_dim = emb;
  p.tt_dim = d;
  p.row_factors.assign(rf, rf + d);
  p.col_factors.assign(cf, cf + d);
  p.ranks.assign(rk, rk + d + 1);
  return p;
}

template <class T>
TtTable<T>& tab(RefTable* t);
template <>
TtTable<float>& tab<float>(RefTable* t) { return *t->f; }
template <>
TtTable<double>& tab<double>(RefTable* t) { return *t->d; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ttrec::plan_shapes (shape_plan.cpp:142-169).  rf_in/cf_in may be null.
int ref_plan_shapes(int64_t rows, int64_t emb, int d, int64_t rank, const int64_t* rf_in,
                    const int64_t* cf_in, int64_t* rf_out, int64_t* cf_out, int64_t* rk_out,
                    int64_t* padded, int64_t* params, int64_t* reduction) {
  return guarded([&] {
    std::optional<std::vector<index_t>> rf, cf;
    if (rf_in) rf = std::vector<index_t>(rf_in, rf_in + d);
    if (cf_in) cf = std::vector<index_t>(cf_in, cf_in + d);
    ShapePlan p = plan_shapes(rows, emb, d, rank, rf, cf);
    std::memcpy(rf_out, p.row_factors.data(), sizeof(int64_t) * d);
    std::memcpy(cf_out, p.col_factors.data(), sizeof(int64_t) * d);
    std::memcpy(rk_out, p.ranks.data(), sizeof(int64_t) * (d + 1));
    *padded = p.padded_rows();
    *params = p.parameter_count();
    *reduction = p.memory_reduction();
  });
}

// ttrec::decompose_index (shape_plan.cpp:171-185)
int ref_decompose_index(int64_t flat, const int64_t* radices, int n, int64_t* out) {
  return guarded([&] {
    auto v = decompose_index(flat, std::span<const index_t>(radices, n));
    std::memcpy(out, v.data(), sizeof(int64_t) * n);
  });
}

int ref_table_create(int64_t rows, int64_t emb, int d, const int64_t* rf, const int64_t* cf,
                     const int64_t* rk, int dtype, const char* name, void** out) {
  return guarded([&] {
    auto* t = new RefTable;
    t->dtype = dtype;
    ShapePlan p = plan_from(rows, emb, d, rf, cf, rk);
    if (dtype)
      t->d = std::make_unique<TtTable<double>>(p, name);
    else
      t->f = std::make_unique<TtTable<float>>(p, name);
    *out = t;
  });
}

void ref_table_destroy(void* t) { delete static_cast<RefTable*>(t); }

int64_t ref_core_size(void* h, int k) {
  auto* t = static_cast<RefTable*>(h);
  return t->dtype ? (int64_t)t->d->core(k).size() : (int64_t)t->f->core(k).size();
}

// Raw bytes of TtTable::core(k) (tt_table.hpp:43-44), (m_k, R_{k-1}, n_k, R_k) layout.
void ref_set_core(void* h, int k, const void* src) {
  auto* t = static_cast<RefTable*>(h);
  if (t->dtype) {
    auto c = t->d->core(k);
    std::memcpy(c.data(), src, c.size() * sizeof(double));
    t->d->mark_mutated();
  } else {
    auto c = t->f->core(k);
    std::memcpy(c.data(), src, c.size() * sizeof(float));
    t->f->mark_mutated();
  }
}

void ref_get_core(void* h, int k, void* dst) {
  auto* t = static_cast<RefTable*>(h);
  if (t->dtype) {
    auto c = t->d->core(k);
    std::memcpy(dst, c.data(), c.size() * sizeof(double));
  } else {
    auto c = t->f->core(k);
    std::memcpy(dst, c.data(), c.size() * sizeof(float));
  }
}

// ttrec::init_tt_cores(table, InitSpec::sampled_gaussian(), seed) (initializer.hpp:143-154)
int ref_init_sampled_gaussian(void* h, uint64_t seed) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    if (t->dtype)
      init_tt_cores(*t->d, InitSpec::sampled_gaussian(), seed);
    else
      init_tt_cores(*t->f, InitSpec::sampled_gaussian(), seed);
  });
}

// oracle_helpers.hpp:55-62 fill_cores: Rng::derive(seed,k).normal()*scale per core
void ref_fill_cores_normal(void* h, uint64_t seed, double scale) {
  auto* t = static_cast<RefTable*>(h);
  const int d = t->plan().tt_dim;
  for (int k = 0; k < d; ++k) {
    Rng rng = Rng::derive(seed, static_cast<uint64_t>(k));
    if (t->dtype)
      for (double& v : t->d->core(k)) v = scale * rng.normal();
    else
      for (float& v : t->f->core(k)) v = static_cast<float>(scale * rng.normal());
  }
  if (t->dtype)
    t->d->mark_mutated();
  else
    t->f->mark_mutated();
}

void ref_set_threads(int n) { omp_set_num_threads(n); }
int ref_max_threads() { return omp_get_max_threads(); }

// ttrec::forward_bags (embedding_ops.hpp:159-253).  *ctx_out receives a
// context usable by ref_backward; free with ref_ctx_destroy.
int ref_forward(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                const double* w, int pooling, int64_t micro_batch, int save, void* out,
                void** ctx_out) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    IndexBatch b = make_batch(idx, L, off, B, w, pooling);
    auto* ctx = new RefCtx;
    ctx->dtype = t->dtype;
    if (t->dtype) {
      auto r = forward_bags(*t->d, b, micro_batch, save != 0);
      std::memcpy(out, r.output.data(), r.output.size() * sizeof(double));
      ctx->d = std::move(r.context);
    } else {
      auto r = forward_bags(*t->f, b, micro_batch, save != 0);
      std::memcpy(out, r.output.data(), r.output.size() * sizeof(float));
      ctx->f = std::move(r.context);
    }
    if (ctx_out)
      *ctx_out = ctx;
    else
      delete ctx;
  });
}

void ref_ctx_destroy(void* c) { delete static_cast<RefCtx*>(c); }

// ttrec::backward_bags (embedding_ops.hpp:260-358).  grads[k] receives core k's
// dense gradient (same layout and size as the core).
int ref_backward(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                 const double* w, int pooling, void* c, const void* grad, int64_t grad_len,
                 void** grads) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    auto* ctx = static_cast<RefCtx*>(c);
    IndexBatch b = make_batch(idx, L, off, B, w, pooling);
    if (t->dtype) {
      auto g = backward_bags(*t->d, b, ctx->d,
                             std::span<const double>((const double*)grad, grad_len));
      for (size_t k = 0; k < g.cores.size(); ++k)
        std::memcpy(grads[k], g.cores[k].data(), g.cores[k].size() * sizeof(double));
    } else {
      auto g = backward_bags(*t->f, b, ctx->f,
                             std::span<const float>((const float*)grad, grad_len));
      for (size_t k = 0; k < g.cores.size(); ++k)
        std::memcpy(grads[k], g.cores[k].data(), g.cores[k].size() * sizeof(float));
    }
  });
}

// ttrec::ref::forward_bags (embedding_ops.hpp:382-423), serial.
int ref_serial_forward(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                       const double* w, int pooling, void* out) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    IndexBatch b = make_batch(idx, L, off, B, w, pooling);
    if (t->dtype) {
      auto o = ref::forward_bags(*t->d, b);
      std::memcpy(out, o.data(), o.size() * sizeof(double));
    } else {
      auto o = ref::forward_bags(*t->f, b);
      std::memcpy(out, o.data(), o.size() * sizeof(float));
    }
  });
}

// ttrec::ref::backward_bags (embedding_ops.hpp:426-490), serial.
int ref_serial_backward(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                        const double* w, int pooling, const void* grad, int64_t grad_len,
                        void** grads) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    IndexBatch b = make_batch(idx, L, off, B, w, pooling);
    if (t->dtype) {
      auto g = ref::backward_bags(*t->d, b,
                                  std::span<const double>((const double*)grad, grad_len));
      for (size_t k = 0; k < g.cores.size(); ++k)
        std::memcpy(grads[k], g.cores[k].data(), g.cores[k].size() * sizeof(double));
    } else {
      auto g = ref::backward_bags(*t->f, b,
                                  std::span<const float>((const float*)grad, grad_len));
      for (size_t k = 0; k < g.cores.size(); ++k)
        std::memcpy(grads[k], g.cores[k].data(), g.cores[k].size() * sizeof(float));
    }
  });
}

// ttrec::sgd_step (embedding_ops.hpp:361-376) with caller-supplied grads.
int ref_sgd(void* h, const void* const* grads, double lr) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    const int d = t->plan().tt_dim;
    if (t->dtype) {
      auto g = CoreGradients<double>::zeros_like(*t->d);
      for (int k = 0; k < d; ++k)
        std::memcpy(g.cores[k].data(), grads[k], g.cores[k].size() * sizeof(double));
      sgd_step(*t->d, g, lr);
    } else {
      auto g = CoreGradients<float>::zeros_like(*t->f);
      for (int k = 0; k < d; ++k)
        std::memcpy(g.cores[k].data(), grads[k], g.cores[k].size() * sizeof(float));
      sgd_step(*t->f, g, lr);
    }
  });
}

// ttrec::lookup_row (embedding_ops.hpp:120-152)
int ref_lookup_row(void* h, int64_t row, void* out) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    if (t->dtype) {
      auto v = lookup_row(*t->d, row);
      std::memcpy(out, v.data(), v.size() * sizeof(double));
    } else {
      auto v = lookup_row(*t->f, row);
      std::memcpy(out, v.data(), v.size() * sizeof(float));
    }
  });
}

// ttrec::reconstruct_full (tt_table.hpp:104-146): dense oracle sharing no code with the chain.
int ref_reconstruct_full(void* h, void* out) {
  return guarded([&] {
    auto* t = static_cast<RefTable*>(h);
    if (t->dtype) {
      auto v = reconstruct_full(*t->d);
      std::memcpy(out, v.data(), v.size() * sizeof(double));
    } else {
      auto v = reconstruct_full(*t->f);
      std::memcpy(out, v.data(), v.size() * sizeof(float));
    }
  });
}

void ref_stats_reset() { EmbeddingStats::reset(); }
uint64_t ref_stats_rows() { return EmbeddingStats::tt_rows_computed(); }

// ---- reference RNG / data streams (rng.hpp, data.cpp) -------------------

void ref_rng_normal(uint64_t seed, int64_t n, double* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.normal();
}

void ref_rng_uniform_int(uint64_t seed, int64_t lo, int64_t hi, int64_t n, int64_t* out) {
  Rng rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = rng.uniform_int(lo, hi);
}

// oracle_helpers.hpp:65-77 random_batch; offsets has room for bags+1, indices/weights
// for bags*max_size.  Returns the lookup count.
// Rng::derive(seed, stream).uniform_int(0, rows) x n (bench.hpp:82-89)
void ref_derived_uniform_int(uint64_t seed, uint64_t stream, int64_t rows, int64_t n, int64_t* out) {
  Rng r = Rng::derive(seed, stream);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform_int(0, rows);
}

int64_t ref_random_batch(uint64_t seed, int64_t rows, int64_t bags, int64_t min_size,
                         int64_t max_size, int weighted, int64_t* idx, int64_t* off,
                         double* w) {
  Rng rng(seed);
  int64_t n = 0;
  off[0] = 0;
  for (int64_t b = 0; b < bags; ++b) {
    const int64_t sz = rng.uniform_int(min_size, max_size + 1);
    for (int64_t t = 0; t < sz; ++t) idx[n++] = rng.uniform_int(0, rows);
    off[b + 1] = n;
  }
  if (weighted)
    for (int64_t t = 0; t < n; ++t) w[t] = rng.uniform(-2.0, 2.0);
  return n;
}

// ZipfianSampler + generate_zipfian_batch (data.cpp:8-47) with Rng(seed).
int ref_zipf_batch(int64_t population, double exponent, uint64_t seed, int64_t bags,
                   int64_t pooling_factor, int64_t* idx, int64_t* off) {
  return guarded([&] {
    ZipfianSampler zs(population, exponent);
    Rng rng(seed);
    IndexBatch b = generate_zipfian_batch(zs, rng, bags, pooling_factor);
    std::memcpy(idx, b.indices.data(), b.indices.size() * sizeof(int64_t));
    std::memcpy(off, b.offsets.data(), b.offsets.size() * sizeof(int64_t));
  });
}

// ---- LFU cache (lfu_cache.hpp / lfu_cache.cpp) ----------------------------

struct RefCache {
  std::unique_ptr<LfuCache<float>> c;
  CachePartition last;
};

int ref_cache_create(int64_t capacity, int64_t emb, int64_t refresh, void** out) {
  return guarded([&] {
    auto* rc = new RefCache;
    rc->c = std::make_unique<LfuCache<float>>(capacity, emb, refresh);
    *out = rc;
  });
}
void ref_cache_destroy(void* c) { delete static_cast<RefCache*>(c); }
int64_t ref_cache_default_capacity(int64_t rows) {
  return LfuCache<float>::default_capacity(rows);
}

// LfuCache::record_and_partition (lfu_cache.hpp:187-219).  Sizes of the two
// parts are returned; fetch them with ref_cache_last_partition.
int ref_cache_record_and_partition(void* c, const int64_t* idx, int64_t L, const int64_t* off,
                                   int64_t B, const double* w, int pooling, int64_t* n_cached,
                                   int64_t* n_tt) {
  return guarded([&] {
    auto* rc = static_cast<RefCache*>(c);
    rc->last = rc->c->record_and_partition(make_batch(idx, L, off, B, w, pooling));
    *n_cached = rc->last.cached.num_lookups();
    *n_tt = rc->last.tt.num_lookups();
  });
}

void ref_cache_last_partition(void* c, int64_t* cached_slots, int64_t* cached_rows,
                              int64_t* cached_off, int64_t* tt_idx, int64_t* tt_off) {
  auto* rc = static_cast<RefCache*>(c);
  const auto& p = rc->last;
  std::memcpy(cached_slots, p.cached.indices.data(), p.cached.indices.size() * 8);
  std::memcpy(cached_rows, p.cached_rows.data(), p.cached_rows.size() * 8);
  std::memcpy(cached_off, p.cached.offsets.data(), p.cached.offsets.size() * 8);
  std::memcpy(tt_idx, p.tt.indices.data(), p.tt.indices.size() * 8);
  std::memcpy(tt_off, p.tt.offsets.data(), p.tt.offsets.size() * 8);
}

void ref_cache_record(void* c, const int64_t* idx, int64_t L) {
  IndexBatch b;
  b.indices.assign(idx, idx + L);
  b.offsets = {0, L};
  static_cast<RefCache*>(c)->c->record(b);
}

int ref_cache_warmup_finalize(void* c, void* t) {
  return guarded([&] {
    static_cast<RefCache*>(c)->c->warmup_finalize(*static_cast<RefTable*>(t)->f);
  });
}

int ref_cache_refresh(void* c, void* t, double* drift) {
  return guarded([&] {
    *drift = static_cast<RefCache*>(c)->c->refresh(*static_cast<RefTable*>(t)->f);
  });
}

int64_t ref_cache_hot_rows(void* c, int64_t* out) {
  auto rows = static_cast<RefCache*>(c)->c->hot_rows();
  if (out) std::memcpy(out, rows.data(), rows.size() * 8);
  return (int64_t)rows.size();
}

int64_t ref_cache_slot_of(void* c, int64_t row) {
  return static_cast<RefCache*>(c)->c->slot_of(row);
}

void ref_cache_row_values(void* c, int64_t slot, float* out) {
  auto v = static_cast<RefCache*>(c)->c->row_values(slot);
  std::memcpy(out, v.data(), v.size() * sizeof(float));
}

double ref_cache_hit_rate(void* c) { return static_cast<RefCache*>(c)->c->hit_rate(); }

uint64_t ref_cache_freq(void* c, int64_t row) {
  return static_cast<RefCache*>(c)->c->freq().count(row);
}

int64_t ref_cache_top_k(void* c, int64_t k, int64_t* out) {
  auto v = static_cast<RefCache*>(c)->c->freq().top_k(static_cast<size_t>(k));
  std::memcpy(out, v.data(), v.size() * 8);
  return (int64_t)v.size();
}

// ---- EmbeddingLayer<float> with a TT table + LFU cache (model.hpp:148-284) --
// The reference's own composition of the cache with forward_bags /
// backward_bags / sgd_step; used to record golden training trajectories.

struct RefLayer {
  std::unique_ptr<EmbeddingLayer<float>> l;
};

int ref_layer_create(int64_t rows, int64_t emb, int tt_dim, const int64_t* rf, const int64_t* cf,
                     const int64_t* rk, int64_t cache_capacity, const char* name, void** out) {
  return guarded([&] {
    ShapePlan p;
    p.num_rows = rows;
    p.emb_dim = emb;
    p.tt_dim = tt_dim;
    p.row_factors.assign(rf, rf + tt_dim);
    p.col_factors.assign(cf, cf + tt_dim);
    p.ranks.assign(rk, rk + tt_dim + 1);
    TableConfig cfg;
    cfg.num_rows = rows;
    cfg.use_tt = true;
    cfg.tt_dim = tt_dim;
    cfg.plan = p;
    cfg.use_cache = cache_capacity >= 0;
    cfg.cache_capacity = cache_capacity > 0 ? cache_capacity : 0;
    auto* rl = new RefLayer;
    rl->l = std::make_unique<EmbeddingLayer<float>>(cfg, emb, name);
    *out = rl;
  });
}
void ref_layer_destroy(void* l) { delete static_cast<RefLayer*>(l); }

int ref_layer_init(void* l, uint64_t seed) {
  return guarded([&] { static_cast<RefLayer*>(l)->l->init(InitSpec::sampled_gaussian(), seed); });
}

int ref_layer_forward(void* l, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                      const double* w, int pooling, float* out) {
  return guarded([&] {
    std::vector<float> o;
    static_cast<RefLayer*>(l)->l->forward(make_batch(idx, L, off, B, w, pooling), o,
                                          kDefaultMicroBatch, true);
    std::memcpy(out, o.data(), o.size() * sizeof(float));
  });
}

int ref_layer_backward(void* l, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                       const double* w, int pooling, const float* grad, int64_t n) {
  return guarded([&] {
    static_cast<RefLayer*>(l)->l->backward(make_batch(idx, L, off, B, w, pooling),
                                           std::span<const float>(grad, static_cast<size_t>(n)));
  });
}

int ref_layer_step(void* l, double lr) {
  return guarded([&] { static_cast<RefLayer*>(l)->l->step(lr); });
}
int ref_layer_finalize_warmup(void* l) {
  return guarded([&] { static_cast<RefLayer*>(l)->l->finalize_warmup(); });
}
int ref_layer_refresh(void* l, double* drift) {
  return guarded([&] { *drift = static_cast<RefLayer*>(l)->l->refresh_cache(); });
}
void ref_layer_get_core(void* l, int k, float* out) {
  const auto& c = static_cast<RefLayer*>(l)->l->tt()->core(k);
  std::memcpy(out, c.data(), c.size() * sizeof(float));
}
void ref_layer_cache_info(void* l, int64_t* resident, uint64_t* accesses, uint64_t* hits,
                          int* active) {
  const auto* c = static_cast<RefLayer*>(l)->l->cache();
  *resident = c->resident_count();
  *accesses = c->active_accesses();
  *hits = c->active_hits();
  *active = c->state() == CacheState::Active ? 1 : 0;
}
int64_t ref_layer_cache_rows(void* l, int64_t* slot_rows, float* values) {
  const auto* c = static_cast<RefLayer*>(l)->l->cache();
  for (int64_t s = 0; s < c->capacity(); ++s) {
    slot_rows[s] = c->row_at(s);
    auto v = c->row_values(s);
    std::memcpy(values + s * c->emb_dim(), v.data(), v.size() * sizeof(float));
  }
  return c->capacity();
}
uint64_t ref_layer_freq(void* l, int64_t row) {
  return static_cast<RefLayer*>(l)->l->cache()->freq().count(row);
}

// ---- CPU baseline timing: the reference's own OpenMP path -----------------
// One step = forward_bags(save=true) + backward_bags + sgd_step, fp32, the
// sequence SURVEY.md §8(d) / BASELINE.md §3 specifies.  Returns the median
// seconds per step over `reps` (after one warm-up step).
double ref_time_step(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                     const float* grad, double lr, int reps, int threads) {
  auto* t = static_cast<RefTable*>(h);
  if (threads > 0) omp_set_num_threads(threads);
  IndexBatch b = make_batch(idx, L, off, B, nullptr, 0);
  std::span<const float> g(grad, static_cast<size_t>(B) * t->f->cols());
  auto step = [&] {
    auto r = forward_bags(*t->f, b, kDefaultMicroBatch, true);
    auto gr = backward_bags(*t->f, b, r.context, g);
    sgd_step(*t->f, gr, lr);
  };
  step();
  std::vector<double> ts;
  for (int i = 0; i < reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    step();
    ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(ts.begin(), ts.end());
  return ts.empty() ? 0.0 : ts[ts.size() / 2];
}

// The serial oracle step: ref::forward_bags + ref::backward_bags (always
// recomputes, embedding_ops.hpp:378-492) + sgd_step -- BASELINE.md §3.2's
// "serial ref::" figure.  Median seconds per step over `reps` after one warm-up.
double ref_time_step_serial(void* h, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                            const float* grad, double lr, int reps) {
  auto* t = static_cast<RefTable*>(h);
  IndexBatch b = make_batch(idx, L, off, B, nullptr, 0);
  std::span<const float> g(grad, static_cast<size_t>(B) * t->f->cols());
  auto step = [&] {
    auto o = ref::forward_bags(*t->f, b);
    auto gr = ref::backward_bags(*t->f, b, g);
    sgd_step(*t->f, gr, lr);
    (void)o;
  };
  step();
  std::vector<double> ts;
  for (int i = 0; i < reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    step();
    ts.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  std::sort(ts.begin(), ts.end());
  return ts.empty() ? 0.0 : ts[ts.size() / 2];
}

#ifdef TTREF_CHECKPOINT
// ---- checkpoint.hpp / src/checkpoint.cpp (TTRECV01) ------------------------
// Checkpoint::put_table for every table (in order), optional f32 arrays
// (name, 1-D length), then save(path).
int ref_checkpoint_save(void* const* tables, int n, const char* const* array_names,
                        const float* const* arrays, const int64_t* array_lens, int na,
                        const char* path) {
  return guarded([&] {
    Checkpoint cp;
    for (int i = 0; i < n; ++i) {
      auto* t = static_cast<RefTable*>(tables[i]);
      if (t->dtype)
        cp.put_table(*t->d);
      else
        cp.put_table(*t->f);
    }
    for (int i = 0; i < na; ++i)
      cp.put_array<float>(array_names[i], {array_lens[i]},
                          std::span<const float>(arrays[i], static_cast<size_t>(array_lens[i])));
    cp.save(path);
  });
}

// Checkpoint::load(path).get_table<T>(name) -> a new RefTable
int ref_checkpoint_load_table(const char* path, const char* name, int dtype, void** out) {
  return guarded([&] {
    Checkpoint cp = Checkpoint::load(path);
    auto* t = new RefTable;
    t->dtype = dtype;
    if (dtype)
      t->d = std::make_unique<TtTable<double>>(cp.get_table<double>(name));
    else
      t->f = std::make_unique<TtTable<float>>(cp.get_table<float>(name));
    *out = t;
  });
}

// Checkpoint::load(path).get_array<float>(name) into out (len elements)
int ref_checkpoint_load_array(const char* path, const char* name, float* out, int64_t len) {
  return guarded([&] {
    Checkpoint cp = Checkpoint::load(path);
    auto v = cp.get_array<float>(name);
    require_arg(static_cast<int64_t>(v.size()) == len, "array length mismatch");
    std::memcpy(out, v.data(), sizeof(float) * v.size());
  });
}

#endif  // TTREF_CHECKPOINT


// ---- DlrmModel<float> + SyntheticDataSource (model.hpp:355-538, data.cpp:49-130) ----
// The reference model, used by tests/test_dlrm_gpu.py as the checker of the GPU
// DlrmModel (paper_2101_11714_b200/dlrm.py): the same minibatches, the
// reference's parameters copied over, then train steps on both.
struct RefModel {
  std::unique_ptr<DlrmModel<float>> m;
};

int ref_model_create(int64_t dense_features, int64_t emb_dim, int ntables, const int64_t* rows,
                     const int* use_tt, const int64_t* ranks, int nbottom, const int64_t* bottom,
                     int ntop, const int64_t* top, int interaction_dot, void** out) {
  return guarded([&] {
    ModelConfig cfg;
    cfg.dense_features = dense_features;
    cfg.emb_dim = emb_dim;
    for (int t = 0; t < ntables; ++t) {
      TableConfig tc;
      tc.num_rows = rows[t];
      tc.use_tt = use_tt[t] != 0;
      tc.tt_dim = 3;
      tc.rank = ranks[t];
      cfg.tables.push_back(tc);
    }
    cfg.bottom_layers.assign(bottom, bottom + nbottom);
    cfg.top_layers.assign(top, top + ntop);
    cfg.interaction = interaction_dot ? InteractionKind::Dot : InteractionKind::Concat;
    auto* rm = new RefModel;
    rm->m = std::make_unique<DlrmModel<float>>(cfg);
    *out = rm;
  });
}
void ref_model_destroy(void* m) { delete static_cast<RefModel*>(m); }

int ref_model_init(void* m, uint64_t seed) {
  return guarded([&] { static_cast<RefModel*>(m)->m->init(seed, InitSpec::sampled_gaussian()); });
}

// parameters through the reference's own checkpoint writer (EmbeddingLayer::put,
// Mlp::put): which 0 bottom.w, 1 bottom.b, 2 top.w, 3 top.b (index = layer),
// 4 TT core k of table index, 5 dense table index (k ignored); returns count
int64_t ref_model_param(void* m, int which, int index, int k, float* out) {
  int64_t n = -1;
  guarded([&] {
    Checkpoint cp;
    static_cast<RefModel*>(m)->m->save_checkpoint(cp);
    std::vector<float> v;
    if (which <= 3) {
      const char* pre = which < 2 ? "bottom" : "top";
      v = cp.get_array<float>(concat(pre, which % 2 == 0 ? ".w" : ".b", index));
    } else if (which == 4) {
      const auto tab = cp.get_table<float>(concat("table", index));
      v.assign(tab.core(k).begin(), tab.core(k).end());
    } else {
      v = cp.get_array<float>(concat("table", index));
    }
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(float));
    n = static_cast<int64_t>(v.size());
  });
  return n;
}

// one training step (train(), model.hpp:566-573): forward, bce_with_logits,
// backward, step.  idx / off: per table, concatenated (table t's lookups at
// lk_off[t], its bs + 1 offsets at t * (bs + 1)).
int ref_model_step(void* m, int64_t bs, const double* dense, const double* labels, int ntables,
                   const int64_t* idx, const int64_t* lk_off, const int64_t* off, double lr,
                   float* logits_out, double* loss_out) {
  return guarded([&] {
    auto& model = *static_cast<RefModel*>(m)->m;
    MiniBatch mb;
    mb.batch_size = bs;
    mb.dense.assign(dense, dense + bs * model.config().dense_features);
    mb.labels.assign(labels, labels + bs);
    for (int t = 0; t < ntables; ++t)
      mb.tables.push_back(make_batch(idx + lk_off[t], lk_off[t + 1] - lk_off[t], off + t * (bs + 1), bs,
                                     nullptr, 0));
    auto logits = model.forward(mb, kDefaultMicroBatch, true);
    std::vector<float> dlogits;
    *loss_out = bce_with_logits<float>(logits, mb.labels, &dlogits);
    if (logits_out) std::memcpy(logits_out, logits.data(), logits.size() * sizeof(float));
    model.backward(mb, dlogits);
    model.step(lr);
  });
}

// SyntheticDataSource minibatches (data.cpp): dense (bs x df), labels (bs),
// per-table lookups (pooling factor pf, so table t's lookups are at t * bs * pf)
// and offsets (t * (bs + 1))
struct RefSource {
  std::unique_ptr<SyntheticDataSource> s;
};
int ref_source_create(int64_t dense_features, int ntables, const int64_t* rows, double zipf,
                      int64_t bs, int64_t pf, uint64_t seed, void** out) {
  return guarded([&] {
    SyntheticConfig c;
    c.dense_features = dense_features;
    c.table_rows.assign(rows, rows + ntables);
    c.zipf_exponent = zipf;
    c.batch_size = bs;
    c.pooling_factor = pf;
    auto* rs = new RefSource;
    rs->s = std::make_unique<SyntheticDataSource>(c, seed);
    *out = rs;
  });
}
void ref_source_destroy(void* s) { delete static_cast<RefSource*>(s); }
int ref_source_next(void* s, int64_t iteration, double* dense, double* labels, int64_t* idx,
                    int64_t* off) {
  return guarded([&] {
    MiniBatch mb = static_cast<RefSource*>(s)->s->next(iteration);
    std::memcpy(dense, mb.dense.data(), mb.dense.size() * sizeof(double));
    std::memcpy(labels, mb.labels.data(), mb.labels.size() * sizeof(double));
    int64_t li = 0;
    for (size_t t = 0; t < mb.tables.size(); ++t) {
      const auto& b = mb.tables[t];
      std::memcpy(idx + li, b.indices.data(), b.indices.size() * 8);
      std::memcpy(off + t * b.offsets.size(), b.offsets.data(), b.offsets.size() * 8);
      li += static_cast<int64_t>(b.indices.size());
    }
  });
}

}  // extern "C"
