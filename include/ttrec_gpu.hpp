// ttrec_gpu.hpp -- C++ drop-in for the reference's TT-EmbeddingBag hot path.
//
// Header-only adapter over the C ABI (ttgpu.h / libttgpu.so).  A maintainer
// puts it next to /root/reference/proj/include/ttrec/embedding_ops.hpp; call
// sites switch by qualifying (or `using`) ttrec::gpu:: instead of ttrec::.
// Nothing here computes: every operation is one or two C-ABI calls.
//
//   ttrec::gpu::TtEmbeddingBagCuda   device-resident table:
//       TtEmbeddingBagCuda(const ShapePlan&, std::string name, int device, void* stream)
//       holds the cores in the reference's physical layout (m_k, R_{k-1}, n_k, R_k)
//       (tt_table.hpp:19-22), so upload/download are byte copies of TtTable::core(k).
//   ttrec::gpu::forward_bags / backward_bags / sgd_step / lookup_row
//       the reference's exact signatures over TtTable<float> (§8(b)(3)):
//         embedding_ops.hpp:159  ForwardResult<T> forward_bags(const TtTable<T>&, const IndexBatch&,
//                                                          index_t micro_batch, bool save)
//         embedding_ops.hpp:260  CoreGradients<T> backward_bags(const TtTable<T>&, const IndexBatch&,
//                                                           const ForwardContext<T>&, span<const T>)
//         embedding_ops.hpp:361  void sgd_step(TtTable<T>&, const CoreGradients<T>&, double)
//         embedding_ops.hpp:120  void lookup_row(const TtTable<T>&, index_t, span<T>)
//       The host TtTable stays authoritative (value semantics, like the
//       reference): a device shadow per table is (re)uploaded whenever the
//       table's mutation counter moves, and sgd_step writes the updated cores
//       back and bumps the counter exactly like the reference.
//
// Errors: status codes are re-thrown as the reference's exception types with
// the library's message (worded like the reference's: table names, "stale").
// Instrumentation: TT rows computed are added to ttrec::EmbeddingStats
// (embedding_ops.hpp:144,230), so acceptance criterion 7's counter works.
#pragma once

#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "ttgpu.h"
#include "ttrec/embedding_ops.hpp"
#include "ttrec/embedding_stats.hpp"

namespace ttrec::gpu {

inline void check(int st) {
  if (st == TTGPU_OK) return;
  const std::string m = ttgpu_last_error();
  if (st == TTGPU_ERR_INVALID_ARGUMENT) throw std::invalid_argument(m);
  if (st == TTGPU_ERR_OUT_OF_RANGE) throw std::out_of_range(m);
  throw std::runtime_error(m);
}

/// One TT table resident on one GPU (cores + gradient buffer + workspace);
/// T = float or double (the reference instantiates both, common.hpp:13-15).
template <typename T = float>
class TtEmbeddingBagCudaT {
 public:
  TtEmbeddingBagCudaT(const ShapePlan& plan, std::string name, int device = 0,
                      void* stream = nullptr)
      : plan_(plan), name_(std::move(name)) {
    check(ttgpu_create(plan.num_rows, plan.emb_dim, plan.tt_dim, plan.row_factors.data(),
                       plan.col_factors.data(), plan.ranks.data(),
                       std::is_same_v<T, double> ? TTGPU_F64 : TTGPU_F32, name_.c_str(),
                       device, stream, &h_));
    check(ttgpu_ctx_create(h_, &ctx_));
  }
  ~TtEmbeddingBagCudaT() {
    if (ctx_) ttgpu_ctx_destroy(ctx_);
    if (h_) ttgpu_destroy(h_);
  }
  TtEmbeddingBagCudaT(const TtEmbeddingBagCudaT&) = delete;
  TtEmbeddingBagCudaT& operator=(const TtEmbeddingBagCudaT&) = delete;

  const ShapePlan& plan() const { return plan_; }
  const std::string& name() const { return name_; }
  ttgpu_table* handle() const { return h_; }
  ttgpu_ctx* context() const { return ctx_; }

  void upload(const TtTable<T>& t) {
    for (int k = 0; k < t.dim(); ++k) check(ttgpu_set_core(h_, k, t.core(k).data()));
  }
  void download(TtTable<T>& t) const {
    for (int k = 0; k < t.dim(); ++k) check(ttgpu_get_core(h_, k, t.core(k).data()));
  }

  /// forward_bags into a host buffer (num_bags x emb_dim); the device context
  /// keeps what backward needs.
  void forward(const IndexBatch& b, index_t micro_batch, bool save, T* out) {
    check(ttgpu_forward(h_, b.indices.data(), b.num_lookups(), b.offsets.data(), b.num_bags(),
                        b.has_weights() ? b.weights.data() : nullptr,
                        b.pooling == Pooling::Mean ? TTGPU_MEAN : TTGPU_SUM, micro_batch,
                        save ? 1 : 0, out, ctx_));
  }
  /// backward_bags: dense gradients into per-core host buffers (may be null)
  void backward(const IndexBatch& b, std::span<const T> grad, T* const* grads_out) {
    check(ttgpu_backward(h_, ctx_, b.num_lookups(), b.num_bags(), grad.data(),
                         static_cast<int64_t>(grad.size()),
                         reinterpret_cast<void* const*>(grads_out)));
  }
  /// fused backward_bags + sgd_step on the device cores
  void backward_sgd(const IndexBatch& b, std::span<const T> grad, double lr) {
    check(ttgpu_backward_sgd(h_, ctx_, b.num_lookups(), b.num_bags(), grad.data(),
                             static_cast<int64_t>(grad.size()), lr));
  }
  void sgd(const CoreGradients<T>& g, double lr) {
    std::vector<const void*> p(g.cores.size());
    for (size_t k = 0; k < p.size(); ++k) p[k] = g.cores[k].data();
    check(ttgpu_sgd_step(h_, p.data(), lr));
  }
  void lookup_row(index_t row, T* out) { check(ttgpu_lookup_row(h_, row, out)); }

 private:
  ShapePlan plan_;
  std::string name_;
  ttgpu_table* h_ = nullptr;
  ttgpu_ctx* ctx_ = nullptr;
};
using TtEmbeddingBagCuda = TtEmbeddingBagCudaT<float>;

namespace detail {

/// Identity of a host table's contents: mutation counter, plan, name, core
/// buffer addresses and a hash of EVERY core element.  The reference allows
/// in-place writes through TtTable::core(k)[i] without mark_mutated() (its own
/// tests do this), so a sampled fingerprint could miss an edit and leave a
/// stale device shadow; the full hash (four independent 64-bit lanes, about
/// 1 ns per 8 bytes) costs less than re-uploading the cores.
template <typename T>
inline std::uint64_t fingerprint(const TtTable<T>& t) {
  std::uint64_t h = 1469598103934665603ull;
  auto mix = [&](std::uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  mix(t.mutation_counter());
  mix(static_cast<std::uint64_t>(t.rows()));
  mix(static_cast<std::uint64_t>(t.cols()));
  for (char c : t.name()) mix(static_cast<unsigned char>(c));
  const ShapePlan& p = t.plan();
  for (int k = 0; k < t.dim(); ++k) {
    mix(static_cast<std::uint64_t>(p.row_factors[k]));
    mix(static_cast<std::uint64_t>(p.col_factors[k]));
    mix(static_cast<std::uint64_t>(p.ranks[k + 1]));
    auto c = t.core(k);
    mix(reinterpret_cast<std::uintptr_t>(c.data()));
    mix(static_cast<std::uint64_t>(c.size()));
    const unsigned char* bytes = reinterpret_cast<const unsigned char*>(c.data());
    const size_t nb = c.size() * sizeof(T), nw = nb / 8;
    constexpr std::uint64_t kMul = 0x9E3779B97F4A7C15ull;
    std::uint64_t lane[4] = {1, 2, 3, 4};
    size_t i = 0;
    for (; i + 4 <= nw; i += 4)
      for (int j = 0; j < 4; ++j) {
        std::uint64_t v;
        std::memcpy(&v, bytes + 8 * (i + j), 8);
        lane[j] = (lane[j] ^ v) * kMul;
        lane[j] ^= lane[j] >> 29;
      }
    for (; i < nw; ++i) {
      std::uint64_t v;
      std::memcpy(&v, bytes + 8 * i, 8);
      lane[0] = ((lane[0] ^ v) * kMul) ^ (lane[0] >> 31);
    }
    for (size_t b = nw * 8; b < nb; ++b) lane[1] = (lane[1] ^ bytes[b]) * kMul;
    for (int j = 0; j < 4; ++j) mix(lane[j]);
  }
  return h;
}

/// Device shadow of a host TtTable<T>, refreshed when its cores change.
template <typename T>
struct Shadow {
  std::unique_ptr<TtEmbeddingBagCudaT<T>> dev;
  std::uint64_t uploaded_at = ~std::uint64_t{0};  // fingerprint of the uploaded cores
  // identity of the forward the device context holds
  const void* idx_data = nullptr;
  index_t L = -1, B = -1;
  std::uint64_t fwd_snapshot = ~std::uint64_t{0};
  bool fwd_saved = false;
};

template <typename T>
inline std::map<const TtTable<T>*, Shadow<T>>& registry() {
  static std::map<const TtTable<T>*, Shadow<T>> r;
  return r;
}

template <typename T>
inline Shadow<T>& shadow_of(const TtTable<T>& t, int device = 0) {
  Shadow<T>& s = registry<T>()[&t];
  const std::uint64_t fp = fingerprint(t);
  if (s.dev && s.uploaded_at != fp) {
    const ShapePlan& a = s.dev->plan();
    const ShapePlan& b = t.plan();
    if (a.num_rows != b.num_rows || a.emb_dim != b.emb_dim || a.row_factors != b.row_factors ||
        a.col_factors != b.col_factors || a.ranks != b.ranks || s.dev->name() != t.name())
      s.dev.reset();  // another table now lives at this address
  }
  if (!s.dev) s.dev = std::make_unique<TtEmbeddingBagCudaT<T>>(t.plan(), t.name(), device);
  if (s.uploaded_at != fp) {
    s.dev->upload(t);
    s.uploaded_at = fp;
    s.idx_data = nullptr;  // device context refers to older cores
  }
  return s;
}

}  // namespace detail

/// Drop the device shadow of a table (e.g. before the table is destroyed).
template <typename T>
inline void release(const TtTable<T>& t) { detail::registry<T>().erase(&t); }

/// embedding_ops.hpp:159-253 on the GPU; bit-identical output.
template <typename T>
inline ForwardResult<T> forward_bags(const TtTable<T>& table, const IndexBatch& batch,
                                     index_t micro_batch = kDefaultMicroBatch,
                                     bool save_intermediates = false) {
  batch.validate(table.rows(), table.name());
  detail::Shadow<T>& s = detail::shadow_of(table);
  ForwardResult<T> r;
  r.output.assign(static_cast<size_t>(batch.num_bags()) * table.cols(), T(0));
  const std::uint64_t before = ttgpu_stats_rows();
  s.dev->forward(batch, micro_batch, save_intermediates, r.output.data());
  EmbeddingStats::add_rows(ttgpu_stats_rows() - before);
  // device workspace high-water mark into the reference's workspace counter
  // (the GPU path does not chunk by micro_batch, so it does not scale with it)
  const auto ws = static_cast<std::size_t>(ttgpu_stats_peak_workspace());
  EmbeddingStats::workspace_add(ws);
  EmbeddingStats::workspace_sub(ws);
  s.idx_data = batch.indices.data();
  s.L = batch.num_lookups();
  s.B = batch.num_bags();
  s.fwd_snapshot = table.mutation_counter();
  s.fwd_saved = save_intermediates;
  r.context.table = &table;
  r.context.num_lookups = batch.num_lookups();
  r.context.num_bags = batch.num_bags();
  r.context.micro_batch = micro_batch;
  r.context.saved = save_intermediates;
  r.context.mutation_snapshot = table.mutation_counter();
  return r;
}

/// embedding_ops.hpp:260-358 on the GPU: the reference's checks (:264-274),
/// then dense CoreGradients in the core layout.
template <typename T>
inline CoreGradients<T> backward_bags(const TtTable<T>& table, const IndexBatch& batch,
                                      const ForwardContext<T>& ctx,
                                      std::span<const T> grad_output) {
  const ShapePlan& plan = table.plan();
  batch.validate(plan.num_rows, table.name());
  require_arg(ctx.table == &table, "forward context belongs to a different table");
  require_arg(ctx.num_lookups == batch.num_lookups() && ctx.num_bags == batch.num_bags(),
              "forward context does not match this batch (", ctx.num_lookups, "/", ctx.num_bags,
              " vs ", batch.num_lookups(), "/", batch.num_bags(), ")");
  require_arg(ctx.mutation_snapshot == table.mutation_counter(), "stale forward context for table '",
              table.name(), "': cores changed since the forward pass");
  require_arg(static_cast<index_t>(grad_output.size()) == batch.num_bags() * plan.emb_dim,
              "grad_output has ", grad_output.size(), " elements, expected ",
              batch.num_bags() * plan.emb_dim);
  detail::Shadow<T>& s = detail::shadow_of(table);
  if (s.idx_data != batch.indices.data() || s.L != batch.num_lookups() ||
      s.B != batch.num_bags() || s.fwd_snapshot != table.mutation_counter()) {
    // the device context holds another forward: rebuild it (not counted as
    // TT rows, like the reference's backward recompute, test_embedding_ops.cpp:341)
    std::vector<T> scratch(static_cast<size_t>(batch.num_bags()) * table.cols());
    s.dev->forward(batch, ctx.micro_batch, true, scratch.data());
    s.idx_data = batch.indices.data();
    s.L = batch.num_lookups();
    s.B = batch.num_bags();
    s.fwd_snapshot = table.mutation_counter();
  }
  CoreGradients<T> g = CoreGradients<T>::zeros_like(table);
  std::vector<T*> p(g.cores.size());
  for (size_t k = 0; k < p.size(); ++k) p[k] = g.cores[k].data();
  s.dev->backward(batch, grad_output, p.data());
  return g;
}

/// embedding_ops.hpp:361-376: core -= T(lr) * grad (separately rounded, like
/// the reference), written back to the host table; invalidates contexts.
template <typename T>
inline void sgd_step(TtTable<T>& table, const CoreGradients<T>& grads, double lr) {
  require_arg(static_cast<int>(grads.cores.size()) == table.dim(), "gradient core count mismatch");
  for (int k = 0; k < table.dim(); ++k)
    require_arg(grads.cores[k].size() == table.core(k).size(), "gradient shape mismatch on core ", k);
  detail::Shadow<T>& s = detail::shadow_of(table);
  s.dev->sgd(grads, lr);
  s.dev->download(table);
  table.mark_mutated();
  s.uploaded_at = detail::fingerprint(table);  // the device already holds these cores
  s.idx_data = nullptr;
}

/// embedding_ops.hpp:120-152 (bit-identical; bumps the row counter by one)
template <typename T>
inline void lookup_row(const TtTable<T>& table, index_t row, std::span<T> out) {
  if (row < 0 || row >= table.plan().num_rows)
    throw std::out_of_range(concat("index ", row, " out of range [0, ", table.plan().num_rows,
                                   ") for table '", table.name(), "'"));
  require_arg(static_cast<index_t>(out.size()) == table.plan().emb_dim, "lookup_row: out has ",
              out.size(), " elements, expected ", table.plan().emb_dim);
  detail::Shadow<T>& s = detail::shadow_of(table);
  s.dev->lookup_row(row, out.data());
  EmbeddingStats::add_rows(1);
}

template <typename T>
inline std::vector<T> lookup_row(const TtTable<T>& table, index_t row) {
  std::vector<T> out(table.cols());
  gpu::lookup_row(table, row, std::span<T>(out));
  return out;
}

}  // namespace ttrec::gpu
