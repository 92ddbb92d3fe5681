// LFU cache -- host side and C ABI (included at the end of ttgpu.cu).
// Mirrors LfuCache<T> (lfu_cache.hpp:134-310) and the cached EmbeddingLayer
// calls (model.hpp:195-284); see lfu_cache.cuh for the device layout.
#include <thrust/iterator/counting_iterator.h>

#include <cub/device/device_select.cuh>

#include "lfu_cache.cuh"

struct ttgpu_cache {
  int64_t capacity = 0, emb_dim = 0, refresh_period = 1000, key_space = 0;
  int dtype = TTGPU_F32;
  size_t esz = 4;
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t last = nullptr;  // stream of the last call that wrote cache state
  bool last_set = false;
  int num_sms = 148;
  bool active = false;
  // frequencies (dense, one counter per row) and counters [accesses, hits]
  DevBuf counts, counters, errs;
  uint64_t accesses = 0;  // partition path: host-side (known L); fast path: counters[0]
  // residency: hash (row -> slot) + slot rows + values; double-buffered for admit
  struct Res {
    DevBuf hkeys, hvals, slot_rows, store;
    int hshift = 63;
    unsigned long long hmask = 1;
    int64_t resident = 0;
  } res[2];
  int cur = 0;
  std::vector<int64_t> prev_top;  // hot_rows() after the last admit (sorted)
  // last partition (device)
  DevBuf lk_slot, flags, hpos, c_idx, c_rows, c_w, c_bag, c_off, t_idx, t_w, t_off;
  int64_t L = 0, B = 0, n_cached = 0, n_tt = 0;
  int pooling = TTGPU_SUM;
  bool has_w = false;
  bool part_valid = false;
  // layer state: chain output / grad_eff / slot gradients
  DevBuf tt_out, grad_eff, skey_in, skey, spos_in, spos, seg_lo, seg_hi, part, sg, tmp;
  bool grads_valid = false;
  // refresh scratch
  DevBuf sel_rows, sel_n, sel_cnt, top_cnt, top_rows, old_slot, fresh, fpos, new_rows, chain;
  // host-API staging
  DevBuf h_idx_stage, h_off_stage, h_w_stage;
  // fast path: the cache consulted inside the fast-path sort (f3_gsort), no
  // host sync; the partition exists only as per-lookup slots on the device
  bool fast_enabled = true;
  bool fast_part = false;  // the last partition came from the fast path
  DevBuf f_slot, f_perm3, f_skey3, f_ncached;
  const int64_t* f_idx = nullptr;  // the last fast forward's device batch (last_partition)
  const int64_t* f_off = nullptr;
  const double* f_w = nullptr;
  // side stream for the slot gradients (forked from / joined to the table's
  // stream: they overlap the chain backward, also inside a captured graph)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ~ttgpu_cache() {
    if (side) cudaStreamDestroy(side);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
  }
  Res& now() { return res[cur]; }
};

namespace ttgpu {
namespace {

int bits_for_slots(int64_t cap) {
  int b = 1;
  while ((int64_t{1} << b) < cap + 1) ++b;
  return b;
}

void cache_ensure_tmp(ttgpu_cache* c, size_t bytes) { c->tmp.ensure(std::max<size_t>(bytes, 256)); }

// The stream a cache call runs on (the table's, when one is involved); it is
// remembered so calls that only touch cache state order after it.
cudaStream_t cache_stream(ttgpu_cache* c, ttgpu_table* t) {
  cudaStream_t s = t ? t->stream : c->stream;
  c->last = s;
  c->last_set = true;
  return s;
}

// Order c->stream after the last stream that wrote cache state (seg_lo, sg,
// slot_rows, store are produced on the table's stream by forward / backward /
// admit, which may differ from the cache's own stream).
void cache_order_after_last(ttgpu_cache* c) {
  if (c->last_set && c->last != c->stream) CK(cudaStreamSynchronize(c->last));
}

void cache_raise(ttgpu_cache* c, cudaStream_t st, const int64_t* host_idx, const char* what) {
  unsigned long long h[2];
  CK(cudaMemcpyAsync(h, c->errs.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] == ULLONG_MAX && h[1] == 0) return;
  unsigned long long init[2] = {ULLONG_MAX, 0};
  CK(cudaMemcpyAsync(c->errs.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  const int sf = static_cast<int>(h[1]);
  if (sf & 1) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets must start at 0");
  if (sf & 2) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing");
  if (sf & 4) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets end does not match the index count");
  const int64_t pos = static_cast<int64_t>(h[0]);
  if (host_idx)
    throw std::out_of_range(cat("index ", host_idx[pos], " out of range [0, ", c->key_space,
                                ") for ", what));
  throw std::out_of_range(cat("index at lookup ", pos, " out of range [0, ", c->key_space,
                              ") for ", what));
}

// record_and_partition on device pointers; returns (with a sync) the part sizes
void cache_partition(ttgpu_cache* c, cudaStream_t st, const int64_t* idx, int64_t L,
                     const int64_t* off, int64_t B, const double* w, int pooling,
                     const int64_t* host_idx, const char* what) {
  require_arg(L >= 0 && B >= 0, "negative batch size");
  require_arg(L < (int64_t{1} << 31), "batch too large for the cache partition");
  c->lk_slot.ensure(4 * std::max<int64_t>(L, 1));
  c->flags.ensure(4 * (L + 1));
  c->hpos.ensure(4 * (L + 1));
  c->c_idx.ensure(8 * std::max<int64_t>(L, 1));
  c->c_rows.ensure(8 * std::max<int64_t>(L, 1));
  c->c_bag.ensure(4 * std::max<int64_t>(L, 1));
  c->t_idx.ensure(8 * std::max<int64_t>(L, 1));
  c->c_off.ensure(8 * (B + 1));
  c->t_off.ensure(8 * (B + 1));
  if (w) {
    c->c_w.ensure(8 * std::max<int64_t>(L, 1));
    c->t_w.ensure(8 * std::max<int64_t>(L, 1));
  }
  if (B > 0)
    lfu::k_check_offsets<<<grid_for(B, kThreads, c->num_sms), kThreads, 0, st>>>(
        off, B, L, reinterpret_cast<int*>(c->errs.as<unsigned long long>() + 1));
  auto& R = c->now();
  const int g = grid_for(std::max<int64_t>(L, 1), kThreads, c->num_sms, 8);
  lfu::k_partition<<<g, kThreads, 0, st>>>(
      idx, L, c->key_space, c->counts.as<unsigned long long>(),
      R.hkeys.as<unsigned long long>(), R.hvals.as<int>(), R.hshift, R.hmask, c->active ? 1 : 0,
      0, c->lk_slot.as<int>(), c->flags.as<int>(), c->errs.as<unsigned long long>(),
      c->counters.as<unsigned long long>() + 1);
  CK(cudaGetLastError());
  size_t tb = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, c->flags.as<int>(), c->hpos.as<int>(),
                                   static_cast<int>(L + 1), st));
  cache_ensure_tmp(c, tb);
  CK(cub::DeviceScan::ExclusiveSum(c->tmp.p, tb, c->flags.as<int>(), c->hpos.as<int>(),
                                   static_cast<int>(L + 1), st));
  lfu::k_split<<<grid_for(std::max<int64_t>(L, B + 1), kThreads, c->num_sms, 8), kThreads, 0, st>>>(
      idx, L, off, B, w, c->lk_slot.as<int>(), c->hpos.as<int>(), c->c_idx.as<int64_t>(),
      c->c_rows.as<int64_t>(), w ? c->c_w.as<double>() : nullptr, c->c_bag.as<int32_t>(),
      c->c_off.as<int64_t>(), c->t_idx.as<int64_t>(), w ? c->t_w.as<double>() : nullptr,
      c->t_off.as<int64_t>());
  CK(cudaGetLastError());
  int nc = 0;
  CK(cudaMemcpyAsync(&nc, c->hpos.as<int>() + L, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c->part_valid = false;
  c->fast_part = false;
  cache_raise(c, st, host_idx, what);
  if (c->active) c->accesses += static_cast<uint64_t>(L);
  c->L = L;
  c->B = B;
  c->n_cached = nc;
  c->n_tt = L - nc;
  c->pooling = pooling;
  c->has_w = w != nullptr;
  c->part_valid = true;
  c->grads_valid = false;
}

// admit(top_k(capacity)) (lfu_cache.hpp:223-243, 266-296) on the device
void cache_admit(ttgpu_cache* c, ttgpu_table* t) {
  cudaStream_t st = t->stream;
  const int64_t K = c->key_space;
  // rows with a count, ascending
  c->sel_rows.ensure(8 * std::max<int64_t>(K, 1));
  c->sel_n.ensure(16);
  size_t tb = 0;
  thrust::counting_iterator<int64_t> rows_it(0);
  lfu::HasCount pred{c->counts.as<unsigned long long>()};
  CK(cub::DeviceSelect::If(nullptr, tb, rows_it, c->sel_rows.as<int64_t>(), c->sel_n.as<int64_t>(),
                           K, pred, st));
  cache_ensure_tmp(c, tb);
  CK(cub::DeviceSelect::If(c->tmp.p, tb, rows_it, c->sel_rows.as<int64_t>(), c->sel_n.as<int64_t>(),
                           K, pred, st));
  int64_t n = 0;
  CK(cudaMemcpyAsync(&n, c->sel_n.p, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // (count desc, row asc): stable descending radix sort of rows already ascending
  c->sel_cnt.ensure(8 * std::max<int64_t>(n, 1));
  c->top_cnt.ensure(8 * std::max<int64_t>(n, 1));
  c->top_rows.ensure(8 * std::max<int64_t>(n, 1));
  if (n > 0) {
    lfu::k_gather_counts<<<grid_for(n, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        c->sel_rows.as<int64_t>(), n, c->counts.as<unsigned long long>(),
        c->sel_cnt.as<unsigned long long>());
    CK(cub::DeviceRadixSort::SortPairsDescending(
        nullptr, tb, c->sel_cnt.as<unsigned long long>(), c->top_cnt.as<unsigned long long>(),
        c->sel_rows.as<int64_t>(), c->top_rows.as<int64_t>(), static_cast<int>(n), 0, 64, st));
    cache_ensure_tmp(c, tb);
    CK(cub::DeviceRadixSort::SortPairsDescending(
        c->tmp.p, tb, c->sel_cnt.as<unsigned long long>(), c->top_cnt.as<unsigned long long>(),
        c->sel_rows.as<int64_t>(), c->top_rows.as<int64_t>(), static_cast<int>(n), 0, 64, st));
  }
  const int64_t k = std::min<int64_t>(n, c->capacity);
  // mark retained / fresh rows against the current residency
  auto& O = c->now();
  auto& N = c->res[1 - c->cur];
  c->old_slot.ensure(4 * std::max<int64_t>(k, 1));
  c->fresh.ensure(4 * (k + 1));
  c->fpos.ensure(4 * (k + 1));
  c->new_rows.ensure(8 * std::max<int64_t>(k, 1));
  const int gk = grid_for(std::max<int64_t>(k, 1), kThreads, c->num_sms);
  lfu::k_admit_mark<<<gk, kThreads, 0, st>>>(
      c->top_rows.as<int64_t>(), k, O.hkeys.as<unsigned long long>(), O.hvals.as<int>(), O.hshift,
      O.hmask, O.resident > 0 ? 1 : 0, c->old_slot.as<int>(), c->fresh.as<int>());
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, c->fresh.as<int>(), c->fpos.as<int>(),
                                   static_cast<int>(k + 1), st));
  cache_ensure_tmp(c, tb);
  CK(cub::DeviceScan::ExclusiveSum(c->tmp.p, tb, c->fresh.as<int>(), c->fpos.as<int>(),
                                   static_cast<int>(k + 1), st));
  lfu::k_admit_compact<<<gk, kThreads, 0, st>>>(c->top_rows.as<int64_t>(), k, c->fresh.as<int>(),
                                                c->fpos.as<int>(), c->new_rows.as<int64_t>());
  int nfresh = 0;
  CK(cudaMemcpyAsync(&nfresh, c->fpos.as<int>() + k, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // chain values of the newly admitted rows: lookup_row (stats += 1 per row, :287)
  c->chain.ensure(c->esz * c->emb_dim * std::max(nfresh, 1));
  if (nfresh > 0) {
    const int s = ttgpu_lookup_rows_device(t, c->new_rows.as<int64_t>(), nfresh, c->chain.p);
    if (s) fail(s, g_last_error);
  }
  // new residency: hash + slot rows + values
  int64_t hcap = 64;
  while (hcap < 2 * c->capacity) hcap <<= 1;
  int lg = 0;
  while ((int64_t{1} << lg) < hcap) ++lg;
  N.hkeys.ensure(8 * hcap);
  N.hvals.ensure(4 * hcap);
  N.slot_rows.ensure(8 * c->capacity);
  N.store.ensure(c->esz * c->capacity * c->emb_dim);
  N.hshift = 64 - lg;
  N.hmask = static_cast<unsigned long long>(hcap - 1);
  CK(cudaMemsetAsync(N.hkeys.p, 0xff, 8 * hcap, st));
  if (k > 0)
    lfu::k_hash_insert<<<gk, kThreads, 0, st>>>(c->top_rows.as<int64_t>(), k,
                                                N.hkeys.as<unsigned long long>(), N.hvals.as<int>(),
                                                N.hshift, N.hmask);
  const int64_t nv = c->capacity * c->emb_dim;
  const int gv = grid_for(nv, kThreads, c->num_sms, 8);
  if (c->dtype == TTGPU_F64)
    lfu::k_admit_fill<double><<<gv, kThreads, 0, st>>>(
        k, c->capacity, static_cast<int>(c->emb_dim), c->top_rows.as<int64_t>(),
        c->old_slot.as<int>(), c->fpos.as<int>(), c->chain.as<double>(), O.store.as<double>(),
        N.store.as<double>(), N.slot_rows.as<int64_t>());
  else
    lfu::k_admit_fill<float><<<gv, kThreads, 0, st>>>(
        k, c->capacity, static_cast<int>(c->emb_dim), c->top_rows.as<int64_t>(),
        c->old_slot.as<int>(), c->fpos.as<int>(), c->chain.as<float>(), O.store.as<float>(),
        N.store.as<float>(), N.slot_rows.as<int64_t>());
  CK(cudaGetLastError());
  N.resident = k;
  c->cur = 1 - c->cur;
  c->grads_valid = false;
  c->part_valid = false;  // slot ids change with the hot set (slots stable only between refreshes)
  std::vector<int64_t> top(static_cast<size_t>(k));
  if (k > 0)
    CK(cudaMemcpyAsync(top.data(), c->top_rows.p, 8 * k, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::sort(top.begin(), top.end());
  c->prev_top.swap(top);
}

double drift_of(std::vector<int64_t> a, std::vector<int64_t> b, int64_t k) {
  require_arg(k > 0, "hot_set_drift needs k > 0");
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  std::vector<int64_t> sym;
  std::set_symmetric_difference(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(sym));
  return static_cast<double>(sym.size()) / (2.0 * static_cast<double>(k));
}

void check_layer(ttgpu_cache* c, ttgpu_table* t) {
  require_arg(t != nullptr, "cached layer needs a table");
  require_arg(t->plan.emb_dim == c->emb_dim,
              cat("cache emb_dim ", c->emb_dim, " does not match table emb_dim ", t->plan.emb_dim));
  require_arg(t->dtype == c->dtype, "cache and table dtypes differ");
  require_arg(t->device == c->device, "cache and table live on different devices");
  require_arg(c->key_space == t->plan.num_rows,
              cat("cache key space ", c->key_space, " does not match table rows ", t->plan.num_rows));
}

// ---- cache fast path: record_and_partition inside f3_gsort ---------------
__device__ unsigned long long g_dev_cached_rows = 0;  // chain rows the fast path did not compute
std::mutex g_fast_dev_mu;
std::vector<int> g_fast_devs;  // devices whose g_dev_cached_rows may be non-zero

}  // namespace

// hits of the cache fast path so far (EmbeddingStats: chain rows it did not
// compute), summed over the devices that ran it; reset zeroes them.  Reads
// after the device work (the legacy-stream copy orders it on blocking streams).
uint64_t cache_fast_rows(bool reset) {
  std::lock_guard<std::mutex> lk(g_fast_dev_mu);
  uint64_t total = 0;
  int cur = 0;
  if (g_fast_devs.empty()) return 0;
  cudaGetDevice(&cur);
  for (int dev : g_fast_devs) {
    cudaSetDevice(dev);
    cudaDeviceSynchronize();
    unsigned long long v = 0;
    if (reset)
      cudaMemcpyToSymbol(g_dev_cached_rows, &v, sizeof(v));
    else if (cudaMemcpyFromSymbol(&v, g_dev_cached_rows, sizeof(v)) == cudaSuccess)
      total += v;
  }
  cudaSetDevice(cur);
  return total;
}

namespace {

bool cache_fast_ok(ttgpu_cache* c, ttgpu_table* t, int64_t L, int64_t B) {
  if (!c->fast_enabled || t->dtype != TTGPU_F32 || c->dtype != TTGPU_F32 || t->force_generic ||
      t->chunked)
    return false;
  if (L <= 0 || B <= 0 || c->emb_dim % 4 != 0 || c->capacity < 1 || c->capacity > 4096) return false;
  if (f3_kind(t) < 0 || !f3_feasible(t, L)) return false;
  int GS = 0, PW = 0;
  gsort_grid(t, make_geo(t), L, static_cast<int>(c->capacity), &GS, &PW);
  return GS > 0;
}

void cache_forward_fast(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const int64_t* idx, int64_t L,
                        const int64_t* off, int64_t B, const double* w, int pooling, bool save,
                        float* out) {
  cudaStream_t st = t->stream;
  cache_stream(c, t);
  const int K3 = static_cast<int>(c->capacity);
  c->f_slot.ensure(4 * L);
  c->f_perm3.ensure(4 * L);
  c->f_skey3.ensure(4 * L);
  c->f_ncached.ensure(16);
  c->seg_lo.ensure(4 * c->capacity);
  c->seg_hi.ensure(4 * c->capacity);
  {
    std::lock_guard<std::mutex> lk(g_fast_dev_mu);
    if (std::find(g_fast_devs.begin(), g_fast_devs.end(), t->device) == g_fast_devs.end())
      g_fast_devs.push_back(t->device);
  }
  unsigned long long* dev_rows = nullptr;
  CK(cudaGetSymbolAddress(reinterpret_cast<void**>(&dev_rows), g_dev_cached_rows));
  F3Cache fc;
  fc.K3 = K3;
  fc.counts = c->counts.as<unsigned long long>();
  auto& R = c->now();
  fc.hkeys = R.hkeys.as<unsigned long long>();
  fc.hvals = R.hvals.as<int>();
  fc.hshift = R.hshift;
  fc.hmask = R.hmask;
  fc.active = c->active && R.resident > 0 ? 1 : 0;
  fc.hits = c->counters.as<unsigned long long>() + 1;
  fc.accesses = fc.active ? c->counters.as<unsigned long long>() : nullptr;  // device-side: graph replays count
  fc.hits2 = dev_rows;
  fc.lk_slot = c->f_slot.as<int>();
  fc.slot_rows = R.slot_rows.as<int64_t>();
  fc.perm3 = c->f_perm3.as<uint32_t>();
  fc.skey3 = c->f_skey3.as<int>();
  fc.seg_lo3 = c->seg_lo.as<int>();
  fc.seg_hi3 = c->seg_hi.as<int>();
  fc.ncached = c->f_ncached.as<int>();
  fc.store = R.store.as<float>();  // read only for hits (none while warming up)
  // ForwardContext bookkeeping of forward_bags(part.tt): the chain part is
  // Sum-pooled with the batch's weights; its size is known on the device only
  ctx->table = t;
  ctx->snapshot = t->generation;
  ctx->L = L;
  ctx->B = B;
  ctx->pooling = TTGPU_SUM;
  ctx->save = false;
  ctx->exact = t->exact;
  ctx->has_w = w != nullptr;
  ctx->w_dev = w;
  ctx->valid = true;
  ctx->fast = true;
  (void)save;
  g_rows.fetch_add(static_cast<uint64_t>(L));  // less the hits, counted on the device
  if (!ctx->f3) ctx->f3 = new F3Bufs;
  ctx->lk_bag.ensure(4 * L);
  ctx->lk_alpha.ensure(4 * L);
  f3_forward(f3_kind(t), t, *ctx->f3, idx, L, off, B, w, pooling, out, t->exact,
             ctx->lk_bag.as<int32_t>(), ctx->lk_alpha.as<float>(), &fc);
  // every bag was pooled by f3_gsort (all lookups cached) or by the last
  // chain lookup in f3_fwd (pool_if_last with the cached rows): no combine pass
  c->L = L;
  c->B = B;
  c->pooling = pooling;
  c->has_w = w != nullptr;
  c->f_idx = idx;
  c->f_off = off;
  c->f_w = w;
  c->fast_part = true;
  c->part_valid = true;
  c->grads_valid = false;
}

void cache_backward_fast(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const float* grad, bool fused,
                         double lr) {
  cudaStream_t st = t->stream;
  cache_stream(c, t);
  const int64_t B = c->B, L = c->L;
  const int N = static_cast<int>(c->emb_dim);
  const float* ge = grad;
  if (c->pooling == TTGPU_MEAN) {
    c->grad_eff.ensure(4 * B * N);
    lfu::k_grad_eff_off<<<grid_for(B * N, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        B, N, c->f_off, grad, c->grad_eff.as<float>());
    ge = c->grad_eff.as<float>();
  }
  // slot gradients (the cached lookups sorted by slot: f3_gsort's key 3) on a
  // side stream, concurrent with the chain part's backward
  if (!c->side) {
    int lo = 0, hi = 0;  // lowest priority: the chain backward is the critical path
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, lo));
    CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  c->sg.ensure(4 * c->capacity * N);
  c->part.ensure(4 * L * N);
  CK(cudaEventRecord(c->ev_fork, st));
  CK(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  const cudaStream_t st_main = st;
  st = c->side;
  const int64_t chunks = (L + lfu::kSlotChunk - 1) / lfu::kSlotChunk;
  lfu::k_slot_chunks<float><<<grid_for(chunks * 32, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
      L, N, c->f_skey3.as<int>(), reinterpret_cast<const int*>(c->f_perm3.as<uint32_t>()), c->f_w,
      ctx->lk_bag.as<int32_t>(), ge, c->seg_lo.as<int>(), c->seg_hi.as<int>(), c->part.as<float>(),
      c->sg.as<float>(), c->now().store.as<float>(), fused ? 1 : 0, static_cast<float>(lr),
      c->f_ncached.as<int>());
  lfu::k_slot_fold<float><<<grid_for(c->capacity * N * 32, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
      c->capacity, N, c->seg_lo.as<int>(), c->seg_hi.as<int>(), c->part.as<float>(), c->sg.as<float>(),
      c->now().store.as<float>(), fused ? 1 : 0, static_cast<float>(lr));
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev_join, st));
  st = st_main;
  // chain part: the fast-path backward over the chain lookups' tiles (the
  // dense gradient, or fused with the SGD)
  f3_backward(t, *ctx->f3, ge, fused ? 1 : 0, static_cast<float>(lr), ctx->lk_bag.as<int32_t>(),
              ctx->lk_alpha.as<float>(), L);
  if (fused) ++t->generation;
  CK(cudaStreamWaitEvent(st, c->ev_join, 0));
  t->mark("cache_bwd");
  c->grads_valid = !fused;
}

// EmbeddingLayer::forward with a cache (model.hpp:210-223), device pointers
template <typename T>
void cache_forward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const int64_t* idx, int64_t L,
                   const int64_t* off, int64_t B, const double* w, int pooling, bool save, T* out,
                   const int64_t* host_idx) {
  check_layer(c, t);
  require_arg(ctx != nullptr, "forward needs a context");
  cudaStream_t st = t->stream;
  if constexpr (std::is_same_v<T, float>) {
    if (cache_fast_ok(c, t, L, B)) {
      cache_forward_fast(c, t, ctx, idx, L, off, B, w, pooling, save, out);
      return;
    }
  }
  c->fast_part = false;
  cache_partition(c, st, idx, L, off, B, w, pooling, host_idx,
                  cat("table '", t->name, "'").c_str());
  const int N = static_cast<int>(c->emb_dim);
  c->tt_out.ensure(sizeof(T) * std::max<int64_t>(B * N, 1));
  forward_impl<T>(t, ctx, c->t_idx.as<int64_t>(), c->n_tt, c->t_off.as<int64_t>(), B,
                  w ? c->t_w.as<double>() : nullptr, TTGPU_SUM, save, c->tt_out.as<T>(), t->exact);
  if (B > 0) {
    lfu::k_combine<T><<<grid_for(B * N, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        B, N, c->c_off.as<int64_t>(), c->c_idx.as<int64_t>(), w ? c->c_w.as<double>() : nullptr,
        c->now().store.as<T>(), c->t_off.as<int64_t>(), c->tt_out.as<T>(),
        pooling == TTGPU_MEAN ? 1 : 0, out);
    CK(cudaGetLastError());
  }
}

// EmbeddingLayer::backward with a cache (model.hpp:237-262) [+ step(), :265-284]
template <typename T>
void cache_backward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const T* grad, bool fused,
                    double lr) {
  check_layer(c, t);
  require_arg(c->part_valid, "cache backward needs the partition of a cached forward");
  check_ctx(t, ctx);
  if constexpr (std::is_same_v<T, float>) {
    if (c->fast_part) {
      cache_backward_fast(c, t, ctx, grad, fused, lr);
      return;
    }
  }
  cudaStream_t st = t->stream;
  const int64_t B = c->B;
  const int N = static_cast<int>(c->emb_dim);
  const T* ge = grad;
  if (c->pooling == TTGPU_MEAN && B > 0) {
    c->grad_eff.ensure(sizeof(T) * B * N);
    lfu::k_grad_eff<T><<<grid_for(B * N, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        B, N, c->c_off.as<int64_t>(), c->t_off.as<int64_t>(), grad, c->grad_eff.as<T>());
    ge = c->grad_eff.as<T>();
  }
  backward_impl<T>(t, ctx, ge, fused ? 1 : 0, lr);
  if (fused) ++t->generation;
  // slot gradients: stable sort of the cached lookups by slot, chunked sums
  const int64_t n = c->n_cached;
  c->seg_lo.ensure(4 * c->capacity);
  c->seg_hi.ensure(4 * c->capacity);
  c->sg.ensure(sizeof(T) * c->capacity * N);
  CK(cudaMemsetAsync(c->seg_lo.p, 0xff, 4 * c->capacity, st));
  if (n > 0) {
    c->skey_in.ensure(4 * n);
    c->skey.ensure(4 * n);
    c->spos_in.ensure(4 * n);
    c->spos.ensure(4 * n);
    c->part.ensure(sizeof(T) * n * N);
    // keys: int32 slot ids; values: cached-lookup positions
    lfu::k_fill_slot_keys<<<grid_for(n, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        c->c_idx.as<int64_t>(), n, c->skey_in.as<int>(), c->spos_in.as<int>());
    const int bits = bits_for_slots(c->capacity);
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, c->skey_in.as<int>(), c->skey.as<int>(),
                                       c->spos_in.as<int>(), c->spos.as<int>(), static_cast<int>(n),
                                       0, bits, st));
    cache_ensure_tmp(c, tb);
    CK(cub::DeviceRadixSort::SortPairs(c->tmp.p, tb, c->skey_in.as<int>(), c->skey.as<int>(),
                                       c->spos_in.as<int>(), c->spos.as<int>(), static_cast<int>(n),
                                       0, bits, st));
    lfu::k_segments<<<grid_for(n, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        c->skey.as<int>(), n, c->seg_lo.as<int>(), c->seg_hi.as<int>());
    const int64_t chunks = (n + lfu::kSlotChunk - 1) / lfu::kSlotChunk;
    lfu::k_slot_chunks<T><<<grid_for(chunks * 32, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        n, N, c->skey.as<int>(), c->spos.as<int>(), c->has_w ? c->c_w.as<double>() : nullptr,
        c->c_bag.as<int32_t>(), ge, c->seg_lo.as<int>(), c->seg_hi.as<int>(), c->part.as<T>(),
        c->sg.as<T>(), c->now().store.as<T>(), fused ? 1 : 0, static_cast<T>(lr));
    lfu::k_slot_fold<T><<<grid_for(c->capacity * N * 32, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        c->capacity, N, c->seg_lo.as<int>(), c->seg_hi.as<int>(), c->part.as<T>(), c->sg.as<T>(),
        c->now().store.as<T>(), fused ? 1 : 0, static_cast<T>(lr));
    CK(cudaGetLastError());
  }
  c->grads_valid = !fused;
}

}  // namespace
}  // namespace ttgpu

// =========================================================================
//                         C ABI: LFU cache
// =========================================================================
extern "C" {

int ttgpu_cache_create(int64_t capacity, int64_t emb_dim, int64_t refresh_period,
                       int64_t key_space, int dtype, int device, void* stream, ttgpu_cache** out) {
  return guarded([&] {
    require_arg(out != nullptr, "null output handle");
    require_arg(capacity >= 1, cat("cache capacity must be >= 1, got ", capacity));
    require_arg(emb_dim >= 1, cat("emb_dim must be >= 1, got ", emb_dim));
    require_arg(emb_dim <= lfu::kSlotMaxN,
                cat("the GPU cache supports emb_dim <= ", lfu::kSlotMaxN, ", got ", emb_dim));
    require_arg(refresh_period >= 1, cat("refresh_period must be >= 1, got ", refresh_period));
    require_arg(key_space >= 1, cat("cache key space must be >= 1, got ", key_space));
    require_arg(capacity < (int64_t{1} << 30), "cache capacity too large");
    require_arg(dtype == TTGPU_F32 || dtype == TTGPU_F64, "dtype must be TTGPU_F32 or TTGPU_F64");
    CK(cudaSetDevice(device));
    auto c = std::make_unique<ttgpu_cache>();
    c->capacity = capacity;
    c->emb_dim = emb_dim;
    c->refresh_period = refresh_period;
    c->key_space = key_space;
    c->dtype = dtype;
    c->esz = dtype == TTGPU_F64 ? 8 : 4;
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device));
    c->counts.ensure(8 * key_space);
    CK(cudaMemsetAsync(c->counts.p, 0, 8 * key_space, c->stream));
    c->counters.ensure(16);
    CK(cudaMemsetAsync(c->counters.p, 0, 16, c->stream));
    c->errs.ensure(16);
    unsigned long long init[2] = {ULLONG_MAX, 0};
    CK(cudaMemcpyAsync(c->errs.p, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    for (auto& r : c->res) {  // empty residency: a 64-entry all-empty hash
      r.hkeys.ensure(8 * 64);
      r.hvals.ensure(4 * 64);
      CK(cudaMemsetAsync(r.hkeys.p, 0xff, 8 * 64, c->stream));
      r.hshift = 64 - 6;
      r.hmask = 63;
      r.slot_rows.ensure(8 * capacity);
      r.store.ensure(c->esz * capacity * emb_dim);
      CK(cudaMemsetAsync(r.slot_rows.p, 0xff, 8 * capacity, c->stream));
      CK(cudaMemsetAsync(r.store.p, 0, c->esz * capacity * emb_dim, c->stream));
    }
    CK(cudaStreamSynchronize(c->stream));
    *out = c.release();
  });
}

int ttgpu_cache_set_fast(ttgpu_cache* c, int enable) {
  return guarded([&] { c->fast_enabled = enable != 0; });
}

int ttgpu_cache_last_counts(ttgpu_cache* c, int64_t* n_cached, int64_t* n_tt, int64_t* bags,
                            int* has_weights, int* pooling) {
  return guarded([&] {
    require_arg(c->part_valid, "no partition recorded");
    int64_t nc = c->n_cached;
    if (c->fast_part) {
      ttgpu::cache_order_after_last(c);
      int v = 0;
      CK(cudaMemcpyAsync(&v, c->f_ncached.p, 4, cudaMemcpyDeviceToHost, c->stream));
      CK(cudaStreamSynchronize(c->stream));
      nc = v;
    }
    if (n_cached) *n_cached = nc;
    if (n_tt) *n_tt = c->L - nc;
    if (bags) *bags = c->B;
    if (has_weights) *has_weights = c->has_w ? 1 : 0;
    if (pooling) *pooling = c->pooling;
  });
}

int ttgpu_cache_destroy(ttgpu_cache* c) {
  return guarded([&] {
    if (!c) return;
    cudaStreamSynchronize(c->stream);
    delete c;
  });
}

int64_t ttgpu_cache_default_capacity(int64_t table_rows) {
  return std::max<int64_t>(1, static_cast<int64_t>(std::llround(1e-4 * static_cast<double>(table_rows))));
}

int ttgpu_cache_set_stream(ttgpu_cache* c, void* stream) {
  return guarded([&] { c->stream = static_cast<cudaStream_t>(stream); });
}

int ttgpu_cache_info(ttgpu_cache* c, int* active, int64_t* resident, uint64_t* accesses,
                     uint64_t* hits) {
  return guarded([&] {
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (active) *active = c->active ? 1 : 0;
    if (resident) *resident = c->now().resident;
    if (accesses) *accesses = c->accesses + h[0];  // partition path (host) + fast path (device)
    if (hits) *hits = h[1];
  });
}

int ttgpu_cache_record(ttgpu_cache* c, const int64_t* host_idx, int64_t L) {
  return guarded([&] {
    require_arg(L >= 0, "negative batch size");
    for (int64_t i = 0; i < L; ++i)
      require_arg(host_idx[i] >= 0, cat("frequency keys must be non-negative, got ", host_idx[i]));
    if (L == 0) return;
    c->t_idx.ensure(8 * L);
    CK(cudaMemcpyAsync(c->t_idx.p, host_idx, 8 * L, cudaMemcpyHostToDevice, c->stream));
    auto& R = c->now();
    ttgpu::lfu::k_partition<<<grid_for(L, kThreads, c->num_sms, 8), kThreads, 0, c->stream>>>(
        c->t_idx.as<int64_t>(), L, c->key_space, c->counts.as<unsigned long long>(),
        R.hkeys.as<unsigned long long>(), R.hvals.as<int>(), R.hshift, R.hmask, 0, 1, nullptr,
        nullptr, c->errs.as<unsigned long long>(), nullptr);
    CK(cudaGetLastError());
    ttgpu::cache_raise(c, c->stream, host_idx, "cache");
    c->part_valid = false;
  });
}

int ttgpu_cache_record_and_partition(ttgpu_cache* c, const int64_t* idx, int64_t L,
                                     const int64_t* off, int64_t B, const double* w, int pooling,
                                     int64_t* n_cached, int64_t* n_tt) {
  return guarded([&] {
    require_arg(off != nullptr && B >= 0, "bad offsets");
    for (int64_t i = 0; i < L; ++i)
      require_arg(idx[i] >= 0, cat("frequency keys must be non-negative, got ", idx[i]));
    // stage the host batch in the partition's own buffers
    c->h_idx_stage.ensure(8 * std::max<int64_t>(L, 1));
    c->h_off_stage.ensure(8 * (B + 1));
    if (L > 0) CK(cudaMemcpyAsync(c->h_idx_stage.p, idx, 8 * L, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->h_off_stage.p, off, 8 * (B + 1), cudaMemcpyHostToDevice, c->stream));
    const double* dw = nullptr;
    if (w) {
      c->h_w_stage.ensure(8 * std::max<int64_t>(L, 1));
      if (L > 0) CK(cudaMemcpyAsync(c->h_w_stage.p, w, 8 * L, cudaMemcpyHostToDevice, c->stream));
      dw = c->h_w_stage.as<double>();
    }
    ttgpu::cache_partition(c, c->stream, c->h_idx_stage.as<int64_t>(), L,
                           c->h_off_stage.as<int64_t>(), B, dw, pooling, idx, "cache");
    if (n_cached) *n_cached = c->n_cached;
    if (n_tt) *n_tt = c->n_tt;
  });
}

int ttgpu_cache_last_partition(ttgpu_cache* c, int64_t* cached_slots, int64_t* cached_rows,
                               int64_t* cached_off, double* cached_w, int64_t* tt_idx,
                               int64_t* tt_off, double* tt_w) {
  return guarded([&] {
    require_arg(c->part_valid, "no partition recorded");
    cudaStream_t st = c->stream;
    if (c->fast_part) {
      // fast path: rebuild CachePartition (lfu_cache.hpp:187-219) from the
      // per-lookup slots and the forward's device batch (still alive)
      cache_order_after_last(c);
      const int64_t L = c->L, B = c->B;
      std::vector<int> slot(static_cast<size_t>(L));
      std::vector<int64_t> idx(static_cast<size_t>(L)), off(static_cast<size_t>(B + 1));
      std::vector<double> w(c->has_w ? static_cast<size_t>(L) : 0);
      CK(cudaMemcpyAsync(slot.data(), c->f_slot.p, 4 * L, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(idx.data(), c->f_idx, 8 * L, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(off.data(), c->f_off, 8 * (B + 1), cudaMemcpyDeviceToHost, st));
      if (c->has_w) CK(cudaMemcpyAsync(w.data(), c->f_w, 8 * L, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      int64_t nc = 0, nt = 0;
      for (int64_t b = 0; b < B; ++b) {
        if (cached_off) cached_off[b] = nc;
        if (tt_off) tt_off[b] = nt;
        for (int64_t l = off[b]; l < off[b + 1]; ++l) {
          if (slot[l] >= 0) {
            if (cached_slots) cached_slots[nc] = slot[l];
            if (cached_rows) cached_rows[nc] = idx[l];
            if (cached_w && c->has_w) cached_w[nc] = w[l];
            ++nc;
          } else {
            if (tt_idx) tt_idx[nt] = idx[l];
            if (tt_w && c->has_w) tt_w[nt] = w[l];
            ++nt;
          }
        }
      }
      if (cached_off) cached_off[B] = nc;
      if (tt_off) tt_off[B] = nt;
      return;
    }
    auto cp = [&](void* dst, const DevBuf& src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src.p, bytes, cudaMemcpyDeviceToHost, st));
    };
    cp(cached_slots, c->c_idx, 8 * c->n_cached);
    cp(cached_rows, c->c_rows, 8 * c->n_cached);
    cp(cached_off, c->c_off, 8 * (c->B + 1));
    cp(tt_idx, c->t_idx, 8 * c->n_tt);
    cp(tt_off, c->t_off, 8 * (c->B + 1));
    if (c->has_w) {
      cp(cached_w, c->c_w, 8 * c->n_cached);
      cp(tt_w, c->t_w, 8 * c->n_tt);
    }
    CK(cudaStreamSynchronize(st));
  });
}

int ttgpu_cache_warmup_finalize(ttgpu_cache* c, ttgpu_table* t) {
  return guarded([&] {
    require_arg(!c->active, "cache already active");
    require_arg(t != nullptr && t->plan.emb_dim == c->emb_dim,
                cat("cache emb_dim ", c->emb_dim, " does not match table emb_dim ",
                    t ? t->plan.emb_dim : 0));
    CK(cudaStreamSynchronize(c->stream));
    ttgpu::cache_admit(c, t);
    c->active = true;
  });
}

int ttgpu_cache_refresh(ttgpu_cache* c, ttgpu_table* t, double* drift) {
  return guarded([&] {
    require_arg(c->active, "refresh before warmup_finalize");
    require_arg(t != nullptr && t->plan.emb_dim == c->emb_dim,
                cat("cache emb_dim ", c->emb_dim, " does not match table emb_dim ",
                    t ? t->plan.emb_dim : 0));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> prev = c->prev_top;
    ttgpu::cache_admit(c, t);
    const double d = ttgpu::drift_of(prev, c->prev_top, c->capacity);
    if (drift) *drift = d;
  });
}

int ttgpu_hot_set_drift(const int64_t* prev, int64_t n_prev, const int64_t* cur, int64_t n_cur,
                        int64_t k, double* out) {
  return guarded([&] {
    *out = ttgpu::drift_of(std::vector<int64_t>(prev, prev + n_prev),
                           std::vector<int64_t>(cur, cur + n_cur), k);
  });
}

int ttgpu_cache_hot_rows(ttgpu_cache* c, int64_t* out, int64_t max, int64_t* n) {
  return guarded([&] {
    const int64_t k = static_cast<int64_t>(c->prev_top.size());
    if (n) *n = k;
    if (out) std::copy(c->prev_top.begin(), c->prev_top.begin() + std::min(k, max), out);
  });
}

int ttgpu_cache_slot_rows(ttgpu_cache* c, int64_t* out) {
  return guarded([&] {
    CK(cudaMemcpyAsync(out, c->now().slot_rows.p, 8 * c->capacity, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_slot_of(ttgpu_cache* c, int64_t row, int64_t* slot) {
  return guarded([&] {
    std::vector<int64_t> rows(static_cast<size_t>(c->capacity));
    CK(cudaMemcpyAsync(rows.data(), c->now().slot_rows.p, 8 * c->capacity, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *slot = -1;
    for (int64_t s = 0; s < c->now().resident; ++s)
      if (rows[s] == row) *slot = s;
  });
}

int ttgpu_cache_get_rows(ttgpu_cache* c, void* host_out) {  // all capacity x emb_dim values
  return guarded([&] {
    CK(cudaMemcpyAsync(host_out, c->now().store.p, c->esz * c->capacity * c->emb_dim,
                       cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_set_row(ttgpu_cache* c, int64_t slot, const void* host_in) {
  return guarded([&] {
    require_arg(slot >= 0 && slot < c->capacity,
                cat("slot ", slot, " outside cache capacity ", c->capacity));
    CK(cudaMemcpyAsync(static_cast<char*>(c->now().store.p) + c->esz * slot * c->emb_dim, host_in,
                       c->esz * c->emb_dim, cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_store_device_ptr(ttgpu_cache* c, void** ptr) {
  return guarded([&] { *ptr = c->now().store.p; });
}

int ttgpu_cache_counts_device_ptr(ttgpu_cache* c, void** ptr, int64_t* n) {
  return guarded([&] {
    *ptr = c->counts.p;
    *n = c->key_space;
  });
}

int ttgpu_cache_freq_count(ttgpu_cache* c, int64_t key, uint64_t* out) {
  return guarded([&] {
    *out = 0;
    if (key < 0 || key >= c->key_space) return;
    CK(cudaMemcpyAsync(out, c->counts.as<unsigned long long>() + key, 8, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_freq_size(ttgpu_cache* c, int64_t* out) {
  return guarded([&] {
    c->sel_n.ensure(16);
    CK(cudaMemsetAsync(c->sel_n.p, 0, 8, c->stream));
    ttgpu::lfu::k_count_nonzero<<<grid_for(c->key_space, kThreads, c->num_sms, 8), kThreads, 0,
                                  c->stream>>>(c->counts.as<unsigned long long>(), c->key_space,
                                               c->sel_n.as<unsigned long long>());
    unsigned long long v = 0;
    CK(cudaMemcpyAsync(&v, c->sel_n.p, 8, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *out = static_cast<int64_t>(v);
  });
}

int ttgpu_cache_freq_decay(ttgpu_cache* c, double factor) {
  return guarded([&] {
    require_arg(factor >= 0.0 && factor <= 1.0,
                cat("decay factor must be in [0, 1], got ", factor));
    ttgpu::lfu::k_decay<<<grid_for(c->key_space, kThreads, c->num_sms, 8), kThreads, 0,
                          c->stream>>>(c->counts.as<unsigned long long>(), c->key_space, factor);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_freq_clear(ttgpu_cache* c) {
  return guarded([&] {
    CK(cudaMemsetAsync(c->counts.p, 0, 8 * c->key_space, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int ttgpu_cache_top_k(ttgpu_cache* c, ttgpu_table* t, int64_t k, int64_t* rows, uint64_t* counts,
                      int64_t* n) {
  return guarded([&] {
    (void)t;
    require_arg(k >= 0, "k must be >= 0");
    // same selection as admit: rows with a count, stable (count desc, row asc)
    cudaStream_t st = c->stream;
    const int64_t K = c->key_space;
    c->sel_rows.ensure(8 * K);
    c->sel_n.ensure(16);
    size_t tb = 0;
    thrust::counting_iterator<int64_t> it(0);
    ttgpu::lfu::HasCount pred{c->counts.as<unsigned long long>()};
    CK(cub::DeviceSelect::If(nullptr, tb, it, c->sel_rows.as<int64_t>(), c->sel_n.as<int64_t>(), K,
                             pred, st));
    ttgpu::cache_ensure_tmp(c, tb);
    CK(cub::DeviceSelect::If(c->tmp.p, tb, it, c->sel_rows.as<int64_t>(), c->sel_n.as<int64_t>(),
                             K, pred, st));
    int64_t m = 0;
    CK(cudaMemcpyAsync(&m, c->sel_n.p, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t kk = std::min(k, m);
    *n = kk;
    if (m == 0 || kk == 0) return;
    c->sel_cnt.ensure(8 * m);
    c->top_cnt.ensure(8 * m);
    c->top_rows.ensure(8 * m);
    ttgpu::lfu::k_gather_counts<<<grid_for(m, kThreads, c->num_sms, 8), kThreads, 0, st>>>(
        c->sel_rows.as<int64_t>(), m, c->counts.as<unsigned long long>(),
        c->sel_cnt.as<unsigned long long>());
    CK(cub::DeviceRadixSort::SortPairsDescending(
        nullptr, tb, c->sel_cnt.as<unsigned long long>(), c->top_cnt.as<unsigned long long>(),
        c->sel_rows.as<int64_t>(), c->top_rows.as<int64_t>(), static_cast<int>(m), 0, 64, st));
    ttgpu::cache_ensure_tmp(c, tb);
    CK(cub::DeviceRadixSort::SortPairsDescending(
        c->tmp.p, tb, c->sel_cnt.as<unsigned long long>(), c->top_cnt.as<unsigned long long>(),
        c->sel_rows.as<int64_t>(), c->top_rows.as<int64_t>(), static_cast<int>(m), 0, 64, st));
    if (rows) CK(cudaMemcpyAsync(rows, c->top_rows.p, 8 * kk, cudaMemcpyDeviceToHost, st));
    if (counts) CK(cudaMemcpyAsync(counts, c->top_cnt.p, 8 * kk, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

// ---- the cached EmbeddingLayer (model.hpp:195-284) ------------------------
int ttgpu_cache_forward_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx,
                               const int64_t* d_idx, int64_t L, const int64_t* d_off, int64_t B,
                               const double* d_w, int pooling, int save, void* d_out) {
  return guarded([&] {
    if (t->dtype == TTGPU_F64)
      ttgpu::cache_forward<double>(c, t, ctx, d_idx, L, d_off, B, d_w, pooling, save != 0,
                                   static_cast<double*>(d_out), nullptr);
    else
      ttgpu::cache_forward<float>(c, t, ctx, d_idx, L, d_off, B, d_w, pooling, save != 0,
                                  static_cast<float*>(d_out), nullptr);
  });
}

int ttgpu_cache_forward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const int64_t* idx,
                        int64_t L, const int64_t* off, int64_t B, const double* w, int pooling,
                        int save, void* out) {
  return guarded([&] {
    require_arg(ctx != nullptr, "forward needs a context");
    ttgpu::validate_host(t, idx, L, off, B);
    ctx->h_idx.ensure(8 * std::max<int64_t>(L, 1));
    ctx->h_off.ensure(8 * (B + 1));
    ctx->h_out.ensure(t->esz * std::max<int64_t>(B * t->plan.emb_dim, 1));
    if (L > 0) CK(cudaMemcpyAsync(ctx->h_idx.p, idx, 8 * L, cudaMemcpyHostToDevice, t->stream));
    CK(cudaMemcpyAsync(ctx->h_off.p, off, 8 * (B + 1), cudaMemcpyHostToDevice, t->stream));
    const double* dw = nullptr;
    if (w) {
      ctx->h_w.ensure(8 * std::max<int64_t>(L, 1));
      if (L > 0) CK(cudaMemcpyAsync(ctx->h_w.p, w, 8 * L, cudaMemcpyHostToDevice, t->stream));
      dw = ctx->h_w.as<double>();
    }
    if (t->dtype == TTGPU_F64)
      ttgpu::cache_forward<double>(c, t, ctx, ctx->h_idx.as<int64_t>(), L, ctx->h_off.as<int64_t>(),
                                   B, dw, pooling, save != 0, ctx->h_out.as<double>(), idx);
    else
      ttgpu::cache_forward<float>(c, t, ctx, ctx->h_idx.as<int64_t>(), L, ctx->h_off.as<int64_t>(),
                                  B, dw, pooling, save != 0, ctx->h_out.as<float>(), idx);
    if (B > 0)
      CK(cudaMemcpyAsync(out, ctx->h_out.p, t->esz * B * t->plan.emb_dim, cudaMemcpyDeviceToHost,
                         t->stream));
    CK(cudaStreamSynchronize(t->stream));
    ttgpu::raise_latched(t, nullptr, 0);
  });
}

// backward: chain gradients into the table's gradient buffer (dense), slot
// gradients into the cache; ttgpu_cache_step applies both (EmbeddingLayer::step)
int ttgpu_cache_backward_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const void* d_grad) {
  return guarded([&] {
    if (t->dtype == TTGPU_F64)
      ttgpu::cache_backward<double>(c, t, ctx, static_cast<const double*>(d_grad), false, 0.0);
    else
      ttgpu::cache_backward<float>(c, t, ctx, static_cast<const float*>(d_grad), false, 0.0);
  });
}

int ttgpu_cache_backward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const void* grad,
                         int64_t grad_len) {
  return guarded([&] {
    require_arg(c->part_valid, "cache backward needs the partition of a cached forward");
    require_arg(grad_len == c->B * c->emb_dim,
                cat("table '", t->name, "': bad gradient size"));
    ctx->h_grad.ensure(t->esz * std::max<int64_t>(grad_len, 1));
    if (grad_len > 0)
      CK(cudaMemcpyAsync(ctx->h_grad.p, grad, t->esz * grad_len, cudaMemcpyHostToDevice, t->stream));
    if (t->dtype == TTGPU_F64)
      ttgpu::cache_backward<double>(c, t, ctx, ctx->h_grad.as<double>(), false, 0.0);
    else
      ttgpu::cache_backward<float>(c, t, ctx, ctx->h_grad.as<float>(), false, 0.0);
    CK(cudaStreamSynchronize(t->stream));
  });
}

// EmbeddingLayer::step (model.hpp:265-284): sgd_step on the chain gradients,
// cached_sgd_update on the touched slots
int ttgpu_cache_step(ttgpu_cache* c, ttgpu_table* t, double lr) {
  return guarded([&] {
    require_arg(c->grads_valid, "cache step needs a cache backward");
    const int s = ttgpu_apply_grad(t, lr);
    if (s) fail(s, g_last_error);
    const int64_t n = c->capacity * c->emb_dim;
    const int g = grid_for(n, kThreads, c->num_sms, 8);
    if (t->dtype == TTGPU_F64)
      ttgpu::lfu::k_slot_sgd<double><<<g, kThreads, 0, t->stream>>>(
          c->capacity, static_cast<int>(c->emb_dim), c->seg_lo.as<int>(), c->sg.as<double>(),
          c->now().store.as<double>(), static_cast<double>(lr));
    else
      ttgpu::lfu::k_slot_sgd<float><<<g, kThreads, 0, t->stream>>>(
          c->capacity, static_cast<int>(c->emb_dim), c->seg_lo.as<int>(), c->sg.as<float>(),
          c->now().store.as<float>(), static_cast<float>(lr));
    CK(cudaGetLastError());
    c->grads_valid = false;
  });
}

// fused backward + step: chain gradients reduced per core slice with the SGD in
// the epilogue, slot gradients applied in their reduction epilogue
int ttgpu_cache_backward_step_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx,
                                     const void* d_grad, double lr) {
  return guarded([&] {
    if (t->dtype == TTGPU_F64)
      ttgpu::cache_backward<double>(c, t, ctx, static_cast<const double*>(d_grad), true, lr);
    else
      ttgpu::cache_backward<float>(c, t, ctx, static_cast<const float*>(d_grad), true, lr);
  });
}

// slot gradients of the last cache backward (test / allreduce access):
// capacity x emb_dim values, touched[s] = 1 for slots with a gradient
int ttgpu_cache_slot_grads(ttgpu_cache* c, void* host_grads, uint8_t* touched) {
  return guarded([&] {
    require_arg(c->grads_valid, "no slot gradients (run ttgpu_cache_backward)");
    ttgpu::cache_order_after_last(c);
    std::vector<int> lo(static_cast<size_t>(c->capacity));
    CK(cudaMemcpyAsync(lo.data(), c->seg_lo.p, 4 * c->capacity, cudaMemcpyDeviceToHost, c->stream));
    if (host_grads)
      CK(cudaMemcpyAsync(host_grads, c->sg.p, c->esz * c->capacity * c->emb_dim,
                         cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (host_grads) {  // untouched slots read as zero
      for (int64_t s = 0; s < c->capacity; ++s)
        if (lo[s] < 0)
          std::memset(static_cast<char*>(host_grads) + c->esz * s * c->emb_dim, 0,
                      c->esz * c->emb_dim);
    }
    if (touched)
      for (int64_t s = 0; s < c->capacity; ++s) touched[s] = lo[s] >= 0 ? 1 : 0;
  });
}

// cached_sgd_update(SlotGradients, lr) with caller rows (lfu_cache.hpp:246-257)
int ttgpu_cache_sgd_update(ttgpu_cache* c, const int64_t* slots, int64_t n, const void* rows,
                           double lr) {
  return guarded([&] {
    ttgpu::cache_order_after_last(c);
    std::vector<int64_t> sr(static_cast<size_t>(c->capacity));
    CK(cudaMemcpyAsync(sr.data(), c->now().slot_rows.p, 8 * c->capacity, cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int64_t i = 0; i < n; ++i)
      require_arg(slots[i] >= 0 && slots[i] < c->capacity && sr[slots[i]] >= 0,
                  cat("cached_sgd_update on empty slot ", slots[i]));
    if (n == 0) return;
    c->skey_in.ensure(8 * n);
    c->part.ensure(c->esz * n * c->emb_dim);
    CK(cudaMemcpyAsync(c->skey_in.p, slots, 8 * n, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->part.p, rows, c->esz * n * c->emb_dim, cudaMemcpyHostToDevice, c->stream));
    const int g = grid_for(n * c->emb_dim, kThreads, c->num_sms, 8);
    if (c->dtype == TTGPU_F64)
      ttgpu::lfu::k_rows_sgd<double><<<g, kThreads, 0, c->stream>>>(
          c->skey_in.as<int64_t>(), n, static_cast<int>(c->emb_dim), c->part.as<double>(),
          c->now().store.as<double>(), static_cast<double>(lr));
    else
      ttgpu::lfu::k_rows_sgd<float><<<g, kThreads, 0, c->stream>>>(
          c->skey_in.as<int64_t>(), n, static_cast<int>(c->emb_dim), c->part.as<float>(),
          c->now().store.as<float>(), static_cast<float>(lr));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
