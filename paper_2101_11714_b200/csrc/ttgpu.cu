// Host side of the B200 TT-EmbeddingBag: the device-resident table
// (TtTable<T> equivalent), forward contexts, the launch pipeline and the C ABI
// declared in include/ttgpu.h.  See tt_kernels.cuh for the algorithm.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <memory>
#include <mutex>
#include <random>
#include <sstream>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/ttgpu.h"
#include "shape_plan.hpp"
#include "tt_kernels.cuh"
#include "head_tc.cuh"
#include "fast3.cuh"
#include "wide3.cuh"

namespace ttgpu {
namespace {

thread_local std::string g_last_error;

// TTGPU_TRACE=1: host-side stage timer for the host-pointer entry points
// (synchronises the stream at every stage; diagnostics only).
struct HostTrace {
  bool on;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit HostTrace(cudaStream_t s) : on(std::getenv("TTGPU_TRACE") != nullptr), st(s) {
    t0 = std::chrono::steady_clock::now();
  }
  void operator()(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto t = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[ttgpu trace] %-24s %9.1f us\n", what,
                 std::chrono::duration<double, std::micro>(t - t0).count());
    t0 = t;
  }
};
std::atomic<uint64_t> g_rows{0};
std::atomic<uint64_t> g_ws_cur{0};
std::atomic<uint64_t> g_ws_peak{0};

template <class... A>
std::string cat(const A&... a) {
  std::ostringstream os;
  (os << ... << a);
  return os.str();
}

struct Error : std::exception {
  int code;
  std::string msg;
  Error(int c, std::string m) : code(c), msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
[[noreturn]] void fail(int code, const std::string& m) { throw Error(code, m); }
void require_arg(bool ok, const std::string& m) {
  if (!ok) fail(TTGPU_ERR_INVALID_ARGUMENT, m);
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(TTGPU_ERR_RUNTIME, cat("CUDA error in ", what, ": ", cudaGetErrorString(e)));
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TTGPU_OK;
  } catch (const Error& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::out_of_range& e) {
    g_last_error = e.what();
    return TTGPU_ERR_OUT_OF_RANGE;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return TTGPU_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TTGPU_ERR_RUNTIME;
  }
}

void ws_add(uint64_t b) {
  const uint64_t cur = g_ws_cur.fetch_add(b) + b;
  uint64_t peak = g_ws_peak.load();
  while (cur > peak && !g_ws_peak.compare_exchange_weak(peak, cur)) {
  }
}
void ws_sub(uint64_t b) { g_ws_cur.fetch_sub(b); }

// Growable device buffer; only reallocates when a call needs more.
// bumped by every workspace (re)allocation: a cached graph of a host-API call
// is replayed only while the buffers it captured are still the current ones
std::atomic<uint64_t> g_alloc_epoch{0};
inline void bump_alloc_epoch() { g_alloc_epoch.fetch_add(1); }

// One instantiated graph of the kernels behind a host-API call (ttgpu_forward /
// ttgpu_backward[_sgd]): the inputs sit in the context's staging buffers, so
// the kernel sequence for a given shape/flags key is replayable.  The first
// call with a key runs eagerly (allocating), the second captures, later ones
// replay -- about 9 launches collapse into one.
struct CachedGraph {
  cudaGraphExec_t exec = nullptr;
  uint64_t key = 0, epoch = 0, seen_key = ~0ull;
  int aux = 0;  // host state the eager path would have set (forward: fast path taken)
  ~CachedGraph() {
    if (exec) cudaGraphExecDestroy(exec);
  }
};

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void ensure(size_t bytes) {
    if (bytes <= cap) return;
    if (p) {
      cudaFree(p);
      ws_sub(cap);
    }
    bytes = std::max<size_t>(bytes, 256);
    CK(cudaMalloc(&p, bytes));
    cap = bytes;
    ws_add(cap);
    bump_alloc_epoch();
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DevBuf() {
    if (p) {
      cudaFree(p);
      ws_sub(cap);
    }
  }
};

constexpr int kTailChunk = 32;   // lookups per CTA in the lookup-level reductions
constexpr int kHeadChunk = 32;   // pairs per CTA in the head kernels
constexpr int kThreads = 256;

int bits_for(uint64_t n) {  // bits needed to represent values < n
  int b = 0;
  while (b < 64 && (1ull << b) < n) ++b;
  return std::max(b, 1);
}

}  // namespace
}  // namespace ttgpu

using namespace ttgpu;

__global__ void k_noop() {}

struct ttgpu_ctx;
struct ttgpu_peers;
void ttgpu_destroy_peers(struct ttgpu_peers*);
struct ttgpu_table {
  void destroy_peers();
  ShapePlan plan;
  std::string name;
  int dtype = TTGPU_F32;
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  size_t esz = 4;
  DevPlan dp{};
  int64_t total = 0;         // total core elements (with alignment padding)
  DevBuf cores, grads, pair_tab, errs, lk_rows, lk_out;
  // destroyed forward contexts keep their device workspace here for the next
  // ttgpu_ctx_create (the reference returns a fresh ForwardContext from every
  // forward_bags call; without recycling each would re-cudaMalloc its buffers)
  std::vector<ttgpu_ctx*> ctx_pool;
  unsigned long long* h_errs = nullptr;  // pinned host mirror of errs
  DevBuf peer_flag_buf;                   // fused peer reduce: flag block (peer_host.inl)
  struct ttgpu_peers* peers = nullptr;
  uint64_t generation = 0;
  bool exact = true;  // forward bit-identical to the reference (no FMA contraction)
  bool force_generic = false;  // route 3-core tables through the generic pipeline (testing)
  bool tensor_head = true;     // head backward on tcgen05 (3xTF32) where the shape allows it
  int pdl = 0;                 // fast-path launches: 0 plain, 1 programmatic dependent launch
  bool grid_sort = true;       // fast path: one-kernel cooperative sort (gsort.cuh) where the batch fits
  bool chunked = false;        // fast path: chunked forward / S+dG1+D0 backward (fastc.cuh; slower, off)
  bool wide3 = true;           // d == 3 wide rows: warp-per-chunk tail kernels (wide3.cuh)
  bool fuse_sb = true;         // fast path: f3_srows + f3_bwd2 in one launch (TTGPU_FUSE_SB=0: two)
  bool fuse_comb = false;      // fast path: f3_bwd1 + f3_combine in one cooperative launch
  bool plan_bwd1 = true;       // fast path: f3_bwd1's ranges planned by f3_srows_bwd2 (TTGPU_PLAN_BWD1=0: in bwd1)
  bool merge1 = true;          // planned f3_bwd1: runs of one-slot tiles of the same (i1, i0) as one unit (TTGPU_MERGE1=0: off)
  int b1tile = 3, b1cont = 1;  // merge-unit range weights (TTGPU_B1COST=tile,cont; swept: 3,1 best at cfg2)
                               // (TTGPU_FUSE_COMB=1; measured slower: the combine tasks get half the warps)
  // optional phase timing (CUDA events between pipeline phases)
  // Marks recorded while the stream is being captured become event-record nodes of
  // the graph (cudaEventRecordExternal) and stay owned by it: every graph launch
  // re-records them, so profile_read can be called after each launch.
  bool prof = false;
  bool graph_marks = false;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;
  std::vector<cudaEvent_t> ev_pool;
  void mark(const char* name) {
    if (!prof) return;
    cudaEvent_t e;
    if (ev_pool.empty()) {
      cudaEventCreate(&e);
    } else {
      e = ev_pool.back();
      ev_pool.pop_back();
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    if (cs == cudaStreamCaptureStatusActive) {
      // an event node at the graph's root fires as soon as the graph is
      // launched, before earlier work on the stream has drained: anchor it
      // behind an empty kernel
      if (marks.empty()) k_noop<<<1, 32, 0, stream>>>();
      cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal);
    }
    else
      cudaEventRecord(e, stream);
    marks.emplace_back(name, e);
  }
  void recycle_marks() {
    for (auto& m : marks) ev_pool.push_back(m.second);
    marks.clear();
    graph_marks = false;
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  ~ttgpu_table() {
    if (h_errs) cudaFreeHost(h_errs);
    destroy_peers();
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto& m : marks) cudaEventDestroy(m.second);
    for (auto e : ev_pool) cudaEventDestroy(e);
  }
  // latched device errors: [0]=first bad lookup, [1]=its value, [2]=struct flags
  unsigned long long* d_bad() { return errs.as<unsigned long long>(); }
  int* d_struct() { return reinterpret_cast<int*>(errs.as<unsigned long long>() + 2); }
};

namespace ttgpu {
struct F3Bufs;
void f3_free(F3Bufs*);
}  // namespace ttgpu

struct ttgpu_ctx {
  ~ttgpu_ctx() {
    if (f3) ttgpu::f3_free(f3);
  }
  ttgpu::F3Bufs* f3 = nullptr;  // fast-path state (3-core tables)
  bool fast = false;
  ttgpu_table* table = nullptr;
  uint64_t snapshot = 0;
  bool valid = false;
  int64_t L = 0, B = 0;
  int pooling = 0;
  bool save = false;
  bool has_w = false;
  bool exact = true;  // rounding mode of the forward that filled this context
  // host-API staging
  DevBuf h_idx, h_off, h_w, h_out, h_grad;
  // forward state
  DevBuf pair_key, iota, s_key, s_lk, tail_dig, lk_bag, lk_alpha, lk_pid, flags, pair_scan,
      pair_key_u, pair_start, counts, H, saved, cub_tmp;
  const double* w_dev = nullptr;
  // backward state
  DevBuf s_dkey, s_dlk, dscan, dseg, pair_i1, scan1, seg1, S, D0, partS, partK, part1;
  // d == 3 wide-row path: per-lookup y rows, dG2 contributions, i2 positions
  DevBuf ybuf, tcontrib, pos2;
  DevBuf w3_slab_base, w3_slab_part, w3_cnt;  // wide3.cuh segsum slabs
  CachedGraph gfwd, gbwd;  // host-API kernel sequences
  size_t cub_bytes = 0;
};

namespace ttgpu {
namespace {

DevPlan make_devplan(const ShapePlan& p, std::vector<int64_t>& coff, int64_t& total) {
  DevPlan d{};
  d.d = p.tt_dim;
  d.N = static_cast<int>(p.emb_dim);
  d.num_rows = p.num_rows;
  int64_t suf = 1;
  for (int k = p.tt_dim - 1; k >= 0; --k) {
    d.suffix[k] = suf;
    suf *= p.row_factors[k];
  }
  int pre = 1;
  int64_t off = 0;
  coff.resize(p.tt_dim);
  d.maxw = 0;
  for (int k = 0; k < p.tt_dim; ++k) {
    d.m[k] = static_cast<int>(p.row_factors[k]);
    d.n[k] = static_cast<int>(p.col_factors[k]);
    d.r[k] = static_cast<int>(p.ranks[k]);
    pre *= d.n[k];
    d.prefix[k] = pre;
    d.slice[k] = static_cast<int>(p.slice_size(k));
    d.coff[k] = off;
    coff[k] = off;
    off += (p.core_size(k) + 63) / 64 * 64;  // 256 B alignment per core (f32)
    d.maxw = std::max<int>(d.maxw, pre * static_cast<int>(p.ranks[k + 1]));
  }
  d.r[p.tt_dim] = 1;
  d.W1 = d.prefix[1] * d.r[2];
  d.C1 = d.n[1] * d.r[2];
  total = off;
  return d;
}

void check_supported(const ShapePlan& p) {
  for (int k = 0; k < p.tt_dim; ++k)
    require_arg(p.row_factors[k] < (1ll << 31) && p.ranks[k + 1] < (1 << 16) &&
                    p.col_factors[k] < (1 << 16),
                "plan dimension too large for the GPU kernels");
  require_arg(static_cast<uint64_t>(p.row_factors[0]) * static_cast<uint64_t>(p.row_factors[1]) <
                  (1ull << 31),
              "m_0 * m_1 must be < 2^31 for the GPU pair table");
  int64_t pre = 1, maxw = 0;
  for (int k = 0; k < p.tt_dim; ++k) {
    pre *= p.col_factors[k];
    maxw = std::max<int64_t>(maxw, pre * p.ranks[k + 1]);
  }
  require_arg(maxw <= (1 << 16), "chain width too large for the GPU kernels");
}

int grid_for(int64_t work, int per_block, int num_sms, int waves = 8) {
  const int64_t g = (work + per_block - 1) / per_block;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(num_sms) * waves)));
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  // dynamic + static shared memory above 48 KB needs the opt-in (static is <= 8 KB here)
  if (bytes > 40 * 1024)
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            static_cast<int>(bytes)));
}

int warps_fitting(size_t per_warp, size_t fixed, size_t limit, int want) {
  int w = want;
  while (w > 1 && fixed + per_warp * w > limit) --w;
  if (fixed + per_warp * w > 227 * 1024) fail(TTGPU_ERR_INVALID_ARGUMENT, "plan too large for shared memory");
  return w;
}

template <typename T>
T* core_ptr(ttgpu_table* t, int k) {
  return t->cores.as<T>() + t->dp.coff[k];
}

}  // namespace
}  // namespace ttgpu

#include "fast3_host.inl"

namespace ttgpu {
namespace {

// The warp-per-chunk wide-row tail kernels (wide3.cuh) serve fp32 3-core
// tables of cfg3's shape class.
bool wide3_ok(const ttgpu_table* t) {
  const DevPlan& P = t->dp;
  return t->dtype == TTGPU_F32 && t->wide3 && P.d == 3 && P.prefix[1] == w3::P1 &&
         P.r[2] == w3::R2 && P.n[2] == w3::N2 && P.r[3] == 1 && P.m[2] <= 1024 * 64;
}

// ------------------------------------------------------------- forward ---
template <typename T>
void forward_impl(ttgpu_table* t, ttgpu_ctx* c, const int64_t* idx, int64_t L, const int64_t* off,
                  int64_t B, const double* w, int pooling, bool save, T* out, bool exact) {
  const DevPlan& P = t->dp;
  cudaStream_t st = t->stream;
  const int d = P.d;
  c->table = t;
  c->snapshot = t->generation;
  c->L = L;
  c->B = B;
  c->pooling = pooling;
  c->save = save && d >= 4;
  c->exact = exact;
  c->has_w = w != nullptr;
  c->w_dev = w;
  c->valid = true;
  g_rows.fetch_add(static_cast<uint64_t>(L));
  if (B == 0) return;
  if (L == 0) {
    CK(cudaMemsetAsync(out, 0, sizeof(T) * B * P.N, st));
    // still validate the offsets structure
    c->lk_bag.ensure(4);
    c->lk_alpha.ensure(sizeof(T));
    k_bags<T><<<grid_for(B, kThreads, t->num_sms), kThreads, 0, st>>>(
        off, B, 0, w, pooling, c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), t->d_struct());
    CK(cudaGetLastError());
    return;
  }
  c->fast = false;
  if constexpr (std::is_same_v<T, float>) {
    const int kind = f3_kind(t);
    if (kind >= 0 && !t->force_generic && f3_feasible(t, L)) {
      if (!c->f3) c->f3 = new F3Bufs;
      c->lk_bag.ensure(4 * L);
      c->lk_alpha.ensure(sizeof(T) * L);
      f3_forward(kind, t, *c->f3, idx, L, off, B, w, pooling, out, exact, c->lk_bag.as<int32_t>(),
                 c->lk_alpha.as<float>());
      c->fast = true;
      return;
    }
  }
  const int64_t m01 = static_cast<int64_t>(P.m[0]) * P.m[1];
  const int64_t ucap = std::min<int64_t>(L, m01);
  c->pair_key.ensure(4 * L);
  c->iota.ensure(4 * L);
  c->s_key.ensure(4 * L);
  c->s_lk.ensure(4 * L);
  c->tail_dig.ensure(4 * L * std::max(1, d - 2));
  c->lk_bag.ensure(4 * L);
  c->lk_alpha.ensure(sizeof(T) * L);
  c->lk_pid.ensure(4 * L);
  c->flags.ensure(8 * L);
  c->pair_scan.ensure(8 * L);
  c->pair_key_u.ensure(4 * ucap);
  c->pair_start.ensure(4 * (ucap + 1));
  c->counts.ensure(64);
  c->H.ensure(sizeof(T) * ucap * P.W1);
  if (c->save) c->saved.ensure(sizeof(T) * (d - 3) * L * P.maxw);
  // CUB scratch (sized for the largest sort/scan we run on L items)
  {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, c->pair_key.as<uint32_t>(), c->s_key.as<uint32_t>(),
                                    c->iota.as<uint32_t>(), c->s_lk.as<uint32_t>(), L, 0, 32, st);
    cub::DeviceScan::InclusiveSum(nullptr, b, c->flags.as<unsigned long long>(),
                                  c->pair_scan.as<unsigned long long>(), L, st);
    c->cub_bytes = std::max(a, b);
    c->cub_tmp.ensure(c->cub_bytes);
  }
  const int gL = grid_for(L, kThreads, t->num_sms);
  t->mark("fwd_begin");
  k_decode<<<gL, kThreads, 0, st>>>(P, idx, L, c->pair_key.as<uint32_t>(), c->iota.as<uint32_t>(),
                                    c->tail_dig.as<uint32_t>(), t->d_bad());
  k_bags<T><<<grid_for(B, kThreads, t->num_sms), kThreads, 0, st>>>(
      off, B, L, w, pooling, c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), t->d_struct());
  t->mark("decode");
  size_t tb = c->cub_bytes;
  CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tb, c->pair_key.as<uint32_t>(),
                                     c->s_key.as<uint32_t>(), c->iota.as<uint32_t>(),
                                     c->s_lk.as<uint32_t>(), L, 0, bits_for(m01), st));
  t->mark("sort_pairs");
  k_run_flags<<<gL, kThreads, 0, st>>>(c->s_key.as<uint32_t>(), nullptr, L, kTailChunk,
                                       c->flags.as<unsigned long long>());
  tb = c->cub_bytes;
  CK(cub::DeviceScan::InclusiveSum(c->cub_tmp.p, tb, c->flags.as<unsigned long long>(),
                                   c->pair_scan.as<unsigned long long>(), L, st));
  k_pairs_compact<<<gL, kThreads, 0, st>>>(
      c->s_key.as<uint32_t>(), c->s_lk.as<uint32_t>(), c->pair_scan.as<unsigned long long>(), L,
      c->pair_key_u.as<uint32_t>(), c->pair_start.as<int32_t>(), c->lk_pid.as<int32_t>(),
      c->counts.as<int>());
  t->mark("pairs_compact");
  // head GEMM per unique pair
  {
    const size_t smem = sizeof(T) * (P.slice[1] + static_cast<size_t>(kHeadChunk) * P.slice[0]);
    auto kern = exact ? k_head_fwd<T, true> : k_head_fwd<T, false>;
    set_smem(kern, smem);
    const int g = grid_for(ucap, kHeadChunk, t->num_sms, 4);
    kern<<<g, kThreads, smem, st>>>(P, t->cores.as<T>(), c->pair_key_u.as<uint32_t>(),
                                    c->counts.as<int>(), kHeadChunk, c->H.as<T>());
  }
  t->mark("head_fwd");
  // d == 3 with wide rows: y per lookup walked in pair order (H staged once per
  // pair run), then pooling in lookup order
  if (d == 3 && sizeof(T) * (P.W1 + P.prefix[1] + 4 + static_cast<size_t>(kTailChunk) * P.slice[2]) <=
                    96 * 1024 &&
      P.W1 >= 32) {
    c->ybuf.ensure(sizeof(T) * L * P.N);
    if (wide3_ok(t)) {  // warp-per-chunk tail (wide3.cuh)
      const int64_t nch = (L + kTailChunk - 1) / kTailChunk;
      const int g = static_cast<int>(std::min<int64_t>((nch + w3::kWarps / 2 - 1) / (w3::kWarps / 2),
                                                       static_cast<int64_t>(t->num_sms) * 3));
      auto kern = exact ? w3::k_w3_fwd<true> : w3::k_w3_fwd<false>;
      set_smem(kern, w3::kFwdSmem);
      kern<<<g, w3::kWarps * 32, w3::kFwdSmem, st>>>(
          reinterpret_cast<const float*>(t->cores.as<T>() + P.coff[2]),
          reinterpret_cast<const float*>(c->H.as<T>()), c->lk_pid.as<int32_t>(),
          c->tail_dig.as<uint32_t>(), c->s_lk.as<uint32_t>(), L, reinterpret_cast<float*>(c->ybuf.as<T>()));
      auto pk = exact ? k_pool_rows<T, true> : k_pool_rows<T, false>;
      pk<<<grid_for(B * P.N, kThreads, t->num_sms), kThreads, 0, st>>>(
          c->ybuf.as<T>(), off, B, L, P.N, w, pooling, out);
      t->mark("tail_pool");
      CK(cudaGetLastError());
      return;
    }
    const size_t smem =
        sizeof(T) * (P.W1 + P.prefix[1] + 4 + static_cast<size_t>(kTailChunk) * P.slice[2]);
    const int cw = std::is_same_v<T, float> ? (P.n[2] % 4 == 0 ? 4 : P.n[2] % 2 == 0 ? 2 : 1) : 1;
    auto kern = cw == 4 ? (exact ? k_pairwalk3<T, 0, true, 4> : k_pairwalk3<T, 0, false, 4>)
              : cw == 2 ? (exact ? k_pairwalk3<T, 0, true, 2> : k_pairwalk3<T, 0, false, 2>)
                        : (exact ? k_pairwalk3<T, 0, true> : k_pairwalk3<T, 0, false>);
    set_smem(kern, smem);
    kern<<<grid_for((L + kTailChunk - 1) / kTailChunk, 1, t->num_sms, 8), 256, smem, st>>>(
        P, t->cores.as<T>(), c->H.as<T>(), c->lk_pid.as<int32_t>(), c->tail_dig.as<uint32_t>(),
        nullptr, nullptr, nullptr, c->s_lk.as<uint32_t>(), nullptr, L, kTailChunk, c->ybuf.as<T>());
    auto pk = exact ? k_pool_rows<T, true> : k_pool_rows<T, false>;
    pk<<<grid_for(B * P.N, kThreads, t->num_sms), kThreads, 0, st>>>(
        c->ybuf.as<T>(), off, B, L, P.N, w, pooling, out);
    t->mark("tail_pool");
    CK(cudaGetLastError());
    return;
  }
  // tail chain + pooling per bag
  {
    const size_t per_warp = sizeof(T) * (2 * P.maxw + P.N);
    const int warps = warps_fitting(per_warp, 0, 96 * 1024, 8);
    const size_t smem = per_warp * warps;
    auto kern = exact ? k_tail_pool<T, true> : k_tail_pool<T, false>;
    set_smem(kern, smem);
    kern<<<grid_for(B, warps, t->num_sms), warps * 32, smem, st>>>(
        P, t->cores.as<T>(), c->H.as<T>(), c->lk_pid.as<int32_t>(), c->tail_dig.as<uint32_t>(),
        off, B, L, w, pooling, out, c->save ? c->saved.as<T>() : nullptr);
  }
  t->mark("tail_pool");
  CK(cudaGetLastError());
}

// ------------------------------------------------------------ backward ---
// mode 0: dense gradient into t->grads; mode 1: fused SGD (lr) on touched slices.
template <typename T>
void backward_impl(ttgpu_table* t, ttgpu_ctx* c, const T* grad, int mode, double lr) {
  const DevPlan& P = t->dp;
  cudaStream_t st = t->stream;
  const int d = P.d;
  const int64_t L = c->L;
  T* cores = t->cores.as<T>();
  T* grads = t->grads.as<T>();
  if constexpr (std::is_same_v<T, float>) {
    if (c->fast && L > 0 && c->B > 0) {
      f3_backward(t, *c->f3, grad, mode, static_cast<float>(lr), c->lk_bag.as<int32_t>(),
                  c->lk_alpha.as<float>(), L);
      return;
    }
  }
  if (mode == 0) CK(cudaMemsetAsync(grads, 0, sizeof(T) * t->total, st));
  // fused mode, d >= 4: the tail cores k >= 2 go through the dense gradient
  // buffer (k_combine<T,0> skips untouched slices, k_sgd applies every slice),
  // so those slices must start at zero -- not at an earlier backward's values
  if (mode == 1 && d >= 4)
    CK(cudaMemsetAsync(grads + P.coff[2], 0, sizeof(T) * (t->total - P.coff[2]), st));
  if (L == 0 || c->B == 0) return;
  const int64_t m01 = static_cast<int64_t>(P.m[0]) * P.m[1];
  const int64_t ucap = std::min<int64_t>(L, m01);
  const int gL = grid_for(L, kThreads, t->num_sms);
  const T tlr = static_cast<T>(lr);
  // ---- tail-digit orderings (k >= 2)
  const int ntail = std::max(0, d - 2);
  if (ntail) {
    c->s_dkey.ensure(4 * L * ntail);
    c->s_dlk.ensure(4 * L * ntail);
    c->dscan.ensure(8 * L * ntail);
    int64_t segsz = 0;
    for (int k = 2; k < d; ++k) segsz += P.m[k] + 1;
    c->dseg.ensure(4 * segsz);
  }
  // ---- pair ordering by i1
  c->pair_i1.ensure(4 * L);
  c->scan1.ensure(8 * L);
  c->seg1.ensure(4 * (P.m[1] + 1));
  c->S.ensure(sizeof(T) * ucap * P.W1);
  c->D0.ensure(sizeof(T) * ucap * P.slice[0]);
  const int64_t nchunksL = (L + kTailChunk - 1) / kTailChunk;
  c->partS.ensure(sizeof(T) * (nchunksL + ucap + 1) * P.W1);
  int64_t partk = 0;
  for (int k = 2; k < d; ++k)
    partk = std::max<int64_t>(partk, (nchunksL + std::min<int64_t>(L, P.m[k]) + 1) * P.slice[k]);
  c->partK.ensure(sizeof(T) * std::max<int64_t>(partk, 1));
  c->part1.ensure(sizeof(T) * ((ucap + kHeadChunk - 1) / kHeadChunk + std::min<int64_t>(ucap, P.m[1]) + 1) *
                  P.slice[1]);

  t->mark("bwd_begin");
  int64_t segoff = 0;
  for (int k = 2; k < d; ++k) {
    const int j = k - 2;
    uint32_t* dk = c->tail_dig.as<uint32_t>() + j * L;
    uint32_t* sk = c->s_dkey.as<uint32_t>() + j * L;
    uint32_t* sl = c->s_dlk.as<uint32_t>() + j * L;
    unsigned long long* sc = c->dscan.as<unsigned long long>() + j * L;
    int32_t* seg = c->dseg.as<int32_t>() + segoff;
    size_t tb = c->cub_bytes;
    CK(cub::DeviceRadixSort::SortPairs(c->cub_tmp.p, tb, dk, sk, c->iota.as<uint32_t>(), sl, L, 0,
                                       bits_for(P.m[k]), st));
    k_run_flags<<<gL, kThreads, 0, st>>>(sk, nullptr, L, kTailChunk, c->flags.as<unsigned long long>());
    tb = c->cub_bytes;
    CK(cub::DeviceScan::InclusiveSum(c->cub_tmp.p, tb, c->flags.as<unsigned long long>(), sc, L, st));
    k_key_bounds<<<gL, kThreads, 0, st>>>(sk, nullptr, L, P.m[k], seg);
    segoff += P.m[k] + 1;
  }
  k_pair_scatter<<<gL, kThreads, 0, st>>>(c->pair_key_u.as<uint32_t>(), c->counts.as<int>(), ucap,
                                          t->pair_tab.as<int32_t>());
  k_pair_i1<<<gL, kThreads, 0, st>>>(c->pair_key_u.as<uint32_t>(), c->counts.as<int>(), L, P.m[0],
                                     c->pair_i1.as<uint32_t>());
  k_run_flags<<<gL, kThreads, 0, st>>>(c->pair_i1.as<uint32_t>(), c->counts.as<int>(), L, kHeadChunk,
                                       c->flags.as<unsigned long long>());
  {
    size_t tb = c->cub_bytes;
    CK(cub::DeviceScan::InclusiveSum(c->cub_tmp.p, tb, c->flags.as<unsigned long long>(),
                                     c->scan1.as<unsigned long long>(), L, st));
  }
  k_key_bounds<<<gL, kThreads, 0, st>>>(c->pair_i1.as<uint32_t>(), c->counts.as<int>(), L, P.m[1],
                                        c->seg1.as<int32_t>());

  t->mark("bwd_prep");
  // ---- S(pair) = sum of D1 over the pair's lookups
  const bool staged3 = d == 3 && P.W1 <= kRun3MaxEPT * 256 && P.slice[2] <= kRun3MaxEPT * 256 &&
                       sizeof(T) * kTailChunk * (P.N + P.slice[2]) <= 96 * 1024 &&
                       sizeof(T) * 8 * (P.W1 + P.N) <= 96 * 1024;
  const bool w3path = staged3 && wide3_ok(t);
  if (w3path) {
    // S partials and the dG2 contributions in one warp-per-chunk pass (wide3.cuh)
    c->pos2.ensure(4 * L);
    c->tcontrib.ensure(sizeof(T) * L * P.slice[2]);
    k_inv_perm<<<gL, kThreads, 0, st>>>(c->s_dlk.as<uint32_t>(), L, c->pos2.as<uint32_t>());
    // pair-aligned warps: S(pair) complete at the end of its walk, no fold
    set_smem(w3::k_w3_bwd_pairs, w3::kBwdSmem);
    const int g = static_cast<int>(std::min<int64_t>((ucap + w3::kWarpsB / 2 - 1) / (w3::kWarpsB / 2),
                                                     static_cast<int64_t>(t->num_sms) * 3));
    w3::k_w3_bwd_pairs<<<g, w3::kWarpsB * 32, w3::kBwdSmem, st>>>(
        reinterpret_cast<const float*>(cores + P.coff[2]), reinterpret_cast<const float*>(c->H.as<T>()),
        c->counts.as<int>(), c->pair_start.as<int32_t>(), c->tail_dig.as<uint32_t>(),
        c->lk_bag.as<int32_t>(), reinterpret_cast<const float*>(c->lk_alpha.as<T>()),
        reinterpret_cast<const float*>(grad), c->s_lk.as<uint32_t>(), c->pos2.as<uint32_t>(),
        reinterpret_cast<float*>(c->S.as<T>()), reinterpret_cast<float*>(c->tcontrib.as<T>()));
  } else if (staged3) {
    const size_t smem = sizeof(T) * kTailChunk * (P.N + P.slice[2]) + 4 * kTailChunk;
    set_smem(k_srun3<T>, smem);
    k_srun3<T><<<grid_for(nchunksL, 1, t->num_sms, 8), 256, smem, st>>>(
        P, cores, c->tail_dig.as<uint32_t>(), c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), grad,
        c->s_key.as<uint32_t>(), c->s_lk.as<uint32_t>(), c->pair_scan.as<unsigned long long>(), L,
        kTailChunk, c->partS.as<T>());
    k_combine<T, 0><<<grid_for(ucap, 1, t->num_sms, 8), 128, 0, st>>>(
        c->partS.as<T>(), c->pair_scan.as<unsigned long long>(), c->pair_start.as<int32_t>(),
        c->counts.as<int>(), 0, P.W1, c->S.as<T>(), T(0));
  } else {
    const int Wc = P.W1;
    const size_t per_warp = sizeof(T) * (Wc + 4 * static_cast<size_t>(P.maxw));
    const int warps = warps_fitting(per_warp, sizeof(T) * Wc, 100 * 1024, 8);
    const size_t smem = sizeof(T) * Wc + per_warp * warps;
    auto kern = k_chunk_reduce<T, 0>;
    set_smem(kern, smem);
    kern<<<grid_for(nchunksL, 1, t->num_sms, 4), warps * 32, smem, st>>>(
        P, cores, c->H.as<T>(), nullptr, c->lk_pid.as<int32_t>(), c->tail_dig.as<uint32_t>(),
        c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), grad, c->s_key.as<uint32_t>(),
        c->s_lk.as<uint32_t>(), c->pair_scan.as<unsigned long long>(), L, kTailChunk, 1, Wc,
        c->partS.as<T>(), c->exact);
    k_combine<T, 0><<<grid_for(ucap, 1, t->num_sms, 8), 128, 0, st>>>(
        c->partS.as<T>(), c->pair_scan.as<unsigned long long>(), c->pair_start.as<int32_t>(),
        c->counts.as<int>(), 0, Wc, c->S.as<T>(), T(0));
  }
  t->mark("bwd_S");
  // ---- tail cores k >= 2 (the fused in-place update is only safe when no
  //      later kernel reads core k, i.e. d == 3)
  const bool fuse_tail = (mode == 1 && d == 3);
  segoff = 0;
  for (int k = 2; k < d; ++k) {
    const int j = k - 2;
    const int Wc = P.slice[k];
    if (w3path) {
      // contributions already at their i2-sorted positions (k_w3_bwd): slab sums
      const int nseg = P.m[k];
      const int64_t max_slabs = (L + w3::kW3Slab - 1) / w3::kW3Slab + nseg;
      c->w3_slab_base.ensure(4 * (nseg + 1));
      c->w3_slab_part.ensure(sizeof(float) * max_slabs * w3::S2);
      if (c->w3_cnt.cap < 4 * static_cast<size_t>(nseg)) {
        c->w3_cnt.ensure(4 * static_cast<size_t>(nseg));
        CK(cudaMemsetAsync(c->w3_cnt.p, 0, c->w3_cnt.cap, st));
      }
      const int32_t* seg = c->dseg.as<int32_t>() + segoff;
      w3::k_w3_slabs<<<1, 1024, 0, st>>>(seg, nseg, c->w3_slab_base.as<int32_t>());
      T* dst = fuse_tail ? cores + P.coff[k] : grads + P.coff[k];
      auto sk = fuse_tail ? w3::k_w3_segsum<1> : w3::k_w3_segsum<0>;
      sk<<<static_cast<int>(max_slabs), 64, 0, st>>>(
          reinterpret_cast<const float*>(c->tcontrib.as<T>()), seg, nseg, c->w3_slab_base.as<int32_t>(),
          c->w3_slab_part.as<float>(), c->w3_cnt.as<int>(), reinterpret_cast<float*>(dst),
          static_cast<float>(lr));
      segoff += P.m[k] + 1;
      continue;
    } else if (staged3) {
      // contributions computed in pair order (H staged per pair run), stored at
      // each lookup's i2-sorted position, then summed per i2 segment in order
      c->pos2.ensure(4 * L);
      c->tcontrib.ensure(sizeof(T) * L * Wc);
      k_inv_perm<<<gL, kThreads, 0, st>>>(c->s_dlk.as<uint32_t>() + j * L, L, c->pos2.as<uint32_t>());
      const size_t smem =
          sizeof(T) * (P.W1 + P.prefix[1] + 4 + static_cast<size_t>(kTailChunk) * P.N);
      const int cw = std::is_same_v<T, float> ? (P.n[2] % 4 == 0 ? 4 : P.n[2] % 2 == 0 ? 2 : 1) : 1;
      auto kern1 = cw == 4 ? k_pairwalk3<T, 1, false, 4>
                 : cw == 2 ? k_pairwalk3<T, 1, false, 2> : k_pairwalk3<T, 1, false>;
      set_smem(kern1, smem);
      kern1<<<grid_for(nchunksL, 1, t->num_sms, 8), 256, smem, st>>>(
          P, cores, c->H.as<T>(), c->lk_pid.as<int32_t>(), c->tail_dig.as<uint32_t>(),
          c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), grad, c->s_lk.as<uint32_t>(),
          c->pos2.as<uint32_t>(), L, kTailChunk, c->tcontrib.as<T>());
      T* dst = fuse_tail ? cores + P.coff[k] : grads + P.coff[k];
      if (fuse_tail)
        k_segsum3<T, 1><<<grid_for(P.m[k], 1, t->num_sms, 16), 256, 0, st>>>(
            c->tcontrib.as<T>(), c->dseg.as<int32_t>() + segoff, P.m[k], Wc, dst, tlr);
      else
        k_segsum3<T, 0><<<grid_for(P.m[k], 1, t->num_sms, 16), 256, 0, st>>>(
            c->tcontrib.as<T>(), c->dseg.as<int32_t>() + segoff, P.m[k], Wc, dst, T(0));
      segoff += P.m[k] + 1;
      continue;
    } else {
      const size_t per_warp = sizeof(T) * (Wc + 4 * static_cast<size_t>(P.maxw));
      const int warps = warps_fitting(per_warp, sizeof(T) * Wc, 100 * 1024, 8);
      const size_t smem = sizeof(T) * Wc + per_warp * warps;
      auto kern = k_chunk_reduce<T, 1>;
      set_smem(kern, smem);
      kern<<<grid_for(nchunksL, 1, t->num_sms, 4), warps * 32, smem, st>>>(
          P, cores, c->H.as<T>(), c->save ? c->saved.as<T>() : nullptr, c->lk_pid.as<int32_t>(),
          c->tail_dig.as<uint32_t>(), c->lk_bag.as<int32_t>(), c->lk_alpha.as<T>(), grad,
          c->s_dkey.as<uint32_t>() + j * L, c->s_dlk.as<uint32_t>() + j * L,
          c->dscan.as<unsigned long long>() + j * L, L, kTailChunk, k, Wc, c->partK.as<T>(),
          c->exact);
    }
    T* dst = fuse_tail ? cores + P.coff[k] : grads + P.coff[k];
    if (fuse_tail)
      k_combine<T, 1><<<grid_for(P.m[k], 1, t->num_sms, 8), 128, 0, st>>>(
          c->partK.as<T>(), c->dscan.as<unsigned long long>() + j * L, c->dseg.as<int32_t>() + segoff,
          nullptr, P.m[k], Wc, dst, tlr);
    else
      k_combine<T, 0><<<grid_for(P.m[k], 1, t->num_sms, 8), 128, 0, st>>>(
          c->partK.as<T>(), c->dscan.as<unsigned long long>() + j * L, c->dseg.as<int32_t>() + segoff,
          nullptr, P.m[k], Wc, dst, T(0));
    segoff += P.m[k] + 1;
  }
  t->mark("bwd_tail");
  // ---- head: D0 per pair, dG1 partials per i1 run
  {
    // the R1 x C1 accumulator lives in registers when a thread can own a column
    const bool reg_acc = P.C1 <= kThreads && P.r[1] <= kHeadMaxR1 && P.n[0] <= kHeadMaxP0;
    const size_t smem = sizeof(T) * ((reg_acc ? 0 : static_cast<size_t>(P.slice[1])) +
                                     static_cast<size_t>(P.C1) * (P.r[1] + 1) + P.W1 +
                                     P.slice[0]);
    if (smem > 227 * 1024) fail(TTGPU_ERR_INVALID_ARGUMENT, "G1 slice too large for shared memory");
    bool launched = false;
    if constexpr (std::is_same_v<T, float>) {
      // tensor-core head (head_tc.cuh): cfg3's shape class, P0 = 4, R1 = 64, C1 = 256
      if (t->tensor_head && d == 3 && P.n[0] == tc::HeadTc::P0 && P.r[1] == tc::HeadTc::R1 &&
          P.C1 == 256 && kHeadChunk <= tc::HeadTc::PAIRS) {
        constexpr int kNT = 512;
        auto kt = tc::k_head_bwd_tc<256, kNT>;
        set_smem(kt, tc::HeadTc::SMEM);
        kt<<<grid_for(ucap, kHeadChunk, t->num_sms, 1), kNT, tc::HeadTc::SMEM, st>>>(
            P, cores, c->S.as<float>(), c->pair_key_u.as<uint32_t>(), c->counts.as<int>(),
            c->scan1.as<unsigned long long>(), kHeadChunk, c->D0.as<float>(), c->part1.as<float>());
        launched = true;
      }
    }
    if (!launched) {
      auto kern = k_head_bwd<T>;
      set_smem(kern, smem);
      kern<<<grid_for(ucap, kHeadChunk, t->num_sms, 2), kThreads, smem, st>>>(
          P, cores, c->S.as<T>(), c->pair_key_u.as<uint32_t>(), c->counts.as<int>(),
          c->scan1.as<unsigned long long>(), kHeadChunk, c->D0.as<T>(), c->part1.as<T>());
    }
  }
  t->mark("bwd_head");
  const bool fuse_head = (mode == 1);
  // wide G1 slices (cfg3: 16,384 floats) are split over CTAs along y
  const dim3 gh(grid_for(P.m[1], 1, t->num_sms, 8),
                static_cast<unsigned>(std::max(1, std::min(16, P.slice[1] / 1024))));
  if (fuse_head)
    k_combine<T, 1><<<gh, 256, 0, st>>>(
        c->part1.as<T>(), c->scan1.as<unsigned long long>(), c->seg1.as<int32_t>(), nullptr, P.m[1],
        P.slice[1], cores + P.coff[1], tlr);
  else
    k_combine<T, 0><<<gh, 256, 0, st>>>(
        c->part1.as<T>(), c->scan1.as<unsigned long long>(), c->seg1.as<int32_t>(), nullptr, P.m[1],
        P.slice[1], grads + P.coff[1], T(0));
  t->mark("bwd_head_combine");
  if (fuse_head)
    k_head_g0<T, 1><<<grid_for(P.m[0], 1, t->num_sms, 8), 128, 0, st>>>(
        P, c->D0.as<T>(), t->pair_tab.as<int32_t>(), c->pair_key_u.as<uint32_t>(), c->counts.as<int>(),
        cores + P.coff[0], tlr);
  else
    k_head_g0<T, 0><<<grid_for(P.m[0], 1, t->num_sms, 8), 128, 0, st>>>(
        P, c->D0.as<T>(), t->pair_tab.as<int32_t>(), c->pair_key_u.as<uint32_t>(), c->counts.as<int>(),
        grads + P.coff[0], T(0));
  t->mark("bwd_g0");
  // fused mode with d >= 4: tail slices were written densely; apply them now
  if (mode == 1 && !fuse_tail && d >= 4) {
    for (int k = 2; k < d; ++k) {
      const int64_t n = P.slice[k] * static_cast<int64_t>(P.m[k]);
      k_sgd<T><<<grid_for(n, kThreads, t->num_sms), kThreads, 0, st>>>(cores + P.coff[k],
                                                                       grads + P.coff[k], n, tlr);
    }
  }
  CK(cudaGetLastError());
}

void check_ctx(ttgpu_table* t, ttgpu_ctx* c) {
  require_arg(c != nullptr && c->valid, "forward context is empty (run forward first)");
  require_arg(c->table == t, "forward context belongs to a different table");
  require_arg(c->snapshot == t->generation,
              cat("stale forward context for table '", t->name,
                  "': cores changed since the forward pass"));
}

// host_idx / host_L: the caller's index array (nullptr for device-side calls).
// The latch can hold a position set by an earlier asynchronous call on a larger
// batch, so the position is bounds-checked before host_idx is read.
void raise_latched(ttgpu_table* t, const int64_t* host_idx, int64_t host_L) {
  if (!t->h_errs) CK(cudaHostAlloc(reinterpret_cast<void**>(&t->h_errs), 32, cudaHostAllocDefault));
  unsigned long long* h = t->h_errs;  // pinned: the read rides the same sync as the caller's copies
  CK(cudaMemcpyAsync(h, t->errs.p, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     t->stream));
  CK(cudaStreamSynchronize(t->stream));
  const int sflags = static_cast<int>(h[2] & 0xffffffffu);
  if (sflags == 0 && h[0] == ULLONG_MAX) return;
  // reset the latch before reporting
  unsigned long long init[3] = {ULLONG_MAX, 0, 0};
  CK(cudaMemcpyAsync(t->errs.p, init, sizeof(init), cudaMemcpyHostToDevice, t->stream));
  CK(cudaStreamSynchronize(t->stream));
  if (sflags & 1) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets must start at 0");
  if (sflags & 2) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing");
  if (sflags & 4) fail(TTGPU_ERR_INVALID_ARGUMENT, "offsets end does not match the index count");
  const int64_t pos = static_cast<int64_t>(h[0]);
  if (host_idx && pos >= 0 && pos < host_L)
    throw std::out_of_range(cat("index ", host_idx[pos], " out of range [0, ", t->plan.num_rows,
                                ") for table '", t->name, "'"));
  throw std::out_of_range(cat("index at lookup ", pos, " out of range [0, ", t->plan.num_rows,
                              ") for table '", t->name, "'"));
}

// Kernels of a host-API call through the context's cached graph (see
// CachedGraph).  Not used while profiling, on the legacy default stream, or
// inside an outer capture.
template <class F>
void run_cached(ttgpu_table* t, CachedGraph& g, uint64_t key, F&& launch) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (t->stream) CK(cudaStreamIsCapturing(t->stream, &cs));
  if (!t->stream || t->prof || cs != cudaStreamCaptureStatusNone) {
    launch();
    return;
  }
  static const bool trace = std::getenv("TTGPU_TRACE") != nullptr;
  if (trace)
    std::fprintf(stderr, "[ttgpu trace] cached graph: exec=%d key=%d epoch=%d seen=%d\n",
                 g.exec != nullptr, g.key == key, g.epoch == g_alloc_epoch.load(), g.seen_key == key);
  if (g.exec && g.key == key && g.epoch == g_alloc_epoch.load()) {
    CK(cudaGraphLaunch(g.exec, t->stream));
    return;
  }
  if (g.seen_key != key) {  // first call with this key: eager, allocates what it needs
    g.seen_key = key;
    launch();
    return;
  }
  const uint64_t ep = g_alloc_epoch.load();
  cudaGraph_t graph = nullptr;
  CK(cudaStreamBeginCapture(t->stream, cudaStreamCaptureModeThreadLocal));
  try {
    launch();
  } catch (...) {
    cudaStreamEndCapture(t->stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  CK(cudaStreamEndCapture(t->stream, &graph));
  if (g_alloc_epoch.load() != ep) {  // a buffer grew while capturing: not replayable
    cudaGraphDestroy(graph);
    launch();
    return;
  }
  if (g.exec) cudaGraphExecDestroy(g.exec);
  g.exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&g.exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    g.exec = nullptr;
    launch();
    return;
  }
  g.key = key;
  g.epoch = ep;
  CK(cudaGraphLaunch(g.exec, t->stream));
}

uint64_t mix_key(std::initializer_list<uint64_t> v) {
  uint64_t h = 1469598103934665603ull;
  for (uint64_t x : v) h = (h ^ x) * 1099511628211ull;
  return h;
}

// Host-side structural validation with the reference's messages
// (index_batch.hpp:41-56); index range is checked on the device.
void validate_host(ttgpu_table* t, const int64_t* idx, int64_t L, const int64_t* off, int64_t B) {
  // O(1) on the good path: the start and end are checked here; monotonicity is
  // checked by the device (f3_hist / k_bags latch "offsets must be
  // non-decreasing", raised after the call with the reference's precedence,
  // and every device loop clamps its range to [0, L)).  The O(B) host scan
  // only runs to pick the reference's message when the end is wrong.
  require_arg(off != nullptr && off[0] == 0, "offsets must start at 0");
  if (off[B] != L) {
    bool monotone = true;
    for (int64_t b = 0; b < B; ++b) monotone &= off[b] <= off[b + 1];
    require_arg(monotone, "offsets must be non-decreasing");
    require_arg(false, cat("offsets end at ", off[B], " but there are ", L, " indices"));
  }
  (void)idx;
  (void)t;
}

}  // namespace
}  // namespace ttgpu

// =========================================================================
//                                 C ABI
// =========================================================================
extern "C" {

const char* ttgpu_last_error(void) { return g_last_error.c_str(); }
int ttgpu_abi_version(void) { return 1; }

int ttgpu_plan_shapes(int64_t num_rows, int64_t emb_dim, int tt_dim, int64_t rank,
                      const int64_t* rf_in, const int64_t* cf_in, int64_t* rf_out, int64_t* cf_out,
                      int64_t* ranks_out) {
  return guarded([&] {
    ShapePlan p = plan_shapes(num_rows, emb_dim, tt_dim, rank, rf_in, cf_in);
    std::copy(p.row_factors.begin(), p.row_factors.end(), rf_out);
    std::copy(p.col_factors.begin(), p.col_factors.end(), cf_out);
    std::copy(p.ranks.begin(), p.ranks.end(), ranks_out);
  });
}

int ttgpu_plan_info(int64_t num_rows, int64_t emb_dim, int tt_dim, const int64_t* rf,
                    const int64_t* cf, const int64_t* ranks, int64_t* padded, int64_t* params,
                    int64_t* reduction) {
  return guarded([&] {
    require_arg(tt_dim >= kMinTtDim && tt_dim <= kMaxTtDim,
                cat("tt_dim must be in [", kMinTtDim, ", ", kMaxTtDim, "], got ", tt_dim));
    ShapePlan p;
    p.num_rows = num_rows;
    p.emb_dim = emb_dim;
    p.tt_dim = tt_dim;
    p.row_factors.assign(rf, rf + tt_dim);
    p.col_factors.assign(cf, cf + tt_dim);
    p.ranks.assign(ranks, ranks + tt_dim + 1);
    p.validate();
    if (padded) *padded = p.padded_rows();
    if (params) *params = p.parameter_count();
    if (reduction) *reduction = p.memory_reduction();
  });
}

int ttgpu_decompose_index(int64_t flat, const int64_t* radices, int n, int64_t* digits) {
  return guarded([&] {
    auto v = decompose_index(flat, radices, n);
    std::copy(v.begin(), v.end(), digits);
  });
}

int ttgpu_recompose_index(const int64_t* digits, const int64_t* radices, int n, int64_t* flat) {
  return guarded([&] { *flat = recompose_index(digits, radices, n); });
}

int ttgpu_create(int64_t num_rows, int64_t emb_dim, int tt_dim, const int64_t* rf,
                 const int64_t* cf, const int64_t* ranks, int dtype, const char* name, int device,
                 void* stream, ttgpu_table** out) {
  return guarded([&] {
    require_arg(dtype == TTGPU_F32 || dtype == TTGPU_F64, "dtype must be TTGPU_F32 or TTGPU_F64");
    require_arg(tt_dim >= kMinTtDim && tt_dim <= kMaxTtDim,
                cat("tt_dim must be in [", kMinTtDim, ", ", kMaxTtDim, "], got ", tt_dim));
    auto t = std::make_unique<ttgpu_table>();
    t->plan.num_rows = num_rows;
    t->plan.emb_dim = emb_dim;
    t->plan.tt_dim = tt_dim;
    t->plan.row_factors.assign(rf, rf + tt_dim);
    t->plan.col_factors.assign(cf, cf + tt_dim);
    t->plan.ranks.assign(ranks, ranks + tt_dim + 1);
    t->plan.validate();
    check_supported(t->plan);
    t->name = name ? name : "tt-table";
    t->dtype = dtype;
    t->esz = dtype == TTGPU_F64 ? 8 : 4;
    t->device = device;
    t->stream = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(device));
    CK(cudaDeviceGetAttribute(&t->num_sms, cudaDevAttrMultiProcessorCount, device));
    {  // TTGPU_PDL: 0 plain launches, nonzero programmatic dependent launch
      const char* e = std::getenv("TTGPU_PDL");
      t->pdl = e ? std::atoi(e) : 0;
      const char* cs = std::getenv("TTGPU_GRID_SORT");
      t->grid_sort = !(cs && std::atoi(cs) == 0);
      const char* ch = std::getenv("TTGPU_CHUNKED");
      t->chunked = ch && std::atoi(ch) != 0;
      const char* fs = std::getenv("TTGPU_FUSE_SB");
      t->fuse_sb = !(fs && std::atoi(fs) == 0);
      const char* fc = std::getenv("TTGPU_FUSE_COMB");
      t->fuse_comb = fc && std::atoi(fc) != 0;
      const char* pb = std::getenv("TTGPU_PLAN_BWD1");
      t->plan_bwd1 = !(pb && std::atoi(pb) == 0);
      const char* mg = std::getenv("TTGPU_MERGE1");
      t->merge1 = !(mg && std::atoi(mg) == 0);
      if (const char* bc = std::getenv("TTGPU_B1COST")) std::sscanf(bc, "%d,%d", &t->b1tile, &t->b1cont);
    }
    std::vector<int64_t> coff;
    t->dp = make_devplan(t->plan, coff, t->total);
    t->cores.ensure(t->esz * t->total);
    t->grads.ensure(t->esz * t->total);
    CK(cudaMemsetAsync(t->cores.p, 0, t->esz * t->total, t->stream));
    CK(cudaMemsetAsync(t->grads.p, 0, t->esz * t->total, t->stream));
    const int64_t m01 = static_cast<int64_t>(t->dp.m[0]) * t->dp.m[1];
    t->pair_tab.ensure(4 * m01);
    CK(cudaMemsetAsync(t->pair_tab.p, 0xff, 4 * m01, t->stream));
    t->errs.ensure(3 * sizeof(unsigned long long));
    unsigned long long init[3] = {ULLONG_MAX, 0, 0};
    CK(cudaMemcpyAsync(t->errs.p, init, sizeof(init), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    *out = t.release();
  });
}

int ttgpu_destroy(ttgpu_table* t) {
  return guarded([&] {
    if (t) {
      cudaStreamSynchronize(t->stream);
      for (ttgpu_ctx* c : t->ctx_pool) delete c;
      t->ctx_pool.clear();
      delete t;
    }
  });
}

int ttgpu_set_stream(ttgpu_table* t, void* stream) {
  return guarded([&] { t->stream = static_cast<cudaStream_t>(stream); });
}

int ttgpu_core_size(const ttgpu_table* t, int k, int64_t* n) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    *n = t->plan.core_size(k);
  });
}

int ttgpu_get_core(ttgpu_table* t, int k, void* dst) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    CK(cudaMemcpyAsync(dst, static_cast<char*>(t->cores.p) + t->esz * t->dp.coff[k],
                       t->esz * t->plan.core_size(k), cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_get_grad(ttgpu_table* t, int k, void* dst) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    CK(cudaMemcpyAsync(dst, static_cast<char*>(t->grads.p) + t->esz * t->dp.coff[k],
                       t->esz * t->plan.core_size(k), cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_set_core(ttgpu_table* t, int k, const void* src) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    CK(cudaMemcpyAsync(static_cast<char*>(t->cores.p) + t->esz * t->dp.coff[k], src,
                       t->esz * t->plan.core_size(k), cudaMemcpyHostToDevice, t->stream));
    CK(cudaStreamSynchronize(t->stream));
    ++t->generation;
  });
}

int ttgpu_core_device_ptr(ttgpu_table* t, int k, void** p) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    *p = static_cast<char*>(t->cores.p) + t->esz * t->dp.coff[k];
  });
}

int ttgpu_grad_device_ptr(ttgpu_table* t, int k, void** p) {
  return guarded([&] {
    require_arg(k >= 0 && k < t->plan.tt_dim, cat("core index ", k, " out of range"));
    *p = static_cast<char*>(t->grads.p) + t->esz * t->dp.coff[k];
  });
}

int ttgpu_set_generic_path(ttgpu_table* t, int on) {
  return guarded([&] { t->force_generic = on != 0; });
}

int ttgpu_fast_path_kind(const ttgpu_table* t, int* kind) {
  return guarded([&] { *kind = t->force_generic ? -1 : f3_kind(t); });
}

int ttgpu_set_chunked(ttgpu_table* t, int on) {
  return guarded([&] { t->chunked = on != 0; });
}

int ttgpu_set_wide3(ttgpu_table* t, int on) {
  return guarded([&] { t->wide3 = on != 0; });
}

int ttgpu_set_grid_sort(ttgpu_table* t, int on) {
  return guarded([&] { t->grid_sort = on != 0; });
}

int ttgpu_set_tensor_path(ttgpu_table* t, int on) {
  return guarded([&] { t->tensor_head = on != 0; });
}

int ttgpu_set_exact_forward(ttgpu_table* t, int on) {
  return guarded([&] { t->exact = on != 0; });
}

int ttgpu_mark_mutated(ttgpu_table* t) {
  return guarded([&] { ++t->generation; });
}

int ttgpu_mutation_counter(const ttgpu_table* t, uint64_t* out) {
  return guarded([&] { *out = t->generation; });
}

int ttgpu_ctx_create(ttgpu_table* t, ttgpu_ctx** out) {
  return guarded([&] {
    ttgpu_ctx* c;
    if (t && !t->ctx_pool.empty()) {  // recycle a destroyed context's workspace
      c = t->ctx_pool.back();
      t->ctx_pool.pop_back();
      c->fast = false;
      c->snapshot = 0;
      c->valid = false;
      c->L = c->B = 0;
      c->pooling = 0;
      c->save = false;
      c->has_w = false;
      c->exact = true;
      c->w_dev = nullptr;
    } else {
      c = new ttgpu_ctx;
    }
    c->table = t;
    *out = c;
  });
}

int ttgpu_ctx_destroy(ttgpu_ctx* c) {
  return guarded([&] {
    if (!c) return;
    ttgpu_table* t = c->table;
    if (t) cudaStreamSynchronize(t->stream);
    if (t && t->ctx_pool.size() < 4) {
      c->valid = false;
      t->ctx_pool.push_back(c);
      return;
    }
    delete c;
  });
}

int ttgpu_forward(ttgpu_table* t, const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                  const double* w, int pooling, int64_t micro_batch, int save, void* out,
                  ttgpu_ctx* c) {
  return guarded([&] {
    require_arg(c != nullptr, "forward needs a context");
    require_arg(L >= 0 && B >= 0, "negative batch size");
    HostTrace tr(t->stream);
    tr("enter");
    validate_host(t, idx, L, off, B);
    tr("validate_host");
    require_arg(micro_batch >= 1, cat("micro_batch must be positive, got ", micro_batch));
    c->valid = false;
    c->h_idx.ensure(8 * std::max<int64_t>(L, 1));
    c->h_off.ensure(8 * (B + 1));
    c->h_out.ensure(t->esz * std::max<int64_t>(B * t->plan.emb_dim, 1));
    CK(cudaMemcpyAsync(c->h_idx.p, idx, 8 * L, cudaMemcpyHostToDevice, t->stream));
    CK(cudaMemcpyAsync(c->h_off.p, off, 8 * (B + 1), cudaMemcpyHostToDevice, t->stream));
    const double* dw = nullptr;
    if (w && L > 0) {
      c->h_w.ensure(8 * L);
      CK(cudaMemcpyAsync(c->h_w.p, w, 8 * L, cudaMemcpyHostToDevice, t->stream));
      dw = c->h_w.as<double>();
    }
    tr("h2d");
    const uint64_t key = mix_key({static_cast<uint64_t>(L), static_cast<uint64_t>(B),
                                  static_cast<uint64_t>(pooling), dw != nullptr ? 1u : 0u,
                                  save != 0 ? 1u : 0u, t->exact ? 1u : 0u,
                                  (t->force_generic ? 1u : 0u) | (t->grid_sort ? 2u : 0u) |
                                      (t->chunked ? 4u : 0u),
                                  static_cast<uint64_t>(t->dtype)});
    const bool replay = c->gfwd.exec && c->gfwd.key == key && c->gfwd.epoch == g_alloc_epoch.load();
    run_cached(t, c->gfwd, key, [&] {
      if (t->dtype == TTGPU_F64)
        forward_impl<double>(t, c, c->h_idx.as<int64_t>(), L, c->h_off.as<int64_t>(), B, dw,
                             pooling, save != 0, c->h_out.as<double>(), t->exact);
      else
        forward_impl<float>(t, c, c->h_idx.as<int64_t>(), L, c->h_off.as<int64_t>(), B, dw,
                            pooling, save != 0, c->h_out.as<float>(), t->exact);
      c->gfwd.aux = c->fast ? 1 : 0;
    });
    if (replay) {  // the host state forward_impl sets, for the replayed kernels
      c->table = t;
      c->snapshot = t->generation;
      c->L = L;
      c->B = B;
      c->pooling = pooling;
      c->save = save != 0 && t->dp.d >= 4;
      c->exact = t->exact;
      c->has_w = dw != nullptr;
      c->w_dev = dw;
      c->valid = true;
      c->fast = c->gfwd.aux != 0;
      g_rows.fetch_add(static_cast<uint64_t>(L));
    }
    tr("kernels");
    if (B > 0)
      CK(cudaMemcpyAsync(out, c->h_out.p, t->esz * B * t->plan.emb_dim, cudaMemcpyDeviceToHost,
                         t->stream));
    tr("d2h");
    try {
      raise_latched(t, idx, L);
      tr("raise_latched");
    } catch (...) {
      c->valid = false;
      throw;
    }
  });
}

int ttgpu_forward_device(ttgpu_table* t, const int64_t* idx, int64_t L, const int64_t* off,
                         int64_t B, const double* w, int pooling, int save, void* out,
                         ttgpu_ctx* c) {
  return guarded([&] {
    require_arg(c != nullptr, "forward needs a context");
    require_arg(L >= 0 && B >= 0, "negative batch size");
    if (t->dtype == TTGPU_F64)
      forward_impl<double>(t, c, idx, L, off, B, w, pooling, save != 0, static_cast<double*>(out),
                           t->exact);
    else
      forward_impl<float>(t, c, idx, L, off, B, w, pooling, save != 0, static_cast<float*>(out),
                          t->exact);
  });
}

int ttgpu_backward(ttgpu_table* t, ttgpu_ctx* c, int64_t L, int64_t B, const void* grad,
                   int64_t grad_len, void* const* grads_out) {
  return guarded([&] {
    check_ctx(t, c);
    require_arg(c->L == L && c->B == B,
                cat("forward context does not match this batch (", c->L, "/", c->B, " vs ", L, "/",
                    B, ")"));
    require_arg(grad_len == B * t->plan.emb_dim,
                cat("grad_output has ", grad_len, " elements, expected ", B * t->plan.emb_dim));
    c->h_grad.ensure(t->esz * std::max<int64_t>(grad_len, 1));
    if (grad_len > 0)
      CK(cudaMemcpyAsync(c->h_grad.p, grad, t->esz * grad_len, cudaMemcpyHostToDevice, t->stream));
    if (t->dtype == TTGPU_F64)
      backward_impl<double>(t, c, c->h_grad.as<double>(), 0, 0.0);
    else
      backward_impl<float>(t, c, c->h_grad.as<float>(), 0, 0.0);
    if (grads_out)
      for (int k = 0; k < t->plan.tt_dim; ++k)
        if (grads_out[k])
          CK(cudaMemcpyAsync(grads_out[k], static_cast<char*>(t->grads.p) + t->esz * t->dp.coff[k],
                             t->esz * t->plan.core_size(k), cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_backward_device(ttgpu_table* t, ttgpu_ctx* c, const void* grad) {
  return guarded([&] {
    check_ctx(t, c);
    if (t->dtype == TTGPU_F64)
      backward_impl<double>(t, c, static_cast<const double*>(grad), 0, 0.0);
    else
      backward_impl<float>(t, c, static_cast<const float*>(grad), 0, 0.0);
  });
}

int ttgpu_backward_sgd_device(ttgpu_table* t, ttgpu_ctx* c, const void* grad, double lr) {
  return guarded([&] {
    check_ctx(t, c);
    if (t->dtype == TTGPU_F64)
      backward_impl<double>(t, c, static_cast<const double*>(grad), 1, lr);
    else
      backward_impl<float>(t, c, static_cast<const float*>(grad), 1, lr);
    ++t->generation;
  });
}

int ttgpu_backward_sgd(ttgpu_table* t, ttgpu_ctx* c, int64_t L, int64_t B, const void* grad,
                       int64_t grad_len, double lr) {
  return guarded([&] {
    check_ctx(t, c);
    require_arg(c->L == L && c->B == B,
                cat("forward context does not match this batch (", c->L, "/", c->B, " vs ", L, "/",
                    B, ")"));
    require_arg(grad_len == B * t->plan.emb_dim,
                cat("grad_output has ", grad_len, " elements, expected ", B * t->plan.emb_dim));
    HostTrace tr(t->stream);
    tr("enter");
    c->h_grad.ensure(t->esz * std::max<int64_t>(grad_len, 1));
    if (grad_len > 0)
      CK(cudaMemcpyAsync(c->h_grad.p, grad, t->esz * grad_len, cudaMemcpyHostToDevice, t->stream));
    tr("h2d");
    uint64_t lrbits;
    std::memcpy(&lrbits, &lr, sizeof(lrbits));
    // everything the captured kernels depend on: the forward's shape and flags
    // (its buffers are the context's own; a reallocation bumps the epoch)
    const uint64_t key = mix_key({static_cast<uint64_t>(c->L), static_cast<uint64_t>(c->B),
                                  static_cast<uint64_t>(c->pooling), c->has_w ? 1u : 0u,
                                  c->save ? 1u : 0u, c->exact ? 1u : 0u, c->fast ? 1u : 0u,
                                  t->force_generic ? 1u : 0u, static_cast<uint64_t>(t->dtype),
                                  1u, lrbits});
    run_cached(t, c->gbwd, key, [&] {
      if (t->dtype == TTGPU_F64)
        backward_impl<double>(t, c, c->h_grad.as<double>(), 1, lr);
      else
        backward_impl<float>(t, c, c->h_grad.as<float>(), 1, lr);
    });
    tr("kernels");
    ++t->generation;
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_grad_buffer(ttgpu_table* t, void** ptr, int64_t* n) {
  return guarded([&] {
    *ptr = t->grads.p;
    *n = t->total;
  });
}

int ttgpu_graph_begin(ttgpu_table* t) {
  return guarded([&] {
    require_arg(t->stream != nullptr, "graph capture needs a non-default stream (ttgpu_set_stream)");
    CK(cudaStreamSynchronize(t->stream));
    if (t->graph_exec) {
      cudaGraphExecDestroy(t->graph_exec);
      t->graph_exec = nullptr;
    }
    if (t->graph) {
      cudaGraphDestroy(t->graph);
      t->graph = nullptr;
    }
    t->recycle_marks();  // marks recorded from here on belong to the new graph
    CK(cudaStreamBeginCapture(t->stream, cudaStreamCaptureModeThreadLocal));
  });
}

int ttgpu_graph_end(ttgpu_table* t, int* kernel_nodes, int* total_nodes) {
  return guarded([&] {
    cudaGraph_t g = nullptr;
    CK(cudaStreamEndCapture(t->stream, &g));
    t->graph = g;
    t->graph_marks = !t->marks.empty();
    CK(cudaGraphInstantiate(&t->graph_exec, g, 0));
    size_t n = 0;
    CK(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes(n);
    if (n) CK(cudaGraphGetNodes(g, nodes.data(), &n));
    int kn = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType ty;
      CK(cudaGraphNodeGetType(nd, &ty));
      if (ty == cudaGraphNodeTypeKernel) ++kn;
    }
    if (kernel_nodes) *kernel_nodes = kn;
    if (total_nodes) *total_nodes = static_cast<int>(n);
  });
}

int ttgpu_graph_launch(ttgpu_table* t) {
  return guarded([&] {
    require_arg(t->graph_exec != nullptr, "no captured graph");
    CK(cudaGraphLaunch(t->graph_exec, t->stream));
  });
}

int ttgpu_apply_grad(ttgpu_table* t, double lr) {
  return guarded([&] {
    for (int k = 0; k < t->plan.tt_dim; ++k) {
      const int64_t n = t->plan.core_size(k);
      if (n == 0) continue;
      const int g = grid_for(n, kThreads, t->num_sms);
      if (t->dtype == TTGPU_F64)
        k_sgd<double><<<g, kThreads, 0, t->stream>>>(t->cores.as<double>() + t->dp.coff[k],
                                                     t->grads.as<double>() + t->dp.coff[k], n,
                                                     static_cast<double>(lr));
      else
        k_sgd<float><<<g, kThreads, 0, t->stream>>>(t->cores.as<float>() + t->dp.coff[k],
                                                    t->grads.as<float>() + t->dp.coff[k], n,
                                                    static_cast<float>(lr));
    }
    CK(cudaGetLastError());
    ++t->generation;
  });
}

int ttgpu_sgd_step(ttgpu_table* t, const void* const* host_grads, double lr) {
  return guarded([&] {
    require_arg(host_grads != nullptr, "gradient core count mismatch");
    for (int k = 0; k < t->plan.tt_dim; ++k) {
      require_arg(host_grads[k] != nullptr, cat("gradient shape mismatch on core ", k));
      CK(cudaMemcpyAsync(static_cast<char*>(t->grads.p) + t->esz * t->dp.coff[k], host_grads[k],
                         t->esz * t->plan.core_size(k), cudaMemcpyHostToDevice, t->stream));
    }
    const int st = ttgpu_apply_grad(t, lr);
    if (st) fail(st, g_last_error);
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_lookup_rows_device(ttgpu_table* t, const int64_t* rows, int64_t n, void* out) {
  return guarded([&] {
    if (n <= 0) return;
    const DevPlan& P = t->dp;
    const size_t per_warp = t->esz * 2 * P.maxw;
    const int warps = warps_fitting(per_warp, 0, 64 * 1024, 8);
    const int g = grid_for(n, warps, t->num_sms);
    if (t->dtype == TTGPU_F64) {
      set_smem(k_lookup_rows<double>, per_warp * warps);
      k_lookup_rows<double><<<g, warps * 32, per_warp * warps, t->stream>>>(
          P, t->cores.as<double>(), rows, n, static_cast<double*>(out), t->d_bad());
    } else {
      set_smem(k_lookup_rows<float>, per_warp * warps);
      k_lookup_rows<float><<<g, warps * 32, per_warp * warps, t->stream>>>(
          P, t->cores.as<float>(), rows, n, static_cast<float*>(out), t->d_bad());
    }
    CK(cudaGetLastError());
    g_rows.fetch_add(static_cast<uint64_t>(n));
  });
}

int ttgpu_lookup_row(ttgpu_table* t, int64_t row, void* out) {
  return guarded([&] {
    if (row < 0 || row >= t->plan.num_rows)
      throw std::out_of_range(cat("index ", row, " out of range [0, ", t->plan.num_rows,
                                  ") for table '", t->name, "'"));
    DevBuf& r = t->lk_rows;
    DevBuf& o = t->lk_out;
    r.ensure(8);
    o.ensure(t->esz * t->plan.emb_dim);
    CK(cudaMemcpyAsync(r.p, &row, 8, cudaMemcpyHostToDevice, t->stream));
    const int st = ttgpu_lookup_rows_device(t, r.as<int64_t>(), 1, o.p);
    if (st) fail(st, g_last_error);
    CK(cudaMemcpyAsync(out, o.p, t->esz * t->plan.emb_dim, cudaMemcpyDeviceToHost, t->stream));
    CK(cudaStreamSynchronize(t->stream));
  });
}

int ttgpu_profile(ttgpu_table* t, int on) {
  return guarded([&] {
    CK(cudaStreamSynchronize(t->stream));
    if (!t->graph_marks) t->recycle_marks();
    t->prof = on != 0;
  });
}

int ttgpu_profile_read(ttgpu_table* t, char* names, int64_t names_len, float* ms, int max_phases,
                       int* n_out) {
  return guarded([&] {
    CK(cudaStreamSynchronize(t->stream));
    std::string all;
    int n = 0;
    for (size_t i = 1; i < t->marks.size() && n < max_phases; ++i) {
      const std::string& nm = t->marks[i].first;
      if (nm == "fwd_begin" || nm == "bwd_begin") continue;
      float v = 0;
      CK(cudaEventElapsedTime(&v, t->marks[i - 1].second, t->marks[i].second));
      ms[n++] = v;
      all += nm;
      all += ';';
    }
    if (names && names_len > 0) {
      std::strncpy(names, all.c_str(), static_cast<size_t>(names_len - 1));
      names[names_len - 1] = 0;
    }
    *n_out = n;
    if (!t->graph_marks) t->recycle_marks();
  });
}

int ttgpu_sync(ttgpu_table* t) {
  return guarded([&] { CK(cudaStreamSynchronize(t->stream)); });
}

int ttgpu_check(ttgpu_table* t) {
  return guarded([&] { raise_latched(t, nullptr, 0); });
}

namespace ttgpu {
uint64_t cache_fast_rows(bool reset);  // lfu_cache_host.inl
}
void ttgpu_stats_reset(void) {
  ttgpu::cache_fast_rows(true);
  g_rows.store(0);
  g_ws_peak.store(g_ws_cur.load());
}
// the cache fast path counts every lookup here and its hits on the device
uint64_t ttgpu_stats_rows(void) { return g_rows.load() - ttgpu::cache_fast_rows(false); }
uint64_t ttgpu_stats_peak_workspace(void) { return g_ws_peak.load(); }
void ttgpu_stats_add_rows(uint64_t n) { g_rows.fetch_add(n); }

// ---- synthetic streams: same algorithms and libstdc++ engines as the
// reference (rng.hpp:10-51, data.cpp:8-47, initializer.hpp:95-154) -------
namespace {
constexpr uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
}  // namespace

int ttgpu_zipf_batch(int64_t population, double s, uint64_t seed, int64_t bags, int64_t pf,
                     int64_t* indices, int64_t* offsets) {
  return guarded([&] {
    require_arg(population >= 1, cat("population must be positive, got ", population));
    require_arg(s >= 0, cat("exponent must be non-negative, got ", s));
    require_arg(bags >= 0, "num_bags must be non-negative");
    require_arg(pf >= 1, cat("pooling_factor must be >= 1, got ", pf));
    std::vector<double> cdf(population);
    double acc = 0.0;
    for (int64_t r = 0; r < population; ++r) {
      acc += std::pow(static_cast<double>(r + 1), -s);
      cdf[r] = acc;
    }
    const double inv = 1.0 / acc;
    for (double& c : cdf) c *= inv;
    cdf.back() = 1.0;
    std::mt19937_64 eng(splitmix(seed));
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    int64_t n = 0;
    offsets[0] = 0;
    for (int64_t b = 0; b < bags; ++b) {
      for (int64_t p = 0; p < pf; ++p) {
        const double u = unit(eng);
        auto it = std::upper_bound(cdf.begin(), cdf.end(), u);
        if (it == cdf.end()) --it;
        indices[n++] = static_cast<int64_t>(it - cdf.begin());
      }
      offsets[b + 1] = n;
    }
  });
}

int ttgpu_uniform_indices(int64_t rows, uint64_t seed, int64_t n, int64_t* out) {
  return guarded([&] {
    require_arg(rows >= 1, "rows must be positive");
    std::mt19937_64 eng(splitmix(seed));
    for (int64_t i = 0; i < n; ++i)
      out[i] = static_cast<int64_t>(
          std::uniform_int_distribution<uint64_t>(0, static_cast<uint64_t>(rows - 1))(eng));
  });
}

int ttgpu_derived_uniform_indices(int64_t rows, uint64_t seed, uint64_t stream, int64_t n,
                                  int64_t* out) {
  return guarded([&] {
    require_arg(rows >= 1, "rows must be positive");
    std::mt19937_64 eng(0);  // Rng::derive(seed, stream) (rng.hpp:25-29)
    eng.seed(splitmix(splitmix(seed) ^ splitmix(stream ^ 0xD1B54A32D192ED03ull)));
    for (int64_t i = 0; i < n; ++i)
      out[i] = static_cast<int64_t>(
          std::uniform_int_distribution<uint64_t>(0, static_cast<uint64_t>(rows - 1))(eng));
  });
}

int ttgpu_init_sampled_gaussian(ttgpu_table* t, uint64_t seed) {
  return guarded([&] {
    // InitSpec::sampled_gaussian(): threshold 2, target 1/(3N), MomentMatched
    const int d = t->plan.tt_dim;
    const double thr = 2.0;
    const double v = 1.0 / (3.0 * static_cast<double>(t->plan.emb_dim));
    const double root = std::pow(v, 1.0 / (2.0 * d));
    const double phi = std::exp(-0.5 * thr * thr) / std::sqrt(2.0 * M_PI);
    const double q = 0.5 * std::erfc(thr / std::sqrt(2.0));
    const double scale = root / std::sqrt(1.0 + thr * phi / q);
    for (int k = 0; k < d; ++k) {
      std::mt19937_64 eng(0);
      eng.seed(splitmix(splitmix(seed) ^ splitmix(static_cast<uint64_t>(k) ^ 0xD1B54A32D192ED03ull)));
      std::normal_distribution<double> nd(0.0, 1.0);
      const int64_t n = t->plan.core_size(k);
      std::vector<double> vals(n);
      for (int64_t i = 0; i < n; ++i) {
        double x = 0;
        int attempt = 0;
        for (; attempt < 10000; ++attempt) {
          x = nd(eng);
          if (std::abs(x) > thr) break;
        }
        if (attempt == 10000) fail(TTGPU_ERR_RUNTIME, "sampled init: no accepted draw");
        vals[i] = x * scale;
      }
      if (t->dtype == TTGPU_F64) {
        if (ttgpu_set_core(t, k, vals.data())) fail(TTGPU_ERR_RUNTIME, g_last_error);
      } else {
        std::vector<float> f(vals.begin(), vals.end());
        if (ttgpu_set_core(t, k, f.data())) fail(TTGPU_ERR_RUNTIME, g_last_error);
      }
    }
  });
}

// Diagnostics (not part of the reference interface): per-CTA timeline of the
// fast-path kernel `kid` (0 f3_gsort, 1 f3_fwd, 2 f3_srows_bwd2, 3 f3_bwd1,
// 4 f3_combine) into the device buffer `dev` (u64 [grid][8]: entry and exit
// global-timer ns, SM id, work note, four marks), or off with dev = NULL.
int ttgpu_debug_cta_times(int kid, void* dev) {
  return guarded([&] {
    require_arg(kid >= 0 && kid < 8, "kernel id out of range");
    unsigned long long* p = static_cast<unsigned long long*>(dev);
    CK(cudaMemcpyToSymbol(f3::g_cta_times, &p, sizeof(p), sizeof(p) * kid));
  });
}

}  // extern "C"

#include "lfu_cache_host.inl"
#include "sampler_host.inl"
#include "peer_host.inl"

void ttgpu_destroy_peers(ttgpu_peers* p) { delete p; }
void ttgpu_table::destroy_peers() { ttgpu_destroy_peers(peers); peers = nullptr; }
#include "dense_host.inl"
