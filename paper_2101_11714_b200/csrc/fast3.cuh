// Fast path for 3-core tables (every BASELINE config): compile-time TT shape,
// 5 kernels per fwd+bwd+SGD step -- f3_gsort (gsort.cuh, replaces the first
// three below when the batch fits one co-resident grid), f3_fwd,
// f3_srows_bwd2 (f3_srows and f3_bwd2 in one launch), f3_bwd1, f3_combine --
// deterministic, no floating-point atomics.
//
//   f3_hist     decode + validate; per-CTA histograms of two sort keys
//               (k1 = i1, k2 = i2); lookup->bag map, backward alpha, solo bags
//   f3_scan     one CTA per kScanKeys keys of either sort key: absolute
//               scatter offsets; tile lists (each key bucket cut into tiles)
//   f3_scatter  stable counting-sort scatter of both keys (warp match_any),
//               plus sorted (lookup, digits, solo) records for f3_fwd
//   f3_fwd      per i1-tile, pipelined one tile ahead: slots = distinct i0
//               (match_any), operands by bulk copy onto mbarriers,
//               H(slot) = G0[i0]·G1[i1], y = H·G2[i2]; bags pooled by their last
//               finished lookup (pool_if_last), single-lookup bags directly
//   f3_srows    warp per i1-tile: S(slot) = Σ D1, D1 = D2·G2ᵀ
//   f3_bwd1     per i1-tile (TMA-staged S and G0 rows): dG1 += Σ G0ᵀS, D0 = S·G1ᵀ;
//               runs of one-slot tiles of one (i1, i0) as one unit on their
//               summed S rows (merge units, planned by plan_bwd1)
//   f3_bwd2     per i2-tile: dG2 += Σ H(lookup)ᵀ D2 (H rows saved by f3_fwd)
//   f3_combine  fixed-order folds of the partials per core slice, fused with
//               the SGD update (or a dense gradient write)
//
// Reference semantics: embedding_ops.hpp:159-376.  In exact mode the forward
// keeps the reference's per-element operation order (separately rounded
// products/sums, p-ascending, lookup-ascending pooling), so outputs are
// bit-identical to ttrec::forward_bags.
#pragma once

#include <cooperative_groups.h>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_reduce.cuh>

#include "tt_kernels.cuh"

namespace ttgpu {
namespace f3 {

// Programmatic dependent launch (the fast-path kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization when the table enables it).
// Every kernel waits for its predecessor grid's completion (griddepcontrol.wait:
// a no-op without PDL) before touching memory, so overlap is limited to launch
// and scheduling.  (An early launch_dependents trigger measured slower and was
// dropped: it also cost every kernel a dependent global load at entry.)
// as soon as every CTA of this one has started.
__device__ __forceinline__ void pdl_entry() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Diagnostics: per-CTA timeline of the fast-path kernels (ttgpu_debug_cta_times),
// compiled in only with -DTTGPU_CTA_TIMES (`make lib-diag`: the reads of the
// pointer table at CTA entry would otherwise cost every kernel a dependent
// global load).  When g_cta_times[kid] is set, thread 0 of every CTA records
// the global timer at entry and at its own exit, the SM id, a kernel-specific
// work note and up to four intermediate marks: u64 [blockIdx][8].
__device__ unsigned long long* g_cta_times[8];
#ifdef TTGPU_CTA_TIMES
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct CtaClock {
  unsigned long long* p;
  __device__ __forceinline__ explicit CtaClock(int kid) {
    p = threadIdx.x == 0 ? g_cta_times[kid] : nullptr;
    if (p) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      p += 8 * static_cast<size_t>(blockIdx.x);
      p[0] = gtimer();
      p[2] = smid;
    }
  }
  __device__ __forceinline__ ~CtaClock() {
    if (p) p[1] = gtimer();
  }
};
__device__ __forceinline__ void cta_note(int kid, unsigned long long v) {
  unsigned long long* p = threadIdx.x == 0 ? g_cta_times[kid] : nullptr;
  if (p) p[8 * static_cast<size_t>(blockIdx.x) + 3] = v;
}
__device__ __forceinline__ void cta_mark(int kid, int m) {  // m in 0..3
  unsigned long long* p = threadIdx.x == 0 ? g_cta_times[kid] : nullptr;
  if (p) p[8 * static_cast<size_t>(blockIdx.x) + 4 + m] = gtimer();
}
#else
struct CtaClock {
  __device__ __forceinline__ explicit CtaClock(int) {}
};
__device__ __forceinline__ void cta_note(int, unsigned long long) {}
__device__ __forceinline__ void cta_mark(int, int) {}
#endif

struct Geo {
  int m0, m1, m2;
  uint32_t m12;  // m1 * m2
  int64_t num_rows;
  int64_t coff0, coff1, coff2;
};

struct Tile {
  int key, start, end, pad;
};

template <int P0_, int R1_, int N1_, int R2_, int N2_, int TT_>
struct Dims {
  static constexpr int P0 = P0_, R1 = R1_, N1 = N1_, R2 = R2_, N2 = N2_, TT = TT_;
  static constexpr int C1 = N1 * R2, S0 = P0 * R1, S1 = R1 * C1, P1 = P0 * N1;
  static constexpr int W1 = P1 * R2, S2 = R2 * N2, N = P1 * N2, C4 = C1 / 4;
  static constexpr int TT2 = 64;  // lookups per i2-tile (f3_bwd2)
  static_assert(N2 == 4, "fast path expects n_2 == 4 (float4 rows)");
  static_assert(C1 % 4 == 0 && R1 % 4 == 0, "C1 and R1 must be multiples of 4");
  static_assert(TT <= 32, "a tile's lookups must fit one warp (slot ballots / match_any)");
};

constexpr int kThreads = 256;

// acc += a * b per component (fmul2_rn / ffma2: tt_kernels.cuh).  Exact: separately
// rounded products and sums (the reference's fp32 loop), products two at a time.
template <typename T, bool kExact>
__device__ __forceinline__ float4 madd4(float a, float4 b, float4 acc) {
  if constexpr (kExact) {
    const float2 p01 = fmul2_rn(a, make_float2(b.x, b.y));
    const float2 p23 = fmul2_rn(a, make_float2(b.z, b.w));
    acc.x = __fadd_rn(acc.x, p01.x);
    acc.y = __fadd_rn(acc.y, p01.y);
    acc.z = __fadd_rn(acc.z, p23.x);
    acc.w = __fadd_rn(acc.w, p23.y);
  } else {
    acc.x = madd<float, kExact>(a, b.x, acc.x);
    acc.y = madd<float, kExact>(a, b.y, acc.y);
    acc.z = madd<float, kExact>(a, b.z, acc.z);
    acc.w = madd<float, kExact>(a, b.w, acc.w);
  }
  return acc;
}

__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Pooling of a multi-lookup bag by its last finished (lookup, row) task: every
// task of a bag's lookups counts itself in bag_cnt[bag] after storing its y row
// (fenced); the task completing the count sums the bag's y rows in lookup
// order -- f3_pool's arithmetic (embedding_ops.hpp:232-249) -- and stores the
// pooled row.  The sort kernel zeroes bag_cnt for every bag of the batch and
// writes the (zero) rows of empty bags, so no separate pooling pass runs.
// Cache mode (lk_slot != nullptr, lfu_cache_host.inl): the bag's cached
// lookups count as already done (f3_gsort presets bag_cnt), and the pooled row
// is cached_out + tt_out, each summed in lookup order (model.hpp:210-223,
// combine_partition_outputs lfu_cache.hpp:106-126).
template <int N, bool kExact>
__device__ __forceinline__ void pool_if_last(int bag, int parts, const int64_t* __restrict__ off,
                                             int64_t L, const double* __restrict__ w, int mean,
                                             const float* y, float* __restrict__ out, int* bag_cnt,
                                             const int* __restrict__ lk_slot = nullptr,
                                             const float* __restrict__ store = nullptr) {
  __threadfence();  // this task's y row before its count
  const int64_t s = off[bag], e = off[bag + 1];
  if (atomicAdd(bag_cnt + bag, 1) != static_cast<int>(e - s) * parts - 1) return;
  __threadfence();  // every other task's row is visible past the count
  const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
  const float inv = static_cast<float>(1.0 / static_cast<double>(e - s));
#pragma unroll
  for (int c = 0; c < N / 4; ++c) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f), cac = acc;
    for (int64_t l = lo; l < hi; ++l) {
      const float a = static_cast<float>(w ? w[l] : 1.0);
      const int slot = lk_slot ? __ldcg(lk_slot + l) : -1;
      if (slot >= 0) {
        const float4 v = reinterpret_cast<const float4*>(store + static_cast<int64_t>(slot) * N)[c];
        cac = make_float4(__fadd_rn(cac.x, __fmul_rn(a, v.x)), __fadd_rn(cac.y, __fmul_rn(a, v.y)),
                          __fadd_rn(cac.z, __fmul_rn(a, v.z)), __fadd_rn(cac.w, __fmul_rn(a, v.w)));
      } else {
        acc = madd4<float, kExact>(a, __ldcg(reinterpret_cast<const float4*>(y + l * N) + c), acc);
      }
    }
    if (lk_slot)
      acc = make_float4(__fadd_rn(cac.x, acc.x), __fadd_rn(cac.y, acc.y), __fadd_rn(cac.z, acc.z),
                        __fadd_rn(cac.w, acc.w));
    if (mean && e - s > 1) {
      acc.x = __fmul_rn(acc.x, inv);
      acc.y = __fmul_rn(acc.y, inv);
      acc.z = __fmul_rn(acc.z, inv);
      acc.w = __fmul_rn(acc.w, inv);
    }
    reinterpret_cast<float4*>(out + static_cast<int64_t>(bag) * N)[c] = acc;
  }
}

// ---- TMA bulk copies (cp.async.bulk, sm_90+/sm_100a) with mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive (count 1) and raise the expected transaction bytes of the current phase
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy; bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Sorted record of key 1 (lookup order within an i1 bucket):
//   x = lookup, y = i0 | i2 << 16, z = bag | (single-lookup bag) << 31, w = alpha bits
__device__ __forceinline__ uint4 make_rec(uint32_t l, uint32_t d02, int32_t solo, int32_t bag, float alpha) {
  return make_uint4(l, d02, static_cast<uint32_t>(bag) | (solo >= 0 ? 0x80000000u : 0u), __float_as_uint(alpha));
}
// the bag a record's lookup is pooled into directly (its only lookup), else -1
__device__ __forceinline__ int rec_solo(const uint4& r) {
  return (r.z >> 31) ? static_cast<int>(r.z & 0x7fffffffu) : -1;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Block-wide exclusive scan of one int per thread (blockDim == kThreads).
__device__ __forceinline__ int block_excl_scan(int v, int* total, int* sm /* >= 33 ints */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sm[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < (kThreads / 32) ? sm[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kThreads / 32) sm[lane] = s;  // inclusive warp totals
    if (lane == kThreads / 32 - 1) sm[32] = s;
  }
  __syncthreads();
  const int base = wid ? sm[wid - 1] : 0;
  const int r = base + x - v;
  *total = sm[32];
  __syncthreads();
  return r;
}

// Copy `n` floats (element e at dst[e]) whose source is src_of(e); U loads in flight.
template <int U, class SrcFn>
__device__ __forceinline__ void gather_to_smem(float* dst, int n, SrcFn src_of) {
  for (int e0 = threadIdx.x; e0 < n; e0 += kThreads * U) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * kThreads;
      v[u] = e < n ? __ldg(src_of(e)) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (e0 + u * kThreads < n) dst[e0 + u * kThreads] = v[u];
  }
}

// ------------------------------------------------------------- f3_hist ---
// 512 * LPT lookups per CTA (LPT lookups per thread, loads batched).
template <typename T, int LPT>
__global__ void __launch_bounds__(512) f3_hist(Geo g, const int64_t* __restrict__ idx, int64_t L,
                                               int NT, const int64_t* __restrict__ off,
                                               int64_t B, const double* __restrict__ w, int mean,
                                               uint16_t* __restrict__ d0, uint16_t* __restrict__ d1,
                                               uint16_t* __restrict__ d2, int32_t* __restrict__ lk_bag,
                                               T* __restrict__ alpha, uint32_t* __restrict__ hist1,
                                               uint32_t* __restrict__ hist2,
                                               uint32_t* __restrict__ tot1, uint32_t* __restrict__ tot2,
                                               unsigned long long* __restrict__ bad,
                                               int* __restrict__ errs, int32_t* __restrict__ solo,
                                               float* __restrict__ out, int N, int* __restrict__ bag_cnt) {
  pdl_entry();
  extern __shared__ uint32_t shist[];  // m1 + m2
  uint32_t* sh1 = shist;
  uint32_t* sh2 = shist + g.m1;
  // this thread's first bag's offsets: loaded now, in flight during the digit phase
  const int64_t b_first = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int64_t s_first = 0, e_first = 0;
  if (b_first < B) {
    s_first = off[b_first];
    e_first = off[b_first + 1];
  }
  for (int k = threadIdx.x; k < g.m1 + g.m2; k += blockDim.x) shist[k] = 0;
  __syncthreads();
  const int tile = blockIdx.x;
  const int lane = threadIdx.x & 31;
  if (tile < NT) {
    int64_t rows[LPT];
    const int64_t base = static_cast<int64_t>(tile) * 512 * LPT + threadIdx.x;
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int64_t l = base + q * 512;
      rows[q] = l < L ? idx[l] : 0;
    }
#pragma unroll
    for (int q = 0; q < LPT; ++q) {
      const int64_t l = base + q * 512;
      uint32_t k1 = 0xffffffffu, k2 = 0xffffffffu;
      if (l < L) {
        int64_t row = rows[q];
        if (row < 0 || row >= g.num_rows) {
          atomicMin(bad, static_cast<unsigned long long>(l));
          row = 0;
        }
        const uint32_t r = static_cast<uint32_t>(row);
        const uint32_t i0 = r / g.m12;
        const uint32_t rem = r - i0 * g.m12;
        const uint32_t i1 = rem / static_cast<uint32_t>(g.m2);
        const uint32_t i2 = rem - i1 * static_cast<uint32_t>(g.m2);
        d0[l] = static_cast<uint16_t>(i0);
        d1[l] = static_cast<uint16_t>(i1);
        d2[l] = static_cast<uint16_t>(i2);
        k1 = i1;
        k2 = i2;
      }
      unsigned peers = __match_any_sync(0xffffffffu, k1);
      if (k1 != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&sh1[k1], __popc(peers));
      peers = __match_any_sync(0xffffffffu, k2);
      if (k2 != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&sh2[k2], __popc(peers));
    }
  }
  __syncthreads();
  if (tile < NT) {
    for (int k = threadIdx.x; k < g.m1; k += blockDim.x) {
      const uint32_t c = sh1[k];
      hist1[static_cast<int64_t>(k) * NT + tile] = c;
      if (c) atomicAdd(tot1 + k, c);
    }
    for (int k = threadIdx.x; k < g.m2; k += blockDim.x) {
      const uint32_t c = sh2[k];
      hist2[static_cast<int64_t>(k) * NT + tile] = c;
      if (c) atomicAdd(tot2 + k, c);
    }
  }
  // bags (grid-stride over all CTAs): offsets checks, lookup->bag, backward alpha
  for (int64_t b = b_first; b < B; b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = b == b_first ? s_first : off[b], e = b == b_first ? e_first : off[b + 1];
    if (b == 0 && s != 0) atomicOr(errs, 1);
    if (e < s) atomicOr(errs, 2);
    if (b == B - 1 && e != L) atomicOr(errs, 4);
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    const double sz = static_cast<double>(e - s);
    bag_cnt[b] = 0;
    if (e == s)  // an empty bag pools to zeros (no lookup will)
      for (int c = 0; c < N; c += 4) reinterpret_cast<float4*>(out + b * N + c)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t l = lo; l < hi; ++l) {
      lk_bag[l] = static_cast<int32_t>(b);
      solo[l] = e - s == 1 ? static_cast<int32_t>(b) : -1;  // pooled by f3_fwd directly
      double a = w ? w[l] : 1.0;
      if (mean) a /= sz;
      alpha[l] = static_cast<T>(a);
    }
  }
}

// ------------------------------------------------------------- f3_scan ---
// One CTA per kScanKeys consecutive keys (CTAs [0, nb1) key 1, then key 2).
// The hist kernel also summed every bucket into tot[k] (integer atomics:
// exact), so each CTA derives its global bases -- lookups, tiles and combine
// groups of all earlier keys -- from tot[] alone, scans its own keys'
// (key-major, K x NT) histogram columns into absolute scatter offsets, and
// cuts its buckets into tiles of <= TT lookups.
struct ScanArgs {
  uint32_t* hist;
  const uint32_t* tot;  // K bucket totals
  int32_t* tile_base;   // K + 1
  int32_t* group_base;  // K + 1: combine groups of <= kGroup tiles per bucket (>= 1 each)
  Tile* tiles;
  int* ntiles;
  int K, TT;
};

// combine: candidate tiles per warp task (dG1 / dG2).  Run partials are sparse
// among a bucket's tiles (one per CTA run), so wide groups keep the number of
// group partials -- and the last arriver's sequential fold -- small.
constexpr int kGroup = 64;
constexpr int kGroup0 = 32;    // combine: candidate CTA blocks per warp task (dG0; dense for hot i0)
static_assert(kGroup0 <= 32, "a dG0 combine task takes its candidates in one 32-lane ballot");
constexpr int kScanKeys = 8;   // keys per f3_scan CTA
constexpr int kScanThreads = 256;

__device__ __forceinline__ int spad(int i) { return i + (i >> 5); }  // bank-conflict-free chunks

__device__ __forceinline__ uint32_t n_groups(uint32_t tk) {
  return tk > kGroup ? (tk + kGroup - 1) / kGroup : 1;
}

__global__ void __launch_bounds__(kScanThreads) f3_scan(ScanArgs a1, ScanArgs a2, int nb1, int NT,
                                                        int64_t L) {
  pdl_entry();
  using Scan = cub::BlockScan<uint32_t, kScanThreads>;
  using Red = cub::BlockReduce<uint32_t, kScanThreads>;
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Red::TempStorage red;
  } tmp;
  __shared__ uint32_t kb[3][kScanKeys + 1];  // per-key lookup / tile / group starts
  extern __shared__ uint32_t sh[];           // spad(kScanKeys * NT) histogram entries
  const bool second = static_cast<int>(blockIdx.x) >= nb1;
  const ScanArgs& A = second ? a2 : a1;
  const int blk = second ? blockIdx.x - nb1 : blockIdx.x;
  const int K = A.K, TT = A.TT;
  const int k0 = blk * kScanKeys, k1 = min(K, k0 + kScanKeys);
  const int tid = threadIdx.x;
  // this CTA's histogram columns: loads issued first, in flight during the bases
  const int n = (k1 - k0) * NT;
  uint32_t* hist = A.hist + static_cast<int64_t>(k0) * NT;
#pragma unroll 4
  for (int i = tid; i < n; i += kScanThreads) sh[spad(i)] = hist[i];
  // global bases: all keys before k0
  uint32_t p = 0, t = 0, gq = 0;
  for (int k = tid; k < k0; k += kScanThreads) {
    const uint32_t c = A.tot[k];
    const uint32_t tk = (c + TT - 1) / TT;
    p += c;
    t += tk;
    gq += n_groups(tk);
  }
  __shared__ uint32_t bases[3];
  {
    const uint32_t v0 = Red(tmp.red).Sum(p);  // aggregates are valid in thread 0 only
    __syncthreads();
    const uint32_t v1 = Red(tmp.red).Sum(t);
    __syncthreads();
    const uint32_t v2 = Red(tmp.red).Sum(gq);
    if (tid == 0) {
      bases[0] = v0;
      bases[1] = v1;
      bases[2] = v2;
    }
    __syncthreads();
  }
  const uint32_t pos_base = bases[0], tile_base = bases[1], group_base = bases[2];
  if (tid < 32) {  // per-key starts within the CTA (one lane per key)
    const int k = k0 + tid;
    const uint32_t c = k < k1 ? A.tot[k] : 0u;
    const uint32_t tk = (c + TT - 1) / TT;
    const uint32_t gk = k < k1 ? n_groups(tk) : 0u;
    uint32_t ic = c, it = tk, ig = gk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y0 = __shfl_up_sync(0xffffffffu, ic, o);
      const uint32_t y1 = __shfl_up_sync(0xffffffffu, it, o);
      const uint32_t y2 = __shfl_up_sync(0xffffffffu, ig, o);
      if (tid >= o) {
        ic += y0;
        it += y1;
        ig += y2;
      }
    }
    if (tid <= kScanKeys) {
      // exclusive starts for keys k0 .. k0 + kScanKeys (the last entry = CTA total)
      kb[0][tid] = pos_base + ic - c;
      kb[1][tid] = tile_base + it - tk;
      kb[2][tid] = group_base + ig - gk;
    }
  }
  // this CTA's histogram columns -> absolute scatter offsets
  __syncthreads();
  const int per = (n + kScanThreads - 1) / kScanThreads;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  uint32_t sacc = 0;
  for (int i = lo; i < hi; ++i) sacc += sh[spad(i)];
  uint32_t ex;
  Scan(tmp.scan).ExclusiveSum(sacc, ex);
  ex += pos_base;
  for (int i = lo; i < hi; ++i) {
    const uint32_t c = sh[spad(i)];
    sh[spad(i)] = ex;
    ex += c;
  }
  __syncthreads();
#pragma unroll 4
  for (int i = tid; i < n; i += kScanThreads) hist[i] = sh[spad(i)];
  // per-key tile / group bases and the tiles themselves
  for (int k = k0 + tid; k < k1; k += kScanThreads) {
    A.tile_base[k] = static_cast<int32_t>(kb[1][k - k0]);
    A.group_base[k] = static_cast<int32_t>(kb[2][k - k0]);
  }
  if (k1 == K && tid == 0) {
    const int j = k1 - k0;
    A.tile_base[K] = static_cast<int32_t>(kb[1][j]);
    A.group_base[K] = static_cast<int32_t>(kb[2][j]);
    *A.ntiles = static_cast<int>(kb[1][j]);
  }
  for (int k = k0; k < k1; ++k) {
    const uint32_t bs = kb[0][k - k0], be = kb[0][k - k0 + 1];
    const uint32_t tb = kb[1][k - k0], tk = kb[1][k - k0 + 1] - tb;
    for (uint32_t q = tid; q < tk; q += kScanThreads) {
      Tile tl;
      tl.key = k;
      tl.start = static_cast<int>(bs + q * TT);
      tl.end = static_cast<int>(min(be, bs + (q + 1) * TT));
      tl.pad = 0;
      A.tiles[tb + q] = tl;
    }
  }
}

// ---------------------------------------------------------- f3_scatter ---
// Stable scatter of one key: 8 warps per CTA, each owning TL/8 consecutive
// lookups, keys loaded 8 rounds at a time.  Run for key 1 then key 2.
__device__ __forceinline__ void scatter_one(const uint16_t* __restrict__ key, int K, int64_t L,
                                            int TL, int NT, const uint32_t* __restrict__ hoff,
                                            uint32_t* __restrict__ perm, uint32_t* wc,
                                            const uint16_t* __restrict__ dg0 = nullptr,
                                            const uint16_t* __restrict__ dg2 = nullptr,
                                            const int32_t* __restrict__ solo = nullptr,
                                            uint4* __restrict__ rec = nullptr,
                                            const int32_t* __restrict__ lk_bag = nullptr,
                                            const float* __restrict__ alpha = nullptr) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int per = TL / 8;
  const int64_t base = static_cast<int64_t>(tile) * TL + static_cast<int64_t>(wid) * per;
  uint32_t* my = wc + static_cast<int64_t>(wid) * K;
  // this CTA's scatter bases (f3_scan) for the first 4 * 256 keys: loads in
  // flight during the counting phase
  uint32_t hpre[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int k = threadIdx.x + j * 256;
    hpre[j] = k < K ? hoff[static_cast<int64_t>(k) * NT + tile] : 0u;
  }
  for (int k = lane; k < K; k += 32) my[k] = 0;
  __syncwarp();
  for (int r0 = 0; r0 < per; r0 += 256) {
    uint32_t ks[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t l = base + r0 + q * 32 + lane;
      ks[q] = (r0 + q * 32 < per && l < L) ? key[l] : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t k = ks[q];
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      if (k != 0xffffffffu && lane == __ffs(peers) - 1) my[k] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  auto bases = [&](int k, uint32_t run) {  // per-warp starts of key k
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = wc[static_cast<int64_t>(w) * K + k];
      wc[static_cast<int64_t>(w) * K + k] = run;
      run += c;
    }
  };
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (threadIdx.x + j * 256 < K) bases(threadIdx.x + j * 256, hpre[j]);
  for (int k = threadIdx.x + 1024; k < K; k += 256) bases(k, hoff[static_cast<int64_t>(k) * NT + tile]);
  __syncthreads();
  const unsigned lt = lanemask_lt();
  for (int r0 = 0; r0 < per; r0 += 256) {
    uint32_t ks[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t l = base + r0 + q * 32 + lane;
      ks[q] = (r0 + q * 32 < per && l < L) ? key[l] : 0xffffffffu;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t k = ks[q];
      const int64_t l = base + r0 + q * 32 + lane;
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      uint32_t pos = 0;
      if (k != 0xffffffffu) pos = my[k] + __popc(peers & lt);
      __syncwarp();
      if (k != 0xffffffffu) {
        perm[pos] = static_cast<uint32_t>(l);
        // sorted record (position -> lookup, i0 | i2 << 16, solo bag) for f3_fwd
        if (rec)
          rec[pos] = make_rec(static_cast<uint32_t>(l), dg0[l] | (static_cast<uint32_t>(dg2[l]) << 16),
                              solo[l], lk_bag[l], alpha[l]);
        if (lane == __ffs(peers) - 1) my[k] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) f3_scatter(Geo g, const uint16_t* __restrict__ d0,
                                                  const uint16_t* __restrict__ d1,
                                                  const uint16_t* __restrict__ d2, int64_t L,
                                                  int TL, int NT, const uint32_t* __restrict__ hoff1,
                                                  const uint32_t* __restrict__ hoff2,
                                                  uint32_t* __restrict__ perm1,
                                                  uint32_t* __restrict__ perm2,
                                                  uint32_t* __restrict__ tot,
                                                  const int32_t* __restrict__ solo,
                                                  uint4* __restrict__ rec1,
                                                  const int32_t* __restrict__ lk_bag,
                                                  const float* __restrict__ alpha) {
  pdl_entry();
  extern __shared__ uint32_t wc[];  // 8 x max(m1, m2)
  // f3_scan has consumed the bucket totals: clear them for the next batch
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < g.m1 + g.m2; k += gridDim.x * blockDim.x)
    tot[k] = 0u;
  scatter_one(d1, g.m1, L, TL, NT, hoff1, perm1, wc, d0, d2, solo, rec1, lk_bag, alpha);
  scatter_one(d2, g.m2, L, TL, NT, hoff2, perm2, wc);
}

// ------------------------------------------------------------- f3_fwd ----
template <class D>
struct FwdSmem {
  // floats: G1s[S1] (TMA) | Hs[TT*HSP] | G0s[TT*S0P] (TMA rows) | G2s[TT*S2P] (TMA rows);
  // then 2 mbarriers + ints (2 metadata buffers)
  static constexpr int R2P = D::R2 + 1;          // padded H rows: (slot, row) -> distinct banks
  static constexpr int HSP = D::P1 * R2P + 1;    // odd slot stride
  static constexpr int HSP4 = (D::TT * HSP + 3) / 4 * 4;
  static constexpr int S0P = D::S0 + 4;          // bulk-copy rows: 16-byte pitch, 2 slots per warp conflict-free
  static constexpr int S2P = D::S2 + 4;          // lookups' float4 rows in distinct bank groups
  static constexpr int MI = 3 * D::TT + 4;       // ints per metadata buffer: lk_l, lk_slot, lk_solo, meta
  static __host__ __device__ size_t floats() {
    size_t f = D::S1 + static_cast<size_t>(HSP4) + static_cast<size_t>(D::TT) * (S0P + S2P);
    return (f + 3) / 4 * 4;
  }
  static __host__ __device__ size_t bytes(int /*m0*/) {
    return floats() * 4 + 16 + sizeof(int) * 2 * MI;
  }
};

// Per i1-tile (CTAs stride over the tiles), software-pipelined one tile ahead:
//   wait A (G1[i1], G0 rows of the slots) -> H(slot) = G0·G1 (all warps)
//   | warp 0: slots of the next tile (distinct i0 numbered by first
//   |   occurrence, match_any; the numbering backward reuses) and its G1/G0
//   |   bulk copies onto A, overlapping ...
//   wait B (G2 rows of the lookups) -> y = H·G2[i2] (warps 1..)
//   then warp 0 issues the next tile's G2 rows onto B (they land during its H).
// Tile descriptors and sorted records (lookup, digits; f3_scatter) are loaded
// two tiles ahead.  Saves H rows and, per lookup, the H row index (hloc) for
// f3_bwd2.
template <class D, bool kExact, bool kCache = false>
__global__ void __launch_bounds__(kThreads) f3_fwd(Geo g, const float* __restrict__ cores,
                                                   const Tile* __restrict__ tiles,
                                                   const int* __restrict__ ntiles,
                                                   const uint4* __restrict__ rec,
                                                   const double* __restrict__ w,
                                                   float* __restrict__ out,
                                                   float* __restrict__ Hbuf, float* __restrict__ y,
                                                   uint32_t* __restrict__ hloc,
                                                   uint16_t* __restrict__ slot_of_pos,
                                                   uint16_t* __restrict__ tile_i0,
                                                   int* __restrict__ tile_nslots,
                                                   int* __restrict__ tile_one,
                                                   const int64_t* __restrict__ off, int64_t L, int mean,
                                                   int* __restrict__ bag_cnt,
                                                   const int* __restrict__ cache_slot,
                                                   const float* __restrict__ store) {
  CtaClock clk_(1);
  pdl_entry();
  using SM = FwdSmem<D>;
  extern __shared__ __align__(128) float sm[];
  float* G1s = sm;
  float* Hs = G1s + D::S1;
  float* G0s = Hs + SM::HSP4;
  float* G2s = G0s + D::TT * SM::S0P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SM::floats());  // [0] G1+G0, [1] G2
  int* mbuf = reinterpret_cast<int*>(bar + 2);                      // 2 x {lk_l, lk_slot, lk_solo, meta}
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  const int nt = *ntiles;
  const int G = static_cast<int>(gridDim.x);
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  // warp 0 state: this lane's lookup of the staged tile (for its G2 copy), the
  // next tile's descriptor + record, the tile after that's descriptor
  bool g2_act = false;
  int g2_i2 = 0, g2_ntl = 0;
  int g1_key = -1;  // the i1 whose G1 slice is in G1s (warp 0)
  Tile ndn{}, nd2{};
  uint4 nrn = make_uint4(0u, 0u, 0u, 0u);
  // slots + metadata of tile u into buffer m, G1/G0 copies onto bar[0]
  auto stage = [&](int u, const Tile& tl, uint4 r, int m) {
    int* lk_l = mbuf + m * SM::MI;
    int* lk_slot = lk_l + D::TT;
    int* lk_solo = lk_slot + D::TT;
    int* meta = lk_solo + D::TT;
    const int ntl = tl.end - tl.start;
    const bool act = lane < ntl;
    const int l = static_cast<int>(r.x), i0 = static_cast<int>(r.y & 0xffffu);
    const unsigned peers = __match_any_sync(0xffffffffu, act ? i0 : -1);
    const int leader = __ffs(peers) - 1;
    const bool is_first = act && leader == lane;
    const unsigned fb = __ballot_sync(0xffffffffu, is_first);
    const int nslots = __popc(fb);
    const int s = __shfl_sync(0xffffffffu, __popc(fb & lanemask_lt()), leader);
    if (act) {
      lk_l[lane] = l;
      lk_slot[lane] = s;
      lk_solo[lane] = static_cast<int>(r.z);  // bag | single-lookup bit (make_rec)
      slot_of_pos[tl.start + lane] = static_cast<uint16_t>(s);
      hloc[l] = static_cast<uint32_t>(tl.start + s);
    }
    if (is_first) tile_i0[tl.start + s] = static_cast<uint16_t>(i0);
    if (lane == 0) {
      tile_nslots[u] = nslots;
      // (i1, i0) of a one-slot tile, for f3_bwd1's merge units (plan_bwd1)
      tile_one[u] = nslots == 1 ? (tl.key << 16) | i0 : -1;
      meta[0] = ntl;
      meta[1] = nslots;
      meta[2] = tl.start;
    }
    g2_act = act;
    g2_i2 = static_cast<int>(r.y >> 16);
    g2_ntl = ntl;
    __syncwarp();
    // G1[i1] stays staged across consecutive tiles of the same bucket (hot
    // buckets under Zipf): only a new i1 is copied
    const bool need_g1 = tl.key != g1_key;
    g1_key = tl.key;
    if (lane == 0) {
      // smem last touched by generic-proxy accesses; order them before the async writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect(bar, ((need_g1 ? D::S1 : 0) + nslots * D::S0) * 4);
      if (need_g1) tma_load(G1s, G1 + static_cast<int64_t>(tl.key) * D::S1, D::S1 * 4, bar);
    }
    __syncwarp();
    if (is_first) tma_load(G0s + s * SM::S0P, G0 + static_cast<int64_t>(i0) * D::S0, D::S0 * 4, bar);
  };
  auto issue_g2 = [&]() {
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect(bar + 1, g2_ntl * D::S2 * 4);
    }
    __syncwarp();
    if (g2_act)
      tma_load(G2s + lane * SM::S2P, G2 + static_cast<int64_t>(g2_i2) * D::S2, D::S2 * 4, bar + 1);
  };
  const int t0 = static_cast<int>(blockIdx.x);
  if (wid == 0 && t0 < nt) {
    const Tile tl = tiles[t0];
    if (t0 + G < nt) ndn = tiles[t0 + G];
    if (t0 + 2 * G < nt) nd2 = tiles[t0 + 2 * G];
    const uint4 r = lane < tl.end - tl.start ? rec[tl.start + lane] : make_uint4(0u, 0u, 0u, 0u);
    if (t0 + G < nt && lane < ndn.end - ndn.start) nrn = rec[ndn.start + lane];
    stage(t0, tl, r, 0);
    issue_g2();
  }
  uint32_t phase = 0;
  int m = 0;
#ifdef TTGPU_CTA_TIMES
  unsigned long long note_t = 0, note_l = 0, note_s = 0;
#endif
  for (int t = t0; t < nt; t += G, phase ^= 1u, m ^= 1) {
    const int* lk_l = mbuf + m * SM::MI;
    const int* lk_slot = lk_l + D::TT;
    const int* lk_solo = lk_slot + D::TT;
    const int* meta = lk_solo + D::TT;
    mbar_wait(bar, phase);
    const int ntl = meta[0], nslots = meta[1], start = meta[2];
#ifdef TTGPU_CTA_TIMES
    if (t == t0) cta_mark(1, 0);
    note_t += 1;
    note_l += ntl;
    note_s += nslots;
#endif
    // H(slot) = G0[i0] (P0 x R1) · G1[i1] (R1 x C1): thread -> (slot, 4 columns), all P0 rows
    for (int q = tid; q < nslots * D::C4; q += kThreads) {
      const int s = q / D::C4, c4 = q - s * D::C4;
      float4 acc[D::P0];
#pragma unroll
      for (int a = 0; a < D::P0; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float* g0 = G0s + s * SM::S0P;
#pragma unroll 8
      for (int p = 0; p < D::R1; ++p) {
        const float4 b = reinterpret_cast<const float4*>(G1s + p * D::C1)[c4];
#pragma unroll
        for (int a = 0; a < D::P0; ++a) acc[a] = madd4<float, kExact>(g0[a * D::R1 + p], b, acc[a]);
      }
      float* hs = Hs + s * SM::HSP;
      float* hg = Hbuf + static_cast<int64_t>(start + s) * D::W1;
#pragma unroll
      for (int a = 0; a < D::P0; ++a) {
        const int c = a * D::C1 + c4 * 4;  // = (row, r) in the (P1 x R2) view
        const float v4[4] = {acc[a].x, acc[a].y, acc[a].z, acc[a].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int row = (c + u) / D::R2, r = (c + u) - row * D::R2;
          hs[row * SM::R2P + r] = v4[u];
        }
        reinterpret_cast<float4*>(hg + c)[0] = acc[a];
      }
    }
    __syncthreads();  // H rows complete; G1s / G0s free
    if (wid == 0) {
      if (t + G < nt) {
        stage(t + G, ndn, nrn, m ^ 1);  // lands during this tile's y phase
        ndn = nd2;
        if (t + 2 * G < nt && lane < ndn.end - ndn.start) nrn = rec[ndn.start + lane];
        if (t + 3 * G < nt) nd2 = tiles[t + 3 * G];
      }
    } else {
      // y = H(slot) (P1 x R2) · G2[i2] (R2 x N2): thread -> (lookup, row a), warps 1..
      mbar_wait(bar + 1, phase);
      for (int q = tid - 32; q < ntl * D::P1; q += kThreads - 32) {
        const int i = q / D::P1, a = q - i * D::P1;
        const float* hrow = Hs + lk_slot[i] * SM::HSP + a * SM::R2P;
        const float4* g2 = reinterpret_cast<const float4*>(G2s + i * SM::S2P);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
        for (int r = 0; r < D::R2; ++r) acc = madd4<float, kExact>(hrow[r], g2[r], acc);
        const int z = lk_solo[i];
        if (z < 0) {  // the bag's only lookup: pooled here, (0 + w·y, the pooling arithmetic)
          const float wl = w ? static_cast<float>(w[lk_l[i]]) : 1.f;
          reinterpret_cast<float4*>(out + static_cast<int64_t>(z & 0x7fffffff) * D::N)[a] =
              madd4<float, kExact>(wl, acc, make_float4(0.f, 0.f, 0.f, 0.f));
        } else {
          reinterpret_cast<float4*>(y + static_cast<int64_t>(lk_l[i]) * D::N)[a] = acc;
          if constexpr (kCache)
            pool_if_last<D::N, kExact>(z, D::P1, off, L, w, mean, y, out, bag_cnt, cache_slot, store);
          else
            pool_if_last<D::N, kExact>(z, D::P1, off, L, w, mean, y, out, bag_cnt);
        }
      }
    }
    __syncthreads();  // G2s / Hs free
    if (wid == 0 && t + G < nt) issue_g2();
  }
#ifdef TTGPU_CTA_TIMES
  cta_note(1, note_t | (note_l << 16) | (note_s << 40));
#endif
}

// ----------------------------------------------------------- f3_srows ----
// One WARP per i1-tile (no block barriers): S(slot) = Σ_{lookups of the slot,
// tile order} D1, D1 = D2·G2[i2]ᵀ, D2 = T(alpha)·grad[bag].  Lane owns the
// elements e = lane + 32k of the (P1 x R2) row (a = e / R2, r = e % R2); the
// members of a slot are walked in tile order, U of them with loads in flight.
// S rows land at the slot's position (start + s), kappa-major: row s holds
// S[a0][c] at a0*C1 + c == a*R2 + r, so f3_bwd1 can bulk-copy a tile's rows.
template <class D>
__device__ __forceinline__ void srows_tile(int t, const float* __restrict__ cores, int64_t coff2,
                                           const Tile* __restrict__ tiles,
                                           const int* __restrict__ ntiles, int max_tiles,
                                           const uint32_t* __restrict__ perm,
                                           const uint16_t* __restrict__ d2,
                                           const int32_t* __restrict__ lk_bag,
                                           const float* __restrict__ alpha,
                                           const float* __restrict__ grad,
                                           const uint16_t* __restrict__ slot_of_pos,
                                           const int* __restrict__ tile_nslots,
                                           float* __restrict__ Sbuf,
                                           const uint4* __restrict__ rec = nullptr) {
  constexpr int EPL = (D::W1 + 31) / 32;  // row elements per lane
  // distinct G2 rows a lane reads per member: r = (lane + 32k) % R2 repeats with period NR
  constexpr int NR = D::R2 > 32 ? D::R2 / 32 : 1;
  static_assert(D::R2 <= 32 ? 32 % D::R2 == 0 : D::R2 % 32 == 0, "lane -> rank column map");
  constexpr int U = 8;  // members with G2 loads in flight
  const int lane = threadIdx.x & 31;
  if (t >= max_tiles) return;
  // the tile count and this tile's descriptor in one round trip (entries past
  // the count are in bounds, just unused)
  const int nt = *ntiles;
  const Tile tl = tiles[t];
  const int nslots = tile_nslots[t];
  if (t >= nt) return;
  const float* G2 = cores + coff2;
  const int ntl = tl.end - tl.start;
  // each lane fetches its own lookup's D2 = T(alpha) * grad[bag] once (one
  // round trip for the whole tile); members' values then move by shuffles
  int my_sl = -1, my_i2 = 0;
  float dmy[D::N];
  if (lane < ntl) {
    // the sorted record (f3_gsort / f3_scatter: lookup, i0 | i2 << 16, bag, alpha)
    // gives i2, bag and alpha in one load; else through the lookup index
    int bag;
    float al;
    my_sl = slot_of_pos[tl.start + lane];
    if (rec) {
      const uint4 r = rec[tl.start + lane];
      my_i2 = static_cast<int>(r.y >> 16);
      bag = static_cast<int>(r.z & 0x7fffffffu);
      al = __uint_as_float(r.w);
    } else {
      const int l = static_cast<int>(perm[tl.start + lane]);
      my_i2 = d2[l];
      bag = lk_bag[l];
      al = alpha[l];
    }
    const float4* grow = reinterpret_cast<const float4*>(grad + static_cast<int64_t>(bag) * D::N);
#pragma unroll
    for (int q = 0; q < D::N / 4; ++q) {
      const float4 gq = __ldg(grow + q);
      dmy[4 * q] = __fmul_rn(al, gq.x);
      dmy[4 * q + 1] = __fmul_rn(al, gq.y);
      dmy[4 * q + 2] = __fmul_rn(al, gq.z);
      dmy[4 * q + 3] = __fmul_rn(al, gq.w);
    }
  } else {
#pragma unroll
    for (int q = 0; q < D::N; ++q) dmy[q] = 0.f;
  }
  // slot-sorted member order (stable: tile order within a slot), so the loads
  // of U consecutive members stay in flight across slot boundaries
  __shared__ int members_all[8][32];
  __shared__ __align__(16) float d2s_all[8][32 * D::N];
  int* members = members_all[(threadIdx.x >> 5) & 7];
  float* d2s = d2s_all[(threadIdx.x >> 5) & 7];
#pragma unroll
  for (int q = 0; q < D::N / 4; ++q)
    reinterpret_cast<float4*>(d2s + lane * D::N)[q] =
        make_float4(dmy[4 * q], dmy[4 * q + 1], dmy[4 * q + 2], dmy[4 * q + 3]);
  {
    const unsigned peers = __match_any_sync(0xffffffffu, my_sl);
    const int rank = __popc(peers & lanemask_lt());
    const unsigned leaders = __ballot_sync(0xffffffffu, my_sl >= 0 && rank == 0);
    // lane s (< nslots): size of slot s (slots are numbered by first occurrence)
    const int lead_s = lane < nslots ? static_cast<int>(__fns(leaders, 0, lane + 1)) : 0;
    const int cnt_s = __shfl_sync(0xffffffffu, __popc(peers), lead_s);
    int inc = lane < nslots ? cnt_s : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int ex = inc - (lane < nslots ? cnt_s : 0);
    const int base = __shfl_sync(0xffffffffu, ex, my_sl >= 0 ? my_sl : 0);
    if (my_sl >= 0) members[base + rank] = lane;
    __syncwarp();
  }
  float acc[EPL];
  int cur = -1;
  for (int j0 = 0; j0 < ntl; j0 += U) {
    int m[U], sl[U];
    float4 g2[U][NR];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      m[u] = j0 + u < ntl ? members[j0 + u] : 0;
      sl[u] = __shfl_sync(0xffffffffu, my_sl, m[u]);
      const int i2 = __shfl_sync(0xffffffffu, my_i2, m[u]);
      if (j0 + u < ntl) {
#pragma unroll
        for (int k = 0; k < NR; ++k)
          g2[u][k] = __ldg(reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(i2) * D::S2) +
                           (lane + 32 * k) % D::R2);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (j0 + u >= ntl) break;
      float dv[D::N];
#pragma unroll
      for (int q = 0; q < D::N / 4; ++q) {
        const float4 x = reinterpret_cast<const float4*>(d2s + m[u] * D::N)[q];
        dv[4 * q] = x.x;
        dv[4 * q + 1] = x.y;
        dv[4 * q + 2] = x.z;
        dv[4 * q + 3] = x.w;
      }
      const bool first = sl[u] != cur;
      if (first) {  // a new slot starts: flush the finished one
        if (cur >= 0) {
          float* dst = Sbuf + static_cast<int64_t>(tl.start + cur) * D::W1;
#pragma unroll
          for (int k = 0; k < EPL; ++k)
            if (lane + 32 * k < D::W1) dst[lane + 32 * k] = acc[k];
        }
        cur = sl[u];
      }
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const int a = ((lane + 32 * k) % D::W1) / D::R2;
        float d4[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // dv[a*4 + j] with a lane-dependent a: select statically
          float x = dv[j];
#pragma unroll
          for (int aa = 1; aa < D::P1; ++aa) x = (a == aa) ? dv[aa * 4 + j] : x;
          d4[j] = x;
        }
        const float4 gk = g2[u][k % NR];
        float v = __fmul_rn(d4[0], gk.x);
        v = __fmaf_rn(d4[1], gk.y, v);
        v = __fmaf_rn(d4[2], gk.z, v);
        v = __fmaf_rn(d4[3], gk.w, v);
        acc[k] = first ? v : __fadd_rn(acc[k], v);
      }
    }
  }
  if (cur >= 0) {
    float* dst = Sbuf + static_cast<int64_t>(tl.start + cur) * D::W1;
#pragma unroll
    for (int k = 0; k < EPL; ++k)
      if (lane + 32 * k < D::W1) dst[lane + 32 * k] = acc[k];
  }
}

// warps of virtual CTAs [vblock, ...) walk the i1-tiles grid-stride (vgrid
// virtual CTAs in all); the per-warp shared rows are reused tile to tile
template <class D>
__device__ __forceinline__ void srows_body(int vblock, int vgrid, const float* __restrict__ cores,
                                           int64_t coff2, const Tile* __restrict__ tiles,
                                           const int* __restrict__ ntiles, int max_tiles,
                                           const uint32_t* __restrict__ perm,
                                           const uint16_t* __restrict__ d2,
                                           const int32_t* __restrict__ lk_bag,
                                           const float* __restrict__ alpha,
                                           const float* __restrict__ grad,
                                           const uint16_t* __restrict__ slot_of_pos,
                                           const int* __restrict__ tile_nslots,
                                           float* __restrict__ Sbuf,
                                           const uint4* __restrict__ rec = nullptr) {
  const int nw = blockDim.x >> 5;
  for (int t = vblock * nw + (threadIdx.x >> 5); t < max_tiles; t += vgrid * nw) {
    srows_tile<D>(t, cores, coff2, tiles, ntiles, max_tiles, perm, d2, lk_bag, alpha, grad, slot_of_pos,
                  tile_nslots, Sbuf, rec);
    __syncwarp();
  }
}

// ------------------------------------------------------------ f3_bwd1 ----
// Per i1-tile, from the S rows of f3_srows:
//   dG1 (R1 x C1) += Σ_kappa G0[i0(kappa)]ᵀ (x) S[kappa]     kappa = (slot, a0)
//   D0[kappa] (R1) = S[kappa] · G1[i1]ᵀ  -> CTA-private D0 block per i0
// Each CTA owns a contiguous tile range.  A tile's S rows are contiguous
// (positions start .. start+nslots) and arrive by one TMA bulk copy; its G0
// rows by one bulk copy per slot; both are issued for tile t+1 as soon as the
// GEMMs of tile t have consumed the buffers.  G1[i1] is staged transposed
// (regular loads) when the tile's bucket differs from the previous one.
// Consecutive tiles of the same i1 keep accumulating the dG1 partial in
// registers; one partial per (CTA, i1 run) is flushed (has1 marks the run's
// first tile).  D0 accumulates per (CTA, i0) in a CTA-private global block,
// stored on first touch (d0mask marks it for f3_combine).  Slots of one tile
// have distinct i0, tiles run in order: every sum has a fixed order.
template <class D>
struct G1Blk {
  static constexpr int RB = D::R1 >= 64 ? 4 : 2;
  static constexpr int CB = D::R1 >= 64 ? 8 : 4;
  static constexpr int TR = D::R1 / RB;  // dG1 threads along r1
  static constexpr int TC = D::C1 / CB;  // dG1 threads along c
  static constexpr int RB0 = D::R1 >= 64 ? 4 : 2;
  static constexpr int TR0 = D::R1 / RB0;  // D0 threads along r1
  static constexpr int KG = 1;             // dG1 partial rows per (CTA, i1 run)
  static_assert(TR * TC <= kThreads, "bad blocking");
  static_assert(D::C1 % CB == 0 && D::R1 % RB == 0 && CB % 4 == 0, "bad blocking");
};

constexpr int kBwd1TileCost = 4;  // f3_bwd1 range weight of a tile: kBwd1TileCost + nslots
constexpr int kBwd1Stages = 2;  // tiles of bulk copies in flight per f3_bwd1 CTA (3: 2 CTAs/SM, slower)

template <class D>
struct Bwd1Smem {
  // floats: NS stages x { S[TT*P0 x C1] (TMA) | G0s[TT*P0 x R1] (TMA) } | G1t[C1 x R1P] ;
  // then NS mbarriers, ints
  static constexpr int NS = kBwd1Stages;
  static constexpr int R1P = D::R1 + 4;
  static constexpr int STAGE = D::TT * D::W1 + D::TT * D::S0;  // floats per stage
  static constexpr int NI = (NS + 1) * D::TT + 16 + 256;  // NS x slot i0 / first-touch flags / misc / bitmap
  static __host__ __device__ size_t floats() {
    size_t f = NS * static_cast<size_t>(STAGE) + static_cast<size_t>(D::C1) * R1P;
    return (f + 3) / 4 * 4;
  }
  static __host__ __device__ size_t bytes() { return floats() * 4 + 8 * NS + sizeof(int) * NI; }
};

template <class D>
__device__ __forceinline__ void bwd1_body(
    Geo g, const float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const float* __restrict__ Sbuf,
    const uint16_t* __restrict__ tile_i0, const int* __restrict__ tile_nslots,
    float* __restrict__ part1, int* __restrict__ has1, float* __restrict__ D0acc,
    unsigned char* __restrict__ d0mask, const int* __restrict__ plan = nullptr,
    const uint8_t* __restrict__ ulen = nullptr) {
  using SM = Bwd1Smem<D>;
  using GB = G1Blk<D>;
  extern __shared__ __align__(128) float sm[];
  constexpr int NS = SM::NS;
  float* G1t = sm + NS * SM::STAGE;                // [c][R1P]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SM::floats());  // NS stages
  int* slot_i0 = reinterpret_cast<int*>(bar + NS);  // NS x TT
  int* d0first = slot_i0 + NS * D::TT;              // TT
  int* misc = d0first + D::TT;  // [2*stage + 0] key, [2*stage + 1] nslots, [8 + stage] unit tiles
  unsigned* d0bits = reinterpret_cast<unsigned*>(misc + 16);
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const int nt = *ntiles;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  int t_lo, t_hi;
  // Contiguous tile ranges balanced by work, not by count: tile t weighs
  // kTileCost + nslots(t) (its GEMMs scale with the slot count), and belongs
  // to the CTA floor(E(t) * grid / W), E = exclusive prefix of the weights.
  // Planned ahead by f3_srows_bwd2's first CTA (plan_bwd1), or else recomputed
  // here by every CTA (the prefix is small); ranges partition the tiles.
  if (plan) {
    t_lo = __ldcg(plan + blockIdx.x);
    t_hi = max(t_lo, __ldcg(plan + blockIdx.x + 1));
  } else {
    constexpr int kTileCost = kBwd1TileCost;
    using Scan = cub::BlockScan<int, kThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int range[2];
    const int per = (nt + kThreads - 1) / kThreads;
    const int a0 = min(nt, tid * per), a1 = min(nt, a0 + per);
    // up to kPer weights per thread are loaded all at once (independent loads,
    // one round trip) and kept in registers for the threshold walk
    constexpr int kPer = 16;
    int wv[kPer];
    int wsum = 0;
    if (per <= kPer) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) wv[j] = a0 + j < a1 ? kTileCost + tile_nslots[a0 + j] : 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) wsum += wv[j];
    } else {
      for (int t = a0; t < a1; ++t) wsum += kTileCost + tile_nslots[t];
    }
    int ex, W;
    Scan(scan_tmp).ExclusiveSum(wsum, ex, W);
    // owner(t) == b  <=>  E(t) in [ceil(b W / G), ceil((b+1) W / G)): the range
    // ends are the first tiles reaching the two thresholds; only the (at most
    // two) threads whose chunk holds a threshold walk their chunk
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t th[2] = {(b * W + G - 1) / G, ((b + 1) * W + G - 1) / G};
    if (tid < 2) range[tid] = th[tid] <= 0 ? 0 : nt;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (ex < th[q] && th[q] <= ex + wsum) {
        int64_t e = ex;
        int t = a0;
        if (per <= kPer) {
#pragma unroll
          for (int j = 0; j < kPer; ++j)
            if (t < a1 && e < th[q]) {
              e += wv[j];
              ++t;
            }
        } else {
          for (; t < a1 && e < th[q]; ++t) e += kTileCost + tile_nslots[t];
        }
        range[q] = t;
      }
    }
    __syncthreads();
    t_lo = range[0];
    t_hi = range[1] > range[0] ? range[1] : range[0];
  }
  unsigned long long note_ns = 0, note_runs = 0;  // diagnostics (cta_note)
  cta_mark(3, 0);
  // prologue loads, all in flight together: warp 0 the descriptors and slot
  // i0s of the first NS + 1 tiles; every thread G1[i1] of the first tile (its
  // transposed staging needs no global round trip at the first tile)
  constexpr int kG1U = 8;
  constexpr bool kG1Pre = D::S1 <= kThreads * kG1U;
  Tile p_d[NS];
  int p_ns[NS], p_i0[NS], p_K[NS];
  int nx_t = t_lo + NS;  // warp 0: first tile of the next unit to fetch
  if (wid == 0) {
    if (ulen) {  // merge units: unit q starts where unit q - 1 ends
      int tq = t_lo;
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        p_K[q] = tq < t_hi ? min(static_cast<int>(ulen[tq]), t_hi - tq) : 0;
        p_d[q] = tq < t_hi ? tiles[tq] : Tile{};
        p_ns[q] = tq < t_hi ? tile_nslots[tq] : 0;
        p_i0[q] = lane < p_ns[q] ? static_cast<int>(tile_i0[p_d[q].start + lane]) : 0;
        tq += p_K[q];
      }
      nx_t = tq;
    } else {
#pragma unroll
      for (int q = 0; q < NS; ++q) {
        p_d[q] = t_lo + q < t_hi ? tiles[t_lo + q] : Tile{};
        p_ns[q] = t_lo + q < t_hi ? tile_nslots[t_lo + q] : 0;
        p_K[q] = t_lo + q < t_hi ? 1 : 0;
      }
#pragma unroll
      for (int q = 0; q < NS; ++q)
        p_i0[q] = lane < p_ns[q] ? static_cast<int>(tile_i0[p_d[q].start + lane]) : 0;
    }
  }
  float g1pre[kG1U];
  int pre_i1 = -1;
  if (kG1Pre && t_lo < t_hi) {
    pre_i1 = __ldg(&tiles[t_lo].key);
    const float* src = G1 + static_cast<int64_t>(pre_i1) * D::S1;
#pragma unroll
    for (int u = 0; u < kG1U; ++u) g1pre[u] = tid + u * kThreads < D::S1 ? __ldg(src + tid + u * kThreads) : 0.f;
  }
  float* d0acc = D0acc + static_cast<int64_t>(blockIdx.x) * g.m0 * D::S0;
  unsigned char* d0m = d0mask + static_cast<int64_t>(blockIdx.x) * g.m0;
  for (int e = tid; e < g.m0; e += kThreads) d0m[e] = 0;
  for (int e = tid; e < 256; e += kThreads) d0bits[e] = 0u;
  if (tid == 0)
    for (int q = 0; q < NS; ++q) mbar_init(bar + q, 1);
  __syncthreads();
  // warp 0 keeps NS tiles of bulk copies in flight: the descriptors of tile
  // t+NS are fetched during tile t, its S rows (one copy) and G0 rows (one per
  // slot) are issued into tile t's stage as soon as tile t's GEMMs are done
  // A merged unit (n_K > 1 one-slot tiles of one i0) copies the S row of each
  // of its tiles (tile q's rows start at its first lookup position, q * TT
  // after the unit's first) and the one G0 row.
  Tile n_d{};
  int n_ns = 0, n_i0 = 0, n_K = 1;
  auto issue = [&](int st) {
    float* Ss = sm + st * SM::STAGE;
    float* G0s = Ss + D::TT * D::W1;
    const int rows = n_K > 1 ? n_K : n_ns;
    if (lane < n_ns) slot_i0[st * D::TT + lane] = n_i0;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect(bar + st, static_cast<uint32_t>(rows * D::W1 + n_ns * D::S0) * 4);
      if (n_K == 1) tma_load(Ss, Sbuf + static_cast<int64_t>(n_d.start) * D::W1, rows * D::W1 * 4, bar + st);
      misc[2 * st] = n_d.key;
      misc[2 * st + 1] = n_ns;
      misc[8 + st] = n_K;
    }
    __syncwarp();
    if (n_K > 1 && lane < n_K)
      tma_load(Ss + lane * D::W1, Sbuf + static_cast<int64_t>(n_d.start + lane * D::TT) * D::W1, D::W1 * 4,
               bar + st);
    if (lane < n_ns)
      tma_load(G0s + lane * D::S0, G0 + static_cast<int64_t>(n_i0) * D::S0, D::S0 * 4, bar + st);
  };
  // descriptor of the tile after the one being fetched (loaded a tile early,
  // so the dependent slot-i0 load of a fetch never waits on it)
  Tile q_d{};
  int q_ns = 0;
  if (wid == 0) {
    if (!ulen && t_lo + NS < t_hi) {
      q_d = tiles[t_lo + NS];
      q_ns = tile_nslots[t_lo + NS];
    }
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      if (p_K[q] > 0) {
        n_d = p_d[q];
        n_ns = p_ns[q];
        n_i0 = p_i0[q];
        n_K = p_K[q];
        issue(q);
      }
    }
  }
  const int r0 = (tid % GB::TR) * GB::RB, cb0 = (tid / GB::TR) * GB::CB;
  const bool g1_on = tid < GB::TR * GB::TC;
  float acc1[GB::RB][GB::CB];
#pragma unroll
  for (int i = 0; i < GB::RB; ++i)
#pragma unroll
    for (int j = 0; j < GB::CB; ++j) acc1[i][j] = 0.f;
  int run_start = t_lo, cur_i1 = -1;
  __syncthreads();  // the prologue's misc / slot_i0 published
  for (int t = t_lo, u = 0; t < t_hi; ++u) {  // unit u: tiles t .. t + K - 1
    const int st = u % NS;
    const uint32_t parity = static_cast<uint32_t>((u / NS) & 1);
    const float* Ss = sm + st * SM::STAGE;
    const float* G0s = Ss + D::TT * D::W1;
    const int* si0 = slot_i0 + st * D::TT;
    // misc / slot_i0 of stage st were written by issue() at the end of tile
    // t - NS (or in the prologue): every thread has passed tile t - 1's
    // barriers since, so no barrier is needed here.  Stage st + 1's misc
    // (the next tile's key) was written at the end of tile t - 1 and is read
    // after this tile's post-wait barrier.
    const int i1 = misc[2 * st], nslots = misc[2 * st + 1], K = misc[8 + st];
    const int nk = nslots * D::P0;
    if (wid == 0 && nx_t < t_hi) {  // unit u+NS's slot i0s in flight during this unit's GEMMs
      if (ulen) {
        n_K = min(static_cast<int>(ulen[nx_t]), t_hi - nx_t);
        n_d = tiles[nx_t];
        n_ns = tile_nslots[nx_t];
      } else {
        n_d = q_d;
        n_ns = q_ns;
        if (nx_t + 1 < t_hi) {
          q_d = tiles[nx_t + 1];
          q_ns = tile_nslots[nx_t + 1];
        }
      }
      n_i0 = lane < n_ns ? static_cast<int>(tile_i0[n_d.start + lane]) : 0;
    }
#ifdef TTGPU_CTA_TIMES
    note_ns += nslots;
    note_runs += i1 != cur_i1;
#endif
    if (kG1Pre && t == t_lo && i1 == pre_i1) {  // the first tile's G1, loaded in the prologue
#pragma unroll
      for (int u = 0; u < kG1U; ++u) {
        const int e = tid + u * kThreads;
        if (e < D::S1) {
          const int r = e / D::C1, c = e - r * D::C1;
          G1t[c * SM::R1P + r] = g1pre[u];
        }
      }
      cur_i1 = i1;
    } else if (i1 != cur_i1) {  // stage G1[i1] transposed (once per bucket run)
      const float* src = G1 + static_cast<int64_t>(i1) * D::S1;
      constexpr int U = 8;
      for (int e0 = tid; e0 < D::S1; e0 += kThreads * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = e0 + u * kThreads < D::S1 ? __ldg(src + e0 + u * kThreads) : 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kThreads;
          if (e < D::S1) {
            const int r = e / D::C1, c = e - r * D::C1;
            G1t[c * SM::R1P + r] = v[u];
          }
        }
      }
      cur_i1 = i1;
    }
    if (wid == 1 && lane < nslots) {  // D0 first touches of this CTA
      const int i0 = si0[lane];
      const unsigned bit = 1u << (i0 & 31);
      const unsigned old = atomicOr(d0bits + (i0 >> 5), bit);
      d0first[lane] = (old & bit) ? 0 : 1;
      if (!(old & bit)) d0m[i0] = 1;
    }
    mbar_wait(bar + st, parity);
    if (t == t_lo) cta_mark(3, 1);
    __syncthreads();  // G1t staged, d0first set, bulk data visible
    const int nxt_i1 = (t + K < t_hi) ? misc[2 * ((st + 1) % NS)] : -1;
    if (K > 1) {  // merged unit: S row 0 = the sum of its K rows (fixed order), then one-slot GEMMs
      static_assert(kThreads % D::W1 == 0, "merge groups");
      constexpr int NG = kThreads / D::W1;
      float* Sw = const_cast<float*>(Ss);
      const int gq = tid / D::W1, e = tid - gq * D::W1;
      float p = 0.f;
      for (int j = gq; j < K; j += NG) p += Sw[j * D::W1 + e];
      if (gq < K) Sw[gq * D::W1 + e] = p;  // row gq is read by this thread only
      __syncthreads();
      if (gq == 0) {
        for (int q = 1; q < min(NG, K); ++q) p += Sw[q * D::W1 + e];
        Sw[e] = p;
      }
      __syncthreads();
    }
    // ---- dG1 partial += Σ_kappa G0s[kappa][r1] (x) S[kappa][c]
    if (g1_on) {
#pragma unroll 2
      for (int k = 0; k < nk; ++k) {
        float a[GB::RB], b[GB::CB];
        const float* ap = G0s + k * D::R1 + r0;
#pragma unroll
        for (int i = 0; i < GB::RB; ++i) a[i] = ap[i];
#pragma unroll
        for (int j = 0; j < GB::CB; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(Ss + k * D::C1 + cb0 + j);
          b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < GB::RB; ++i)
#pragma unroll
          for (int j = 0; j < GB::CB; j += 2) ffma2(a[i], b[j], b[j + 1], acc1[i][j], acc1[i][j + 1]);
      }
    }
    // ---- D0[kappa][r1] = Σ_c S[kappa][c] · G1[r1][c]; thread = (kappa, RB0 r1)
    constexpr int KPT = kThreads / GB::TR0;  // kappas per pass
    constexpr int NP = (D::P0 * D::TT + KPT - 1) / KPT;
    float dv[NP][GB::RB0];
    int my_i0[NP], my_first[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int k = q * KPT + tid / GB::TR0, rb = (tid % GB::TR0) * GB::RB0;
#pragma unroll
      for (int i = 0; i < GB::RB0; ++i) dv[q][i] = 0.f;
      my_i0[q] = k < nk ? si0[k / D::P0] : 0;
      my_first[q] = k < nk ? d0first[k / D::P0] : 0;
      if (q * KPT < nk && k < nk) {
        const float* srow = Ss + k * D::C1;
#pragma unroll 4
        for (int c = 0; c < D::C1; c += 4) {
          const float4 s4 = *reinterpret_cast<const float4*>(srow + c);
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float* gp = G1t + (c + cc) * SM::R1P + rb;
#pragma unroll
            for (int i = 0; i < GB::RB0; i += 2) ffma2(sv[cc], gp[i], gp[i + 1], dv[q][i], dv[q][i + 1]);
          }
        }
      }
    }
    __syncthreads();  // stage st / slot lists consumed
    if (wid == 0 && nx_t < t_hi) {
      issue(st);
      nx_t += n_K;
    }
    // ---- D0 into the CTA block (slots of one tile have distinct i0)
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int k = q * KPT + tid / GB::TR0, rb = (tid % GB::TR0) * GB::RB0;
      if (k < nk) {
        const int a0 = k % D::P0;
        float* dst = d0acc + my_i0[q] * D::S0 + a0 * D::R1 + rb;
        if (my_first[q]) {
#pragma unroll
          for (int i = 0; i < GB::RB0; ++i) dst[i] = dv[q][i];
        } else {
#pragma unroll
          for (int i = 0; i < GB::RB0; ++i) dst[i] += dv[q][i];
        }
      }
    }
    // ---- end of an i1 run (or of this CTA's range): flush the dG1 partial
    if (tid < K) has1[t + tid] = (t + tid == run_start) ? 1 : 0;
    if (nxt_i1 != i1 || t + K == t_hi) {
      float* dst = part1 + static_cast<int64_t>(run_start) * D::S1;
      if (g1_on) {
#pragma unroll
        for (int i = 0; i < GB::RB; ++i)
#pragma unroll
          for (int j = 0; j < GB::CB; j += 4)
            *reinterpret_cast<float4*>(dst + (r0 + i) * D::C1 + cb0 + j) =
                make_float4(acc1[i][j], acc1[i][j + 1], acc1[i][j + 2], acc1[i][j + 3]);
      }
#pragma unroll
      for (int i = 0; i < GB::RB; ++i)
#pragma unroll
        for (int j = 0; j < GB::CB; ++j) acc1[i][j] = 0.f;
      run_start = t + K;
    }
    t += K;
  }
  cta_mark(3, 2);
  cta_note(3, static_cast<unsigned long long>(t_hi - t_lo) | (note_ns << 16) | (note_runs << 40));
}

// ------------------------------------------------------------ f3_bwd2 ----
// Per i2-tile (<= TT2 lookups with the same i2): dG2 contribution
// Σ_l H(l)ᵀ (R2 x P1) · D2_l (P1 x N2).  4 warps split the lookups
// (l = w, w+4, ...), 4 lookups' loads in flight per warp; lanes own rank
// columns (float4 over j2); warp sums are folded in warp order.  Consecutive
// tiles of the same i2 in a CTA's range accumulate; one partial per run
// (has2 marks its first tile).
template <class D>
__device__ __forceinline__ void bwd2_body(
    int vblock, int vgrid, Geo g, const Tile* __restrict__ tiles, const int* __restrict__ ntiles,
    const uint32_t* __restrict__ perm, const uint32_t* __restrict__ hloc,
    const int32_t* __restrict__ lk_bag, const float* __restrict__ alpha,
    const float* __restrict__ grad, const float* __restrict__ Hbuf, float* __restrict__ part2,
    int* __restrict__ has2) {
  constexpr int NW = 4, U = 4;
  constexpr int CH = (D::R2 + 31) / 32;
  __shared__ float4 red[NW][CH * 32];
  __shared__ int hl[D::TT2], bg[D::TT2];
  __shared__ float al[D::TT2];
  const int nt = *ntiles;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int t_lo = static_cast<int>(static_cast<int64_t>(vblock) * nt / vgrid);
  const int t_hi = static_cast<int>(static_cast<int64_t>(vblock + 1) * nt / vgrid);
  float4 acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
  int run_start = t_lo;
  // the next tile's descriptor (loaded during this tile) and its lookups
  // (loaded after this tile's loads): only the last hop is exposed per tile
  Tile nx{};
  int nl = 0;
  for (int t = t_lo; t < t_hi; ++t) {
    const Tile tl = t == t_lo ? tiles[t] : nx;
    const int ntl = tl.end - tl.start;
    if (tid < ntl) {
      const int l = t == t_lo ? static_cast<int>(perm[tl.start + tid]) : nl;
      hl[tid] = static_cast<int>(hloc[l]);
      bg[tid] = lk_bag[l];
      al[tid] = alpha[l];
    }
    if (t + 1 < t_hi) nx = tiles[t + 1];
    __syncthreads();
    for (int i0 = wid * U; i0 < ntl; i0 += NW * U) {
      float4 d[U][D::P1];
      float h[U][CH][D::P1];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u;
        if (i < ntl) {
          const float4* grow = reinterpret_cast<const float4*>(grad + static_cast<int64_t>(bg[i]) * D::N);
          const float* hrow = Hbuf + static_cast<int64_t>(hl[i]) * D::W1;
#pragma unroll
          for (int a = 0; a < D::P1; ++a) d[u][a] = __ldg(grow + a);
#pragma unroll
          for (int c = 0; c < CH; ++c)
#pragma unroll
            for (int a = 0; a < D::P1; ++a)
              h[u][c][a] = (c * 32 + lane < D::R2) ? __ldg(hrow + a * D::R2 + c * 32 + lane) : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + u;
        if (i < ntl) {
          const float a0 = al[i];
#pragma unroll
          for (int a = 0; a < D::P1; ++a) {
            const float2 d01 = fmul2_rn(a0, make_float2(d[u][a].x, d[u][a].y));
            const float2 d23 = fmul2_rn(a0, make_float2(d[u][a].z, d[u][a].w));
            const float4 dv = make_float4(d01.x, d01.y, d23.x, d23.y);
#pragma unroll
            for (int c = 0; c < CH; ++c) {
              ffma2(h[u][c][a], dv.x, dv.y, acc[c].x, acc[c].y);
              ffma2(h[u][c][a], dv.z, dv.w, acc[c].z, acc[c].w);
            }
          }
        }
      }
    }
    if (t + 1 < t_hi && tid < nx.end - nx.start) nl = static_cast<int>(perm[nx.start + tid]);
    const bool last = (t + 1 == t_hi) || (nx.key != tl.key);
    if (tid == 0) has2[t] = (t == run_start) ? 1 : 0;
    if (last) {
#pragma unroll
      for (int c = 0; c < CH; ++c) red[wid][c * 32 + lane] = acc[c];
      __syncthreads();
      if (wid == 0) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
          const int r = c * 32 + lane;
          float4 s = red[0][c * 32 + lane];
          for (int w = 1; w < NW; ++w) add4(s, red[w][c * 32 + lane]);
          if (r < D::R2)
            reinterpret_cast<float4*>(part2 + static_cast<int64_t>(run_start) * D::S2)[r] = s;
        }
      }
#pragma unroll
      for (int c = 0; c < CH; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      run_start = t + 1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------- f3_combine ---
// Fixed-order list reductions, one WARP per (output slice, 128-column
// chunk) task: the warp scans its candidates 32 at a time, ballots the live
// ones and sums their rows 4 loads at a time (lanes own float4 columns).
// No block barriers.  Task ranges:
//   [0, m1*C1c)      dG1[i1]   candidates: i1-tiles of bucket i1 (has1), KG rows each
//   [.., + m2*C2c)   dG2[i2]   candidates: i2-tiles of bucket i2 (has2)
//   [.., + m0*C0c)   dG0[i0]   candidates: f3_bwd1 CTAs (d0mask)
// MODE 0 writes dense gradients (zeros if untouched), 1 applies SGD in place.
template <class RowFn>
__device__ __forceinline__ void sum_live(unsigned live, int cand0, int col4, bool colok, RowFn row_of,
                                         float4& acc) {
  while (live) {
    int idx[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      idx[u] = -1;
      if (live) {
        idx[u] = cand0 + __ffs(live) - 1;
        live &= live - 1;
      }
    }
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      v[u] = (idx[u] >= 0 && colok) ? __ldcg(reinterpret_cast<const float4*>(row_of(idx[u])) + col4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (idx[u] >= 0) add4(acc, v[u]);
  }
}

// ---- kernel wrappers of the two independent backward stages, and their
// horizontal fusion: f3_srows (per i1-tile) and f3_bwd2 (per i2-tile) read
// only the forward's outputs and grad_out, so one launch runs both -- the first
// nb2 CTAs as f3_bwd2, the rest as f3_srows warps -- and their tails overlap.
template <class D>
__global__ void __launch_bounds__(256, 2) f3_srows(const float* __restrict__ cores, int64_t coff2,
                                                const Tile* __restrict__ tiles,
                                                const int* __restrict__ ntiles, int max_tiles,
                                                const uint32_t* __restrict__ perm,
                                                const uint16_t* __restrict__ d2,
                                                const int32_t* __restrict__ lk_bag,
                                                const float* __restrict__ alpha,
                                                const float* __restrict__ grad,
                                                const uint16_t* __restrict__ slot_of_pos,
                                                const int* __restrict__ tile_nslots,
                                                float* __restrict__ Sbuf) {
  pdl_entry();
  srows_body<D>(blockIdx.x, gridDim.x, cores, coff2, tiles, ntiles, max_tiles, perm, d2, lk_bag, alpha,
                grad, slot_of_pos, tile_nslots, Sbuf);
}

template <class D>
__global__ void __launch_bounds__(128) f3_bwd2(
    Geo g, const Tile* __restrict__ tiles, const int* __restrict__ ntiles,
    const uint32_t* __restrict__ perm, const uint32_t* __restrict__ hloc,
    const int32_t* __restrict__ lk_bag, const float* __restrict__ alpha,
    const float* __restrict__ grad, const float* __restrict__ Hbuf, float* __restrict__ part2,
    int* __restrict__ has2) {
  pdl_entry();
  bwd2_body<D>(blockIdx.x, gridDim.x, g, tiles, ntiles, perm, hloc, lk_bag, alpha, grad, Hbuf, part2,
               has2);
}

struct SrowsArgs {
  const float* cores;
  int64_t coff2;
  const Tile* tiles;
  const int* ntiles;
  int max_tiles;
  const uint32_t* perm;
  const uint16_t* d2;
  const uint16_t* slot_of_pos;
  const int* tile_nslots;
  float* Sbuf;
  int* b1range;  // f3_bwd1's tile ranges, planned by CTA 0 (nullptr: bwd1 plans itself)
  int b1grid;
  const uint4* rec;  // sorted key-1 records (nullptr: through perm / d2 / lk_bag / alpha)
  uint8_t* b1ulen;   // f3_bwd1 merge units planned with the ranges (nullptr: one tile per unit)
  const int* tile_one;  // (i1 << 16 | i0) of one-slot tiles, else -1 (f3_fwd)
  int b1tile, b1cont;   // merge-unit range weights: a tile b1tile + nslots, a continuing tile b1cont
};
struct Bwd2Args {
  const Tile* tiles;
  const int* ntiles;
  const uint32_t* perm;
  const uint32_t* hloc;
  const float* Hbuf;
  float* part2;
  int* has2;
};

// f3_bwd1's contiguous tile ranges, balanced by weight kBwd1TileCost + nslots
// (tile t belongs to CTA b iff its exclusive weight prefix E(t) lies in
// [ceil(bW/G), ceil((b+1)W/G))): range[b] = first tile with E >= ceil(bW/G),
// range[G] = nt.  One 128-thread CTA; each thread walks its chunk of tiles
// once for every threshold that falls inside it.  Same partition as the
// in-kernel planning of bwd1_body (used when no plan is given) unless ulen
// is given:
//
// Merge units (ulen != nullptr).  Under Zipf most i1-tiles of a hot (i0, i1)
// pair hold that single slot (cfg2: 939 of 2,157 tiles are pair (0, 0)), and
// f3_bwd1 pays its per-tile pipeline (bulk copies, barriers, the D0
// read-modify-write) for each.  By linearity their GEMMs can run once on the
// sum of their S rows: tile t CONTINUES tile t - 1 when both hold one slot of
// the same i1 and i0 (bwd1 copies the K S rows of a unit one by one: a
// tile's rows start at its first lookup position).  A run of continuing
// tiles is cut into units of <= kCap tiles (counted from the run's first
// tile); ulen[t] = tiles from t to the end of its unit, so a CTA whose range
// starts inside a unit starts a shorter one there.  A continuing tile weighs
// wcont (default kBwd1ContCost) instead of wtile + 1 (default kBwd1TileCost + 1).
constexpr int kBwd1ContCost = 1;

template <int kCap>
__device__ __forceinline__ void plan_bwd1(const int* __restrict__ ntiles,
                                          const int* __restrict__ tile_nslots, int* __restrict__ range,
                                          int G, const int* __restrict__ tile_one,
                                          uint8_t* __restrict__ ulen, int wtile, int wcont) {
  using Scan = cub::BlockScan<int, 128>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int run_first[128], run_last[128];
  const int nt = *ntiles;
  const int tid = threadIdx.x;
  const int per = (nt + 127) / 128;
  const int a0 = min(nt, tid * per), a1 = min(nt, a0 + per);
  constexpr int kPer = 32;
  const bool merge = ulen != nullptr && per <= kPer;
  int wv[kPer];
  int wsum = 0;
  unsigned cont = 0;  // bit j: tile a0 + j continues tile a0 + j - 1
  if (merge) {
    // tile_one: (i1 << 16 | i0) of a one-slot tile, else -1; all loads of a
    // batch of 16 tiles (and tile a0 - 1) in one round trip
    int prev = a0 > 0 && a0 < a1 ? tile_one[a0 - 1] : -1;
#pragma unroll
    for (int b0 = 0; b0 < kPer; b0 += 16) {
      int ns[16], on[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = a0 + b0 + j;
        ns[j] = t < a1 ? tile_nslots[t] : 0;
        on[j] = t < a1 ? tile_one[t] : -1;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int jj = b0 + j;
        const bool c = on[j] >= 0 && on[j] == prev;
        if (c) cont |= 1u << jj;
        wv[jj] = a0 + jj < a1 ? (c ? wcont : wtile + ns[j]) : 0;
        prev = on[j];
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < kPer; ++j) wv[j] = a0 + j < a1 ? kBwd1TileCost + tile_nslots[a0 + j] : 0;
  }
#pragma unroll
  for (int j = 0; j < kPer; ++j) wsum += wv[j];
  if (per > kPer)
    for (int t = a0 + kPer; t < a1; ++t) wsum += kBwd1TileCost + tile_nslots[t];
  int ex, W;
  Scan(scan_tmp).ExclusiveSum(wsum, ex, W);
  if (tid == 0) {
    range[0] = 0;
    range[G] = nt;
  }
  if (W == 0) {
    for (int b = tid + 1; b < G; b += 128) range[b] = nt;
  } else {
    // thresholds th_b = ceil(b W / G) with ex < th_b <= ex + wsum (b in 1 .. G-1)
    const int64_t Wl = W, Gl = G;
    int64_t b = static_cast<int64_t>(ex) * Gl / Wl + 1;
    const int64_t b_end = min(Gl - 1, (static_cast<int64_t>(ex) + wsum) * Gl / Wl);
    int64_t e = ex;
    int t = a0, j = 0;
    // With merge units the boundary is placed by tile MIDPOINTS (a tile goes
    // to the CTA holding E(t) + w(t)/2): once the hot one-slot runs are cheap,
    // the big multi-slot tiles set the longest CTA, and the first-tile rule
    // lets one overshoot its CTA's share by up to a whole tile weight.
    const bool mid = ulen != nullptr;
    for (; b <= b_end; ++b) {
      const int64_t th = (b * Wl + Gl - 1) / Gl;
      while (t < a1) {
        const int w = j < kPer ? wv[j] : kBwd1TileCost + tile_nslots[t];
        if (mid ? 2 * e + w >= 2 * th : e >= th) break;
        e += w;
        ++t;
        ++j;
      }
      range[b] = t;
    }
  }
  if (ulen == nullptr) return;
  // unit lengths: a tile's run starts at the last non-continuing tile <= t and
  // ends before the first non-continuing tile > t (searched across chunks)
  const int n = a1 - a0;
  const unsigned live = n >= 32 ? 0xffffffffu : ((1u << n) - 1u);
  const unsigned starts = merge ? (~cont & live) : live;  // non-continuing tiles of the chunk
  run_last[tid] = starts ? a0 + 31 - __clz(starts) : -1;
  run_first[tid] = starts ? a0 + __ffs(starts) - 1 : INT_MAX;
  __syncthreads();
  if (!merge) {
    for (int t = a0; t < a1; ++t) ulen[t] = 1;
    return;
  }
  int rs = -1;  // run start carried into the chunk
  for (int q = tid - 1; q >= 0 && rs < 0; --q) rs = run_last[q];
  int re_after = nt;  // first run start after the chunk
  for (int q = tid + 1; q < 128 && re_after == nt; ++q)
    if (run_first[q] != INT_MAX) re_after = run_first[q];
  for (int j = 0; j < n; ++j) {
    const int t = a0 + j;
    if (!((cont >> j) & 1u)) rs = t;
    const unsigned later = j + 1 < 32 ? (starts >> (j + 1)) : 0u;
    const int re = later ? t + __ffs(later) : re_after;
    const int ce = rs + kCap * ((t - rs) / kCap + 1);
    ulen[t] = static_cast<uint8_t>(min(ce, re) - t);
  }
}

// CTA roles interleave (even: f3_bwd2 CTA, odd: 4 f3_srows warps) while both
// have work left, so both stages spread over every SM from the first wave.
// With sa.b1range, the grid's first CTA plans f3_bwd1's tile ranges instead.
template <class D>
__global__ void __launch_bounds__(128, 4) f3_srows_bwd2(Geo g, SrowsArgs sa, Bwd2Args ba, int nb2, int nbs,
                                                    const int32_t* __restrict__ lk_bag,
                                                    const float* __restrict__ alpha,
                                                    const float* __restrict__ grad) {
  CtaClock clk_(2);
  pdl_entry();
  int b = static_cast<int>(blockIdx.x);
  if (sa.b1range) {  // CTA 0 (first wave) plans f3_bwd1; the roles start at CTA 1
    if (b == 0) {
      plan_bwd1<D::TT>(sa.ntiles, sa.tile_nslots, sa.b1range, sa.b1grid, sa.tile_one, sa.b1ulen, sa.b1tile,
                       sa.b1cont);
      return;
    }
    --b;
  }
  const int m = min(nb2, nbs);
  bool is_b2;
  int idx;
  if (b < 2 * m) {
    is_b2 = (b & 1) == 0;
    idx = b >> 1;
  } else {
    is_b2 = nb2 > nbs;
    idx = m + (b - 2 * m);
  }
  if (is_b2)
    bwd2_body<D>(idx, nb2, g, ba.tiles, ba.ntiles, ba.perm, ba.hloc, lk_bag, alpha, grad, ba.Hbuf,
                 ba.part2, ba.has2);
  else
    srows_body<D>(idx, nbs, sa.cores, sa.coff2, sa.tiles, sa.ntiles, sa.max_tiles, sa.perm, sa.d2, lk_bag,
                  alpha, grad, sa.slot_of_pos, sa.tile_nslots, sa.Sbuf, sa.rec);
}

__device__ __forceinline__ void store_slice(float4 s, bool touched, float* out_core, float* out_grad,
                                            int col4, bool colok, int mode, float lr) {
  if (!colok) return;
  if (mode == 0) {
    reinterpret_cast<float4*>(out_grad)[col4] = s;
  } else if (touched) {
    float4 c = reinterpret_cast<float4*>(out_core)[col4];
    c.x = __fadd_rn(c.x, -__fmul_rn(lr, s.x));
    c.y = __fadd_rn(c.y, -__fmul_rn(lr, s.y));
    c.z = __fadd_rn(c.z, -__fmul_rn(lr, s.z));
    c.w = __fadd_rn(c.w, -__fmul_rn(lr, s.w));
    reinterpret_cast<float4*>(out_core)[col4] = c;
  }
}

struct CombineArgs {
  const int32_t *tile_base1, *tile_base2, *group_base1, *group_base2;
  const float *part1, *part2, *D0acc;
  const int *has1, *has2;
  const unsigned char* d0mask;
  float* gpart;        // one 128-column chunk per warp task
  int* gtouch;         // per warp task
  int* counters;       // per (slice, chunk); zero between launches
  int maxg1, maxg2, nbwd;
};

// Warp task (role, slice, group, chunk).  A slice's candidate list is cut into
// groups of <= kGroup; each group is summed by its own warp.  Single-group
// slices are applied directly; otherwise the last warp to finish (atomic
// counter) folds the group partials in group order -- deterministic.
template <int W>
__device__ __forceinline__ void finish_task(float4 acc, bool touched, int task_first, int ng, int gi,
                                            int ch, int nch, int* counter, const CombineArgs& A,
                                            float* core, float* grad, int mode, float lr) {
  const int lane = threadIdx.x & 31;
  const int col4 = ch * 32 + lane;
  const bool colok = col4 < W / 4;
  if (ng == 1) {
    store_slice(acc, touched, core, grad, col4, colok, mode, lr);
    return;
  }
  const int task = task_first + gi * nch + ch;
  reinterpret_cast<float4*>(A.gpart + static_cast<int64_t>(task) * 128)[lane] = acc;
  if (lane == 0) A.gtouch[task] = touched ? 1 : 0;
  __threadfence();
  int prev = 0;
  if (lane == 0) prev = atomicAdd(counter, 1);
  prev = __shfl_sync(0xffffffffu, prev, 0);
  if (prev != ng - 1) return;
  __threadfence();
  float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
  bool any = false;
  // 8 group partials in flight per round, added in group order
  for (int q0 = 0; q0 < ng; q0 += 8) {
    float4 v[8];
    int tch[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int tq = task_first + (q0 + u) * nch + ch;
      const bool ok = q0 + u < ng;
      v[u] = ok ? __ldcg(reinterpret_cast<const float4*>(A.gpart + static_cast<int64_t>(tq) * 128) + lane)
                : make_float4(0.f, 0.f, 0.f, 0.f);
      tch[u] = ok ? __ldcg(A.gtouch + tq) : 0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (q0 + u < ng) add4(sum, v[u]);
      any |= tch[u] != 0;
    }
  }
  store_slice(sum, any, core, grad, col4, colok, mode, lr);
  if (lane == 0) *counter = 0;  // ready for the next launch
}

__device__ __forceinline__ int find_slice(const int32_t* base, int K, int x) {
  int lo = 0, hi = K;  // base[lo] <= x < base[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (base[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// One combine warp task (task = slice group x 128-column chunk of dG1, dG2 or
// dG0).  gb1 / gb2: the group bases of both keys (shared memory copies).
template <class D>
__device__ __forceinline__ void combine_task(int task, const int* gb1, const int* gb2, Geo g,
                                             float* __restrict__ cores, float* __restrict__ grads,
                                             const CombineArgs& A, float lr, int MODE) {
  const int lane = threadIdx.x & 31;
  constexpr int C1c = (D::S1 + 127) / 128, C2c = (D::S2 + 127) / 128, C0c = (D::S0 + 127) / 128;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool touched = false;
  if (task < A.maxg1 * C1c) {
    const int gidx = task / C1c, ch = task - gidx * C1c;
    if (gidx >= gb1[g.m1]) return;
    const int i1 = find_slice(gb1, g.m1, gidx);
    const int gfirst = gb1[i1], ng = gb1[i1 + 1] - gfirst, gi = gidx - gfirst;
    const int col4 = ch * 32 + lane;
    const bool colok = col4 < D::S1 / 4;
    auto row = [&](int t) { return A.part1 + static_cast<int64_t>(t) * D::S1; };
    const int t0 = A.tile_base1[i1] + gi * kGroup;
    const int t1 = min(A.tile_base1[i1 + 1], t0 + kGroup);
    for (int c0 = t0; c0 < t1; c0 += 32) {
      const int t = c0 + lane;
      const unsigned live = __ballot_sync(0xffffffffu, t < t1 && A.has1[t] != 0);
      touched |= live != 0;
      sum_live(live, c0, col4, colok, row, acc);
    }
    finish_task<D::S1>(acc, touched, gfirst * C1c, ng, gi, ch, C1c, A.counters + i1 * C1c + ch, A,
                       cores + g.coff1 + static_cast<int64_t>(i1) * D::S1,
                       grads + g.coff1 + static_cast<int64_t>(i1) * D::S1, MODE, lr);
    return;
  }
  task -= A.maxg1 * C1c;
  if (task < A.maxg2 * C2c) {
    const int gidx = task / C2c, ch = task - gidx * C2c;
    if (gidx >= gb2[g.m2]) return;
    const int i2 = find_slice(gb2, g.m2, gidx);
    const int gfirst = gb2[i2], ng = gb2[i2 + 1] - gfirst, gi = gidx - gfirst;
    const int col4 = ch * 32 + lane;
    const bool colok = col4 < D::S2 / 4;
    auto row = [&](int t) { return A.part2 + static_cast<int64_t>(t) * D::S2; };
    const int t0 = A.tile_base2[i2] + gi * kGroup;
    const int t1 = min(A.tile_base2[i2 + 1], t0 + kGroup);
    for (int c0 = t0; c0 < t1; c0 += 32) {
      const int t = c0 + lane;
      const unsigned live = __ballot_sync(0xffffffffu, t < t1 && A.has2[t] != 0);
      touched |= live != 0;
      sum_live(live, c0, col4, colok, row, acc);
    }
    finish_task<D::S2>(acc, touched, A.maxg1 * C1c + gfirst * C2c, ng, gi, ch, C2c,
                       A.counters + g.m1 * C1c + i2 * C2c + ch, A,
                       cores + g.coff2 + static_cast<int64_t>(i2) * D::S2,
                       grads + g.coff2 + static_cast<int64_t>(i2) * D::S2, MODE, lr);
    return;
  }
  task -= A.maxg2 * C2c;
  const int ng0 = (A.nbwd + kGroup0 - 1) / kGroup0;
  const int gidx = task / C0c, ch = task - gidx * C0c;
  if (gidx >= g.m0 * ng0) return;
  const int i0 = gidx / ng0, gi = gidx - i0 * ng0;
  const int col4 = ch * 32 + lane;
  const bool colok = col4 < D::S0 / 4;
  auto row = [&](int c) { return A.D0acc + (static_cast<int64_t>(c) * g.m0 + i0) * D::S0; };
  const int c0 = gi * kGroup0, c1 = min(A.nbwd, c0 + kGroup0);
  {
    const int c = c0 + lane;
    const unsigned live =
        __ballot_sync(0xffffffffu, c < c1 && A.d0mask[static_cast<int64_t>(c) * g.m0 + i0] != 0);
    touched |= live != 0;
    sum_live(live, c0, col4, colok, row, acc);
  }
  finish_task<D::S0>(acc, touched, A.maxg1 * C1c + A.maxg2 * C2c + i0 * ng0 * C0c, ng0, gi, ch, C0c,
                     A.counters + g.m1 * C1c + g.m2 * C2c + i0 * C0c + ch, A,
                     cores + g.coff0 + static_cast<int64_t>(i0) * D::S0,
                     grads + g.coff0 + static_cast<int64_t>(i0) * D::S0, MODE, lr);
}

template <class D>
__global__ void __launch_bounds__(kThreads, D::R1 <= 32 ? 3 : 1) f3_bwd1(
    Geo g, const float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const float* __restrict__ Sbuf,
    const uint16_t* __restrict__ tile_i0, const int* __restrict__ tile_nslots,
    float* __restrict__ part1, int* __restrict__ has1, float* __restrict__ D0acc,
    unsigned char* __restrict__ d0mask, const int* __restrict__ plan, const uint8_t* __restrict__ ulen) {
  CtaClock clk_(3);
  pdl_entry();
  bwd1_body<D>(g, cores, tiles, ntiles, Sbuf, tile_i0, tile_nslots, part1, has1, D0acc, d0mask, plan, ulen);
}

// f3_bwd1 and f3_combine in ONE cooperative launch (the bwd1 grid is exactly
// the co-resident CTAs): after its tiles every CTA meets a grid barrier, then
// its warps take the combine tasks (grid-stride).  Saves the combine launch
// and its ramp; the combine's partial loads are L2-coherent (__ldcg).
template <class D>
__global__ void __launch_bounds__(kThreads, D::R1 <= 32 ? 3 : 1) f3_bwd1_comb(
    Geo g, float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const float* __restrict__ Sbuf,
    const uint16_t* __restrict__ tile_i0, const int* __restrict__ tile_nslots,
    float* __restrict__ part1, int* __restrict__ has1, float* __restrict__ D0acc,
    unsigned char* __restrict__ d0mask, float* __restrict__ grads, CombineArgs A, float lr, int mode,
    int ntasks) {
  pdl_entry();
  bwd1_body<D>(g, cores, tiles, ntiles, Sbuf, tile_i0, tile_nslots, part1, has1, D0acc, d0mask);
  cooperative_groups::this_grid().sync();
  extern __shared__ __align__(128) float sm[];
  int* gb1 = reinterpret_cast<int*>(sm);
  int* gb2 = gb1 + g.m1 + 1;
  for (int e = threadIdx.x; e < g.m1 + 1; e += blockDim.x) gb1[e] = __ldcg(A.group_base1 + e);
  for (int e = threadIdx.x; e < g.m2 + 1; e += blockDim.x) gb2[e] = __ldcg(A.group_base2 + e);
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int task = blockIdx.x * nw + (threadIdx.x >> 5); task < ntasks; task += gridDim.x * nw)
    combine_task<D>(task, gb1, gb2, g, cores, grads, A, lr, mode);
}

template <class D, int MODE>
__global__ void __launch_bounds__(kThreads, 6) f3_combine(Geo g, float* __restrict__ cores,
                                                       float* __restrict__ grads, CombineArgs A,
                                                       float lr) {
  CtaClock clk_(4);
  pdl_entry();
  // the group bases of both keys in shared memory: a warp's slice lookup is a
  // binary search there instead of ~8 dependent global loads
  extern __shared__ int cb_sm[];
  int* gb1 = cb_sm;
  int* gb2 = cb_sm + g.m1 + 1;
  for (int e = threadIdx.x; e < g.m1 + 1; e += blockDim.x) gb1[e] = A.group_base1[e];
  for (int e = threadIdx.x; e < g.m2 + 1; e += blockDim.x) gb2[e] = A.group_base2[e];
  __syncthreads();
  cta_mark(4, 0);
  combine_task<D>((blockIdx.x * blockDim.x + threadIdx.x) >> 5, gb1, gb2, g, cores, grads, A, lr, MODE);
}

}  // namespace f3
}  // namespace ttgpu
#include "gsort.cuh"
#include "fastc.cuh"
