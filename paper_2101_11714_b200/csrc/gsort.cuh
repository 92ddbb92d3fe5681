// One-kernel two-key stable counting sort for the 3-core fast path (replaces
// f3_hist + f3_scan + f3_scatter when the batch fits one co-resident grid).
//
// A cooperative grid of G <= #SMs CTAs x 512 threads; CTA c owns the lookups
// [c*16*PW, (c+1)*16*PW), warp w of it a run of PW consecutive lookups walked
// 32 at a time, so (CTA, warp, round, lane) is lookup order.  Phases:
//   A  decode + range check (d2 digits), per-warp key counts (match_any
//      leaders, warp-private smem counters); the CTA's count of every key
//      into hist[k][c] (key-major); bags: offsets checks, lookup->bag, alpha,
//      solo flags, pooling counters zeroed, empty bags' rows zeroed
//   -- grid barrier --
//   B1 one warp per key (keys spread over the grid): exclusive scan of the
//      key's G CTA counts in place, key total into tot[k]
//   -- grid barrier --
//   B2 every CTA scans the K key totals (lookups, tiles, combine groups) into
//      the bucket / tile / group bases (CTA 0 publishes them, every CTA
//      writes its share of the tile lists) and adds its own CTA prefix
//   C  stable scatter of both keys from the per-warp starts, plus the sorted
//      (lookup, i0 | i2 << 16, bag | solo, alpha) records of key 1 (make_rec)
// Keys and digits stay in registers between A and C; no memsets, so the
// kernel replays from a CUDA graph.  Outputs are
// exactly those of f3_hist + f3_scan + f3_scatter, so the kernels after the
// sort are unchanged.  Reference semantics: decompose_row
// (embedding_ops.hpp:98-108), offsets checks (index_batch.hpp:33-55),
// backward alpha (embedding_ops.hpp:283-296).
#pragma once

#include <cooperative_groups.h>

#include "lfu_cache.cuh"

namespace ttgpu {
namespace f3 {

constexpr int kGsThreads = 512;
constexpr int kGsWarps = kGsThreads / 32;
constexpr int kGsMaxRounds = 8;  // lookups per thread (PW <= 256)
constexpr int kGsMaxGridChunks = 5;  // G <= 160 CTAs

struct GsortArgs {
  Geo g;
  const int64_t* idx;
  int64_t L;
  const int64_t* off;
  int64_t B;
  const double* w;
  int mean;
  int PW;  // lookups per warp, multiple of 32, <= 32 * kGsMaxRounds
  int TT1, TT2;
  double inv_m12, inv_m2;  // 1 / m12, 1 / m2 (decode by multiply + correction)
  uint16_t* d2;
  int32_t* lk_bag;
  float* alpha;
  int32_t* solo;
  uint32_t* hist;  // [K][G] CTA counts -> exclusive CTA prefixes
  uint32_t* tot;   // [K] key totals
  uint32_t* perm1;
  uint32_t* perm2;
  uint4* rec1;
  Tile* tiles1;
  Tile* tiles2;
  int32_t *tile_base1, *tile_base2, *group_base1, *group_base2;
  int* ntiles;
  unsigned long long* bad;
  int* errs;
  float* out;    // pooled rows: empty bags are written here (zeros)
  int N;         // embedding dim
  int* bag_cnt;  // [B] pooling counters (pool_if_last), zeroed here
  // LFU cache consulted before decompression (cache mode; K3 == 0 and
  // counts == nullptr: no cache).  record_and_partition (lfu_cache.hpp:187-219)
  // happens here: every valid lookup counts its row, an Active cache's hash is
  // probed, and a hit becomes a key-3 (slot) record instead of a TT lookup.
  int K3;                            // cache capacity (key-3 buckets); 0 = no cache
  unsigned long long* counts;        // [rows] frequencies (record), or nullptr
  const unsigned long long* hkeys;   // residency hash (lfu_cache.cuh probe)
  const int* hvals;
  int hshift;
  unsigned long long hmask;
  int active;                        // probe the hash (CacheState::Active)
  unsigned long long* hits;          // += hits of this batch
  unsigned long long* hits2;         // += hits (the chain rows not computed: EmbeddingStats)
  unsigned long long* accesses;      // += L (Active accesses), or nullptr
  const int64_t* slot_rows;          // [K3] row of each slot (frequency of cached rows)
  int* lk_slot;                      // [L] slot of a cached lookup, -1 for the chain
  uint32_t* perm3;                   // cached lookups, stable by slot
  int* skey3;                        // their slots
  int* seg_lo3;                      // [K3] first sorted position of a slot, -1 if none
  int* seg_hi3;                      // [K3] one past the last
  int* ncached;                      // [1] cached lookups in the batch
  const float* store;                // [K3][N] cached rows (single-lookup bags pooled here)
  int pool_mean;                     // the batch's Mean pooling (cache mode: all-cached bags)
  int parts;                         // pool_if_last tasks per lookup (f3_fwd: P1)
};

// dynamic shared memory: wc[16][K] | ctot[K] | base[K] | gb1 tb1 [K1+1] | gb2 tb2 [K2+1]
// (K = K1 + K2 + K3; key 3 = cache slots)
__host__ __device__ constexpr size_t gsort_smem_bytes(int K1, int K2, int K3 = 0) {
  return 4 * (static_cast<size_t>(kGsWarps + 2) * (K1 + K2 + K3) + 2 * (K1 + 1) + 2 * (K2 + 1));
}

// largest i in [0, n) with a[i] <= x (a ascending, a[0] <= x)
__device__ __forceinline__ int upper_slot(const uint32_t* a, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// q = x / d, r = x % d for x, d < 2^32 (inv = 1.0 / d): the double product is
// within one of the quotient; one correction step makes it exact.
__device__ __forceinline__ uint32_t div_fix(uint32_t x, uint32_t d, double inv, uint32_t& r) {
  uint32_t q = static_cast<uint32_t>(static_cast<double>(x) * inv);
  int64_t rr = static_cast<int64_t>(x) - static_cast<int64_t>(q) * d;
  if (rr < 0) {
    --q;
    rr += d;
  } else if (rr >= d) {
    ++q;
    rr -= d;
  }
  r = static_cast<uint32_t>(rr);
  return q;
}

// RMAX: rounds (lookups per thread) compiled in -- the host picks the smallest
// power of two >= the batch's rounds, so a one-round batch (cfg2) runs a
// kernel without the unrolled code of eight (instruction-cache pressure);
// kCache: the LFU cache code (key 3) compiled in only where a cache is used
template <int RMAX, bool kCache>
__global__ void __launch_bounds__(kGsThreads, 1) f3_gsort(GsortArgs a) {
  CtaClock clk_(0);
  constexpr int QC = RMAX < 4 ? RMAX : 4;  // rounds whose index loads are batched
  namespace cg = cooperative_groups;
  const int c = blockIdx.x, G = gridDim.x;
  const int K1 = a.g.m1, K2 = a.g.m2, K12 = K1 + K2, K3 = kCache ? a.K3 : 0, K = K12 + K3;
  extern __shared__ __align__(16) uint32_t gs_sm[];
  uint32_t* wc = gs_sm;                  // [16][K] per-warp counts -> per-warp starts
  uint32_t* ctot = wc + kGsWarps * K;    // [K] this CTA's count per key
  uint32_t* base = ctot + K;             // [K] this CTA's absolute start per key
  uint32_t* gb1 = base + K;              // [K1+1] bucket starts, key 1
  uint32_t* tb1 = gb1 + K1 + 1;          // [K1+1] tile starts, key 1
  uint32_t* gb2 = tb1 + K1 + 1;          // [K2+1]
  uint32_t* tb2 = gb2 + K2 + 1;          // [K2+1]
  __shared__ uint32_t wsum[32][3];
  __shared__ uint32_t k1tot[3];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int R = a.PW >> 5;
  const int64_t wbase = (static_cast<int64_t>(c) * kGsWarps + wid) * a.PW;

  // ---- phase A: keys (loads of 4 rounds in flight), counts, bags
  // this thread's first bag's offsets: in flight during the key phase
  const int64_t b_first = static_cast<int64_t>(c) * kGsThreads + tid;
  int64_t s_first = 0, e_first = 0;
  if (b_first < a.B) {
    s_first = a.off[b_first];
    e_first = a.off[b_first + 1];
  }
  for (int i = tid; i < kGsWarps * K; i += kGsThreads) wc[i] = 0u;
  // per round: k1 = i1 (0xffffffff: no lookup), d02 = i0 | i2 << 16
  // cached lookups: k1 = 0x80000000 | slot
  uint32_t k1[RMAX], d02[RMAX];
  uint32_t* mywc = wc + wid * K;
  unsigned my_hits = 0;
  __shared__ unsigned cta_hits;
  if (tid == 0) cta_hits = 0u;
#pragma unroll
  for (int q0 = 0; q0 < RMAX; q0 += QC) {
    int64_t rows[QC];
#pragma unroll
    for (int u = 0; u < QC; ++u) {
      const int64_t l = wbase + (q0 + u) * 32 + lane;
      rows[u] = (q0 + u < R && l < a.L) ? a.idx[l] : 0;
    }
    if (q0 == 0) __syncthreads();  // counters zeroed
#pragma unroll
    for (int u = 0; u < QC; ++u) {
      const int q = q0 + u;
      k1[q] = 0xffffffffu;
      d02[q] = 0u;
      if (q < R) {  // warp-uniform
        const int64_t l = wbase + q * 32 + lane;
        const bool in = l < a.L;
        int64_t row = rows[u];
        bool ok = in;
        if (in && (row < 0 || row >= a.g.num_rows)) {
          atomicMin(a.bad, static_cast<unsigned long long>(l));
          ok = false;
        }
        if (!ok) row = 0;
        int slot = -1;
        if (kCache && a.active && ok)
          slot = lfu::probe(a.hkeys, a.hvals, a.hshift, a.hmask, static_cast<unsigned long long>(row));
        // FreqTable::increment: chain rows warp-aggregated here; the cached (hot)
        // rows once per CTA from the slot counts below (no same-address storm)
        if (kCache && a.counts) {
          const unsigned long long key = ok && slot < 0 ? static_cast<unsigned long long>(row) : ~0ull;
          const unsigned pr = __match_any_sync(0xffffffffu, key);
          if (key != ~0ull && lane == __ffs(pr) - 1)
            atomicAdd(a.counts + row, static_cast<unsigned long long>(__popc(pr)));
        }
        if (in) {
          if (kCache && a.lk_slot) a.lk_slot[l] = slot;
          if (slot >= 0) {
            k1[q] = 0x80000000u | static_cast<uint32_t>(slot);
            ++my_hits;
          } else {
            uint32_t rem, i2;
            const uint32_t i0 = div_fix(static_cast<uint32_t>(row), a.g.m12, a.inv_m12, rem);
            const uint32_t i1 = div_fix(rem, static_cast<uint32_t>(a.g.m2), a.inv_m2, i2);
            a.d2[l] = static_cast<uint16_t>(i2);
            k1[q] = i1;
            d02[q] = i0 | (i2 << 16);
          }
        }
        const bool tt = k1[q] < 0x80000000u;
        const uint32_t x1 = tt ? k1[q] : 0xffffffffu;
        const uint32_t x2 = tt ? d02[q] >> 16 : 0xffffffffu;
        unsigned p = __match_any_sync(0xffffffffu, x1);
        if (tt && lane == __ffs(p) - 1) mywc[x1] += __popc(p);
        p = __match_any_sync(0xffffffffu, x2);
        if (tt && lane == __ffs(p) - 1) mywc[K1 + x2] += __popc(p);
        if (K3) {
          const bool ca = k1[q] != 0xffffffffu && !tt;
          const uint32_t x3 = ca ? (k1[q] & 0x7fffffffu) : 0xffffffffu;
          p = __match_any_sync(0xffffffffu, x3);
          if (ca && lane == __ffs(p) - 1) mywc[K12 + x3] += __popc(p);
        }
        __syncwarp();
      }
    }
  }
  // bags (grid-stride over the whole grid).  Cache mode: a single-lookup bag
  // whose lookup this very thread decoded (every bag when bags are singles and
  // the batch is laid out one lookup per thread) knows its slot already and is
  // pooled here; any other bag sets need_c and is handled after the grid
  // barriers, when every lookup's slot is visible
  bool need_c = false;
  int32_t loc_bag = -1;  // bag of this thread's first-round lookup when it is a single-lookup bag
  float loc_alpha = 0.f;
  for (int64_t b = b_first; b < a.B; b += static_cast<int64_t>(G) * kGsThreads) {
    const int64_t s = b == b_first ? s_first : a.off[b], e = b == b_first ? e_first : a.off[b + 1];
    if (b == 0 && s != 0) atomicOr(a.errs, 1);
    if (e < s) atomicOr(a.errs, 2);
    if (b == a.B - 1 && e != a.L) atomicOr(a.errs, 4);
    const int64_t lo = s < 0 ? 0 : s, hi = e > a.L ? a.L : e;
    a.bag_cnt[b] = 0;
    if (e == s)  // an empty bag pools to zeros (no lookup will)
      for (int c = 0; c < a.N; c += 4)
        reinterpret_cast<float4*>(a.out + b * a.N + c)[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (e - s == 1 && hi - lo == 1) {  // the common single-lookup bag
      a.lk_bag[lo] = static_cast<int32_t>(b);
      a.solo[lo] = static_cast<int32_t>(b);
      const float wl = a.w ? static_cast<float>(a.w[lo]) : 1.f;
      a.alpha[lo] = wl;
      if (lo == wbase + lane) {  // this thread's own first-round lookup: keep it for phase C
        loc_bag = static_cast<int32_t>(b);
        loc_alpha = wl;
      }
      if (K3) {
        if (lo == wbase + lane && k1[0] != 0xffffffffu) {
          if (k1[0] >= 0x80000000u) {  // cached: out = (0 + w·row) + 0
            const float4* src =
                reinterpret_cast<const float4*>(a.store + static_cast<int64_t>(k1[0] & 0x7fffffffu) * a.N);
            float4* dst = reinterpret_cast<float4*>(a.out + b * a.N);
            for (int j = 0; j < a.N / 4; ++j) {
              const float4 v = src[j];
              dst[j] = make_float4(__fadd_rn(__fadd_rn(0.f, __fmul_rn(wl, v.x)), 0.f),
                                   __fadd_rn(__fadd_rn(0.f, __fmul_rn(wl, v.y)), 0.f),
                                   __fadd_rn(__fadd_rn(0.f, __fmul_rn(wl, v.z)), 0.f),
                                   __fadd_rn(__fadd_rn(0.f, __fmul_rn(wl, v.w)), 0.f));
            }
          }
        } else {
          need_c = true;
        }
      }
      continue;
    }
    if (K3) need_c = true;
    const double sz = static_cast<double>(e - s);
    for (int64_t l = lo; l < hi; ++l) {
      a.lk_bag[l] = static_cast<int32_t>(b);
      a.solo[l] = -1;
      double al = a.w ? a.w[l] : 1.0;
      if (a.mean) al /= sz;
      a.alpha[l] = static_cast<float>(al);
    }
  }
  if (kCache && a.hits) {
    unsigned h = my_hits;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if (lane == 0 && h) atomicAdd(&cta_hits, h);
  }
  __syncthreads();
  if (kCache && a.accesses && c == 0 && tid == 0) atomicAdd(a.accesses, static_cast<unsigned long long>(a.L));
  if (kCache && a.hits && tid == 0 && cta_hits) {
    atomicAdd(a.hits, static_cast<unsigned long long>(cta_hits));
    if (a.hits2) atomicAdd(a.hits2, static_cast<unsigned long long>(cta_hits));
  }
  // per-warp exclusive starts within the CTA; CTA counts out
  for (int k = tid; k < K; k += kGsThreads) {
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kGsWarps; ++w) {
      const uint32_t v = wc[w * K + k];
      wc[w * K + k] = run;
      run += v;
    }
    ctot[k] = run;
    a.hist[static_cast<int64_t>(k) * G + c] = run;
    if (k >= K12 && run && a.counts)  // this CTA's hits of slot k - K12
      atomicAdd(a.counts + a.slot_rows[k - K12], static_cast<unsigned long long>(run));
  }
  cg::grid_group grid = cg::this_grid();
  cta_mark(0, 0);
  grid.sync();
  cta_mark(0, 1);

  // ---- phase B1: per key, exclusive scan over the CTAs (warp per key)
  for (int k = c * kGsWarps + wid; k < K; k += G * kGsWarps) {
    uint32_t* row = a.hist + static_cast<int64_t>(k) * G;
    uint32_t v[kGsMaxGridChunks];  // all loads first: one round trip
#pragma unroll
    for (int j = 0; j < kGsMaxGridChunks; ++j) v[j] = j * 32 + lane < G ? __ldcg(row + j * 32 + lane) : 0u;
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < kGsMaxGridChunks; ++j) {
      uint32_t x = v[j];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (j * 32 + lane < G) row[j * 32 + lane] = run + x - v[j];
      run += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) a.tot[k] = run;
  }
  grid.sync();
  cta_mark(0, 2);

  // ---- phase B2: bases from the totals plus this CTA's prefix.  Block scan
  // of (lookups, tiles, groups) over [key 1 | key 2], IPT consecutive keys
  // per thread.
  const int IPT = (K12 + kGsThreads - 1) / kGsThreads;
  const int k_lo = min(K12, tid * IPT), k_hi = min(K12, k_lo + IPT);
  uint32_t t0 = 0, t1 = 0, t2 = 0;
  for (int k = k_lo; k < k_hi; ++k) {
    const uint32_t T = __ldcg(a.tot + k);
    const uint32_t TT = k >= K1 ? a.TT2 : a.TT1;
    const uint32_t tk = (T + TT - 1) / TT;
    t0 += T;
    t1 += tk;
    t2 += n_groups(tk);
    // the key total, until the scan is done; this CTA's prefix (B1) in flight
    base[k] = T;
  }
  uint32_t pre[4];  // IPT <= 4 (K1 + K2 <= 2048)
#pragma unroll
  for (int j = 0; j < 4; ++j)
    pre[j] = k_lo + j < k_hi && ctot[k_lo + j] ? __ldcg(a.hist + static_cast<int64_t>(k_lo + j) * G + c) : 0u;
  uint32_t s0 = t0, s1 = t1, s2 = t2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y0 = __shfl_up_sync(0xffffffffu, s0, o);
    const uint32_t y1 = __shfl_up_sync(0xffffffffu, s1, o);
    const uint32_t y2 = __shfl_up_sync(0xffffffffu, s2, o);
    if (lane >= o) {
      s0 += y0;
      s1 += y1;
      s2 += y2;
    }
  }
  if (lane == 31) {
    wsum[wid][0] = s0;
    wsum[wid][1] = s1;
    wsum[wid][2] = s2;
  }
  __syncthreads();
  if (wid == 0) {
    uint32_t v[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) v[j] = lane < kGsWarps ? wsum[lane][j] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v[j], o);
        if (lane >= o) v[j] += y;
      }
    }
    __syncwarp();
    if (lane < kGsWarps)
#pragma unroll
      for (int j = 0; j < 3; ++j) wsum[lane][j] = v[j];
  }
  __syncthreads();
  // exclusive running values at this thread's first key
  uint32_t e0 = s0 - t0, e1 = s1 - t1, e2 = s2 - t2;
  if (wid > 0) {
    e0 += wsum[wid - 1][0];
    e1 += wsum[wid - 1][1];
    e2 += wsum[wid - 1][2];
  }
  // key-2 entries restart at zero: key 1's totals are the running values at
  // k = K1, found by the thread whose key range holds K1 (K2 >= 1)
  if (k_lo <= K1 && K1 < k_hi) {
    uint32_t r0 = e0, r1 = e1, r2 = e2;
    for (int k = k_lo; k < K1; ++k) {
      const uint32_t T = base[k];
      const uint32_t tk = (T + a.TT1 - 1) / a.TT1;
      r0 += T;
      r1 += tk;
      r2 += n_groups(tk);
    }
    k1tot[0] = r0;
    k1tot[1] = r1;
    k1tot[2] = r2;
  }
  __syncthreads();
  for (int k = k_lo; k < k_hi; ++k) {
    const bool second = k >= K1;
    const uint32_t T = base[k];
    const uint32_t TT = second ? a.TT2 : a.TT1;
    const uint32_t tk = (T + TT - 1) / TT;
    const uint32_t b0 = second ? e0 - k1tot[0] : e0;
    const uint32_t b1 = second ? e1 - k1tot[1] : e1;
    const uint32_t b2 = second ? e2 - k1tot[2] : e2;
    if (!second) {
      gb1[k] = b0;
      tb1[k] = b1;
    } else {
      gb2[k - K1] = b0;
      tb2[k - K1] = b1;
    }
    if (c == 0) {
      (second ? a.tile_base2 : a.tile_base1)[second ? k - K1 : k] = static_cast<int32_t>(b1);
      (second ? a.group_base2 : a.group_base1)[second ? k - K1 : k] = static_cast<int32_t>(b2);
    }
    base[k] = b0 + pre[k - k_lo];  // this CTA's start of the key
    e0 += T;
    e1 += tk;
    e2 += n_groups(tk);
    if (k == K1 - 1) {
      gb1[K1] = e0;
      tb1[K1] = e1;
      if (c == 0) {
        a.tile_base1[K1] = static_cast<int32_t>(e1);
        a.group_base1[K1] = static_cast<int32_t>(e2);
        a.ntiles[0] = static_cast<int>(e1);
      }
    }
    if (k == K12 - 1) {
      gb2[K2] = e0 - k1tot[0];
      tb2[K2] = e1 - k1tot[1];
      if (c == 0) {
        a.tile_base2[K2] = static_cast<int32_t>(e1 - k1tot[1]);
        a.group_base2[K2] = static_cast<int32_t>(e2 - k1tot[2]);
        a.ntiles[1] = static_cast<int>(e1 - k1tot[1]);
      }
    }
  }
  __syncthreads();
  // tile lists, split over the grid; the key of a tile by binary search
  {
    const uint32_t nt1 = tb1[K1], nt2 = tb2[K2];
    for (uint32_t t = static_cast<uint32_t>(c) * kGsThreads + tid; t < nt1 + nt2;
         t += static_cast<uint32_t>(G) * kGsThreads) {
      const bool s = t >= nt1;
      const uint32_t tt = s ? t - nt1 : t;
      const uint32_t* tb = s ? tb2 : tb1;
      const uint32_t* gb = s ? gb2 : gb1;
      const int kk = upper_slot(tb, s ? K2 : K1, tt);
      const uint32_t TTk = s ? a.TT2 : a.TT1;
      Tile tl;
      tl.key = kk;
      tl.start = static_cast<int>(gb[kk] + (tt - tb[kk]) * TTk);
      tl.end = static_cast<int>(min(gb[kk + 1], gb[kk] + (tt - tb[kk] + 1) * TTk));
      tl.pad = 0;
      (s ? a.tiles2 : a.tiles1)[tt] = tl;
    }
  }
  __syncthreads();
  // key 3 (cache slots): bucket bases by a block scan of the slot totals, IPT3
  // consecutive slots per thread; CTA 0 publishes the per-slot segments
  if (K3) {
    const int IPT3 = (K3 + kGsThreads - 1) / kGsThreads;
    const int s_lo = min(K3, tid * IPT3), s_hi = min(K3, s_lo + IPT3);
    uint32_t sum = 0;
    for (int s = s_lo; s < s_hi; ++s) {
      const uint32_t T = __ldcg(a.tot + K12 + s);
      base[K12 + s] = T;
      sum += T;
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid][0] = x;
    __syncthreads();
    if (wid == 0) {
      uint32_t v = lane < kGsWarps ? wsum[lane][0] : 0u;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      __syncwarp();
      if (lane < kGsWarps) wsum[lane][1] = v;
    }
    __syncthreads();
    uint32_t e = x - sum + (wid > 0 ? wsum[wid - 1][1] : 0u);
    for (int s = s_lo; s < s_hi; ++s) {
      const uint32_t T = base[K12 + s];
      if (c == 0) {
        a.seg_lo3[s] = T ? static_cast<int>(e) : -1;
        a.seg_hi3[s] = static_cast<int>(e + T);
      }
      base[K12 + s] = e + (ctot[K12 + s] ? __ldcg(a.hist + static_cast<int64_t>(K12 + s) * G + c) : 0u);
      e += T;
    }
    if (c == 0 && tid == kGsThreads - 1) *a.ncached = static_cast<int>(wsum[kGsWarps - 1][1]);
    __syncthreads();
  }

  cta_mark(0, 3);
  // ---- phase C: stable scatter of both keys
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int q = 0; q < RMAX; ++q) {
    if (q < R) {
      const int64_t l = wbase + q * 32 + lane;
      const bool tt = k1[q] < 0x80000000u;
      const uint32_t x = tt ? k1[q] : 0xffffffffu;
      unsigned p = __match_any_sync(0xffffffffu, x);
      if (tt) {
        const uint32_t pos = base[x] + mywc[x] + __popc(p & lt);
        a.perm1[pos] = static_cast<uint32_t>(l);
        // the bag fields of a lookup whose single-lookup bag this thread set
        // up are in registers; others were written by another thread (phase A)
        a.rec1[pos] = q == 0 && loc_bag >= 0
                          ? make_rec(static_cast<uint32_t>(l), d02[q], loc_bag, loc_bag, loc_alpha)
                          : make_rec(static_cast<uint32_t>(l), d02[q], __ldcg(a.solo + l),
                                     __ldcg(a.lk_bag + l), __ldcg(a.alpha + l));
      }
      __syncwarp();
      if (tt && lane == __ffs(p) - 1) mywc[x] += __popc(p);
      const uint32_t y = tt ? d02[q] >> 16 : 0xffffffffu;
      p = __match_any_sync(0xffffffffu, y);
      if (tt) {
        const uint32_t pos = base[K1 + y] + mywc[K1 + y] + __popc(p & lt);
        a.perm2[pos] = static_cast<uint32_t>(l);
      }
      __syncwarp();
      if (tt && lane == __ffs(p) - 1) mywc[K1 + y] += __popc(p);
      __syncwarp();
      if (K3) {
        const bool ca = k1[q] != 0xffffffffu && !tt;
        const uint32_t z = ca ? (k1[q] & 0x7fffffffu) : 0xffffffffu;
        p = __match_any_sync(0xffffffffu, z);
        if (ca) {
          const uint32_t pos = base[K12 + z] + mywc[K12 + z] + __popc(p & lt);
          a.perm3[pos] = static_cast<uint32_t>(l);
          a.skey3[pos] = static_cast<int>(z);
        }
        __syncwarp();
        if (ca && lane == __ffs(p) - 1) mywc[K12 + z] += __popc(p);
        __syncwarp();
      }
    }
  }
  // cache mode: a bag whose lookups ALL hit the cache pools here (cached_out =
  // Σ w·row in lookup order, out = cached_out + 0, the Mean rescale:
  // model.hpp:210-223 with an empty chain part); a bag with chain lookups
  // presets its pooling counter with its cached lookups, so its last chain
  // lookup pools it in f3_fwd (pool_if_last)
  if (kCache && K3 && need_c) {
    for (int64_t b = static_cast<int64_t>(c) * kGsThreads + tid; b < a.B;
         b += static_cast<int64_t>(G) * kGsThreads) {
      const int64_t s = a.off[b], e = a.off[b + 1];
      if (e - s < 1 || s < 0 || e > a.L) continue;
      if (e - s == 1 && s == wbase + lane) continue;  // pooled in phase A
      int nc = 0;
      for (int64_t l = s; l < e; ++l) nc += __ldcg(a.lk_slot + l) >= 0 ? 1 : 0;
      if (nc < e - s) {
        if (e - s > 1) a.bag_cnt[b] = nc * a.parts;
        continue;
      }
      const float inv = static_cast<float>(1.0 / static_cast<double>(e - s));
      for (int j = 0; j < a.N / 4; ++j) {
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int64_t l = s; l < e; ++l) {
          const float wl = a.w ? static_cast<float>(a.w[l]) : 1.f;
          const float4 v = reinterpret_cast<const float4*>(a.store + static_cast<int64_t>(__ldcg(a.lk_slot + l)) * a.N)[j];
          acc = make_float4(__fadd_rn(acc.x, __fmul_rn(wl, v.x)), __fadd_rn(acc.y, __fmul_rn(wl, v.y)),
                            __fadd_rn(acc.z, __fmul_rn(wl, v.z)), __fadd_rn(acc.w, __fmul_rn(wl, v.w)));
        }
        acc = make_float4(__fadd_rn(acc.x, 0.f), __fadd_rn(acc.y, 0.f), __fadd_rn(acc.z, 0.f),
                          __fadd_rn(acc.w, 0.f));  // + tt_out (zero)
        if (a.pool_mean && e - s > 1)
          acc = make_float4(__fmul_rn(acc.x, inv), __fmul_rn(acc.y, inv), __fmul_rn(acc.z, inv),
                            __fmul_rn(acc.w, inv));
        reinterpret_cast<float4*>(a.out + b * a.N)[j] = acc;
      }
    }
  }
}

}  // namespace f3
}  // namespace ttgpu
