// Fast path for 3-core tables (every BASELINE config): compile-time TT shape,
// 7 kernels per fwd+bwd+SGD step, deterministic, no floating-point atomics.
//
//   f3_hist    decode + validate + per-CTA histogram of the tile key
//              key = (i2 / BLK) * m1 + i1, lookup->bag map and backward alpha
//   f3_scan    one CTA: exclusive scan of the (key, CTA) histogram, bucket
//              tile list (buckets cut into tiles of <= TT lookups)
//   f3_scatter stable counting-sort scatter (warp match_any ranks)
//   f3_fwd     per tile: G1[i1] staged in smem once, tile-local dedup of i0
//              ("slots"), H(slot) = G0[i0]·G1[i1], y = H·G2[i2] per lookup
//   f3_pool    per bag, lookup order: out = Σ T(w)·y (Mean rescale)
//   f3_bwd     per tile: dG2 partial (BLK i2 slices in smem), S(slot) = Σ D1,
//              dG1 partial = Σ G0ᵀ S, D0(slot) = S·G1ᵀ
//   f3_combine fixed-order folds of the tile partials per core slice, fused
//              with the SGD update (or a dense gradient write)
//
// Reference semantics: embedding_ops.hpp:159-376.  In exact mode the forward
// keeps the reference's per-element operation order (separately rounded
// products/sums, p-ascending, lookup-ascending pooling), so outputs are
// bit-identical to ttrec::forward_bags.
#pragma once

#include <cub/block/block_scan.cuh>

#include "tt_kernels.cuh"

namespace ttgpu {
namespace f3 {

struct Geo {
  int m0, m1, m2;
  uint32_t m12;   // m1 * m2
  int blk;        // i2 block size (<= 64)
  int nblk;       // ceil(m2 / blk)
  int K;          // nblk * m1 tile keys
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
  static constexpr int W1P = W1 + 1;  // odd slot strides: conflict-free across slots
  static constexpr int S0P = S0 + 1;
  static constexpr int S2P = S2 + 4;  // 16 B pad: float4 rows land in distinct bank groups
  static constexpr int C1P = C1 + 1;
  static_assert(N2 == 4, "fast path expects n_2 == 4 (float4 rows)");
  static_assert(C1 % 4 == 0, "C1 must be a multiple of 4");
  static_assert((C1 & (C1 - 1)) == 0, "C1 must be a power of two (rotated D0 reads)");
};

constexpr int kThreads = 256;

template <typename T, bool kExact>
__device__ __forceinline__ float4 madd4(float a, float4 b, float4 acc) {
  acc.x = madd<float, kExact>(a, b.x, acc.x);
  acc.y = madd<float, kExact>(a, b.y, acc.y);
  acc.z = madd<float, kExact>(a, b.z, acc.z);
  acc.w = madd<float, kExact>(a, b.w, acc.w);
  return acc;
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

// ------------------------------------------------------------- f3_hist ---
// TL = 512 * LPT lookups per CTA (LPT lookups per thread, loads batched).
template <typename T, int LPT>
__global__ void __launch_bounds__(512) f3_hist(Geo g, const int64_t* __restrict__ idx, int64_t L,
                                               int NT, const int64_t* __restrict__ off,
                                               int64_t B, const double* __restrict__ w, int mean,
                                               uint32_t* __restrict__ key, uint16_t* __restrict__ d0,
                                               uint16_t* __restrict__ d2, int32_t* __restrict__ lk_bag,
                                               T* __restrict__ alpha, uint32_t* __restrict__ hist,
                                               unsigned long long* __restrict__ bad,
                                               int* __restrict__ errs) {
  extern __shared__ uint32_t shist[];
  for (int k = threadIdx.x; k < g.K; k += blockDim.x) shist[k] = 0;
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
      uint32_t k = 0xffffffffu;
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
        k = (i2 / static_cast<uint32_t>(g.blk)) * static_cast<uint32_t>(g.m1) + i1;
        key[l] = k;
        d0[l] = static_cast<uint16_t>(i0);
        d2[l] = static_cast<uint16_t>(i2);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      if (k != 0xffffffffu && lane == __ffs(peers) - 1) atomicAdd(&shist[k], __popc(peers));
    }
  }
  __syncthreads();
  if (tile < NT)
    for (int k = threadIdx.x; k < g.K; k += blockDim.x)
      hist[static_cast<int64_t>(k) * NT + tile] = shist[k];
  // bags (grid-stride over all CTAs): offsets checks, lookup->bag, backward alpha
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = off[b], e = off[b + 1];
    if (b == 0 && s != 0) atomicOr(errs, 1);
    if (e < s) atomicOr(errs, 2);
    if (b == B - 1 && e != L) atomicOr(errs, 4);
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    const double sz = static_cast<double>(e - s);
    for (int64_t l = lo; l < hi; ++l) {
      lk_bag[l] = static_cast<int32_t>(b);
      double a = w ? w[l] : 1.0;
      if (mean) a /= sz;
      alpha[l] = static_cast<T>(a);
    }
  }
}

// ------------------------------------------------------------- f3_scan ---
// One CTA of 1024 threads; the (K x NT, key-major) histogram is staged in
// shared memory with coalesced loads, scanned there, and written back as
// exclusive offsets.  Also emits the tile list (buckets cut into <= TT).
__global__ void __launch_bounds__(1024) f3_scan(Geo g, int NT, int TT, int64_t L,
                                                uint32_t* __restrict__ hist,
                                                int32_t* __restrict__ tile_base,
                                                Tile* __restrict__ tiles, int* __restrict__ ntiles) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  extern __shared__ uint32_t sh[];  // n entries
  const int n = g.K * NT;
  const int tid = threadIdx.x;
#pragma unroll 8
  for (int i = tid; i < n; i += 1024) sh[i] = hist[i];
  __syncthreads();
  const int per = (n + 1023) / 1024;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += sh[i];
  uint32_t ex;
  Scan(tmp).ExclusiveSum(s, ex);
  for (int i = lo; i < hi; ++i) {
    const uint32_t c = sh[i];
    sh[i] = ex;
    ex += c;
  }
  __syncthreads();
#pragma unroll 8
  for (int i = tid; i < n; i += 1024) hist[i] = sh[i];
  // tiles per bucket
  const int perk = (g.K + 1023) / 1024;
  const int klo = min(g.K, tid * perk), khi = min(g.K, klo + perk);
  uint32_t nt = 0;
  for (int k = klo; k < khi; ++k) {
    const uint32_t bs = sh[k * NT];
    const uint32_t be = k + 1 < g.K ? sh[(k + 1) * NT] : static_cast<uint32_t>(L);
    nt += (be - bs + TT - 1) / TT;
  }
  uint32_t tex;
  __syncthreads();
  Scan(tmp).ExclusiveSum(nt, tex);
  uint32_t* tb = sh + n;  // K + 1 tile bases
  for (int k = klo; k < khi; ++k) {
    const uint32_t bs = sh[k * NT];
    const uint32_t be = k + 1 < g.K ? sh[(k + 1) * NT] : static_cast<uint32_t>(L);
    tb[k] = tex;
    tile_base[k] = static_cast<int32_t>(tex);
    tex += (be - bs + TT - 1) / TT;
  }
  if (tid == 1023) {
    tb[g.K] = tex;
    tile_base[g.K] = static_cast<int32_t>(tex);
    *ntiles = static_cast<int>(tex);
  }
  __syncthreads();
  // one thread per tile: find its bucket by binary search over the tile bases
  const uint32_t total = tb[g.K];
  for (uint32_t t = tid; t < total; t += 1024) {
    int lo = 0, hi = g.K;  // invariant: tb[lo] <= t < tb[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (tb[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t bs = sh[lo * NT];
    const uint32_t be = lo + 1 < g.K ? sh[(lo + 1) * NT] : static_cast<uint32_t>(L);
    Tile tl;
    tl.key = lo;
    tl.start = static_cast<int>(bs + (t - tb[lo]) * TT);
    tl.end = static_cast<int>(min(be, bs + (t - tb[lo] + 1) * TT));
    tl.pad = 0;
    tiles[t] = tl;
  }
}

// ---------------------------------------------------------- f3_scatter ---
// Stable scatter: 8 warps per CTA, each owning TL/8 consecutive lookups,
// keys loaded 8 rounds at a time.
__global__ void __launch_bounds__(256) f3_scatter(Geo g, const uint32_t* __restrict__ key, int64_t L,
                                                  int TL, int NT, const uint32_t* __restrict__ hoff,
                                                  uint32_t* __restrict__ perm) {
  extern __shared__ uint32_t wc[];  // 8 x K
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int per = TL / 8;
  const int64_t base = static_cast<int64_t>(tile) * TL + static_cast<int64_t>(wid) * per;
  uint32_t* my = wc + static_cast<int64_t>(wid) * g.K;
  for (int k = lane; k < g.K; k += 32) my[k] = 0;
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
  for (int k = threadIdx.x; k < g.K; k += blockDim.x) {
    uint32_t run = hoff[static_cast<int64_t>(k) * NT + tile];
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = wc[static_cast<int64_t>(w) * g.K + k];
      wc[static_cast<int64_t>(w) * g.K + k] = run;
      run += c;
    }
  }
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
        if (lane == __ffs(peers) - 1) my[k] += __popc(peers);
      }
      __syncwarp();
    }
  }
}

// --------------------------------------------------------- smem layouts ---
template <class D>
struct FwdSmem {
  // floats: G1s[S1] (TMA) | Hs[TT*W1P] | G0s[TT*S0] ; then mbarrier + ints
  static constexpr int W1P = D::W1 + 1;  // odd: lookups of different slots hit different banks
  static __host__ __device__ size_t floats() {
    size_t f = D::S1 + static_cast<size_t>(D::TT) * (W1P + D::S0);
    return (f + 3) / 4 * 4;
  }
  static __host__ __device__ size_t bytes(int m0) {
    return floats() * 4 + 16 + sizeof(int) * (static_cast<size_t>(m0) + 5 * D::TT + 40);
  }
};

// ------------------------------------------------------------- f3_fwd ----
// Per tile: TMA G1[i1] (issued first, overlaps the index gathers); dedup i0
// -> slots (ascending i0, the numbering backward reuses); H(slot) = G0·G1
// with G1 from smem; y = H·G2[i2] per lookup (G2 rows straight from L1/L2).
template <class D, bool kExact>
__global__ void __launch_bounds__(kThreads) f3_fwd(Geo g, const float* __restrict__ cores,
                                                   const Tile* __restrict__ tiles,
                                                   const int* __restrict__ ntiles,
                                                   const uint32_t* __restrict__ perm,
                                                   const uint16_t* __restrict__ d0,
                                                   const uint16_t* __restrict__ d2,
                                                   float* __restrict__ Hbuf, float* __restrict__ y,
                                                   uint16_t* __restrict__ slot_of_pos,
                                                   uint16_t* __restrict__ tile_i0,
                                                   int* __restrict__ tile_nslots) {
  using SM = FwdSmem<D>;
  extern __shared__ __align__(128) float sm[];
  float* G1s = sm;
  float* Hs = G1s + D::S1;
  float* G0s = Hs + D::TT * SM::W1P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SM::floats());
  int* flags = reinterpret_cast<int*>(bar + 2);
  int* lk_l = flags + g.m0;
  int* lk_i0 = lk_l + D::TT;
  int* lk_i2 = lk_i0 + D::TT;
  int* lk_slot = lk_i2 + D::TT;
  int* slot_i0 = lk_slot + D::TT;
  int* scr = slot_i0 + D::TT;  // 40 ints scan scratch
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  const int nt = *ntiles;
  const int tid = threadIdx.x;
  if (tid == 0) mbar_init(bar, 1);
  for (int i = tid; i < g.m0; i += kThreads) flags[i] = 0;
  __syncthreads();
  uint32_t phase = 0;
  for (int t = blockIdx.x; t < nt; t += gridDim.x, phase ^= 1u) {
    const Tile tl = tiles[t];
    const int i1 = tl.key % g.m1;
    const int ntl = tl.end - tl.start;
    if (tid == 0) {
      // smem last touched by generic-proxy accesses; order them before the TMA write
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect(bar, D::S1 * 4);
      tma_load(G1s, G1 + static_cast<int64_t>(i1) * D::S1, D::S1 * 4, bar);
    }
    if (tid < ntl) {
      const int l = static_cast<int>(perm[tl.start + tid]);
      const int i0 = d0[l];
      const int i2 = d2[l];
      lk_l[tid] = l;
      lk_i0[tid] = i0;
      lk_i2[tid] = i2;
      flags[i0] = 1;
    }
    __syncthreads();
    int nslots;
    {
      const int per = (g.m0 + kThreads - 1) / kThreads;
      const int lo = min(g.m0, tid * per), hi = min(g.m0, lo + per);
      int c = 0;
      for (int i = lo; i < hi; ++i) c += flags[i];
      int ex = block_excl_scan(c, &nslots, scr);
      for (int i = lo; i < hi; ++i) {
        if (flags[i]) {
          slot_i0[ex] = i;
          flags[i] = ex++;
        }
      }
    }
    __syncthreads();
    if (tid < ntl) {
      const int s = flags[lk_i0[tid]];
      lk_slot[tid] = s;
      slot_of_pos[tl.start + tid] = static_cast<uint16_t>(s);
    }
    if (tid < nslots) tile_i0[tl.start + tid] = static_cast<uint16_t>(slot_i0[tid]);
    if (tid == 0) tile_nslots[t] = nslots;
    // G0 rows of the slots (independent loads, batched)
    {
      constexpr int U = 8;
      for (int e0 = tid; e0 < nslots * D::S0; e0 += kThreads * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kThreads;
          v[u] = 0.f;
          if (e < nslots * D::S0) {
            const int s = e / D::S0;
            v[u] = __ldg(G0 + static_cast<int64_t>(slot_i0[s]) * D::S0 + (e - s * D::S0));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (e0 + u * kThreads < nslots * D::S0) G0s[e0 + u * kThreads] = v[u];
      }
    }
    __syncthreads();
    if (tid < nslots) flags[slot_i0[tid]] = 0;  // ready for the next tile
    mbar_wait(bar, phase);
    // H(slot) = G0[i0] (P0 x R1) · G1[i1] (R1 x C1): thread -> (slot, 4 columns), all P0 rows
    for (int q = tid; q < nslots * D::C4; q += kThreads) {
      const int s = q / D::C4, c4 = q - s * D::C4;
      float4 acc[D::P0];
#pragma unroll
      for (int a = 0; a < D::P0; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float* g0 = G0s + s * D::S0;
#pragma unroll 8
      for (int p = 0; p < D::R1; ++p) {
        const float4 b = reinterpret_cast<const float4*>(G1s + p * D::C1)[c4];
#pragma unroll
        for (int a = 0; a < D::P0; ++a) acc[a] = madd4<float, kExact>(g0[a * D::R1 + p], b, acc[a]);
      }
      float* hrow = Hs + s * SM::W1P;
      float* hg = Hbuf + static_cast<int64_t>(tl.start + s) * D::W1;
#pragma unroll
      for (int a = 0; a < D::P0; ++a) {
        const int c = a * D::C1 + c4 * 4;
        hrow[c] = acc[a].x;
        hrow[c + 1] = acc[a].y;
        hrow[c + 2] = acc[a].z;
        hrow[c + 3] = acc[a].w;
        reinterpret_cast<float4*>(hg + c)[0] = acc[a];
      }
    }
    __syncthreads();
    // y = H(slot) (P1 x R2) · G2[i2] (R2 x N2): thread -> (lookup, row a)
    for (int q = tid; q < ntl * D::P1; q += kThreads) {
      const int i = q / D::P1, a = q - i * D::P1;
      const float* hrow = Hs + lk_slot[i] * SM::W1P + a * D::R2;
      const float4* g2 = reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(lk_i2[i]) * D::S2);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int r = 0; r < D::R2; ++r) acc = madd4<float, kExact>(hrow[r], __ldg(g2 + r), acc);
      reinterpret_cast<float4*>(y + static_cast<int64_t>(lk_l[i]) * D::N)[a] = acc;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- f3_pool ---
// One thread per (bag, float4 column chunk); lookup-ascending accumulation.
template <int N, bool kExact>
__global__ void f3_pool(const int64_t* __restrict__ off, int64_t B, int64_t L,
                        const double* __restrict__ w, int mean, const float* __restrict__ y,
                        float* __restrict__ out) {
  constexpr int Q = N / 4;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < B * Q;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / Q;
    const int c = static_cast<int>(q - b * Q);
    const int64_t s = off[b], e = off[b + 1];
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t l = lo; l < hi; ++l) {
      const float a = static_cast<float>(w ? w[l] : 1.0);
      acc = madd4<float, kExact>(a, reinterpret_cast<const float4*>(y + l * N)[c], acc);
    }
    if (mean && e - s > 1) {
      const float inv = static_cast<float>(1.0 / static_cast<double>(e - s));
      acc.x = __fmul_rn(acc.x, inv);
      acc.y = __fmul_rn(acc.y, inv);
      acc.z = __fmul_rn(acc.z, inv);
      acc.w = __fmul_rn(acc.w, inv);
    }
    reinterpret_cast<float4*>(out + b * N)[c] = acc;
  }
}

// -------------------------------------------------------------- f3_bwd ---
template <class D>
struct BwdSmem {
  // floats: G1t[C1*R1P] (G1 slice transposed) | S[TT*W1] | P2[BLK*S2] | G0s[TT*S0]
  //         | d0tmp[TT*S0] ; then u64 mask + ints
  static constexpr int R1P = D::R1 + 4;
  static __host__ __device__ size_t floats(int blk) {
    size_t f = static_cast<size_t>(D::C1) * R1P + static_cast<size_t>(D::TT) * D::W1 +
               static_cast<size_t>(blk) * D::S2 + 2 * static_cast<size_t>(D::TT) * D::S0;
    return (f + 3) / 4 * 4;
  }
  static __host__ __device__ size_t bytes(int m0, int blk) {
    (void)m0;
    return floats(blk) * 4 + 16 + sizeof(int) * (5 * static_cast<size_t>(D::TT) + 8);
  }
};

// Each CTA owns a contiguous range of tiles.  Consecutive tiles of the same
// bucket keep accumulating the dG1 partial (registers) and the dG2 partial
// (smem); one partial per (CTA, bucket run) is flushed, stored at the run's
// first tile (has1 / mask2 mark it).  D0 accumulates per (CTA, i0) in a
// CTA-private global block.  Within a tile, warp w owns the dG2 slices
// j = w (mod 8) and the slots s = w (mod 8): each warp walks the tile's
// lookups in order and updates only what it owns, so every accumulation
// happens in one fixed order (deterministic) with no atomics.
template <class D>
__global__ void __launch_bounds__(kThreads) f3_bwd(
    Geo g, const float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const uint32_t* __restrict__ perm,
    const uint16_t* __restrict__ d2, const int32_t* __restrict__ lk_bag,
    const float* __restrict__ alpha, const float* __restrict__ grad,
    const float* __restrict__ Hbuf, const uint16_t* __restrict__ slot_of_pos,
    const uint16_t* __restrict__ tile_i0, const int* __restrict__ tile_nslots,
    float* __restrict__ part1, int* __restrict__ has1, float* __restrict__ part2,
    unsigned long long* __restrict__ mask2, float* __restrict__ D0acc,
    unsigned char* __restrict__ d0mask) {
  using SM = BwdSmem<D>;
  constexpr int NW = kThreads / 32;
  extern __shared__ __align__(128) float sm[];
  float* G1t = sm;                                   // C1 x R1P
  float* S = G1t + D::C1 * SM::R1P;                  // TT x W1
  float* P2 = S + D::TT * D::W1;                     // BLK x S2
  const int p2sz = g.blk * D::S2;
  float* G0s = P2 + p2sz;                            // TT x S0
  float* d0tmp = G0s + D::TT * D::S0;                // TT x S0
  unsigned long long* tmask = reinterpret_cast<unsigned long long*>(sm + SM::floats(g.blk));
  int* lk_slot = reinterpret_cast<int*>(tmask + 1);
  int* lk_i2 = lk_slot + D::TT;
  int* lk_bg = lk_i2 + D::TT;
  float* lk_al = reinterpret_cast<float*>(lk_bg + D::TT);
  int* slot_i0 = reinterpret_cast<int*>(lk_al + D::TT);
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  const int nt = *ntiles;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const int t_lo = static_cast<int>(static_cast<int64_t>(blockIdx.x) * nt / gridDim.x);
  const int t_hi = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * nt / gridDim.x);
  float* d0acc = D0acc + static_cast<int64_t>(blockIdx.x) * g.m0 * D::S0;
  unsigned char* d0m = d0mask + static_cast<int64_t>(blockIdx.x) * g.m0;
  for (int e = tid; e < g.m0 * D::S0; e += kThreads) d0acc[e] = 0.f;
  for (int e = tid; e < g.m0; e += kThreads) d0m[e] = 0;
  // dG1 partial: thread owns (r1, 4 consecutive columns) items, float4 each
  constexpr int ITEMS1 = D::R1 * D::C4;
  constexpr int PER1 = (ITEMS1 + kThreads - 1) / kThreads;
  float4 acc1[PER1];
#pragma unroll
  for (int x = 0; x < PER1; ++x) acc1[x] = make_float4(0.f, 0.f, 0.f, 0.f);
  int run_start = t_lo;
  for (int e = tid; e < p2sz; e += kThreads) P2[e] = 0.f;
  if (tid == 0) *tmask = 0ull;
  __syncthreads();
  for (int t = t_lo; t < t_hi; ++t) {
    const Tile tl = tiles[t];
    const int i1 = tl.key % g.m1;
    const int i2base = (tl.key / g.m1) * g.blk;
    const int ntl = tl.end - tl.start;
    const int nslots = tile_nslots[t];
    if (tid < ntl) {
      const int l = static_cast<int>(perm[tl.start + tid]);
      lk_slot[tid] = slot_of_pos[tl.start + tid];
      const int i2 = d2[l];
      lk_i2[tid] = i2;
      lk_bg[tid] = lk_bag[l];
      lk_al[tid] = alpha[l];
      atomicOr(tmask, 1ull << (i2 - i2base));
    }
    if (tid < nslots) slot_i0[tid] = tile_i0[tl.start + tid];
    // G1[i1] transposed into smem (c-major, padded rows): coalesced, batched loads
    {
      constexpr int U = (D::S1 / kThreads) > 8 ? 8 : (D::S1 / kThreads > 0 ? D::S1 / kThreads : 1);
      const float* src = G1 + static_cast<int64_t>(i1) * D::S1;
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
    }
    __syncthreads();
    {
      constexpr int U = 8;
      for (int e0 = tid; e0 < nslots * D::S0; e0 += kThreads * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kThreads;
          v[u] = 0.f;
          if (e < nslots * D::S0) {
            const int s = e / D::S0;
            v[u] = __ldg(G0 + static_cast<int64_t>(slot_i0[s]) * D::S0 + (e - s * D::S0));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (e0 + u * kThreads < nslots * D::S0) G0s[e0 + u * kThreads] = v[u];
      }
    }
    for (int e = tid; e < nslots * D::W1; e += kThreads) S[e] = 0.f;
    __syncthreads();
    // dG2 (warp owns slices j = w mod NW) and S (warp owns slots s = w mod NW);
    // lane owns rank column r.  D2 = alpha * grad row, recomputed per use.
    for (int i = 0; i < ntl; ++i) {
      const int j = lk_i2[i] - i2base;
      const int s = lk_slot[i];
      const bool own_j = (j % NW) == wid, own_s = (s % NW) == wid;
      if (!own_j && !own_s) continue;
      const float al = lk_al[i];
      const float4* grow = reinterpret_cast<const float4*>(grad + static_cast<int64_t>(lk_bg[i]) * D::N);
      float4 d[D::P1];
#pragma unroll
      for (int a = 0; a < D::P1; ++a) {
        const float4 gv = __ldg(grow + a);
        d[a] = make_float4(__fmul_rn(al, gv.x), __fmul_rn(al, gv.y), __fmul_rn(al, gv.z),
                           __fmul_rn(al, gv.w));
      }
      for (int r = lane; r < D::R2; r += 32) {
        if (own_j) {
          // P2[j][r][:] += Σ_a H[a][r] · D2[a][:]
          const float* hrow = Hbuf + static_cast<int64_t>(tl.start + s) * D::W1 + r;
          float h[D::P1];
#pragma unroll
          for (int a = 0; a < D::P1; ++a) h[a] = __ldg(hrow + a * D::R2);
          float4* p = reinterpret_cast<float4*>(P2 + j * D::S2 + r * D::N2);
          float4 v = *p;
#pragma unroll
          for (int a = 0; a < D::P1; ++a) {
            v.x = __fmaf_rn(h[a], d[a].x, v.x);
            v.y = __fmaf_rn(h[a], d[a].y, v.y);
            v.z = __fmaf_rn(h[a], d[a].z, v.z);
            v.w = __fmaf_rn(h[a], d[a].w, v.w);
          }
          *p = v;
        }
        if (own_s) {
          // S[s][a][r] += Σ_j2 D2[a][j2] · G2[i2][r][j2]
          const float4 gv = __ldg(reinterpret_cast<const float4*>(
              G2 + static_cast<int64_t>(lk_i2[i]) * D::S2) + r);
          float* srow = S + s * D::W1 + r;
#pragma unroll
          for (int a = 0; a < D::P1; ++a) {
            float v = __fmul_rn(d[a].x, gv.x);
            v = __fmaf_rn(d[a].y, gv.y, v);
            v = __fmaf_rn(d[a].z, gv.z, v);
            v = __fmaf_rn(d[a].w, gv.w, v);
            srow[a * D::R2] += v;
          }
        }
      }
    }
    __syncthreads();
    // dG1 partial += Σ_slots G0[i0]ᵀ (R1 x P0) · S (P0 x C1)
#pragma unroll
    for (int x = 0; x < PER1; ++x) {
      const int item = tid + x * kThreads;
      if (item < ITEMS1) {
        const int r1 = item / D::C4, c4 = item - r1 * D::C4;
        float4 a4 = acc1[x];
        for (int s = 0; s < nslots; ++s) {
#pragma unroll
          for (int a = 0; a < D::P0; ++a) {
            const float gv = G0s[s * D::S0 + a * D::R1 + r1];
            const float4 sv = reinterpret_cast<const float4*>(S + s * D::W1 + a * D::C1)[c4];
            a4.x = __fmaf_rn(gv, sv.x, a4.x);
            a4.y = __fmaf_rn(gv, sv.y, a4.y);
            a4.z = __fmaf_rn(gv, sv.z, a4.z);
            a4.w = __fmaf_rn(gv, sv.w, a4.w);
          }
        }
        acc1[x] = a4;
      }
    }
    // D0(slot) (P0 x R1) = S (P0 x C1) · G1[i1]ᵀ: item (slot, a, 4 r1) over c
    {
      constexpr int R4 = D::R1 / 4;
      for (int q = tid; q < nslots * D::P0 * R4; q += kThreads) {
        const int sa = q / R4, r4 = q - sa * R4;
        const float* srow = S + (sa / D::P0) * D::W1 + (sa % D::P0) * D::C1;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
        for (int c = 0; c < D::C1; ++c) {
          const float sv = srow[c];
          const float4 gt = reinterpret_cast<const float4*>(G1t + c * SM::R1P)[r4];
          v.x = __fmaf_rn(sv, gt.x, v.x);
          v.y = __fmaf_rn(sv, gt.y, v.y);
          v.z = __fmaf_rn(sv, gt.z, v.z);
          v.w = __fmaf_rn(sv, gt.w, v.w);
        }
        reinterpret_cast<float4*>(d0tmp + sa * D::R1)[r4] = v;
      }
    }
    __syncthreads();
    // batched read-modify-write of this CTA's private D0 accumulator
    {
      constexpr int U = 4;
      for (int q0 = tid; q0 < nslots * D::S0; q0 += kThreads * U) {
        float cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + u * kThreads;
          if (q < nslots * D::S0) {
            const int s = q / D::S0, e = q - s * D::S0;
            cur[u] = d0acc[slot_i0[s] * D::S0 + e];
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = q0 + u * kThreads;
          if (q < nslots * D::S0) {
            const int s = q / D::S0, e = q - s * D::S0;
            d0acc[slot_i0[s] * D::S0 + e] = cur[u] + d0tmp[q];
            if (e == 0) d0m[slot_i0[s]] = 1;
          }
        }
      }
    }
    // end of a bucket run (or of this CTA's range): flush the run partials
    const bool last = (t + 1 == t_hi) || (tiles[t + 1].key != tl.key);
    if (tid == 0) {
      has1[t] = (t == run_start) ? 1 : 0;
      if (t != run_start) mask2[t] = 0ull;
    }
    __syncthreads();
    if (last) {
#pragma unroll
      for (int x = 0; x < PER1; ++x) {
        const int item = tid + x * kThreads;
        if (item < ITEMS1) {
          reinterpret_cast<float4*>(part1 + static_cast<int64_t>(run_start) * D::S1)[item] = acc1[x];
          acc1[x] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      const unsigned long long tm = *tmask;
      for (int e = tid; e < p2sz; e += kThreads) {
        const int j = e / D::S2;
        if ((tm >> j) & 1ull) part2[static_cast<int64_t>(run_start) * p2sz + e] = P2[e];
        P2[e] = 0.f;
      }
      __syncthreads();
      if (tid == 0) {
        mask2[run_start] = tm;
        *tmask = 0ull;
      }
      run_start = t + 1;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------- f3_combine ---
// Fixed-order list reductions.  One CTA per (output slice, 128-column chunk):
// warp w scans candidate chunks of 32 (w, w+8, ...), ballots the live
// candidates, and sums their rows 4 loads at a time (lanes own float4
// columns); warp sums are folded in warp order.  Roles by blockIdx:
//   [0, m1*C1c)            dG1[i1]   candidates: tiles of buckets (blk, i1), has1
//   [.., + m2*C2c)         dG2[i2]   candidates: tiles of blk(i2) buckets, mask2 bit
//   [.., + m0*C0c)         dG0[i0]   candidates: bwd CTAs, d0mask
// MODE 0 writes dense gradients (zeros if untouched), 1 applies SGD in place.
__device__ __forceinline__ void add4(float4& a, const float4 b) {
  a.x += b.x;
  a.y += b.y;
  a.z += b.z;
  a.w += b.w;
}

// Sum rows row_of(k) (float4 column col4) over the set bits k of `live`
// (relative to cand0), 4 independent loads in flight.
template <class RowFn>
__device__ __forceinline__ void sum_live(unsigned live, int cand0, int col4, bool colok, RowFn row_of,
                                         float4& acc) {
  while (live) {
    int idx[4];
    int n = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      idx[u] = -1;
      if (live) {
        idx[u] = cand0 + __ffs(live) - 1;
        live &= live - 1;
        ++n;
      }
    }
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      v[u] = (idx[u] >= 0 && colok) ? __ldg(reinterpret_cast<const float4*>(row_of(idx[u])) + col4)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 4; ++u) add4(acc, v[u]);
  }
}

template <int W>
__device__ __forceinline__ void fold_store(float4 v, bool touched, float4* red, float* out_core,
                                           float* out_grad, int col4, int mode, float lr,
                                           int* touched_sm) {
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  red[wid * 32 + lane] = v;
  if (touched) atomicOr(touched_sm, 1);
  __syncthreads();
  if (wid == 0 && col4 < W / 4) {
    float4 s = red[lane];
    for (int w = 1; w < kThreads / 32; ++w) add4(s, red[w * 32 + lane]);
    if (mode == 0) {
      reinterpret_cast<float4*>(out_grad)[col4] = s;
    } else if (*touched_sm) {
      float4 c = reinterpret_cast<float4*>(out_core)[col4];
      c.x = __fadd_rn(c.x, -__fmul_rn(lr, s.x));
      c.y = __fadd_rn(c.y, -__fmul_rn(lr, s.y));
      c.z = __fadd_rn(c.z, -__fmul_rn(lr, s.z));
      c.w = __fadd_rn(c.w, -__fmul_rn(lr, s.w));
      reinterpret_cast<float4*>(out_core)[col4] = c;
    }
  }
}

template <class D, int MODE>
__global__ void __launch_bounds__(kThreads) f3_combine(
    Geo g, float* __restrict__ cores, float* __restrict__ grads, const int* __restrict__ ntiles,
    const int32_t* __restrict__ tile_base, const float* __restrict__ part1,
    const int* __restrict__ has1, const float* __restrict__ part2,
    const unsigned long long* __restrict__ mask2, const float* __restrict__ D0acc,
    const unsigned char* __restrict__ d0mask, int nbwd, float lr) {
  __shared__ float4 red[kThreads];
  __shared__ int touched_sm;
  constexpr int NW = kThreads / 32;
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int C1c = (D::S1 + 127) / 128, C2c = (D::S2 + 127) / 128, C0c = (D::S0 + 127) / 128;
  if (threadIdx.x == 0) touched_sm = 0;
  __syncthreads();
  int bid = blockIdx.x;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  bool touched = false;
  if (bid < g.m1 * C1c) {
    const int i1 = bid / C1c, ch = bid - i1 * C1c;
    const int col4 = ch * 32 + lane;
    const bool colok = col4 < D::S1 / 4;
    auto row = [&](int t) { return part1 + static_cast<int64_t>(t) * D::S1; };
    for (int b = 0; b < g.nblk; ++b) {
      const int key = b * g.m1 + i1;
      const int t0 = tile_base[key], t1 = tile_base[key + 1];
      for (int c0 = t0 + wid * 32; c0 < t1; c0 += NW * 32) {
        const int t = c0 + lane;
        const unsigned live = __ballot_sync(0xffffffffu, t < t1 && has1[t] != 0);
        touched |= live != 0;
        sum_live(live, c0, col4, colok, row, acc);
      }
    }
    fold_store<D::S1>(acc, touched, red, cores + g.coff1 + static_cast<int64_t>(i1) * D::S1,
                      grads + g.coff1 + static_cast<int64_t>(i1) * D::S1, col4, MODE, lr,
                      &touched_sm);
    return;
  }
  bid -= g.m1 * C1c;
  if (bid < g.m2 * C2c) {
    const int i2 = bid / C2c, ch = bid - i2 * C2c;
    const int b = i2 / g.blk, j = i2 - b * g.blk;
    const int col4 = ch * 32 + lane;
    const bool colok = col4 < D::S2 / 4;
    const int t0 = tile_base[b * g.m1], t1 = tile_base[b * g.m1 + g.m1];
    const int p2sz = g.blk * D::S2;
    auto row = [&](int t) { return part2 + static_cast<int64_t>(t) * p2sz + j * D::S2; };
    for (int c0 = t0 + wid * 32; c0 < t1; c0 += NW * 32) {
      const int t = c0 + lane;
      const unsigned live = __ballot_sync(0xffffffffu, t < t1 && ((mask2[t] >> j) & 1ull));
      touched |= live != 0;
      sum_live(live, c0, col4, colok, row, acc);
    }
    fold_store<D::S2>(acc, touched, red, cores + g.coff2 + static_cast<int64_t>(i2) * D::S2,
                      grads + g.coff2 + static_cast<int64_t>(i2) * D::S2, col4, MODE, lr,
                      &touched_sm);
    return;
  }
  bid -= g.m2 * C2c;
  const int i0 = bid / C0c, ch = bid - i0 * C0c;
  if (i0 >= g.m0) return;
  const int col4 = ch * 32 + lane;
  const bool colok = col4 < D::S0 / 4;
  auto row = [&](int c) { return D0acc + (static_cast<int64_t>(c) * g.m0 + i0) * D::S0; };
  for (int c0 = wid * 32; c0 < nbwd; c0 += NW * 32) {
    const int c = c0 + lane;
    const unsigned live =
        __ballot_sync(0xffffffffu, c < nbwd && d0mask[static_cast<int64_t>(c) * g.m0 + i0] != 0);
    touched |= live != 0;
    sum_live(live, c0, col4, colok, row, acc);
  }
  fold_store<D::S0>(acc, touched, red, cores + g.coff0 + static_cast<int64_t>(i0) * D::S0,
                    grads + g.coff0 + static_cast<int64_t>(i0) * D::S0, col4, MODE, lr,
                    &touched_sm);
}

}  // namespace f3
}  // namespace ttgpu
