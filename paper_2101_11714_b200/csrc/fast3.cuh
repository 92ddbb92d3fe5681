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
template <typename T>
__global__ void __launch_bounds__(512) f3_hist(Geo g, const int64_t* __restrict__ idx, int64_t L,
                                               int TL, int NT, const int64_t* __restrict__ off,
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
    for (int i = threadIdx.x; i < TL; i += blockDim.x) {  // TL % blockDim == 0: warp-uniform
      const int64_t l = static_cast<int64_t>(tile) * TL + i;
      uint32_t k = 0xffffffffu;
      if (l < L) {
        int64_t row = idx[l];
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
    for (int k = threadIdx.x; k < g.K; k += blockDim.x) hist[static_cast<int64_t>(k) * NT + tile] = shist[k];
  // bags (grid-stride over all CTAs)
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
// One CTA of 1024 threads.  hist (K x NT, key-major) becomes exclusive offsets.
__global__ void __launch_bounds__(1024) f3_scan(Geo g, int NT, int TT, int64_t L,
                                                uint32_t* __restrict__ hist,
                                                int32_t* __restrict__ tile_base,
                                                Tile* __restrict__ tiles, int* __restrict__ ntiles) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int n = g.K * NT;
  const int per = (n + 1023) / 1024;
  const int lo = min(n, static_cast<int>(threadIdx.x) * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (int i = lo; i < hi; ++i) s += hist[i];
  uint32_t ex;
  Scan(tmp).ExclusiveSum(s, ex);
  __syncthreads();
  for (int i = lo; i < hi; ++i) {
    const uint32_t c = hist[i];
    hist[i] = ex;
    ex += c;
  }
  __syncthreads();
  // tiles per bucket
  const int perk = (g.K + 1023) / 1024;
  const int klo = min(g.K, static_cast<int>(threadIdx.x) * perk), khi = min(g.K, klo + perk);
  uint32_t nt = 0;
  for (int k = klo; k < khi; ++k) {
    const uint32_t bs = hist[static_cast<int64_t>(k) * NT];
    const uint32_t be = k + 1 < g.K ? hist[static_cast<int64_t>(k + 1) * NT] : static_cast<uint32_t>(L);
    nt += (be - bs + TT - 1) / TT;
  }
  uint32_t tex;
  __syncthreads();
  Scan(tmp).ExclusiveSum(nt, tex);
  for (int k = klo; k < khi; ++k) {
    const uint32_t bs = hist[static_cast<int64_t>(k) * NT];
    const uint32_t be = k + 1 < g.K ? hist[static_cast<int64_t>(k + 1) * NT] : static_cast<uint32_t>(L);
    tile_base[k] = static_cast<int32_t>(tex);
    for (uint32_t st = bs; st < be; st += TT) {
      Tile t;
      t.key = k;
      t.start = static_cast<int>(st);
      t.end = static_cast<int>(min(be, st + TT));
      t.pad = 0;
      tiles[tex++] = t;
    }
  }
  if (threadIdx.x == 1023) {
    tile_base[g.K] = static_cast<int32_t>(tex);
    *ntiles = static_cast<int>(tex);
  }
}

// ---------------------------------------------------------- f3_scatter ---
// Stable scatter: 8 warps per CTA, each owning TL/8 consecutive lookups.
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
  for (int r = 0; r < per; r += 32) {
    const int64_t l = base + r + lane;
    const uint32_t k = l < L ? key[l] : 0xffffffffu;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    if (k != 0xffffffffu && lane == __ffs(peers) - 1) my[k] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int k = threadIdx.x; k < g.K; k += blockDim.x) {
    uint32_t run = hoff[static_cast<int64_t>(k) * NT + tile];
    for (int w = 0; w < 8; ++w) {
      const uint32_t c = wc[static_cast<int64_t>(w) * g.K + k];
      wc[static_cast<int64_t>(w) * g.K + k] = run;
      run += c;
    }
  }
  __syncthreads();
  const unsigned lt = lanemask_lt();
  for (int r = 0; r < per; r += 32) {
    const int64_t l = base + r + lane;
    const uint32_t k = l < L ? key[l] : 0xffffffffu;
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

// --------------------------------------------------------- smem layouts ---
template <class D>
struct FwdSmem {
  // floats: G1s[S1] | Hs[TT*W1P] | G0s[TT*S0P] | G2s[TT*S2P] ; ints after
  static __host__ __device__ size_t floats() {
    return D::S1 + static_cast<size_t>(D::TT) * (D::W1P + D::S0P + D::S2P);
  }
  static __host__ __device__ size_t bytes(int m0) {
    return floats() * 4 + sizeof(int) * (static_cast<size_t>(m0) + 5 * D::TT + 40);
  }
};

// ------------------------------------------------------------- f3_fwd ----
// Per tile: stage G1[i1]; dedup i0 -> slots (numbered by ascending i0 -> the
// same numbering in backward); H(slot); y per lookup.  Saves H, slot maps.
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
  extern __shared__ __align__(16) float sm[];
  float* G1s = sm;
  float* Hs = G1s + D::S1;
  float* G0s = Hs + D::TT * D::W1P;
  float* G2s = G0s + D::TT * D::S0P;
  int* flags = reinterpret_cast<int*>(G2s + D::TT * D::S2P);
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
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const Tile tl = tiles[t];
    const int i1 = tl.key % g.m1;
    const int ntl = tl.end - tl.start;
    {
      const float4* src = reinterpret_cast<const float4*>(G1 + static_cast<int64_t>(i1) * D::S1);
      for (int e = tid; e < D::S1 / 4; e += kThreads) reinterpret_cast<float4*>(G1s)[e] = src[e];
    }
    for (int i = tid; i < g.m0; i += kThreads) flags[i] = 0;
    __syncthreads();
    for (int i = tid; i < ntl; i += kThreads) {
      const int l = static_cast<int>(perm[tl.start + i]);
      lk_l[i] = l;
      const int i0 = d0[l];
      lk_i0[i] = i0;
      const int i2 = d2[l];
      lk_i2[i] = i2;
      flags[i0] = 1;
      // stage G2[i2] (float4 rows, padded stride)
    }
    __syncthreads();
    // slot numbering: ascending i0 (deterministic)
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
        } else {
          flags[i] = -1;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < ntl; i += kThreads) lk_slot[i] = flags[lk_i0[i]];
    for (int e = tid; e < nslots * D::S0; e += kThreads) {
      const int s = e / D::S0, q = e - s * D::S0;
      G0s[s * D::S0P + q] = G0[static_cast<int64_t>(slot_i0[s]) * D::S0 + q];
    }
    for (int e = tid; e < ntl * (D::S2 / 4); e += kThreads) {
      const int i = e / (D::S2 / 4), q = e - i * (D::S2 / 4);
      reinterpret_cast<float4*>(G2s + i * D::S2P)[q] =
          reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(lk_i2[i]) * D::S2)[q];
    }
    __syncthreads();
    // H(slot) = G0[i0] (P0 x R1) · G1[i1] (R1 x C1): thread -> (slot, 4 columns), all P0 rows
    for (int q = tid; q < nslots * D::C4; q += kThreads) {
      const int s = q / D::C4, c4 = q - s * D::C4;
      float4 acc[D::P0];
#pragma unroll
      for (int a = 0; a < D::P0; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      const float* g0 = G0s + s * D::S0P;
#pragma unroll 8
      for (int p = 0; p < D::R1; ++p) {
        const float4 b = reinterpret_cast<const float4*>(G1s + p * D::C1)[c4];
#pragma unroll
        for (int a = 0; a < D::P0; ++a) acc[a] = madd4<float, kExact>(g0[a * D::R1 + p], b, acc[a]);
      }
      float* hrow = Hs + s * D::W1P;
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
    for (int s = tid; s < nslots; s += kThreads) tile_i0[tl.start + s] = static_cast<uint16_t>(slot_i0[s]);
    for (int i = tid; i < ntl; i += kThreads) slot_of_pos[tl.start + i] = static_cast<uint16_t>(lk_slot[i]);
    if (tid == 0) tile_nslots[t] = nslots;
    __syncthreads();
    // y = H(slot) (P1 x R2) · G2[i2] (R2 x N2): thread -> (lookup, row a)
    for (int q = tid; q < ntl * D::P1; q += kThreads) {
      const int i = q / D::P1, a = q - i * D::P1;
      const float* hrow = Hs + lk_slot[i] * D::W1P + a * D::R2;
      const float4* g2 = reinterpret_cast<const float4*>(G2s + i * D::S2P);
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
      for (int r = 0; r < D::R2; ++r) acc = madd4<float, kExact>(hrow[r], g2[r], acc);
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
  // floats: G1s[R1*C1P] | A[TT*W1P] (H then S) | Bq[max(BLK*S2, TT*S2P)] (P2 then G2s)
  //         | D2s[TT*N] | G0s[TT*S0P] ; ints after
  static __host__ __device__ size_t floats(int blk) {
    const size_t b1 = static_cast<size_t>(blk) * D::S2, b2 = static_cast<size_t>(D::TT) * D::S2P;
    return static_cast<size_t>(D::R1) * D::C1P + static_cast<size_t>(D::TT) * D::W1P +
           (b1 > b2 ? b1 : b2) + static_cast<size_t>(D::TT) * (D::N + D::S0P);
  }
  static __host__ __device__ size_t bytes(int m0, int blk) {
    return floats(blk) * 4 + sizeof(int) * (static_cast<size_t>(m0) + 4 * D::TT + 8);
  }
};

template <class D>
__global__ void __launch_bounds__(kThreads) f3_bwd(
    Geo g, const float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const uint32_t* __restrict__ perm,
    const uint16_t* __restrict__ d2, const int32_t* __restrict__ lk_bag,
    const float* __restrict__ alpha, const float* __restrict__ grad,
    const float* __restrict__ Hbuf, const uint16_t* __restrict__ slot_of_pos,
    const uint16_t* __restrict__ tile_i0, const int* __restrict__ tile_nslots,
    float* __restrict__ part1, float* __restrict__ part2, unsigned long long* __restrict__ mask2,
    float* __restrict__ D0buf, int* __restrict__ tab0, int tab_stride) {
  extern __shared__ __align__(16) float sm[];
  float* G1s = sm;                                   // R1 x C1P
  float* A = G1s + D::R1 * D::C1P;                   // TT x W1P  (H, then S)
  float* Bq = A + D::TT * D::W1P;                    // P2 (BLK x S2), then G2s (TT x S2P)
  const int bq = (g.blk * D::S2 > D::TT * D::S2P) ? g.blk * D::S2 : D::TT * D::S2P;
  float* D2s = Bq + bq;                              // TT x N
  float* G0s = D2s + D::TT * D::N;                   // TT x S0P
  int* slotmap = reinterpret_cast<int*>(G0s + D::TT * D::S0P);  // m0
  int* lk_slot = slotmap + g.m0;
  int* lk_i2 = lk_slot + D::TT;
  int* lk_l = lk_i2 + D::TT;
  int* slot_i0 = lk_l + D::TT;
  unsigned long long* tmask = reinterpret_cast<unsigned long long*>(slot_i0 + D::TT + 2);
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  const int nt = *ntiles;
  const int tid = threadIdx.x;
  for (int t = blockIdx.x; t < nt; t += gridDim.x) {
    const Tile tl = tiles[t];
    const int i1 = tl.key % g.m1;
    const int i2base = (tl.key / g.m1) * g.blk;
    const int ntl = tl.end - tl.start;
    const int nslots = tile_nslots[t];
    for (int e = tid; e < D::S1; e += kThreads) {
      const int r = e / D::C1, c = e - r * D::C1;
      G1s[r * D::C1P + c] = G1[static_cast<int64_t>(i1) * D::S1 + e];
    }
    for (int i = tid; i < g.m0; i += kThreads) slotmap[i] = -1;
    for (int e = tid; e < g.blk * D::S2; e += kThreads) Bq[e] = 0.f;
    if (tid == 0) *tmask = 0ull;
    for (int i = tid; i < ntl; i += kThreads) {
      const int l = static_cast<int>(perm[tl.start + i]);
      lk_l[i] = l;
      lk_i2[i] = d2[l];
      lk_slot[i] = slot_of_pos[tl.start + i];
    }
    __syncthreads();
    for (int s = tid; s < nslots; s += kThreads) {
      const int i0 = tile_i0[tl.start + s];
      slot_i0[s] = i0;
      slotmap[i0] = s;
    }
    for (int e = tid; e < ntl * D::N; e += kThreads) {
      const int i = e / D::N, j = e - i * D::N;
      const int l = lk_l[i];
      D2s[e] = __fmul_rn(alpha[l], grad[static_cast<int64_t>(lk_bag[l]) * D::N + j]);
    }
    for (int e = tid; e < nslots * D::W1; e += kThreads) {
      const int s = e / D::W1, q = e - s * D::W1;
      A[s * D::W1P + q] = Hbuf[static_cast<int64_t>(tl.start + s) * D::W1 + q];
    }
    __syncthreads();
    // dG2 partial: slice j = i2 - i2base, element e = (r, j2); groups split lookups by i2 parity
    {
      constexpr int NG = kThreads / D::S2 > 0 ? kThreads / D::S2 : 1;
      const int e = tid % D::S2, grp = tid / D::S2;
      if (grp < NG) {
        const int r = e / D::N2, j2 = e - r * D::N2;
        for (int i = 0; i < ntl; ++i) {
          const int j = lk_i2[i] - i2base;
          if (j % NG != grp) continue;
          const float* hrow = A + lk_slot[i] * D::W1P + r;
          const float* d = D2s + i * D::N + j2;
          float v = Bq[j * D::S2 + e];
#pragma unroll
          for (int a = 0; a < D::P1; ++a) v = __fmaf_rn(hrow[a * D::R2], d[a * D::N2], v);
          Bq[j * D::S2 + e] = v;
        }
      }
      for (int i = tid; i < ntl; i += kThreads) atomicOr(tmask, 1ull << (lk_i2[i] - i2base));
    }
    __syncthreads();
    const unsigned long long tm = *tmask;
    for (int e = tid; e < g.blk * D::S2; e += kThreads) {
      const int j = e / D::S2;
      if ((tm >> j) & 1ull) part2[static_cast<int64_t>(t) * g.blk * D::S2 + e] = Bq[e];
    }
    if (tid == 0) mask2[t] = tm;
    __syncthreads();
    // stage G2 slices (reuse Bq) and zero S (reuse A)
    for (int e = tid; e < ntl * (D::S2 / 4); e += kThreads) {
      const int i = e / (D::S2 / 4), q = e - i * (D::S2 / 4);
      reinterpret_cast<float4*>(Bq + i * D::S2P)[q] =
          reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(lk_i2[i]) * D::S2)[q];
    }
    for (int e = tid; e < nslots * D::W1P; e += kThreads) A[e] = 0.f;
    __syncthreads();
    // S(slot) += D1 = D2 (P1 x N2) · G2[i2]ᵀ (N2 x R2); element e = (a, r); groups by slot parity
    {
      constexpr int NG = kThreads / D::W1 > 0 ? kThreads / D::W1 : 1;
      for (int e0 = tid; e0 < D::W1 * NG; e0 += kThreads) {
        const int e = e0 % D::W1, grp = e0 / D::W1;
        const int a = e / D::R2, r = e - a * D::R2;
        for (int i = 0; i < ntl; ++i) {
          const int s = lk_slot[i];
          if (s % NG != grp) continue;
          const float4 gv = reinterpret_cast<const float4*>(Bq + i * D::S2P)[r];
          const float4 dv = reinterpret_cast<const float4*>(D2s + i * D::N)[a];
          float v = __fmul_rn(dv.x, gv.x);
          v = __fmaf_rn(dv.y, gv.y, v);
          v = __fmaf_rn(dv.z, gv.z, v);
          v = __fmaf_rn(dv.w, gv.w, v);
          A[s * D::W1P + e] += v;
        }
      }
    }
    for (int e = tid; e < nslots * D::S0; e += kThreads) {
      const int s = e / D::S0, q = e - s * D::S0;
      G0s[s * D::S0P + q] = G0[static_cast<int64_t>(slot_i0[s]) * D::S0 + q];
    }
    __syncthreads();
    // dG1 partial (R1 x C1) = Σ_slots G0[i0]ᵀ (R1 x P0) · S (P0 x C1)
    {
      constexpr int PER = D::S1 / kThreads > 0 ? D::S1 / kThreads : 1;
      for (int e0 = tid * PER; e0 < D::S1; e0 += kThreads * PER) {
        const int r1 = e0 / D::C1, c0 = e0 - r1 * D::C1;
        float acc[PER];
#pragma unroll
        for (int x = 0; x < PER; ++x) acc[x] = 0.f;
        for (int s = 0; s < nslots; ++s) {
          const float* srow = A + s * D::W1P;
#pragma unroll
          for (int a = 0; a < D::P0; ++a) {
            const float gv = G0s[s * D::S0P + a * D::R1 + r1];
#pragma unroll
            for (int x = 0; x < PER; ++x) acc[x] = __fmaf_rn(gv, srow[a * D::C1 + c0 + x], acc[x]);
          }
        }
        float* dst = part1 + static_cast<int64_t>(t) * D::S1 + e0;
#pragma unroll
        for (int x = 0; x < PER; ++x) dst[x] = acc[x];
      }
    }
    // D0(slot) (P0 x R1) = S (P0 x C1) · G1[i1]ᵀ (C1 x R1)
    for (int q = tid; q < nslots * D::S0; q += kThreads) {
      const int s = q / D::S0, e = q - s * D::S0;
      const int a = e / D::R1, r1 = e - a * D::R1;
      const float* srow = A + s * D::W1P + a * D::C1;
      const float* grow = G1s + r1 * D::C1P;
      float v = 0.f;
#pragma unroll 8
      for (int c = 0; c < D::C1; ++c) v = __fmaf_rn(srow[c], grow[c], v);
      D0buf[static_cast<int64_t>(tl.start + s) * D::S0 + e] = v;
    }
    for (int i0 = tid; i0 < g.m0; i0 += kThreads)
      tab0[static_cast<int64_t>(i0) * tab_stride + t] = slotmap[i0];
    __syncthreads();
  }
}

// ---------------------------------------------------------- f3_combine ---
// CTA roles: [0, m1) dG1 slices, [m1, m1+m2) dG2 slices, [m1+m2, +m0) dG0.
// MODE 0: dense gradient write (zeros for untouched slices); 1: SGD in place.
template <class D, int MODE>
__global__ void __launch_bounds__(kThreads) f3_combine(
    Geo g, float* __restrict__ cores, float* __restrict__ grads, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const int32_t* __restrict__ tile_base,
    const float* __restrict__ part1, const float* __restrict__ part2,
    const unsigned long long* __restrict__ mask2, const float* __restrict__ D0buf,
    const int* __restrict__ tab0, int tab_stride, float lr) {
  extern __shared__ int lst[];  // compacted (tile, slot) lists
  __shared__ int cnt_sm[40];
  const int tid = threadIdx.x;
  const int nt = *ntiles;
  const int bid = blockIdx.x;
  if (bid < g.m1) {
    const int i1 = bid;
    for (int e = tid; e < D::S1; e += kThreads) {
      float sum = 0.f;
      bool touched = false;
      for (int b = 0; b < g.nblk; ++b) {
        const int key = b * g.m1 + i1;
        for (int t = tile_base[key]; t < tile_base[key + 1]; ++t) {
          sum += part1[static_cast<int64_t>(t) * D::S1 + e];
          touched = true;
        }
      }
      const int64_t o = g.coff1 + static_cast<int64_t>(i1) * D::S1 + e;
      if (MODE == 0)
        grads[o] = sum;
      else if (touched)
        cores[o] = __fadd_rn(cores[o], -__fmul_rn(lr, sum));
    }
    return;
  }
  if (bid < g.m1 + g.m2) {
    const int i2 = bid - g.m1;
    const int b = i2 / g.blk, j = i2 - b * g.blk;
    const int t0 = tile_base[b * g.m1], t1 = tile_base[b * g.m1 + g.m1];
    // compact the tiles that touched slice j, in tile order
    int n = 0;
    for (int base = t0; base < t1; base += kThreads) {
      const int t = base + tid;
      const int f = (t < t1) && ((mask2[t] >> j) & 1ull);
      int tot;
      const int pos = block_excl_scan(f, &tot, cnt_sm);
      if (f) lst[n + pos] = t;
      n += tot;
    }
    __syncthreads();
    constexpr int NG = kThreads / D::S2 > 0 ? kThreads / D::S2 : 1;
    float* red = reinterpret_cast<float*>(lst + n + 4);
    const int e = tid % D::S2, grp = tid / D::S2;
    float sum = 0.f;
    if (grp < NG)
      for (int k = grp; k < n; k += NG)
        sum += part2[(static_cast<int64_t>(lst[k]) * g.blk + j) * D::S2 + e];
    if (grp < NG) red[grp * D::S2 + e] = sum;
    __syncthreads();
    if (tid < D::S2) {
      float s = red[tid];
      for (int q = 1; q < NG; ++q) s += red[q * D::S2 + tid];
      const int64_t o = g.coff2 + static_cast<int64_t>(i2) * D::S2 + tid;
      if (MODE == 0)
        grads[o] = s;
      else if (n > 0)
        cores[o] = __fadd_rn(cores[o], -__fmul_rn(lr, s));
    }
    return;
  }
  const int i0 = bid - g.m1 - g.m2;
  if (i0 >= g.m0) return;
  int n = 0;
  const int* row = tab0 + static_cast<int64_t>(i0) * tab_stride;
  for (int base = 0; base < nt; base += kThreads) {
    const int t = base + tid;
    const int s = t < nt ? row[t] : -1;
    int tot;
    const int pos = block_excl_scan(s >= 0 ? 1 : 0, &tot, cnt_sm);
    if (s >= 0) lst[n + pos] = tiles[t].start + s;
    n += tot;
  }
  __syncthreads();
  constexpr int NG = kThreads / D::S0 > 0 ? kThreads / D::S0 : 1;
  float* red = reinterpret_cast<float*>(lst + n + 4);
  const int e = tid % D::S0, grp = tid / D::S0;
  float sum = 0.f;
  if (grp < NG)
    for (int k = grp; k < n; k += NG) sum += D0buf[static_cast<int64_t>(lst[k]) * D::S0 + e];
  if (grp < NG) red[grp * D::S0 + e] = sum;
  __syncthreads();
  if (tid < D::S0) {
    float s = red[tid];
    for (int q = 1; q < NG; ++q) s += red[q * D::S0 + tid];
    const int64_t o = g.coff0 + static_cast<int64_t>(i0) * D::S0 + tid;
    if (MODE == 0)
      grads[o] = s;
    else if (n > 0)
      cores[o] = __fadd_rn(cores[o], -__fmul_rn(lr, s));
  }
}

}  // namespace f3
}  // namespace ttgpu
