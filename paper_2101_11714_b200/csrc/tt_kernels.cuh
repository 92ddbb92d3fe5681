// sm_100a kernels for the TT-EmbeddingBag hot path.
//
// Algorithm: the reference evaluates the rank-R chain
// G0[i0]·G1[i1]·…·G_{d-1}[i_{d-1}] once per lookup (embedding_ops.hpp:213-229)
// and scatters per-lookup gradients into per-worker dense copies
// (:320-357).  Here the widest, most expensive stage -- the "head"
// H(i0,i1) = G0[i0]·G1[i1] -- is evaluated once per UNIQUE (i0,i1) pair, and
// every gradient is reduced per unique core slice by a deterministic
// sort-by-key / chunked segmented reduction (no floating-point atomics):
//
//   forward : decode -> sort lookups by pair key (i1-major) -> head GEMM per
//             unique pair -> per-bag tail chain + pooling in lookup order
//   backward: S(pair)  = Σ_{lookups of pair} D1          (segmented, by pair)
//             dG_k[i]  = Σ_{lookups with i_k=i} u_{k-1}ᵀ D_k  (segmented, k>=2)
//             dG1[i1]  = Σ_{pairs with i1} G0[i0]ᵀ S      (segmented over pairs)
//             D0(pair) = S · G1[i1]ᵀ ;  dG0[i0] = Σ_{i1} D0   (dense pair table)
//
// All reductions combine their per-chunk partials in a fixed order, so the
// result is bit-reproducible run to run.  Forward kernels take a kExact flag:
// with it, products and sums are separately rounded in the reference's loop
// order (gemm.hpp:15-31, embedding_ops.hpp:232-249), which makes forward and
// lookup_row bit-identical to the reference; without it they use FFMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ttgpu {

constexpr int kMaxD = 8;

// Shape of one table as the kernels see it (shape_plan.hpp:19-46 +
// embedding_ops.hpp:27-47 ChainDims).
struct DevPlan {
  int d;
  int N;                    // emb_dim
  int64_t num_rows;
  int64_t suffix[kMaxD];    // row-digit place values (tt_table.hpp:30-33)
  int m[kMaxD];             // row factors
  int n[kMaxD];             // col factors
  int r[kMaxD + 1];         // ranks
  int prefix[kMaxD];        // prod_{j<=k} n_j
  int slice[kMaxD];         // R_k n_k R_{k+1}
  int64_t coff[kMaxD];      // element offset of core k in the core buffer
  int W1;                   // head width prefix[1]*R_2 (== N when d == 2)
  int C1;                   // G1 slice columns n_1*R_2
  int maxw;                 // max chain width
};

// ---------------------------------------------------------------- helpers --
// Packed fp32 pairs (sm_100a).  fmul2_rn: mul.rn.f32x2 = FMUL2, the same IEEE
// products as two FMULs; exact sums stay scalar (ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2, which would not be bit-exact).
__device__ __forceinline__ float2 fmul2_rn(float a, float2 b) {
  unsigned long long aa, bb, m;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(b.x), "f"(b.y));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(aa), "l"(bb));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(m));
  return r;
}

// (c.x, c.y) += a * (b.x, b.y), one fma.rn.f32x2 (FFMA2): per lane the same
// IEEE fma as __fmaf_rn, half the issue slots.
__device__ __forceinline__ void ffma2(float a, float bx, float by, float& cx, float& cy) {
  unsigned long long aa, bb, cc, d;
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("mov.b64 %0, {%1, %2};" : "=l"(bb) : "f"(bx), "f"(by));
  asm("mov.b64 %0, {%1, %2};" : "=l"(cc) : "f"(cx), "f"(cy));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(aa), "l"(bb), "l"(cc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(cx), "=f"(cy) : "l"(d));
}

template <typename T, bool kExact>
__device__ __forceinline__ T madd(T a, T b, T acc);
template <>
__device__ __forceinline__ float madd<float, true>(float a, float b, float acc) {
  return __fadd_rn(acc, __fmul_rn(a, b));
}
template <>
__device__ __forceinline__ float madd<float, false>(float a, float b, float acc) {
  return __fmaf_rn(a, b, acc);
}
template <>
__device__ __forceinline__ double madd<double, true>(double a, double b, double acc) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}
template <>
__device__ __forceinline__ double madd<double, false>(double a, double b, double acc) {
  return __fma_rn(a, b, acc);
}
template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

__device__ __forceinline__ void decode_row(const DevPlan& P, int64_t row, int* dig) {
#pragma unroll
  for (int k = 0; k < kMaxD; ++k) {
    if (k >= P.d) break;
    const int64_t q = row / P.suffix[k];
    dig[k] = static_cast<int>(q);
    row -= q * P.suffix[k];
  }
}

// C[M x Nc] = A[M x K] · B[K x Nc] by one warp, p-ascending accumulation from
// zero per output (gemm.hpp:15-31 order).  A, C: shared; B: global/shared.
template <typename T, bool kExact>
__device__ __forceinline__ void warp_mm(const T* A, const T* __restrict__ B, T* C, int M, int K,
                                        int Nc, int lane) {
  for (int e = lane; e < M * Nc; e += 32) {
    const int i = e / Nc, j = e - i * Nc;
    const T* a = A + i * K;
    T acc = T(0);
    for (int p = 0; p < K; ++p) acc = madd<T, kExact>(a[p], B[p * Nc + j], acc);
    C[e] = acc;
  }
}

// C[M x K] = A[M x Nc] · B[K x Nc]ᵀ by one warp (gemm.hpp:47-60 order).
template <typename T>
__device__ __forceinline__ void warp_mm_abt(const T* A, const T* __restrict__ B, T* C, int M,
                                            int Nc, int K, int lane) {
  for (int e = lane; e < M * K; e += 32) {
    const int i = e / K, q = e - i * K;
    const T* a = A + i * Nc;
    const T* b = B + q * Nc;
    T acc = T(0);
    for (int j = 0; j < Nc; ++j) acc = madd<T, false>(a[j], b[j], acc);
    C[e] = acc;
  }
}

// ---------------------------------------------------------- batch decode --
// One pass over the lookups: range check (index_batch.hpp:49-54 -- the first
// offending lookup is latched), mixed-radix decode, pair key (i1-major so
// pairs sharing G1[i1] are adjacent after sorting) and tail digits.
__global__ void k_decode(DevPlan P, const int64_t* __restrict__ idx, int64_t L,
                         uint32_t* __restrict__ pair_key, uint32_t* __restrict__ iota,
                         uint32_t* __restrict__ tail_dig, unsigned long long* __restrict__ bad) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
       l += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = idx[l];
    if (row < 0 || row >= P.num_rows) {
      atomicMin(bad, static_cast<unsigned long long>(l));
      row = 0;
    }
    int dig[kMaxD];
    decode_row(P, row, dig);
    pair_key[l] = static_cast<uint32_t>(dig[1]) * static_cast<uint32_t>(P.m[0]) +
                  static_cast<uint32_t>(dig[0]);
    iota[l] = static_cast<uint32_t>(l);
    for (int k = 2; k < P.d; ++k) tail_dig[(k - 2) * L + l] = static_cast<uint32_t>(dig[k]);
  }
}

// Per bag: structural offsets checks (index_batch.hpp:42-46), lookup->bag map
// and the backward scale alpha = T(w / bag_size) computed in double
// (embedding_ops.hpp:329-333).
template <typename T>
__global__ void k_bags(const int64_t* __restrict__ off, int64_t B, int64_t L,
                       const double* __restrict__ w, int mean, int32_t* __restrict__ lk_bag,
                       T* __restrict__ lk_alpha, int* __restrict__ err_struct) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = off[b], e = off[b + 1];
    if (b == 0 && s != 0) atomicOr(err_struct, 1);
    if (e < s) atomicOr(err_struct, 2);
    if (b == B - 1 && e != L) atomicOr(err_struct, 4);
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    const double inv = mean ? static_cast<double>(e - s) : 1.0;
    for (int64_t l = lo; l < hi; ++l) {
      lk_bag[l] = static_cast<int32_t>(b);
      double a = w ? w[l] : 1.0;
      if (mean) a /= inv;
      lk_alpha[l] = static_cast<T>(a);
    }
  }
}

// ---------------------------------------------- segment / run bookkeeping --
// Items sorted by key are cut into fixed chunks of C positions; a "run" is a
// maximal piece of one segment inside one chunk.  packed[s] = head | run-head<<32
// is scanned (inclusive) to give segment and run ordinals per position.
__global__ void k_run_flags(const uint32_t* __restrict__ keys, const int* __restrict__ n_dev,
                            int64_t n_host, int C, unsigned long long* __restrict__ packed) {
  const int64_t n = n_dev ? *n_dev : n_host;
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n_host;
       s += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = 0;
    if (s < n) {
      const bool head = (s == 0) || keys[s] != keys[s - 1];
      const bool run = head || (s % C == 0);
      v = (head ? 1ull : 0ull) | ((run ? 1ull : 0ull) << 32);
    }
    packed[s] = v;
  }
}

// Unique pairs from the sorted lookup keys.
__global__ void k_pairs_compact(const uint32_t* __restrict__ s_key,
                                const uint32_t* __restrict__ s_lk,
                                const unsigned long long* __restrict__ scan, int64_t L,
                                uint32_t* __restrict__ pair_key_u, int32_t* __restrict__ pair_start,
                                int32_t* __restrict__ lk_pid,
                                int* __restrict__ counts /* [0]=U, [1]=runs */) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < L;
       s += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = scan[s];
    const int pid = static_cast<int>(v & 0xffffffffull) - 1;
    const uint32_t key = s_key[s];
    if (s == 0 || s_key[s - 1] != key) {
      pair_key_u[pid] = key;
      pair_start[pid] = static_cast<int32_t>(s);
    }
    lk_pid[s_lk[s]] = pid;
    if (s == L - 1) {
      counts[0] = pid + 1;
      counts[1] = static_cast<int>(v >> 32);
      pair_start[pid + 1] = static_cast<int32_t>(L);
    }
  }
}

// CSR over a dense key space [0, K) from keys sorted ascending: seg[v] = first
// position with key >= v, seg[K] = n.
__global__ void k_key_bounds(const uint32_t* __restrict__ keys, const int* __restrict__ n_dev,
                             int64_t n_host, int K, int32_t* __restrict__ seg) {
  const int64_t n = n_dev ? *n_dev : n_host;
  if (n == 0) {
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v <= K; v += gridDim.x * blockDim.x)
      seg[v] = 0;
    return;
  }
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n;
       s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = keys[s];
    const int64_t prev = s == 0 ? -1 : static_cast<int64_t>(keys[s - 1]);
    for (int64_t v = prev + 1; v <= k; ++v) seg[v] = static_cast<int32_t>(s);
    if (s == n - 1)
      for (int64_t v = k + 1; v <= K; ++v) seg[v] = static_cast<int32_t>(n);
  }
}

// Dense pair table key -> pid for this context's pairs (the table is shared
// by all contexts of a table, so it is refreshed before each backward).
__global__ void k_pair_scatter(const uint32_t* __restrict__ pair_key_u,
                               const int* __restrict__ counts, int64_t cap,
                               int32_t* __restrict__ pair_tab) {
  const int U = counts[0];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cap && p < U;
       p += (int64_t)gridDim.x * blockDim.x)
    pair_tab[pair_key_u[p]] = static_cast<int32_t>(p);
}

// i1 of each unique pair (pid order == (i1, i0) order).
__global__ void k_pair_i1(const uint32_t* __restrict__ pair_key_u, const int* __restrict__ counts,
                          int64_t cap, int m0, uint32_t* __restrict__ out) {
  const int U = counts[0];
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cap;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = p < U ? pair_key_u[p] / static_cast<uint32_t>(m0) : 0xffffffffu;
}

// ------------------------------------------------------------ forward: head --
// H[pid] = G0[i0] (P0 x R1) · G1[i1] (R1 x C1) for every unique pair.  Pairs
// are processed in chunks of CH; G1[i1] is staged in shared memory once per
// i1 run inside the chunk (pairs are i1-major, so runs are long).
__device__ __forceinline__ void cp_async16_g(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <typename T, bool kExact>
__global__ void k_head_fwd(DevPlan P, const T* __restrict__ cores,
                           const uint32_t* __restrict__ pair_key_u,
                           const int* __restrict__ counts, int CH, T* __restrict__ H) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* g1s = reinterpret_cast<T*>(smem_raw);                 // R1 x C1
  T* g0s = g1s + P.r[1] * P.C1;                            // CH x P0 x R1
  const int U = counts[0];
  const int P0 = P.n[0], R1 = P.r[1], C1 = P.C1;
  const int s0 = P.slice[0], s1 = P.slice[1];
  const T* G0 = cores + P.coff[0];
  const T* G1 = cores + P.coff[1];
  const int nchunks = (U + CH - 1) / CH;
  // contiguous chunk ranges per CTA: consecutive chunks usually share i1 (pairs
  // are i1-major), so the staged G1[i1] is reused across them
  const int ch_lo = static_cast<int>(static_cast<int64_t>(blockIdx.x) * nchunks / gridDim.x);
  const int ch_hi = static_cast<int>(static_cast<int64_t>(blockIdx.x + 1) * nchunks / gridDim.x);
  // fp32 operands with 16-byte rows are staged by cp.async (no register round trip)
  bool async16 = false;
  if constexpr (std::is_same_v<T, float>) async16 = (s0 % 4) == 0 && (s1 % 4) == 0;
  uint32_t staged_i1 = 0xffffffffu;
  for (int ch = ch_lo; ch < ch_hi; ++ch) {
    const int p0 = ch * CH, p1 = min(U, p0 + CH);
    __syncthreads();
    if (async16) {
      const int q4 = s0 / 4;
      for (int e = threadIdx.x; e < (p1 - p0) * q4; e += blockDim.x) {
        const int q = e / q4;
        const uint32_t i0 = pair_key_u[p0 + q] % static_cast<uint32_t>(P.m[0]);
        cp_async16_g(g0s + 4 * e, G0 + static_cast<int64_t>(i0) * s0 + 4 * (e - q * q4));
      }
    } else {
      for (int e = threadIdx.x; e < (p1 - p0) * s0; e += blockDim.x) {
        const int q = e / s0;
        const uint32_t i0 = pair_key_u[p0 + q] % static_cast<uint32_t>(P.m[0]);
        g0s[e] = G0[i0 * s0 + (e - q * s0)];
      }
    }
    int run_lo = p0;
    while (run_lo < p1) {
      const uint32_t i1 = pair_key_u[run_lo] / static_cast<uint32_t>(P.m[0]);
      int run_hi = run_lo + 1;
      while (run_hi < p1 && pair_key_u[run_hi] / static_cast<uint32_t>(P.m[0]) == i1) ++run_hi;
      __syncthreads();
      if (i1 != staged_i1) {
        if (async16) {
          for (int e = threadIdx.x; e < s1 / 4; e += blockDim.x)
            cp_async16_g(g1s + 4 * e, G1 + static_cast<int64_t>(i1) * s1 + 4 * e);
        } else {
          for (int e = threadIdx.x; e < s1; e += blockDim.x) g1s[e] = G1[(int64_t)i1 * s1 + e];
        }
        staged_i1 = i1;
      }
      if (async16) cp_async_wait_all();
      __syncthreads();
      const int outs = P0 * C1;
      bool quad_done = false, block4 = false;
      if constexpr (std::is_same_v<T, float>) {
        quad_done = (C1 & 3) == 0;
        block4 = quad_done && P0 == 4;
      }
      if (block4) {
        // fp32, P0 == 4 (cfg3): a thread owns all 4 rows x 4 adjacent columns
        // of one pair; per p one 16-byte G1 load and the 4 G0 values (read as
        // broadcasts) feed 16 products -- the same per-element p-ascending chain
        const int C4 = C1 >> 2;
        for (int e = threadIdx.x; e < (run_hi - run_lo) * C4; e += blockDim.x) {
          const int q = e / C4, c = (e - q * C4) * 4;
          const float* arow = reinterpret_cast<const float*>(g0s) + (run_lo - p0 + q) * s0;
          const float* gcol = reinterpret_cast<const float*>(g1s) + c;
          float v[4][4];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int u = 0; u < 4; ++u) v[a][u] = 0.f;
#pragma unroll 4
          for (int p = 0; p < R1; ++p) {
            const float4 g = *reinterpret_cast<const float4*>(gcol + p * C1);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
              const float x = arow[a * R1 + p];
              if (kExact) {
                const float2 p01 = fmul2_rn(x, make_float2(g.x, g.y));
                const float2 p23 = fmul2_rn(x, make_float2(g.z, g.w));
                v[a][0] = __fadd_rn(v[a][0], p01.x);
                v[a][1] = __fadd_rn(v[a][1], p01.y);
                v[a][2] = __fadd_rn(v[a][2], p23.x);
                v[a][3] = __fadd_rn(v[a][3], p23.y);
              } else {
                ffma2(x, g.x, g.y, v[a][0], v[a][1]);
                ffma2(x, g.z, g.w, v[a][2], v[a][3]);
              }
            }
          }
          float* hrow = reinterpret_cast<float*>(H) + static_cast<int64_t>(run_lo + q) * P.W1 + c;
#pragma unroll
          for (int a = 0; a < 4; ++a)
            *reinterpret_cast<float4*>(hrow + a * C1) = make_float4(v[a][0], v[a][1], v[a][2], v[a][3]);
        }
      } else if (quad_done) {
        // fp32: four adjacent columns per thread, products two at a time
        // (FMUL2 / FFMA2), the same per-element p-ascending chain
        const int outs4 = outs >> 2;
        for (int e = threadIdx.x; e < (run_hi - run_lo) * outs4; e += blockDim.x) {
          const int q = e / outs4, rem = (e - q * outs4) * 4;
          const int a = rem / C1, c = rem - a * C1;
          const float* arow = reinterpret_cast<const float*>(g0s) + (run_lo - p0 + q) * s0 + a * R1;
          const float* gcol = reinterpret_cast<const float*>(g1s) + c;
          float v[4] = {0.f, 0.f, 0.f, 0.f};
          for (int p = 0; p < R1; ++p) {
            const float4 g = *reinterpret_cast<const float4*>(gcol + p * C1);
            const float x = arow[p];
            if (kExact) {
              const float2 p01 = fmul2_rn(x, make_float2(g.x, g.y));
              const float2 p23 = fmul2_rn(x, make_float2(g.z, g.w));
              v[0] = __fadd_rn(v[0], p01.x);
              v[1] = __fadd_rn(v[1], p01.y);
              v[2] = __fadd_rn(v[2], p23.x);
              v[3] = __fadd_rn(v[3], p23.y);
            } else {
              ffma2(x, g.x, g.y, v[0], v[1]);
              ffma2(x, g.z, g.w, v[2], v[3]);
            }
          }
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(H) + static_cast<int64_t>(run_lo + q) * P.W1 +
                                     rem) = make_float4(v[0], v[1], v[2], v[3]);
        }
      } else {
        for (int e = threadIdx.x; e < (run_hi - run_lo) * outs; e += blockDim.x) {
          const int q = e / outs, rem = e - q * outs;
          const int a = rem / C1, c = rem - a * C1;
          const T* arow = g0s + (run_lo - p0 + q) * s0 + a * R1;
          T acc = T(0);
          for (int p = 0; p < R1; ++p) acc = madd<T, kExact>(arow[p], g1s[p * C1 + c], acc);
          H[static_cast<int64_t>(run_lo + q) * P.W1 + rem] = acc;
        }
      }
      run_lo = run_hi;
    }
  }
}

// ---------------------------------------------------- forward: tail + pool --
// One warp per bag: for each lookup in ascending order, chain the head row
// through G_2..G_{d-1} and pool out[b] += T(w)·y (embedding_ops.hpp:232-237),
// then the Mean rescale (:240-249).  Saves u_k (2 <= k <= d-2) when requested.
template <typename T, bool kExact>
__global__ void k_tail_pool(DevPlan P, const T* __restrict__ cores, const T* __restrict__ H,
                            const int32_t* __restrict__ lk_pid, const uint32_t* __restrict__ tail_dig,
                            const int64_t* __restrict__ off, int64_t B, int64_t L,
                            const double* __restrict__ w, int mean, T* __restrict__ out,
                            T* __restrict__ saved /* (d-3) x L x maxw or null */) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* buf = reinterpret_cast<T*>(smem_raw) + static_cast<int64_t>(wid) * (2 * P.maxw + P.N);
  T* ping = buf;
  T* pong = buf + P.maxw;
  T* acc = buf + 2 * P.maxw;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * warps + wid; b < B;
       b += static_cast<int64_t>(gridDim.x) * warps) {
    for (int j = lane; j < P.N; j += 32) acc[j] = T(0);
    const int64_t s = off[b], e = off[b + 1];
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    for (int64_t l = lo; l < hi; ++l) {
      const T* u = H + static_cast<int64_t>(lk_pid[l]) * P.W1;
      if (P.d > 2) {
        const T* src = u;
        T* dst = ping;
        for (int k = 2; k < P.d; ++k) {
          const int i_k = static_cast<int>(tail_dig[(k - 2) * L + l]);
          const T* G = cores + P.coff[k] + static_cast<int64_t>(i_k) * P.slice[k];
          __syncwarp();
          warp_mm<T, kExact>(src, G, dst, P.prefix[k - 1], P.r[k], P.n[k] * P.r[k + 1], lane);
          __syncwarp();
          if (saved && k <= P.d - 2) {
            const int wk = P.prefix[k] * P.r[k + 1];
            T* sv = saved + (static_cast<int64_t>(k - 2) * L + l) * P.maxw;
            for (int x = lane; x < wk; x += 32) sv[x] = dst[x];
          }
          src = dst;
          dst = (dst == ping) ? pong : ping;
        }
        u = src;
      }
      const T a = static_cast<T>(w ? w[l] : 1.0);
      for (int j = lane; j < P.N; j += 32) acc[j] = madd<T, kExact>(a, u[j], acc[j]);
      __syncwarp();
    }
    T scale = T(1);
    const bool do_scale = mean && (e - s) > 1;
    if (do_scale) scale = static_cast<T>(1.0 / static_cast<double>(e - s));
    for (int j = lane; j < P.N; j += 32)
      out[b * P.N + j] = do_scale ? mul_rn<T>(acc[j], scale) : acc[j];
    __syncwarp();
  }
}

// ------------------------------------------------ backward: chain helpers --
// D_{k-1} = D_k · G_k[i_k]ᵀ for k = kfrom..kto+1 (descending), starting from
// D_{d-1} = alpha * g[bag].  Result left in *res (ping/pong owned by caller).
template <typename T>
__device__ __forceinline__ const T* bwd_chain(const DevPlan& P, const T* __restrict__ cores,
                                              const uint32_t* __restrict__ tail_dig, int64_t L,
                                              int64_t l, const T* __restrict__ grow, T alpha,
                                              int kto, T* ping, T* pong, int lane) {
  for (int j = lane; j < P.N; j += 32) ping[j] = mul_rn<T>(alpha, grow[j]);
  __syncwarp();
  T* cur = ping;
  T* nxt = pong;
  for (int k = P.d - 1; k > kto; --k) {
    const int i_k = static_cast<int>(tail_dig[(k - 2) * L + l]);
    const T* G = cores + P.coff[k] + static_cast<int64_t>(i_k) * P.slice[k];
    warp_mm_abt<T>(cur, G, nxt, P.prefix[k - 1], P.n[k] * P.r[k + 1], P.r[k], lane);
    __syncwarp();
    T* t = cur;
    cur = nxt;
    nxt = t;
  }
  return cur;
}

// u_{kk} for one lookup from its head row (forward chain k = 2..kk), or the
// saved partial.
template <typename T>
__device__ __forceinline__ const T* fwd_partial(const DevPlan& P, const T* __restrict__ cores,
                                                const T* __restrict__ H, const int32_t* lk_pid,
                                                const uint32_t* __restrict__ tail_dig, int64_t L,
                                                int64_t l, int kk, const T* __restrict__ saved,
                                                T* ping, T* pong, int lane, bool exact) {
  const T* src = H + static_cast<int64_t>(lk_pid[l]) * P.W1;
  if (kk <= 1) return src;
  if (saved) return saved + (static_cast<int64_t>(kk - 2) * L + l) * P.maxw;
  T* dst = ping;
  for (int k = 2; k <= kk; ++k) {
    const int i_k = static_cast<int>(tail_dig[(k - 2) * L + l]);
    const T* G = cores + P.coff[k] + static_cast<int64_t>(i_k) * P.slice[k];
    // same rounding as the forward that produced (or would have saved) it
    if (exact)
      warp_mm<T, true>(src, G, dst, P.prefix[k - 1], P.r[k], P.n[k] * P.r[k + 1], lane);
    else
      warp_mm<T, false>(src, G, dst, P.prefix[k - 1], P.r[k], P.n[k] * P.r[k + 1], lane);
    __syncwarp();
    src = dst;
    dst = (dst == ping) ? pong : ping;
  }
  return src;
}

// ---------------------------------------- backward: chunked segmented sums --
// Generic chunked reduction over items sorted by segment.  Each CTA owns one
// chunk of C consecutive sorted positions; each of its warps produces the
// contribution vector (width Wc) of one item into a shared slot; the CTA then
// folds the slots in position order into a shared accumulator and emits one
// partial per run.  MODE selects the contribution:
//   0: S pairs   item = lookup (pair order)    contrib = D1 (P1 x R2) [d>=3], alpha*g [d==2]
//   1: tail core item = lookup (i_k order)     contrib = u_{k-1}ᵀ D_k  (R_k x n_k R_{k+1})
template <typename T, int MODE>
__global__ void k_chunk_reduce(DevPlan P, const T* __restrict__ cores, const T* __restrict__ H,
                               const T* __restrict__ saved, const int32_t* __restrict__ lk_pid,
                               const uint32_t* __restrict__ tail_dig, const int32_t* lk_bag,
                               const T* __restrict__ lk_alpha, const T* __restrict__ grad,
                               const uint32_t* __restrict__ s_key, const uint32_t* __restrict__ s_lk,
                               const unsigned long long* __restrict__ scan, int64_t L, int C,
                               int kcore, int Wc, T* __restrict__ partials, bool exact) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* acc = reinterpret_cast<T*>(smem_raw);                  // Wc
  T* slots = acc + Wc;                                      // warps x Wc
  T* scratch = slots + static_cast<int64_t>(warps) * Wc;    // warps x 4 x maxw
  T* my = scratch + static_cast<int64_t>(wid) * 4 * P.maxw;
  const int64_t nchunks = (L + C - 1) / C;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * C, c1 = (L < c0 + C ? L : c0 + C);
    int run = static_cast<int>(scan[c0] >> 32) - 1;
    for (int e = threadIdx.x; e < Wc; e += blockDim.x) acc[e] = T(0);
    for (int64_t g0 = c0; g0 < c1; g0 += warps) {
      const int64_t s = g0 + wid;
      if (s < c1) {
        const int64_t l = s_lk[s];
        const T alpha = lk_alpha[l];
        const T* grow = grad + static_cast<int64_t>(lk_bag[l]) * P.N;
        T* slot = slots + static_cast<int64_t>(wid) * Wc;
        if (MODE == 0) {
          const T* D = bwd_chain<T>(P, cores, tail_dig, L, l, grow, alpha, 1, my, my + P.maxw,
                                    lane);
          for (int e = lane; e < Wc; e += 32) slot[e] = D[e];
        } else {
          // contribution u_{k-1}ᵀ · D_k : (R_k x P_{k-1}) · (P_{k-1} x n_k R_{k+1})
          const T* D = bwd_chain<T>(P, cores, tail_dig, L, l, grow, alpha, kcore, my,
                                    my + P.maxw, lane);
          const T* u = fwd_partial<T>(P, cores, H, lk_pid, tail_dig, L, l, kcore - 1, saved,
                                      my + 2 * P.maxw, my + 3 * P.maxw, lane, exact);
          const int pk = P.prefix[kcore - 1], rk = P.r[kcore], wk = P.n[kcore] * P.r[kcore + 1];
          for (int e = lane; e < rk * wk; e += 32) {
            const int q = e / wk, j = e - q * wk;
            T a = T(0);
            for (int i = 0; i < pk; ++i) a = madd<T, false>(u[i * rk + q], D[i * wk + j], a);
            slot[e] = a;
          }
        }
      }
      __syncthreads();
      const int ng = static_cast<int>((warps < c1 - g0 ? (int64_t)warps : c1 - g0));
      for (int q = 0; q < ng; ++q) {
        const int64_t s = g0 + q;
        const bool new_run = (s != c0) && (s_key[s] != s_key[s - 1]);
        if (new_run) {
          for (int e = threadIdx.x; e < Wc; e += blockDim.x) {
            partials[static_cast<int64_t>(run) * Wc + e] = acc[e];
            acc[e] = T(0);
          }
          ++run;
        }
        const T* slot = slots + static_cast<int64_t>(q) * Wc;
        for (int e = threadIdx.x; e < Wc; e += blockDim.x) acc[e] += slot[e];
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < Wc; e += blockDim.x)
      partials[static_cast<int64_t>(run) * Wc + e] = acc[e];
    __syncthreads();
  }
}

// ------------------------------------- backward, d == 3: staged chunk sums --
// Same contract as k_chunk_reduce (one chunk of C sorted positions per CTA
// iteration, one partial per run, runs numbered from scan[c0] >> 32) and the
// same per-element arithmetic, restructured for wide rows (cfg3: W1 = 1024):
// the chunk's small per-lookup operands are staged once in shared memory and
// every thread keeps ITS output elements of the running sum in registers, so
// no per-lookup row is materialised or folded through shared memory.
//   k_srun3  (S per pair run):   contrib[a][r] = Σ_j D2[a][j] · G2[i2][r][j]
//   k_trun3  (dG2 per i2 run):   contrib[q][j] = Σ_a H[pair][a][q] · D2[a][j]
// D2 = T(alpha) * grad[bag] (bwd_chain), products accumulated from zero with
// FMA in the same order as warp_mm_abt / the MODE 1 loop of k_chunk_reduce.
constexpr int kRun3MaxEPT = 8;   // output elements per thread (row width <= 8 x 256)
constexpr int kQuadPT = 2;       // k_srun3 fp32 quad path: column quads per thread

template <typename T>
__global__ void __launch_bounds__(256) k_srun3(DevPlan P, const T* __restrict__ cores,
                                               const uint32_t* __restrict__ tail_dig,
                                               const int32_t* __restrict__ lk_bag,
                                               const T* __restrict__ lk_alpha,
                                               const T* __restrict__ grad,
                                               const uint32_t* __restrict__ s_key,
                                               const uint32_t* __restrict__ s_lk,
                                               const unsigned long long* __restrict__ scan,
                                               int64_t L, int C, T* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = P.N, R2 = P.r[2], n2 = P.n[2], S2 = P.slice[2], W = P.W1;
  T* d2s = reinterpret_cast<T*>(smem_raw);               // C x N
  T* g2s = d2s + static_cast<int64_t>(C) * N;            // C x S2
  uint32_t* keys = reinterpret_cast<uint32_t*>(g2s + static_cast<int64_t>(C) * S2);  // C
  __shared__ int qbag[64], qi2[64];
  __shared__ T qal[64];
  const T* G2 = cores + P.coff[2];
  const int64_t nchunks = (L + C - 1) / C;
  // quad path (fp32, n2 == 4): a thread owns quads (a, r..r+3); G2 slices are
  // staged transposed ([j][r]) so a quad's 4 columns are one 16-byte load, and
  // the products go two lanes at a time (FFMA2).  Per element the same fma
  // chain over j, then acc += v, as the scalar form.
  const bool quad = std::is_same_v<T, float> && n2 == 4 && (R2 & 3) == 0 && W <= 4 * kQuadPT * 256;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * C;
    const int n = static_cast<int>(L - c0 < C ? L - c0 : C);
    __syncthreads();
    // per-position indices once (one round trip), then the row copies
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int64_t l = s_lk[c0 + q];
      keys[q] = s_key[c0 + q];
      qbag[q] = lk_bag[l];
      qi2[q] = static_cast<int>(tail_dig[l]);
      qal[q] = lk_alpha[l];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < n * N; e += blockDim.x) {
      const int q = e / N, j = e - q * N;
      d2s[e] = mul_rn<T>(qal[q], grad[static_cast<int64_t>(qbag[q]) * N + j]);
    }
    if constexpr (std::is_same_v<T, float>) {
      if (quad) {  // row r of slice i2 -> column r of the [j][r] block
        for (int e = threadIdx.x; e < n * R2; e += blockDim.x) {
          const int q = e / R2, r = e - q * R2;
          const float4 v =
              __ldg(reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(qi2[q]) * S2) + r);
          float* gt = reinterpret_cast<float*>(g2s) + q * S2 + r;
          gt[0] = v.x;
          gt[R2] = v.y;
          gt[2 * R2] = v.z;
          gt[3 * R2] = v.w;
        }
      } else if ((S2 & 3) == 0) {
        const int S4 = S2 >> 2;
        for (int e = threadIdx.x; e < n * S4; e += blockDim.x) {
          const int q = e / S4, j = e - q * S4;
          reinterpret_cast<float4*>(g2s)[e] =
              __ldg(reinterpret_cast<const float4*>(G2 + static_cast<int64_t>(qi2[q]) * S2) + j);
        }
      } else {
        for (int e = threadIdx.x; e < n * S2; e += blockDim.x) {
          const int q = e / S2, j = e - q * S2;
          g2s[e] = G2[static_cast<int64_t>(qi2[q]) * S2 + j];
        }
      }
    } else {
      for (int e = threadIdx.x; e < n * S2; e += blockDim.x) {
        const int q = e / S2, j = e - q * S2;
        g2s[e] = G2[static_cast<int64_t>(qi2[q]) * S2 + j];
      }
    }
    __syncthreads();
    const int run0 = static_cast<int>(scan[c0] >> 32) - 1;
    if constexpr (std::is_same_v<T, float>) {
      if (quad) {
        const int R4 = R2 >> 2, NQ = W >> 2;
        float4 qa[kQuadPT];
        int doff[kQuadPT], goff[kQuadPT], ooff[kQuadPT];
#pragma unroll
        for (int k = 0; k < kQuadPT; ++k) {
          qa[k] = make_float4(0.f, 0.f, 0.f, 0.f);
          const int g = threadIdx.x + k * blockDim.x;
          const int a = g / R4, r4 = g - a * R4;
          doff[k] = a * 4;
          goff[k] = r4 * 4;
          ooff[k] = a * R2 + r4 * 4;
        }
        int run = run0;
        for (int q = 0; q < n; ++q) {
          if (q > 0 && keys[q] != keys[q - 1]) {
#pragma unroll
            for (int k = 0; k < kQuadPT; ++k) {
              if (threadIdx.x + k * blockDim.x < NQ)
                *reinterpret_cast<float4*>(partials + static_cast<int64_t>(run) * W + ooff[k]) = qa[k];
              qa[k] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            ++run;
          }
          const float* d = reinterpret_cast<const float*>(d2s) + q * N;
          const float* gt = reinterpret_cast<const float*>(g2s) + q * S2;
#pragma unroll
          for (int k = 0; k < kQuadPT; ++k) {
            if (threadIdx.x + k * blockDim.x < NQ) {
              const float4 dv = *reinterpret_cast<const float4*>(d + doff[k]);
              const float dj[4] = {dv.x, dv.y, dv.z, dv.w};
              float v0 = 0.f, v1 = 0.f, v2 = 0.f, v3 = 0.f;
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const float4 gv = *reinterpret_cast<const float4*>(gt + j * R2 + goff[k]);
                ffma2(dj[j], gv.x, gv.y, v0, v1);
                ffma2(dj[j], gv.z, gv.w, v2, v3);
              }
              qa[k].x += v0;
              qa[k].y += v1;
              qa[k].z += v2;
              qa[k].w += v3;
            }
          }
        }
#pragma unroll
        for (int k = 0; k < kQuadPT; ++k)
          if (threadIdx.x + k * blockDim.x < NQ)
            *reinterpret_cast<float4*>(partials + static_cast<int64_t>(run) * W + ooff[k]) = qa[k];
        continue;
      }
    }
    T acc[kRun3MaxEPT];
    int aoff[kRun3MaxEPT], roff[kRun3MaxEPT];  // element -> (a*n2, r*n2), hoisted
#pragma unroll
    for (int k = 0; k < kRun3MaxEPT; ++k) {
      acc[k] = T(0);
      const int e = threadIdx.x + k * blockDim.x;
      const int a = e / R2;
      aoff[k] = a * n2;
      roff[k] = (e - a * R2) * n2;
    }
    int run = run0;
    for (int q = 0; q < n; ++q) {
      if (q > 0 && keys[q] != keys[q - 1]) {
#pragma unroll
        for (int k = 0; k < kRun3MaxEPT; ++k) {
          const int e = threadIdx.x + k * blockDim.x;
          if (e < W) partials[static_cast<int64_t>(run) * W + e] = acc[k];
          acc[k] = T(0);
        }
        ++run;
      }
      const T* d = d2s + q * N;
      const T* gg = g2s + q * S2;
#pragma unroll
      for (int k = 0; k < kRun3MaxEPT; ++k) {
        const int e = threadIdx.x + k * blockDim.x;
        if (e < W) {
          T v = T(0);
          if constexpr (std::is_same_v<T, float>) {
            if (n2 == 4) {  // rows of 4: one 16-byte load per operand
              const float4 dv = *reinterpret_cast<const float4*>(d + aoff[k]);
              const float4 gv = *reinterpret_cast<const float4*>(gg + roff[k]);
              v = __fmaf_rn(dv.x, gv.x, v);
              v = __fmaf_rn(dv.y, gv.y, v);
              v = __fmaf_rn(dv.z, gv.z, v);
              v = __fmaf_rn(dv.w, gv.w, v);
              acc[k] += v;
              continue;
            }
          }
          if (n2 == 4) {
#pragma unroll
            for (int j = 0; j < 4; ++j) v = madd<T, false>(d[aoff[k] + j], gg[roff[k] + j], v);
          } else {
            for (int j = 0; j < n2; ++j) v = madd<T, false>(d[aoff[k] + j], gg[roff[k] + j], v);
          }
          acc[k] += v;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kRun3MaxEPT; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < W) partials[static_cast<int64_t>(run) * W + e] = acc[k];
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) k_trun3(DevPlan P, const T* __restrict__ H,
                                               const int32_t* __restrict__ lk_pid,
                                               const int32_t* __restrict__ lk_bag,
                                               const T* __restrict__ lk_alpha,
                                               const T* __restrict__ grad,
                                               const uint32_t* __restrict__ s_key,
                                               const uint32_t* __restrict__ s_lk,
                                               const unsigned long long* __restrict__ scan,
                                               int64_t L, int C, int sub, T* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = P.N, R2 = P.r[2], n2 = P.n[2], P1 = P.prefix[1], W1 = P.W1, Wc = P.slice[2];
  T* hs = reinterpret_cast<T*>(smem_raw);                // sub x W1
  T* d2s = hs + static_cast<int64_t>(sub) * W1;          // sub x N
  uint32_t* keys = reinterpret_cast<uint32_t*>(d2s + static_cast<int64_t>(sub) * N);  // C
  const int64_t nchunks = (L + C - 1) / C;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * C;
    const int n = static_cast<int>(L - c0 < C ? L - c0 : C);
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) keys[q] = s_key[c0 + q];
    const int run0 = static_cast<int>(scan[c0] >> 32) - 1;
    T acc[kRun3MaxEPT];
#pragma unroll
    for (int k = 0; k < kRun3MaxEPT; ++k) acc[k] = T(0);
    int run = run0;
    for (int q0 = 0; q0 < n; q0 += sub) {
      const int m = n - q0 < sub ? n - q0 : sub;
      __syncthreads();  // previous sub-batch consumed (and keys staged)
      for (int e = threadIdx.x; e < m * W1; e += blockDim.x) {
        const int q = e / W1, x = e - q * W1;
        const int64_t l = s_lk[c0 + q0 + q];
        hs[e] = H[static_cast<int64_t>(lk_pid[l]) * W1 + x];
      }
      for (int e = threadIdx.x; e < m * N; e += blockDim.x) {
        const int q = e / N, j = e - q * N;
        const int64_t l = s_lk[c0 + q0 + q];
        d2s[e] = mul_rn<T>(lk_alpha[l], grad[static_cast<int64_t>(lk_bag[l]) * N + j]);
      }
      __syncthreads();
      for (int qq = 0; qq < m; ++qq) {
        const int q = q0 + qq;
        if (q > 0 && keys[q] != keys[q - 1]) {
#pragma unroll
          for (int k = 0; k < kRun3MaxEPT; ++k) {
            const int e = threadIdx.x + k * blockDim.x;
            if (e < Wc) partials[static_cast<int64_t>(run) * Wc + e] = acc[k];
            acc[k] = T(0);
          }
          ++run;
        }
        const T* u = hs + qq * W1;
        const T* d = d2s + qq * N;
#pragma unroll
        for (int k = 0; k < kRun3MaxEPT; ++k) {
          const int e = threadIdx.x + k * blockDim.x;
          if (e < Wc) {
            const int qr = e / n2, j = e - qr * n2;
            T v = T(0);
            for (int i = 0; i < P1; ++i) v = madd<T, false>(u[i * R2 + qr], d[i * n2 + j], v);
            acc[k] += v;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kRun3MaxEPT; ++k) {
      const int e = threadIdx.x + k * blockDim.x;
      if (e < Wc) partials[static_cast<int64_t>(run) * Wc + e] = acc[k];
    }
  }
}

// ------------------------ d == 3, wide rows: work in pair order, H staged --
// The tail contractions need the pair's head row H (P1 x R2; 4 KB at cfg3).
// Walking lookups in i2 order re-reads H per lookup from HBM (H of all pairs
// does not fit L2); walking them in PAIR order stages H once per pair run.
// Per-lookup results go to a buffer (y rows for pooling; dG2 contributions
// at the lookup's position in the i2 order), then a fixed-order segmented
// sum / pooling pass produces the outputs -- deterministic.
__global__ void k_inv_perm(const uint32_t* __restrict__ sorted_lk, int64_t L,
                           uint32_t* __restrict__ pos_of) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < L;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x)
    pos_of[sorted_lk[p]] = static_cast<uint32_t>(p);
}

// MODE 0: y[l][a*n2 + j] = Σ_r H[a][r] · G2[i2][r][j] (forward, kExact rounding)
// MODE 1: C[pos2[l]][q*n2 + j] = Σ_a H[a][q] · D2[a][j]   (dG2 contribution)
// CW (float, n2 % CW == 0): a thread owns CW = 2 or 4 adjacent output columns
// and forms their products two at a time (FMUL2 / FFMA2), same per-element
// arithmetic and order as the scalar form (CW = 1).
template <typename T, int MODE, bool kExact, int CW = 1>
__global__ void __launch_bounds__(256) k_pairwalk3(DevPlan P, const T* __restrict__ cores,
                                                   const T* __restrict__ H,
                                                   const int32_t* __restrict__ lk_pid,
                                                   const uint32_t* __restrict__ tail_dig,
                                                   const int32_t* __restrict__ lk_bag,
                                                   const T* __restrict__ lk_alpha,
                                                   const T* __restrict__ grad,
                                                   const uint32_t* __restrict__ s_lk,
                                                   const uint32_t* __restrict__ pos2, int64_t L,
                                                   int C, T* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = P.N, R2 = P.r[2], n2 = P.n[2], S2 = P.slice[2], W1 = P.W1, P1 = P.prefix[1];
  const int OW = MODE == 0 ? N : S2;             // output row width per lookup
  const int XW = MODE == 0 ? S2 : N;             // per-lookup operand (G2 slice / D2 row)
  // H row staged with an odd pitch per a-row (R2 + 1): MODE 0 lanes read
  // hs[a][r] for 8 different a at once, which would share one bank otherwise
  const int R2p = R2 + 1;
  T* hs = reinterpret_cast<T*>(smem_raw);        // P1 x R2p (current pair's H row)
  T* xs = hs + (P1 * R2p + 3) / 4 * 4;           // C x XW, 16-byte aligned for the vector stores
  __shared__ int cur_pid;
  __shared__ int pids[64];                       // pair of each chunk position (C <= 64)
  __shared__ int qlk[64], qrow[64];              // lookup, G2 slice (MODE 0) / bag (MODE 1)
  __shared__ T qal[64];
  const int64_t nchunks = (L + C - 1) / C;
  const int OWt = OW / CW;  // threads per lookup
  const int per = blockDim.x / OWt > 0 ? blockDim.x / OWt : 1;  // lookups in flight
  const int e = (threadIdx.x % OWt) * CW, slot = threadIdx.x / OWt;
  const bool on_e = threadIdx.x < per * OWt;
  // element -> operand offsets (hoisted)
  const int ra = MODE == 0 ? (e / n2) * R2p : e / n2;  // MODE0: a*R2p  MODE1: q
  const int rj = e % n2;
  if (threadIdx.x == 0) cur_pid = -1;
  for (int64_t ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int64_t c0 = ch * C;
    const int n = static_cast<int>(L - c0 < C ? L - c0 : C);
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += blockDim.x) {  // per-position indices, one round trip
      const int64_t l = s_lk[c0 + q];
      qlk[q] = static_cast<int>(l);
      pids[q] = lk_pid[l];
      qrow[q] = MODE == 0 ? static_cast<int>(tail_dig[l]) : lk_bag[l];
      if (MODE == 1) qal[q] = lk_alpha[l];
    }
    __syncthreads();
    const T* src = MODE == 0 ? cores + P.coff[2] : grad;
    bool vec = false;
    if constexpr (std::is_same_v<T, float>) vec = (XW & 3) == 0;
    if (vec) {
      const int X4 = XW >> 2;
      for (int x = threadIdx.x; x < n * X4; x += blockDim.x) {
        const int q = x / X4, j = x - q * X4;
        float4 v = __ldg(reinterpret_cast<const float4*>(src + static_cast<int64_t>(qrow[q]) * XW) + j);
        if (MODE == 1) {
          const float a = static_cast<float>(qal[q]);
          v = make_float4(__fmul_rn(a, v.x), __fmul_rn(a, v.y), __fmul_rn(a, v.z), __fmul_rn(a, v.w));
        }
        reinterpret_cast<float4*>(xs)[x] = v;
      }
    } else {
      for (int x = threadIdx.x; x < n * XW; x += blockDim.x) {
        const int q = x / XW, j = x - q * XW;
        const T v = src[static_cast<int64_t>(qrow[q]) * XW + j];
        xs[x] = MODE == 0 ? v : mul_rn<T>(qal[q], v);
      }
    }
    __syncthreads();
    // one pair run of this chunk at a time: stage its H row once, then every
    // thread walks its lookups of the run (slot, slot + per, ...)
    for (int q0 = 0; q0 < n;) {
      const int pid0 = pids[q0];
      int q1 = q0 + 1;
      while (q1 < n && pids[q1] == pid0) ++q1;
      if (cur_pid != pid0) {
        __syncthreads();  // the previous run's readers are done with hs
        for (int x = threadIdx.x; x < W1; x += blockDim.x)
          hs[(x / R2) * R2p + x % R2] = H[static_cast<int64_t>(pid0) * W1 + x];
        __syncthreads();
        if (threadIdx.x == 0) cur_pid = pid0;
      }
      if (on_e) {
        for (int q = q0 + slot; q < q1; q += per) {
          const int64_t l = qlk[q];
          const T* x = xs + q * XW;
          if constexpr (CW == 4) {
            float v[4] = {0.f, 0.f, 0.f, 0.f};
            if (MODE == 0) {
              for (int r = 0; r < R2; ++r) {
                const float4 xv = *reinterpret_cast<const float4*>(x + r * n2 + rj);
                const float h = hs[ra + r];
                if (kExact) {
                  const float2 p01 = fmul2_rn(h, make_float2(xv.x, xv.y));
                  const float2 p23 = fmul2_rn(h, make_float2(xv.z, xv.w));
                  v[0] = __fadd_rn(v[0], p01.x);
                  v[1] = __fadd_rn(v[1], p01.y);
                  v[2] = __fadd_rn(v[2], p23.x);
                  v[3] = __fadd_rn(v[3], p23.y);
                } else {
                  ffma2(h, xv.x, xv.y, v[0], v[1]);
                  ffma2(h, xv.z, xv.w, v[2], v[3]);
                }
              }
              *reinterpret_cast<float4*>(out + l * N + e) = make_float4(v[0], v[1], v[2], v[3]);
            } else {
              for (int i = 0; i < P1; ++i) {
                const float4 xv = *reinterpret_cast<const float4*>(x + i * n2 + rj);
                const float h = hs[i * R2p + ra];
                ffma2(h, xv.x, xv.y, v[0], v[1]);
                ffma2(h, xv.z, xv.w, v[2], v[3]);
              }
              *reinterpret_cast<float4*>(out + static_cast<int64_t>(pos2[l]) * S2 + e) =
                  make_float4(v[0], v[1], v[2], v[3]);
            }
          } else if constexpr (CW == 2) {
            float v0 = 0.f, v1 = 0.f;
            if (MODE == 0) {
              for (int r = 0; r < R2; ++r) {
                const float2 xv = *reinterpret_cast<const float2*>(x + r * n2 + rj);
                if (kExact) {
                  const float2 pr = fmul2_rn(hs[ra + r], xv);
                  v0 = __fadd_rn(v0, pr.x);
                  v1 = __fadd_rn(v1, pr.y);
                } else {
                  ffma2(hs[ra + r], xv.x, xv.y, v0, v1);
                }
              }
              *reinterpret_cast<float2*>(out + l * N + e) = make_float2(v0, v1);
            } else {
              for (int i = 0; i < P1; ++i) {
                const float2 xv = *reinterpret_cast<const float2*>(x + i * n2 + rj);
                ffma2(hs[i * R2p + ra], xv.x, xv.y, v0, v1);
              }
              *reinterpret_cast<float2*>(out + static_cast<int64_t>(pos2[l]) * S2 + e) =
                  make_float2(v0, v1);
            }
          } else {
            T v = T(0);
            if (MODE == 0) {
              for (int r = 0; r < R2; ++r) v = madd<T, kExact>(hs[ra + r], x[r * n2 + rj], v);
              out[l * N + e] = v;
            } else {
              for (int i = 0; i < P1; ++i) v = madd<T, false>(hs[i * R2p + ra], x[i * n2 + rj], v);
              out[static_cast<int64_t>(pos2[l]) * S2 + e] = v;
            }
          }
        }
      }
      __syncthreads();  // cur_pid update visible; xs rows of this run consumed
      q0 = q1;
    }
  }
}

// Σ over the sorted positions of each segment (i2 bucket) of the dG2
// contributions, in position order; OUT_MODE 0 dense slice, 1 fused SGD.
template <typename T, int OUT_MODE>
__global__ void k_segsum3(const T* __restrict__ contrib, const int32_t* __restrict__ seg, int nseg,
                          int Wc, T* __restrict__ out, T lr) {
  for (int g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int first = seg[g], last = seg[g + 1];
    if (last <= first) continue;
    for (int e = threadIdx.x; e < Wc; e += blockDim.x) {
      T sum = contrib[static_cast<int64_t>(first) * Wc + e];
      for (int p = first + 1; p < last; ++p) sum += contrib[static_cast<int64_t>(p) * Wc + e];
      if (OUT_MODE == 0)
        out[static_cast<int64_t>(g) * Wc + e] = sum;
      else
        out[static_cast<int64_t>(g) * Wc + e] =
            add_rn<T>(out[static_cast<int64_t>(g) * Wc + e], -mul_rn<T>(lr, sum));
    }
  }
}

// Pooling of per-lookup rows y (L x N) per bag in lookup order (reference
// embedding_ops.hpp:232-249): out[b] = Σ T(w)·y, Mean rescale.
template <typename T, bool kExact>
__global__ void k_pool_rows(const T* __restrict__ y, const int64_t* __restrict__ off, int64_t B,
                            int64_t L, int N, const double* __restrict__ w, int mean,
                            T* __restrict__ out) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < B * N;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / N;
    const int j = static_cast<int>(q - b * N);
    const int64_t s = off[b], e = off[b + 1];
    const int64_t lo = s < 0 ? 0 : s, hi = e > L ? L : e;
    T acc = T(0);
    for (int64_t l = lo; l < hi; ++l)
      acc = madd<T, kExact>(static_cast<T>(w ? w[l] : 1.0), y[l * N + j], acc);
    if (mean && e - s > 1) acc = mul_rn<T>(acc, static_cast<T>(1.0 / static_cast<double>(e - s)));
    out[b * N + j] = acc;
  }
}

// Fold the partials of each segment in order.  Segment g spans sorted
// positions [first, last]; its runs are run(first)..run(last).
//   OUT_MODE 0: out[g*Wc + e] = sum      (S per pair; dense gradient slices)
//   OUT_MODE 1: core[g*Wc + e] -= lr*sum (fused SGD on touched slices)
template <typename T, int OUT_MODE>
__global__ void k_combine(const T* __restrict__ partials, const unsigned long long* __restrict__ scan,
                          const int32_t* __restrict__ seg, const int* __restrict__ nseg_dev,
                          int nseg_host, int Wc, T* __restrict__ out, T lr) {
  const int nseg = nseg_dev ? *nseg_dev : nseg_host;
  // gridDim.y > 1 splits a wide row's elements over several CTAs
  for (int g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int first = seg[g], last = seg[g + 1] - 1;
    if (last < first) continue;  // empty segment: untouched slice
    const int r0 = static_cast<int>(scan[first] >> 32) - 1;
    const int r1 = static_cast<int>(scan[last] >> 32) - 1;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < Wc; e += blockDim.x * gridDim.y) {
      T sum = partials[static_cast<int64_t>(r0) * Wc + e];
      for (int r = r0 + 1; r <= r1; ++r) sum += partials[static_cast<int64_t>(r) * Wc + e];
      if (OUT_MODE == 0)
        out[static_cast<int64_t>(g) * Wc + e] = sum;
      else
        out[static_cast<int64_t>(g) * Wc + e] =
            add_rn<T>(out[static_cast<int64_t>(g) * Wc + e], -mul_rn<T>(lr, sum));
    }
  }
}

// ------------------------------------------------- backward: head (pairs) --
// Over pairs in pid order (i1-major), chunks of CH pairs, runs by i1:
//   D0[pid] = S[pid] (P0 x C1) · G1[i1]ᵀ (C1 x R1)
//   partial(run) = Σ_pairs G0[i0]ᵀ (R1 x P0) · S[pid] (P0 x C1)
constexpr int kHeadMaxR1 = 64, kHeadMaxP0 = 4;

template <typename T>
__global__ void k_head_bwd(DevPlan P, const T* __restrict__ cores, const T* __restrict__ S,
                           const uint32_t* __restrict__ pair_key_u, const int* __restrict__ counts,
                           const unsigned long long* __restrict__ scan1, int CH,
                           T* __restrict__ D0, T* __restrict__ partials) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R1 = P.r[1], C1 = P.C1, P0 = P.n[0], s0 = P.slice[0], s1 = P.slice[1];
  // G1[i1] staged transposed with an odd row pitch (C1 x (R1+1)): the D0
  // loop's lanes walk r, so reads are conflict-free (row-major R1 x C1 with
  // C1 a multiple of 32 put every lane of a warp in the same bank)
  const int R1p = R1 + 1;
  T* g1t = reinterpret_cast<T*>(smem_raw);              // C1 x R1p
  T* sps = g1t + static_cast<int64_t>(C1) * R1p;        // P0 x C1: S row of the pair
  T* g0s = sps + P.W1;                                  // P0 x R1: G0[i0]
  T* acc = g0s + s0;                                    // R1 x C1 (only without reg_acc)
  const T* G0 = cores + P.coff[0];
  const T* G1 = cores + P.coff[1];
  const int U = counts[0];
  const int nchunks = (U + CH - 1) / CH;
  const uint32_t m0 = static_cast<uint32_t>(P.m[0]);
  // dG1 run accumulator in registers when one thread can own a whole column
  // (C1 <= blockDim, R1 <= kHeadMaxR1, P0 <= kHeadMaxP0: cfg3's 4 x 64 x 256)
  const bool reg_acc = C1 <= static_cast<int>(blockDim.x) && R1 <= kHeadMaxR1 && P0 <= kHeadMaxP0;
  T racc[kHeadMaxR1];
#pragma unroll
  for (int rr = 0; rr < kHeadMaxR1; ++rr) racc[rr] = T(0);
  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int p0 = ch * CH, p1 = min(U, p0 + CH);
    int run = static_cast<int>(scan1[p0] >> 32) - 1;
    int lo = p0;
    while (lo < p1) {
      const uint32_t i1 = pair_key_u[lo] / m0;
      int hi = lo + 1;
      while (hi < p1 && pair_key_u[hi] / m0 == i1) ++hi;
      __syncthreads();
      for (int e = threadIdx.x; e < s1; e += blockDim.x) {
        const int rr = e / C1, c = e - rr * C1;
        g1t[c * R1p + rr] = G1[static_cast<int64_t>(i1) * s1 + e];
        if (!reg_acc) acc[e] = T(0);
      }
      __syncthreads();
      for (int p = lo; p < hi; ++p) {
        const uint32_t i0 = pair_key_u[p] % m0;
        // the pair's S row and G0[i0] staged once (every thread reads them)
        for (int e = threadIdx.x; e < P.W1; e += blockDim.x)
          sps[e] = S[static_cast<int64_t>(p) * P.W1 + e];
        for (int e = threadIdx.x; e < s0; e += blockDim.x)
          g0s[e] = G0[static_cast<int64_t>(i0) * s0 + e];
        __syncthreads();
        // D0[p][a][r] = sum_c S[a][c] * G1[r][c]
        for (int e = threadIdx.x; e < P0 * R1; e += blockDim.x) {
          const int a = e / R1, rr = e - a * R1;
          const T* sa = sps + a * C1;
          // four independent chains over c (c mod 4), folded in a fixed order
          T v[4] = {T(0), T(0), T(0), T(0)};
          int c = 0;
          for (; c + 4 <= C1; c += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = madd<T, false>(sa[c + u], g1t[(c + u) * R1p + rr], v[u]);
          }
          for (; c < C1; ++c) v[0] = madd<T, false>(sa[c], g1t[c * R1p + rr], v[0]);
          D0[static_cast<int64_t>(p) * s0 + e] = (v[0] + v[1]) + (v[2] + v[3]);
        }
        // acc[r][c] += sum_a G0[a][r] * S[a][c]
        if (reg_acc) {  // thread = column c, the whole r column in registers
          const int c = threadIdx.x;
          if (c < C1) {
            T sv[kHeadMaxP0];
#pragma unroll
            for (int a = 0; a < kHeadMaxP0; ++a) sv[a] = a < P0 ? sps[a * C1 + c] : T(0);
            bool paired = false;
            if constexpr (std::is_same_v<T, float>)
              paired = (R1 & 1) == 0 && ((C1 * R1p + P.W1) & 1) == 0;  // 8-byte aligned G0 pairs
            if (paired) {  // (r, r+1) two lanes at a time: FFMA2, same per-element chain
              if constexpr (std::is_same_v<T, float>) {
#pragma unroll
                for (int rr = 0; rr < kHeadMaxR1; rr += 2) {
                  if (rr < R1) {
#pragma unroll
                    for (int a = 0; a < kHeadMaxP0; ++a)
                      if (a < P0) {
                        const float2 g = *reinterpret_cast<const float2*>(g0s + a * R1 + rr);
                        ffma2(sv[a], g.x, g.y, racc[rr], racc[rr + 1]);
                      }
                  }
                }
              }
            } else {
#pragma unroll
              for (int rr = 0; rr < kHeadMaxR1; ++rr) {
                if (rr < R1) {
                  T v = racc[rr];
#pragma unroll
                  for (int a = 0; a < kHeadMaxP0; ++a)
                    if (a < P0) v = madd<T, false>(g0s[a * R1 + rr], sv[a], v);
                  racc[rr] = v;
                }
              }
            }
          }
        } else {
          for (int e = threadIdx.x; e < s1; e += blockDim.x) {
            const int rr = e / C1, c = e - rr * C1;
            T v = acc[e];
            for (int a = 0; a < P0; ++a) v = madd<T, false>(g0s[a * R1 + rr], sps[a * C1 + c], v);
            acc[e] = v;
          }
        }
        __syncthreads();  // sps / g0s are restaged for the next pair
      }
      __syncthreads();
      if (reg_acc) {
        const int c = threadIdx.x;
        if (c < C1) {
#pragma unroll
          for (int rr = 0; rr < kHeadMaxR1; ++rr) {
            if (rr < R1) partials[static_cast<int64_t>(run) * s1 + rr * C1 + c] = racc[rr];
            racc[rr] = T(0);
          }
        }
      } else {
        for (int e = threadIdx.x; e < s1; e += blockDim.x)
          partials[static_cast<int64_t>(run) * s1 + e] = acc[e];
      }
      ++run;
      lo = hi;
    }
  }
}

// dG0[i0] = Σ_{i1 ascending} D0[pair(i0,i1)] via the dense pair table; entries
// from earlier batches are rejected by checking the pair key back.
// OUT_MODE 0 writes the dense slice, 1 applies SGD to touched slices.
template <typename T, int OUT_MODE>
__global__ void __launch_bounds__(128) k_head_g0(DevPlan P, const T* __restrict__ D0,
                                                 const int32_t* __restrict__ pair_tab,
                                                 const uint32_t* __restrict__ pair_key_u,
                                                 const int* __restrict__ counts, T* __restrict__ out,
                                                 T lr) {
  // the pair ids of a tile of i1 values are resolved by all threads at once
  // (one round trip) and compacted in i1 order; every thread then sums its
  // elements over them with kU independent D0 loads in flight
  constexpr int kTile = 1024, kEPT = 4, kU = 16;
  __shared__ int pids[kTile];
  __shared__ int wcnt[4];
  const int U = counts[0];
  const int s0 = P.slice[0], m0 = P.m[0], m1 = P.m[1];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i0 = blockIdx.x; i0 < m0; i0 += gridDim.x) {
    for (int e0 = 0; e0 < s0; e0 += kEPT * blockDim.x) {
      T sum[kEPT];
#pragma unroll
      for (int k = 0; k < kEPT; ++k) sum[k] = T(0);
      bool touched = false;
      for (int b = 0; b < m1; b += kTile) {
        const int nb = m1 - b < kTile ? m1 - b : kTile;
        __syncthreads();
        // thread j resolves i1 = b + j.. (blockDim-strided chunks, each chunk
        // compacted in order by a ballot prefix)
        int nvalid = 0;
        for (int j0 = 0; j0 < nb; j0 += blockDim.x) {
          const int j = j0 + threadIdx.x;
          int pid = -1;
          if (j < nb) {
            const uint32_t key = static_cast<uint32_t>(b + j) * static_cast<uint32_t>(m0) + i0;
            pid = pair_tab[key];
            if (pid < 0 || pid >= U || pair_key_u[pid] != key) pid = -1;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, pid >= 0);
          if (lane == 0) wcnt[wid] = __popc(bal);
          __syncthreads();
          int before = nvalid;
          for (int w = 0; w < wid; ++w) before += wcnt[w];
          int total = nvalid;
          for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) total += wcnt[w];
          if (pid >= 0) pids[before + __popc(bal & ((1u << lane) - 1u))] = pid;
          nvalid = total;
          __syncthreads();
        }
        if (nvalid) touched = true;
        for (int j = 0; j < nvalid; j += kU) {
          T v[kU][kEPT];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int pid = j + u < nvalid ? pids[j + u] : -1;
#pragma unroll
            for (int k = 0; k < kEPT; ++k) {
              const int e = e0 + k * blockDim.x + threadIdx.x;
              v[u][k] = (pid >= 0 && e < s0) ? D0[static_cast<int64_t>(pid) * s0 + e] : T(0);
            }
          }
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (j + u < nvalid)
#pragma unroll
              for (int k = 0; k < kEPT; ++k) sum[k] += v[u][k];
        }
      }
#pragma unroll
      for (int k = 0; k < kEPT; ++k) {
        const int e = e0 + k * blockDim.x + threadIdx.x;
        if (e >= s0) continue;
        if (OUT_MODE == 0)
          out[static_cast<int64_t>(i0) * s0 + e] = sum[k];
        else if (touched)
          out[static_cast<int64_t>(i0) * s0 + e] =
              add_rn<T>(out[static_cast<int64_t>(i0) * s0 + e], -mul_rn<T>(lr, sum[k]));
      }
    }
  }
}

// ------------------------------------------------------------------ misc --
// sgd_step element update c -= T(lr) * g, separately rounded like the
// reference's `c[i] -= step * g[i]` (embedding_ops.hpp:372-373).
template <typename T>
__global__ void k_sgd(T* __restrict__ c, const T* __restrict__ g, int64_t n, T step) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    c[i] = add_rn<T>(c[i], -mul_rn<T>(step, g[i]));
}

// lookup_row for a list of rows (embedding_ops.hpp:120-152), one warp per row,
// bit-identical to the reference (kExact).  Rows are pre-validated on the host
// or latched into *bad.
template <typename T>
__global__ void k_lookup_rows(DevPlan P, const T* __restrict__ cores, const int64_t* __restrict__ rows,
                              int64_t n, T* __restrict__ out, unsigned long long* bad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warps = blockDim.x >> 5, wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* ping = reinterpret_cast<T*>(smem_raw) + static_cast<int64_t>(wid) * 2 * P.maxw;
  T* pong = ping + P.maxw;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * warps + wid; q < n;
       q += static_cast<int64_t>(gridDim.x) * warps) {
    int64_t row = rows[q];
    if (row < 0 || row >= P.num_rows) {
      if (lane == 0 && bad) atomicMin(bad, static_cast<unsigned long long>(q));
      row = 0;
    }
    int dig[kMaxD];
    decode_row(P, row, dig);
    const T* src = cores + P.coff[0] + static_cast<int64_t>(dig[0]) * P.slice[0];
    T* dst = ping;
    for (int k = 1; k < P.d; ++k) {
      const T* G = cores + P.coff[k] + static_cast<int64_t>(dig[k]) * P.slice[k];
      T* target = (k == P.d - 1) ? out + q * P.N : dst;
      warp_mm<T, true>(src, G, target, P.prefix[k - 1], P.r[k], P.n[k] * P.r[k + 1], lane);
      __syncwarp();
      src = target;
      dst = (dst == ping) ? pong : ping;
    }
  }
}

}  // namespace ttgpu
