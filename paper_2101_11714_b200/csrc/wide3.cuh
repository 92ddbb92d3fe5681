// Wide-row 3-core tail kernels, warp per chunk (cfg3's shape class: fp32,
// P1 = n0·n1 = 16, R2 = 64, n2 = 4, so H rows are 16 x 64 = 4 KB, G2 slices
// 64 x 4 = 1 KB, output rows 64 floats).
//
// The generic d == 3 wide-row path (tt_kernels.cuh k_pairwalk3 / k_srun3)
// stages a CTA's operands in shared memory and reads them back for every
// multiply-add, so it is bound by shared-memory bandwidth (cfg3: forward tail
// 1.7 ms, S 2.2 ms, dG2 walk 1.5 ms).  Here one WARP owns one chunk of
// kTailChunk = 32 pair-sorted lookups (the same chunks, runs and partial rows
// as the generic path, so the downstream folds are unchanged) and keeps the
// reused operand in REGISTERS:
//
//   k_w3_fwd  (forward tail)  lane = lookup.  y[a][j] = Σ_r H[a][r]·G2[i2][r][j]
//             with H of the lane's pair broadcast from shared memory (one 4 KB
//             row per pair run) and the lane's own G2 rows streamed from L2.
//             Exact mode keeps the reference's per-element order (r ascending,
//             separately rounded products and sums: gemm.hpp:15-31), so the
//             pooled output stays bit-identical.
//   k_w3_bwd_pairs (backward tail) two warps per PAIR, lane = one column r
//             of the 64.  The lane holds H[a][r] and the running S[a][r] (16 a)
//             in registers as f32x2 pairs; per lookup (D2 = T(alpha)·grad[bag]
//             staged per 32-lookup chunk in shared memory, read as broadcasts):
//               S[a][r]  += Σ_j D2[a][j]·G2[i2][r][j]     (S = Σ D1, D1 = D2·G2ᵀ)
//               C[r][j]   = Σ_a H[a][r]·D2[a][j]          (dG2 contribution)
//             S(pair) is written once, complete; C goes to the lookup's
//             i2-sorted position, summed per i2 by k_w3_segsum.
//   k_w3_segsum  dG2[i2] = Σ C over the i2 segment in position order, split
//             into slabs of kW3Slab rows so every SM streams (the generic
//             k_segsum3 runs one CTA per i2 with 2,000-long dependent chains);
//             slab partials are folded in slab order by the last slab to
//             finish (deterministic), fused with the SGD when asked.
//
// Reference: embedding_ops.hpp:213-229 (forward chain), :335-347 (backward
// chain, k = 2 and the D1 that feeds S), :355-357 (gradients summed over all
// lookups).
#pragma once

namespace ttgpu {
namespace w3 {

constexpr int P1 = 16, R2 = 64, N2 = 4, N = P1 * N2, W1 = P1 * R2, S2 = R2 * N2;
constexpr int kWarps = 8;      // warps per CTA
constexpr int kChunk = 32;     // lookups per warp work unit (== kTailChunk)
constexpr int kW3Slab = 64;    // rows of C per segsum slab

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Packed fp32 pairs held in 64-bit registers (sm_100a f32x2 ops).
__device__ __forceinline__ unsigned long long pk(float x, float y) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(x), "f"(y));
  return r;
}
__device__ __forceinline__ float2 upk(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b,
                                                   unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ unsigned long long add2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// ---------------------------------------------------------------- forward --
// Up to kRunsPerPass pair runs of a chunk are staged at once (H transposed,
// [r][a]), so every lane of the chunk computes in the same pass.
constexpr int kRunsPerPass = 2;
constexpr int kRB = 8;          // G2 rows per staged block
constexpr int kGsStride = 9;    // float4 per staged lookup block (8 rows + 1 pad: no bank conflicts)
constexpr int kAH = P1 / 2;     // output rows a per warp (two warps per chunk)
constexpr size_t kFwdWarpFloats = kRunsPerPass * R2 * kAH + 2 * kChunk * kGsStride * 4;
constexpr size_t kFwdSmem = sizeof(float) * kWarps * kFwdWarpFloats;  // 104 KB

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N_>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N_) : "memory"); }

// Two warps per chunk: warp half h computes rows a in [8h, 8h + 8) of every
// lookup's y (lane = lookup), so a lane keeps 8 x 4 accumulators.
template <bool kExact>
__global__ void __launch_bounds__(kWarps * 32, 2) k_w3_fwd(const float* __restrict__ G2,
                                                           const float* __restrict__ H,
                                                           const int32_t* __restrict__ lk_pid,
                                                           const uint32_t* __restrict__ tail_dig,
                                                           const uint32_t* __restrict__ s_lk,
                                                           int64_t L, float* __restrict__ y) {
  // per warp: [kRunsPerPass][R2][kAH] H rows (transposed) | 2 x [kChunk][kGsStride] float4 G2
  // blocks (double-buffered: block rb + 1 lands by cp.async while block rb is used)
  extern __shared__ __align__(16) float w3f_dyn[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = wid & 1, a0 = half * kAH;
  float* hs_w = w3f_dyn + wid * kFwdWarpFloats;
  float4* gs = reinterpret_cast<float4*>(hs_w + kRunsPerPass * R2 * kAH);
  const int64_t nchunks = (L + kChunk - 1) / kChunk;
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * (kWarps / 2) + (wid >> 1); ch < nchunks;
       ch += static_cast<int64_t>(gridDim.x) * (kWarps / 2)) {
    const int64_t c0 = ch * kChunk;
    const int n = static_cast<int>(L - c0 < kChunk ? L - c0 : kChunk);
    int l = 0, pid = -1, i2 = 0;
    if (lane < n) {
      l = static_cast<int>(s_lk[c0 + lane]);
      pid = lk_pid[l];
      i2 = static_cast<int>(tail_dig[l]);
    }
    // run starts: lane q starts a run iff its pair differs from lane q - 1's
    const int prev = __shfl_up_sync(0xffffffffu, pid, 1);
    const unsigned starts = __ballot_sync(0xffffffffu, lane < n && (lane == 0 || prev != pid));
    const int my_run = __popc(starts & ((2u << lane) - 1u)) - 1;  // this lane's run ordinal
    const int nruns = __popc(starts);
    for (int r0 = 0; r0 < nruns; r0 += kRunsPerPass) {
      const int rn = min(kRunsPerPass, nruns - r0);
      __syncwarp();
      for (int k = 0; k < rn; ++k) {
        // the k-th run's pair: the lane at the (r0 + k)-th set bit of starts
        unsigned m = starts;
        for (int z = 0; z < r0 + k; ++z) m &= m - 1;
        const int p = __shfl_sync(0xffffffffu, pid, __ffs(m) - 1);
        const float* hp = H + static_cast<int64_t>(p) * W1 + a0 * R2;
        float* hs = hs_w + k * R2 * kAH;
        // column r = it % 2 * 32 + lane, a-group g = it / 2 (of this warp's 8 rows):
        // 4 coalesced loads, one 16-byte store into the [r][a] layout
#pragma unroll
        for (int it = 0; it < 2 * (kAH / 4); ++it) {
          const int r = (it & 1) * 32 + lane, g = it >> 1;
          const float4 v = make_float4(__ldg(hp + (4 * g + 0) * R2 + r), __ldg(hp + (4 * g + 1) * R2 + r),
                                       __ldg(hp + (4 * g + 2) * R2 + r), __ldg(hp + (4 * g + 3) * R2 + r));
          *reinterpret_cast<float4*>(hs + r * kAH + 4 * g) = v;
        }
      }
      const int k = my_run - r0;
      const bool act = lane < n && k >= 0 && k < rn;
      const float* hs = hs_w + (act ? k : 0) * R2 * kAH;
      float4 acc[kAH];
#pragma unroll
      for (int a = 0; a < kAH; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      // G2 rows [rb, rb + kRB) of every lookup of the chunk: 4 lookups x 128 B per
      // warp copy (coalesced), lane q then reads its own block
      auto stage = [&](int rb, int buf) {
        float4* gb = gs + buf * kChunk * kGsStride;
#pragma unroll
        for (int it = 0; it < kChunk / 4; ++it) {
          const int qq = it * 4 + (lane >> 3), piece = lane & 7;
          const int iq = __shfl_sync(0xffffffffu, i2, qq);
          if (qq < n) cp_async16(gb + qq * kGsStride + piece, G2 + static_cast<int64_t>(iq) * S2 + (rb + piece) * N2);
        }
        cp_async_commit();
      };
      __syncwarp();
      stage(0, 0);
      for (int rb = 0; rb < R2; rb += kRB) {
        const int buf = (rb / kRB) & 1;
        if (rb + kRB < R2) {
          stage(rb + kRB, buf ^ 1);
          cp_async_wait<1>();
        } else {
          cp_async_wait<0>();
        }
        __syncwarp();
        const float4* gb = gs + buf * kChunk * kGsStride;
        if (act) {
#pragma unroll
          for (int rr = 0; rr < kRB; ++rr) {
            const float4 g = gb[lane * kGsStride + rr];
            const float4* h4 = reinterpret_cast<const float4*>(hs + (rb + rr) * kAH);
#pragma unroll
            for (int a4 = 0; a4 < kAH / 4; ++a4) {
              const float4 h = h4[a4];
              const float hv[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                float4& c = acc[a4 * 4 + u];
                if constexpr (kExact) {
                  const float2 p01 = fmul2_rn(hv[u], make_float2(g.x, g.y));
                  const float2 p23 = fmul2_rn(hv[u], make_float2(g.z, g.w));
                  c.x = __fadd_rn(c.x, p01.x);
                  c.y = __fadd_rn(c.y, p01.y);
                  c.z = __fadd_rn(c.z, p23.x);
                  c.w = __fadd_rn(c.w, p23.y);
                } else {
                  ffma2(hv[u], g.x, g.y, c.x, c.y);
                  ffma2(hv[u], g.z, g.w, c.z, c.w);
                }
              }
            }
          }
        }
        __syncwarp();  // every lane is done with this buffer before it is restaged
      }
      if (act) {
        float4* yo = reinterpret_cast<float4*>(y + static_cast<int64_t>(l) * N) + a0;
#pragma unroll
        for (int a = 0; a < kAH; ++a) yo[a] = acc[a];
      }
    }
  }
}

// --------------------------------------------------------------- backward --
// Two warps per chunk, each owning 32 of the 64 columns r (lane = one column):
// per pair run the lane holds H[a][r] and the running S[a][r] for the 16 a in
// registers as (a, a+1) pairs.  D2 is staged per warp as [j][a], so
// (D2[a][j], D2[a+1][j]) is a natural f32x2 operand; the only packed value is
// the lane's G2 row duplicated per j, once per lookup.  Per lookup:
//   S[a][r]  += Σ_j D2[a][j]·G2[i2][r][j]       (fma chain over j from zero)
//   C[r][j]   = Σ_a H[a][r]·D2[a][j]            (even / odd a accumulated apart)
constexpr int kWarpsB = 8;                              // 4 chunks x 2 column halves
constexpr size_t kBwdSmem = sizeof(float) * kWarpsB * kChunk * N;  // 64 KB: [warp][q][j][a]

// A warp pair owns whole PAIRS (grid-stride over the unique pairs, positions
// pair_start[p] .. pair_start[p + 1]), walked in chunks of kChunk lookups, so
// S(p) is complete when its walk ends and is written straight to S[p] -- no
// partial rows and no separate fold.  S sums over the pair's lookups in sorted
// order.
__global__ void __launch_bounds__(kWarpsB * 32, 3) k_w3_bwd_pairs(
    const float* __restrict__ G2, const float* __restrict__ H, const int* __restrict__ counts,
    const int32_t* __restrict__ pair_start, const uint32_t* __restrict__ tail_dig,
    const int32_t* __restrict__ lk_bag, const float* __restrict__ lk_alpha,
    const float* __restrict__ grad, const uint32_t* __restrict__ s_lk,
    const uint32_t* __restrict__ pos2, float* __restrict__ S, float* __restrict__ contrib) {
  extern __shared__ __align__(16) float w3p_dyn[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* d2s = w3p_dyn + wid * kChunk * N;  // this warp's [q][j][a]
  const int half = wid & 1;
  const int r = half * 32 + lane;  // this lane's column
  const int U = counts[0];
  for (int p = blockIdx.x * (kWarpsB / 2) + (wid >> 1); p < U; p += gridDim.x * (kWarpsB / 2)) {
    const int ps = pair_start[p], pe = pair_start[p + 1];
    unsigned long long h[P1 / 2], s[P1 / 2];
    {
      const float* hp = H + static_cast<int64_t>(p) * W1 + r;
#pragma unroll
      for (int a2 = 0; a2 < P1 / 2; ++a2) {
        h[a2] = pk(__ldg(hp + (2 * a2) * R2), __ldg(hp + (2 * a2 + 1) * R2));
        s[a2] = 0ull;
      }
    }
    for (int c0 = ps; c0 < pe; c0 += kChunk) {
      const int n = pe - c0 < kChunk ? pe - c0 : kChunk;
      int i2 = 0, bag = 0;
      uint32_t p2 = 0;
      float al = 0.f;
      __syncwarp();
      if (lane < n) {
        const int l = static_cast<int>(s_lk[c0 + lane]);
        i2 = static_cast<int>(tail_dig[l]);
        p2 = pos2[l];
        bag = lk_bag[l];
        al = lk_alpha[l];
      }
#pragma unroll 4
      for (int it = 0; it < kChunk / 2; ++it) {
        const int qq = it * 2 + (lane >> 4), k4 = lane & 15;
        const int bq = __shfl_sync(0xffffffffu, bag, qq);
        const float aq = __shfl_sync(0xffffffffu, al, qq);
        if (qq < n) {
          const float4 v = __ldg(reinterpret_cast<const float4*>(grad + static_cast<int64_t>(bq) * N) + k4);
          float* dq = d2s + qq * N + k4;  // [j][a]: j * 16 + a
          dq[0 * P1] = __fmul_rn(aq, v.x);
          dq[1 * P1] = __fmul_rn(aq, v.y);
          dq[2 * P1] = __fmul_rn(aq, v.z);
          dq[3 * P1] = __fmul_rn(aq, v.w);
        }
      }
      __syncwarp();
      float4 gn = ld4(G2 + static_cast<int64_t>(__shfl_sync(0xffffffffu, i2, 0)) * S2 + r * N2);
      float4 gnn = ld4(G2 + static_cast<int64_t>(__shfl_sync(0xffffffffu, i2, 1)) * S2 + r * N2);
      for (int q = 0; q < n; ++q) {
        const uint32_t pq = __shfl_sync(0xffffffffu, p2, q);
        const float4 g = gn;
        gn = gnn;
        {
          const int i2q = __shfl_sync(0xffffffffu, i2, (q + 2) & 31);
          if (q + 2 < n) gnn = ld4(G2 + static_cast<int64_t>(i2q) * S2 + r * N2);
        }
        const unsigned long long g0 = pk(g.x, g.x), g1 = pk(g.y, g.y), g2 = pk(g.z, g.z), g3 = pk(g.w, g.w);
        unsigned long long c0v = 0ull, c1v = 0ull, c2v = 0ull, c3v = 0ull;
        const float* dq = d2s + q * N;
#pragma unroll
        for (int a2 = 0; a2 < P1 / 2; ++a2) {
          const unsigned long long d0 = *reinterpret_cast<const unsigned long long*>(dq + 0 * P1 + 2 * a2);
          const unsigned long long d1 = *reinterpret_cast<const unsigned long long*>(dq + 1 * P1 + 2 * a2);
          const unsigned long long d2 = *reinterpret_cast<const unsigned long long*>(dq + 2 * P1 + 2 * a2);
          const unsigned long long d3 = *reinterpret_cast<const unsigned long long*>(dq + 3 * P1 + 2 * a2);
          unsigned long long v = fma2(d0, g0, 0ull);
          v = fma2(d1, g1, v);
          v = fma2(d2, g2, v);
          v = fma2(d3, g3, v);
          s[a2] = add2(s[a2], v);
          c0v = fma2(h[a2], d0, c0v);
          c1v = fma2(h[a2], d1, c1v);
          c2v = fma2(h[a2], d2, c2v);
          c3v = fma2(h[a2], d3, c3v);
        }
        const float2 e0 = upk(c0v), e1 = upk(c1v), e2 = upk(c2v), e3 = upk(c3v);
        *reinterpret_cast<float4*>(contrib + static_cast<int64_t>(pq) * S2 + r * N2) =
            make_float4(e0.x + e0.y, e1.x + e1.y, e2.x + e2.y, e3.x + e3.y);
      }
    }
    float* so = S + static_cast<int64_t>(p) * W1 + r;
#pragma unroll
    for (int a2 = 0; a2 < P1 / 2; ++a2) {
      const float2 sv = upk(s[a2]);
      so[(2 * a2) * R2] = sv.x;
      so[(2 * a2 + 1) * R2] = sv.y;
    }
  }
}

// dG2 per i2 segment: slab partials, folded in slab order by the last slab.
// Thread = 4 columns of the 256; a CTA of 64 threads per slab.
template <int OUT_MODE>
__global__ void __launch_bounds__(64) k_w3_segsum(const float* __restrict__ contrib,
                                                   const int32_t* __restrict__ seg, int nseg,
                                                   const int32_t* __restrict__ slab_base,
                                                   float* __restrict__ slab_part, int* __restrict__ cnt,
                                                   float* __restrict__ out, float lr) {
  const int task = blockIdx.x;
  // segment of this slab: slab_base is the exclusive prefix of slabs per segment
  int lo = 0, hi = nseg;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (slab_base[mid] <= task) lo = mid; else hi = mid;
  }
  const int g = lo, si = task - slab_base[g], ns = slab_base[g + 1] - slab_base[g];
  if (si >= ns) return;  // past the last slab (the grid is sized for the worst case)
  const int first = seg[g] + si * kW3Slab, last = min(seg[g + 1], first + kW3Slab);
  const int e = threadIdx.x * 4;
  float4 acc = __ldcg(reinterpret_cast<const float4*>(contrib + static_cast<int64_t>(first) * S2 + e));
#pragma unroll 8
  for (int p = first + 1; p < last; ++p) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(contrib + static_cast<int64_t>(p) * S2 + e));
    acc.x += v.x;
    acc.y += v.y;
    acc.z += v.z;
    acc.w += v.w;
  }
  if (ns > 1) {
    reinterpret_cast<float4*>(slab_part + static_cast<int64_t>(task) * S2)[threadIdx.x] = acc;
    __threadfence();
    __shared__ int last_one;
    __syncthreads();
    if (threadIdx.x == 0) last_one = atomicAdd(cnt + g, 1) == ns - 1;
    __syncthreads();
    if (!last_one) return;
    __threadfence();
    acc = __ldcg(reinterpret_cast<const float4*>(slab_part + static_cast<int64_t>(slab_base[g]) * S2) +
                 threadIdx.x);
    for (int k = 1; k < ns; ++k) {
      const float4 v = __ldcg(
          reinterpret_cast<const float4*>(slab_part + static_cast<int64_t>(slab_base[g] + k) * S2) +
          threadIdx.x);
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    if (threadIdx.x == 0) cnt[g] = 0;  // ready for the next launch
  }
  float4* o = reinterpret_cast<float4*>(out + static_cast<int64_t>(g) * S2) + threadIdx.x;
  if (OUT_MODE == 0) {
    *o = acc;
  } else {
    float4 cv = *o;
    cv.x = __fadd_rn(cv.x, -__fmul_rn(lr, acc.x));
    cv.y = __fadd_rn(cv.y, -__fmul_rn(lr, acc.y));
    cv.z = __fadd_rn(cv.z, -__fmul_rn(lr, acc.z));
    cv.w = __fadd_rn(cv.w, -__fmul_rn(lr, acc.w));
    *o = cv;
  }
}

// slabs per i2 segment -> exclusive prefix (one thread per segment, then a
// block scan; nseg <= 4096 here)
__global__ void k_w3_slabs(const int32_t* __restrict__ seg, int nseg, int32_t* __restrict__ slab_base) {
  __shared__ int32_t sm[1024];
  const int per = (nseg + blockDim.x - 1) / blockDim.x;
  const int g0 = threadIdx.x * per;
  int32_t tot = 0;
  for (int g = g0; g < min(nseg, g0 + per); ++g) {
    const int len = seg[g + 1] - seg[g];
    tot += (len + kW3Slab - 1) / kW3Slab;
  }
  sm[threadIdx.x] = tot;
  __syncthreads();
  for (int o = 1; o < blockDim.x; o <<= 1) {
    const int32_t v = threadIdx.x >= o ? sm[threadIdx.x - o] : 0;
    __syncthreads();
    sm[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = sm[threadIdx.x] - tot;
  for (int g = g0; g < min(nseg, g0 + per); ++g) {
    slab_base[g] = run;
    const int len = seg[g + 1] - seg[g];
    run += (len + kW3Slab - 1) / kW3Slab;
  }
  if (threadIdx.x == blockDim.x - 1) slab_base[nseg] = sm[threadIdx.x];
}

}  // namespace w3
}  // namespace ttgpu
