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
//   k_w3_bwd  (backward tail) lane = 2 columns r of the 64.  Per pair run the
//             lane holds H[a][r] (16 x 2) and the running S[a][r] (16 x 2) in
//             registers; per lookup (D2 = T(alpha)·grad[bag] staged once per
//             chunk in shared memory, read as broadcasts):
//               S[a][r]  += Σ_j D2[a][j]·G2[i2][r][j]     (S = Σ D1, D1 = D2·G2ᵀ)
//               C[r][j]   = Σ_a H[a][r]·D2[a][j]          (dG2 contribution)
//             S is written once per run (partial row, folded by k_combine as
//             before); C goes to the lookup's i2-sorted position, summed per i2
//             by k_w3_segsum.  Per element the same fma chains as k_srun3 /
//             k_pairwalk3 MODE 1, so gradients are bitwise those of the generic
//             kernels.
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
constexpr size_t kFwdSmem =
    sizeof(float) * kWarps * (kRunsPerPass * W1 + kChunk * kGsStride * 4);  // 64 + 36 KB

template <bool kExact>
__global__ void __launch_bounds__(kWarps * 32, 2) k_w3_fwd(const float* __restrict__ G2,
                                                        const float* __restrict__ H,
                                                        const int32_t* __restrict__ lk_pid,
                                                        const uint32_t* __restrict__ tail_dig,
                                                        const uint32_t* __restrict__ s_lk, int64_t L,
                                                        float* __restrict__ y) {
  // per warp: [kRunsPerPass][R2][P1] H rows (transposed) | [kChunk][kGsStride] float4 G2 block
  extern __shared__ __align__(16) float w3f_dyn[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* hs_w = w3f_dyn + wid * (kRunsPerPass * W1 + kChunk * kGsStride * 4);
  float4* gs = reinterpret_cast<float4*>(hs_w + kRunsPerPass * W1);
  const int64_t nchunks = (L + kChunk - 1) / kChunk;
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * kWarps + wid; ch < nchunks;
       ch += static_cast<int64_t>(gridDim.x) * kWarps) {
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
        const float* hp = H + static_cast<int64_t>(p) * W1;
        float* hs = hs_w + k * W1;
        // column r = it % 2 * 32 + lane, a-group g = it / 2: 4 coalesced loads,
        // one 16-byte store into the [r][a] layout
#pragma unroll
        for (int it = 0; it < 2 * (P1 / 4); ++it) {
          const int r = (it & 1) * 32 + lane, g = it >> 1;
          const float4 v = make_float4(__ldg(hp + (4 * g + 0) * R2 + r), __ldg(hp + (4 * g + 1) * R2 + r),
                                       __ldg(hp + (4 * g + 2) * R2 + r), __ldg(hp + (4 * g + 3) * R2 + r));
          *reinterpret_cast<float4*>(hs + r * P1 + 4 * g) = v;
        }
      }
      const int k = my_run - r0;
      const bool act = lane < n && k >= 0 && k < rn;
      const float* hs = hs_w + (act ? k : 0) * W1;
      float4 acc[P1];
#pragma unroll
      for (int a = 0; a < P1; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int rb = 0; rb < R2; rb += kRB) {
        // G2 rows [rb, rb + kRB) of every lookup of the chunk: 4 lookups x 128 B
        // per warp load (coalesced), lane q then reads its own block
        __syncwarp();
#pragma unroll
        for (int it = 0; it < kChunk / 4; ++it) {
          const int qq = it * 4 + (lane >> 3), piece = lane & 7;
          const int iq = __shfl_sync(0xffffffffu, i2, qq);
          if (qq < n) gs[qq * kGsStride + piece] = ld4(G2 + static_cast<int64_t>(iq) * S2 + (rb + piece) * N2);
        }
        __syncwarp();
        if (act) {
#pragma unroll
          for (int rr = 0; rr < kRB; ++rr) {
            const float4 g = gs[lane * kGsStride + rr];
            const float4* h4 = reinterpret_cast<const float4*>(hs + (rb + rr) * P1);
#pragma unroll
            for (int a4 = 0; a4 < P1 / 4; ++a4) {
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
      }
      if (act) {
        float4* yo = reinterpret_cast<float4*>(y + static_cast<int64_t>(l) * N);
#pragma unroll
        for (int a = 0; a < P1; ++a) yo[a] = acc[a];
      }
    }
  }
}

// --------------------------------------------------------------- backward --
// D2 is staged as DUPLICATED pairs (d, d), so every f32x2 operand is a natural
// register pair: no packing moves in the inner loop.
constexpr int kWarpsB = 4;
constexpr int kDdStride = N + 2;  // pairs per staged lookup (+16 B: conflict-free 16-byte stores)
constexpr size_t kBwdSmem = sizeof(unsigned long long) * kWarpsB * kChunk * kDdStride;  // 66 KB

__global__ void __launch_bounds__(kWarpsB * 32, 3) k_w3_bwd(
    const float* __restrict__ G2, const float* __restrict__ H, const int32_t* __restrict__ lk_pid,
    const uint32_t* __restrict__ tail_dig, const int32_t* __restrict__ lk_bag,
    const float* __restrict__ lk_alpha, const float* __restrict__ grad,
    const uint32_t* __restrict__ s_lk, const unsigned long long* __restrict__ scan,
    const uint32_t* __restrict__ pos2, int64_t L, float* __restrict__ partS,
    float* __restrict__ contrib) {
  extern __shared__ __align__(16) float w3b_dyn[];  // [kWarpsB][kChunk][P1][N2] (d, d) pairs
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long* dd = reinterpret_cast<unsigned long long*>(w3b_dyn) + wid * kChunk * kDdStride;
  const int r0 = 2 * lane;  // this lane's two columns r0, r0 + 1
  const int64_t nchunks = (L + kChunk - 1) / kChunk;
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * kWarpsB + wid; ch < nchunks;
       ch += static_cast<int64_t>(gridDim.x) * kWarpsB) {
    const int64_t c0 = ch * kChunk;
    const int n = static_cast<int>(L - c0 < kChunk ? L - c0 : kChunk);
    int pid = -1, i2 = 0, run = 0, bag = 0;
    uint32_t p2 = 0;
    float al = 0.f;
    __syncwarp();
    if (lane < n) {
      const int l = static_cast<int>(s_lk[c0 + lane]);
      pid = lk_pid[l];
      i2 = static_cast<int>(tail_dig[l]);
      run = static_cast<int>(scan[c0 + lane] >> 32) - 1;
      p2 = pos2[l];
      bag = lk_bag[l];
      al = lk_alpha[l];
    }
    // D2 = T(alpha)·grad[bag] as (d, d) pairs: two lookups' rows (2 x 256 B)
    // per warp load, lanes 16 B apart (coalesced and conflict-free)
#pragma unroll 4
    for (int it = 0; it < kChunk / 2; ++it) {
      const int qq = it * 2 + (lane >> 4), k4 = lane & 15;
      const int bq = __shfl_sync(0xffffffffu, bag, qq);
      const float aq = __shfl_sync(0xffffffffu, al, qq);
      if (qq < n) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(grad + static_cast<int64_t>(bq) * N) + k4);
        const float x = __fmul_rn(aq, v.x), yv = __fmul_rn(aq, v.y), z = __fmul_rn(aq, v.z),
                    w = __fmul_rn(aq, v.w);
        ulonglong2* dst = reinterpret_cast<ulonglong2*>(dd + qq * kDdStride + 4 * k4);
        dst[0] = make_ulonglong2(pk(x, x), pk(yv, yv));
        dst[1] = make_ulonglong2(pk(z, z), pk(w, w));
      }
    }
    __syncwarp();
    unsigned long long h[P1], s[P1];
    int cur = -1;
    int i2n = __shfl_sync(0xffffffffu, i2, 0);
    float4 ga = ld4(G2 + static_cast<int64_t>(i2n) * S2 + r0 * N2);
    float4 gb = ld4(G2 + static_cast<int64_t>(i2n) * S2 + (r0 + 1) * N2);
    for (int q = 0; q < n; ++q) {
      const int p = __shfl_sync(0xffffffffu, pid, q);
      const int rq = __shfl_sync(0xffffffffu, run, q);
      const uint32_t pq = __shfl_sync(0xffffffffu, p2, q);
      // G2 column pairs (G2[r0][j], G2[r0+1][j]) of this lookup
      const unsigned long long gp0 = pk(ga.x, gb.x), gp1 = pk(ga.y, gb.y), gp2 = pk(ga.z, gb.z),
                               gp3 = pk(ga.w, gb.w);
      if (q + 1 < n) {
        i2n = __shfl_sync(0xffffffffu, i2, q + 1);
        ga = ld4(G2 + static_cast<int64_t>(i2n) * S2 + r0 * N2);
        gb = ld4(G2 + static_cast<int64_t>(i2n) * S2 + (r0 + 1) * N2);
      }
      if (p != cur) {  // a new pair run: its H column pairs into registers, S from zero
        const float* hp = H + static_cast<int64_t>(p) * W1 + r0;
#pragma unroll
        for (int a = 0; a < P1; ++a) {
          h[a] = __ldg(reinterpret_cast<const unsigned long long*>(hp + a * R2));
          s[a] = 0ull;
        }
        cur = p;
      }
      unsigned long long c0v = 0ull, c1v = 0ull, c2v = 0ull, c3v = 0ull;
      const ulonglong2* d2 = reinterpret_cast<const ulonglong2*>(dd + q * kDdStride);
#pragma unroll
      for (int a = 0; a < P1; ++a) {
        const ulonglong2 d01 = d2[2 * a], d23 = d2[2 * a + 1];  // (D2[a][j], D2[a][j]) pairs
        // S: v = Σ_j D2[a][j]·G2[r][j] (fma chain from zero), S += v
        unsigned long long v = fma2(d01.x, gp0, 0ull);
        v = fma2(d01.y, gp1, v);
        v = fma2(d23.x, gp2, v);
        v = fma2(d23.y, gp3, v);
        s[a] = add2(s[a], v);
        // C[r][j] += H[a][r]·D2[a][j] (a ascending from zero)
        c0v = fma2(h[a], d01.x, c0v);
        c1v = fma2(h[a], d01.y, c1v);
        c2v = fma2(h[a], d23.x, c2v);
        c3v = fma2(h[a], d23.y, c3v);
      }
      // C rows r0, r0 + 1 (4 columns each) at the lookup's i2-sorted position
      const float2 e0 = upk(c0v), e1 = upk(c1v), e2 = upk(c2v), e3 = upk(c3v);
      float4* co = reinterpret_cast<float4*>(contrib + static_cast<int64_t>(pq) * S2 + r0 * N2);
      co[0] = make_float4(e0.x, e1.x, e2.x, e3.x);
      co[1] = make_float4(e0.y, e1.y, e2.y, e3.y);
      // the run ends here: its S partial row (a-major, [a][r])
      const int pn = q + 1 < n ? __shfl_sync(0xffffffffu, pid, q + 1) : -2;
      if (pn != p) {
        float* so = partS + static_cast<int64_t>(rq) * W1 + r0;
#pragma unroll
        for (int a = 0; a < P1; ++a) *reinterpret_cast<unsigned long long*>(so + a * R2) = s[a];
      }
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
