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
constexpr size_t kBwdSmem = sizeof(float) * kWarps * kChunk * N;  // 64 KB

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// ---------------------------------------------------------------- forward --
template <bool kExact>
__global__ void __launch_bounds__(kWarps * 32) k_w3_fwd(const float* __restrict__ G2,
                                                        const float* __restrict__ H,
                                                        const int32_t* __restrict__ lk_pid,
                                                        const uint32_t* __restrict__ tail_dig,
                                                        const uint32_t* __restrict__ s_lk, int64_t L,
                                                        float* __restrict__ y) {
  __shared__ __align__(16) float hs_all[kWarps][R2 * P1];  // H staged transposed: [r][a]
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* hs = hs_all[wid];
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
    const float* g2 = G2 + static_cast<int64_t>(i2) * S2;
    for (int q0 = 0; q0 < n;) {
      const int p = __shfl_sync(0xffffffffu, pid, q0);
      const unsigned same = __ballot_sync(0xffffffffu, lane < n && pid == p);
      const int q1 = 32 - __clz(same);  // runs are contiguous: last member + 1
      __syncwarp();
      // H[p] (P1 x R2, a-major) -> hs[r][a]
      const float* hp = H + static_cast<int64_t>(p) * W1;
#pragma unroll
      for (int k = 0; k < W1 / 32 / 4; ++k) {
        const int e = (k * 32 + lane) * 4;  // 4 consecutive r of one a
        const float4 v = ld4(hp + e);
        const int a = e / R2, r = e - a * R2;
        hs[(r + 0) * P1 + a] = v.x;
        hs[(r + 1) * P1 + a] = v.y;
        hs[(r + 2) * P1 + a] = v.z;
        hs[(r + 3) * P1 + a] = v.w;
      }
      __syncwarp();
      if (lane >= q0 && lane < q1) {
        float4 acc[P1];
#pragma unroll
        for (int a = 0; a < P1; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (int r = 0; r < R2; ++r) {
          const float4 g = ld4(g2 + r * N2);
          const float4* h4 = reinterpret_cast<const float4*>(hs + r * P1);
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
        float4* yo = reinterpret_cast<float4*>(y + static_cast<int64_t>(l) * N);
#pragma unroll
        for (int a = 0; a < P1; ++a) yo[a] = acc[a];
      }
      q0 = q1;
    }
  }
}

// --------------------------------------------------------------- backward --
__global__ void __launch_bounds__(kWarps * 32, 2) k_w3_bwd(
    const float* __restrict__ G2, const float* __restrict__ H, const int32_t* __restrict__ lk_pid,
    const uint32_t* __restrict__ tail_dig, const int32_t* __restrict__ lk_bag,
    const float* __restrict__ lk_alpha, const float* __restrict__ grad,
    const uint32_t* __restrict__ s_lk, const unsigned long long* __restrict__ scan,
    const uint32_t* __restrict__ pos2, int64_t L, float* __restrict__ partS,
    float* __restrict__ contrib) {
  extern __shared__ __align__(16) float w3_dyn[];  // [kWarps][kChunk * N]: the chunk's D2 rows
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* d2s = w3_dyn + wid * kChunk * N;
  const int r0 = 2 * lane;  // this lane's two columns r0, r0 + 1
  const int64_t nchunks = (L + kChunk - 1) / kChunk;
  for (int64_t ch = static_cast<int64_t>(blockIdx.x) * kWarps + wid; ch < nchunks;
       ch += static_cast<int64_t>(gridDim.x) * kWarps) {
    const int64_t c0 = ch * kChunk;
    const int n = static_cast<int>(L - c0 < kChunk ? L - c0 : kChunk);
    int pid = -1, i2 = 0, run = 0;
    uint32_t p2 = 0;
    __syncwarp();
    if (lane < n) {
      const int l = static_cast<int>(s_lk[c0 + lane]);
      pid = lk_pid[l];
      i2 = static_cast<int>(tail_dig[l]);
      run = static_cast<int>(scan[c0 + lane] >> 32) - 1;
      p2 = pos2[l];
      // D2 = T(alpha)·grad[bag], one row per lane
      const float al = lk_alpha[l];
      const float4* gr = reinterpret_cast<const float4*>(grad + static_cast<int64_t>(lk_bag[l]) * N);
      float4* dst = reinterpret_cast<float4*>(d2s + lane * N);
#pragma unroll
      for (int k = 0; k < N / 4; ++k) {
        const float4 v = __ldg(gr + k);
        dst[k] = make_float4(__fmul_rn(al, v.x), __fmul_rn(al, v.y), __fmul_rn(al, v.z),
                             __fmul_rn(al, v.w));
      }
    }
    __syncwarp();
    float2 h[P1], s[P1];
    int cur = -1;
    // G2 rows of the first lookup; later ones are loaded one lookup ahead
    int i2n = __shfl_sync(0xffffffffu, i2, 0);
    float4 ga = ld4(G2 + static_cast<int64_t>(i2n) * S2 + r0 * N2);
    float4 gb = ld4(G2 + static_cast<int64_t>(i2n) * S2 + (r0 + 1) * N2);
    for (int q = 0; q < n; ++q) {
      const int p = __shfl_sync(0xffffffffu, pid, q);
      const int rq = __shfl_sync(0xffffffffu, run, q);
      const uint32_t pq = __shfl_sync(0xffffffffu, p2, q);
      const float4 g0 = ga, g1 = gb;
      if (q + 1 < n) {
        i2n = __shfl_sync(0xffffffffu, i2, q + 1);
        ga = ld4(G2 + static_cast<int64_t>(i2n) * S2 + r0 * N2);
        gb = ld4(G2 + static_cast<int64_t>(i2n) * S2 + (r0 + 1) * N2);
      }
      if (p != cur) {  // a new pair run: its H columns into registers, S from zero
        const float* hp = H + static_cast<int64_t>(p) * W1 + r0;
#pragma unroll
        for (int a = 0; a < P1; ++a) {
          h[a] = __ldg(reinterpret_cast<const float2*>(hp + a * R2));
          s[a] = make_float2(0.f, 0.f);
        }
        cur = p;
      }
      float2 c[N2];
#pragma unroll
      for (int j = 0; j < N2; ++j) c[j] = make_float2(0.f, 0.f);
      const float4* d4 = reinterpret_cast<const float4*>(d2s + q * N);
#pragma unroll
      for (int a = 0; a < P1; ++a) {
        const float4 d = d4[a];  // D2[a][0..3] (broadcast)
        // S: v = Σ_j D2[a][j]·G2[r][j] (fma chain from zero), S += v
        float v0 = 0.f, v1 = 0.f;
        ffma2(d.x, g0.x, g1.x, v0, v1);
        ffma2(d.y, g0.y, g1.y, v0, v1);
        ffma2(d.z, g0.z, g1.z, v0, v1);
        ffma2(d.w, g0.w, g1.w, v0, v1);
        s[a].x += v0;
        s[a].y += v1;
        // C[r][j] += H[a][r]·D2[a][j] (a ascending from zero)
        ffma2(d.x, h[a].x, h[a].y, c[0].x, c[0].y);
        ffma2(d.y, h[a].x, h[a].y, c[1].x, c[1].y);
        ffma2(d.z, h[a].x, h[a].y, c[2].x, c[2].y);
        ffma2(d.w, h[a].x, h[a].y, c[3].x, c[3].y);
      }
      // C rows r0, r0 + 1 (4 columns each) at the lookup's i2-sorted position
      float4* co = reinterpret_cast<float4*>(contrib + static_cast<int64_t>(pq) * S2 + r0 * N2);
      co[0] = make_float4(c[0].x, c[1].x, c[2].x, c[3].x);
      co[1] = make_float4(c[0].y, c[1].y, c[2].y, c[3].y);
      // the run ends here: its S partial row (a-major, [a][r])
      const int pn = q + 1 < n ? __shfl_sync(0xffffffffu, pid, q + 1) : -2;
      if (pn != p) {
        float* so = partS + static_cast<int64_t>(rq) * W1 + r0;
#pragma unroll
        for (int a = 0; a < P1; ++a) *reinterpret_cast<float2*>(so + a * R2) = s[a];
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
