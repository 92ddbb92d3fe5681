// Head backward of 3-core tables on the 5th-gen tensor cores (tcgen05,
// kind::tf32, error-compensated 3xTF32, accumulators in TMEM).
//
// Same contract as k_head_bwd (tt_kernels.cuh) -- the reference chain
// embedding_ops.hpp:335-347 at k = 1, per unique pair p = (i0, i1):
//   D0[p]          = S[p] (P0 x C1) · G1[i1]ᵀ (C1 x R1)          (D = D1 · G1ᵀ)
//   partial(run)  += Σ_{p in run} G0[i0]ᵀ (R1 x P0) · S[p]        (dG1 += u0ᵀ D1)
// over pairs in pid order, chunks of CH pairs, one partial per (chunk, i1 run)
// -- so scan1 / seg1 / k_combine downstream are unchanged.
//
// One work unit = one i1 run inside one chunk (np <= 32 pairs).  Its C1
// columns are streamed in chunks of KC = 32; per chunk (double-buffered):
//   A_S  (128 x KC, K-major over c)       rows (p, a): the S rows      -> D0 A operand
//   B_S  (KC x 128, K-major over (p, a))  the same values transposed   -> dG1 B operand
//   B_G1 (R1 x KC, K-major over c)        G1[i1] rows                  -> D0 B operand
// plus, once per unit, A_G0 (R1 x 128, K-major over (p, a)) = G0[i0]ᵀ stacked.
//   D0  (M=128, N=R1=64) accumulates over the C1 chunks       (TMEM cols [0, 64))
//   dG1 (M=R1=64, N=KC)  one accumulator per chunk            (TMEM cols 64 + c)
// Every operand is staged by the threads as hi/lo tf32 parts (tc_tf32.cuh);
// each product is hi·hi + hi·lo + lo·hi in fp32 (relative error ~1e-6, the
// backward's tolerance is 1e-4).  Padded rows (p >= np) are zero.
#pragma once

#include "tc_tf32.cuh"

namespace ttgpu {
namespace tc {

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

struct HeadTc {
  static constexpr int R1 = 64, P0 = 4, KC = 32, ROWS = 128, PAIRS = ROWS / P0;
  static constexpr uint32_t AS_B = ROWS * KC * 4;   // 16 KB
  static constexpr uint32_t BS_B = KC * ROWS * 4;   // 16 KB
  static constexpr uint32_t BG_B = R1 * KC * 4;     //  8 KB
  static constexpr uint32_t STAGE_B = 2 * (AS_B + BS_B + BG_B);
  static constexpr uint32_t AG_B = R1 * ROWS * 4;   // 32 KB
  static constexpr uint32_t SMEM = 2 * STAGE_B + 2 * AG_B;
  // K-major strides (bytes): 4-wide k groups adjacent (LBO 128), 8-row groups after all k
  static constexpr uint32_t LBO = 128;
  static constexpr uint32_t SBO_KC = (KC / 4) * 128;      // operands with K = KC
  static constexpr uint32_t SBO_KR = (ROWS / 4) * 128;    // operands with K = ROWS
  static constexpr int TMEM_COLS = 512;
};

template <int C1>
__global__ void __launch_bounds__(256, 1) k_head_bwd_tc(
    DevPlan P, const float* __restrict__ cores, const float* __restrict__ S,
    const uint32_t* __restrict__ pair_key_u, const int* __restrict__ counts,
    const unsigned long long* __restrict__ scan1, int CH, float* __restrict__ D0,
    float* __restrict__ partials) {
  using H = HeadTc;
  constexpr int R1 = H::R1, P0 = H::P0, KC = H::KC, NKC = C1 / KC;
  static_assert(C1 % KC == 0 && 64 + C1 <= H::TMEM_COLS, "C1 layout");
  constexpr int S0 = P0 * R1, S1 = R1 * C1, W1 = P0 * C1;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  unsigned char* stage[2] = {sm, sm + H::STAGE_B};
  unsigned char* AGh = sm + 2 * H::STAGE_B;
  unsigned char* AGl = AGh + H::AG_B;
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  const float* G0 = cores + P.coff[0];
  const float* G1 = cores + P.coff[1];
  if (tid == 0) {
    mbar_init1(&bar[0]);
    mbar_init1(&bar[1]);
  }
  if (wid == 0) tmem_alloc(&tbase, H::TMEM_COLS);
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tm = tbase;
  uint32_t ph[2] = {0u, 0u};
  bool pend[2] = {false, false};
  const int U = counts[0];
  const int nchunks = (U + CH - 1) / CH;
  const uint32_t m0 = static_cast<uint32_t>(P.m[0]);
  constexpr uint32_t id_d0 = idesc_tf32(128, R1, 0, 0);
  constexpr uint32_t id_g1 = idesc_tf32(R1, KC, 0, 0);

  for (int ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const int p0 = ch * CH, p1 = min(U, p0 + CH);
    int run = static_cast<int>(scan1[p0] >> 32) - 1;
    int lo = p0;
    while (lo < p1) {
      const uint32_t i1 = pair_key_u[lo] / m0;
      int hi = lo + 1;
      while (hi < p1 && pair_key_u[hi] / m0 == i1) ++hi;
      const int np = hi - lo;  // <= CH <= 32
      const int rows = P0 * np;
      const int ksteps_g1 = (rows + 7) / 8;
      // ---- A_G0 = G0[i0(p)]ᵀ stacked: (r1, k = 4p + a), zero for p >= np
      for (int e = tid; e < R1 * H::PAIRS; e += blockDim.x) {
        const int p = e / R1, r = e - p * R1;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (p < np) {
          const uint32_t i0 = pair_key_u[lo + p] % m0;
          const float* g = G0 + static_cast<int64_t>(i0) * S0 + r;
#pragma unroll
          for (int a = 0; a < P0; ++a) v[a] = __ldg(g + a * R1);
        }
        float4 h4, l4;
        split_tf32(v[0], h4.x, l4.x);
        split_tf32(v[1], h4.y, l4.y);
        split_tf32(v[2], h4.z, l4.z);
        split_tf32(v[3], h4.w, l4.w);
        const uint32_t o = kmaj_off(r, P0 * p, H::LBO, H::SBO_KR);
        *reinterpret_cast<float4*>(AGh + o) = h4;
        *reinterpret_cast<float4*>(AGl + o) = l4;
      }
      const float* Sp = S + static_cast<int64_t>(lo) * W1;
      const float* G1i = G1 + static_cast<int64_t>(i1) * S1;
      for (int kc = 0; kc < NKC; ++kc) {
        const int b = kc & 1;
        if (pend[b]) {  // the MMAs of chunk kc-2 read this buffer
          mbar_wait_parity(&bar[b], ph[b] & 1u);
          ++ph[b];
          pend[b] = false;
        }
        unsigned char* ASh = stage[b];
        unsigned char* ASl = ASh + H::AS_B;
        unsigned char* BSh = ASl + H::AS_B;
        unsigned char* BSl = BSh + H::BS_B;
        unsigned char* BGh = BSl + H::BS_B;
        unsigned char* BGl = BGh + H::BG_B;
        const int c0 = kc * KC;
        // S chunk: row = (p, a) = 4p + a, 4 consecutive columns per item
        for (int e = tid; e < H::ROWS * (KC / 4); e += blockDim.x) {
          const int row = e / (KC / 4), q = e - row * (KC / 4);
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (row < rows) v = __ldg(reinterpret_cast<const float4*>(Sp + static_cast<int64_t>(row) * C1 + c0) + q);
          float4 h4, l4;
          split_tf32(v.x, h4.x, l4.x);
          split_tf32(v.y, h4.y, l4.y);
          split_tf32(v.z, h4.z, l4.z);
          split_tf32(v.w, h4.w, l4.w);
          const uint32_t oa = kmaj_off(row, 4 * q, H::LBO, H::SBO_KC);
          *reinterpret_cast<float4*>(ASh + oa) = h4;
          *reinterpret_cast<float4*>(ASl + oa) = l4;
          // transposed copy: (n = c, k = row)
          const float hv[4] = {h4.x, h4.y, h4.z, h4.w}, lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t ob = kmaj_off(4 * q + j, row, H::LBO, H::SBO_KR);
            *reinterpret_cast<float*>(BSh + ob) = hv[j];
            *reinterpret_cast<float*>(BSl + ob) = lv[j];
          }
        }
        // G1 chunk: (n = r1, k = c)
        for (int e = tid; e < R1 * (KC / 4); e += blockDim.x) {
          const int r = e / (KC / 4), q = e - r * (KC / 4);
          const float4 v = __ldg(reinterpret_cast<const float4*>(G1i + static_cast<int64_t>(r) * C1 + c0) + q);
          float4 h4, l4;
          split_tf32(v.x, h4.x, l4.x);
          split_tf32(v.y, h4.y, l4.y);
          split_tf32(v.z, h4.z, l4.z);
          split_tf32(v.w, h4.w, l4.w);
          const uint32_t o = kmaj_off(r, 4 * q, H::LBO, H::SBO_KC);
          *reinterpret_cast<float4*>(BGh + o) = h4;
          *reinterpret_cast<float4*>(BGl + o) = l4;
        }
        fence_smem_to_async();
        __syncthreads();
        if (tid == 0) {
          fence_after_sync();
          // D0 (128 x 64) += S_chunk (128 x KC) · G1_chunkᵀ (KC x 64)
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint32_t o = ks * 256;
            const uint64_t ah = smem_desc(smem_addr(ASh + o), H::LBO, H::SBO_KC);
            const uint64_t al = smem_desc(smem_addr(ASl + o), H::LBO, H::SBO_KC);
            const uint64_t bh = smem_desc(smem_addr(BGh + o), H::LBO, H::SBO_KC);
            const uint64_t bl = smem_desc(smem_addr(BGl + o), H::LBO, H::SBO_KC);
            const uint32_t first = (kc == 0 && ks == 0) ? 0u : 1u;
            mma_tf32(tm, al, bh, id_d0, first);
            mma_tf32(tm, ah, bl, id_d0, 1u);
            mma_tf32(tm, ah, bh, id_d0, 1u);
          }
          // dG1[:, c0:c0+KC] (64 x KC) = G0stackᵀ (64 x rows) · S_chunk (rows x KC)
          const uint32_t dg = tm + 64 + static_cast<uint32_t>(c0);
          for (int ks = 0; ks < ksteps_g1; ++ks) {
            const uint32_t o = ks * 256;
            const uint64_t ah = smem_desc(smem_addr(AGh + o), H::LBO, H::SBO_KR);
            const uint64_t al = smem_desc(smem_addr(AGl + o), H::LBO, H::SBO_KR);
            const uint64_t bh = smem_desc(smem_addr(BSh + o), H::LBO, H::SBO_KR);
            const uint64_t bl = smem_desc(smem_addr(BSl + o), H::LBO, H::SBO_KR);
            mma_tf32(dg, al, bh, id_g1, ks == 0 ? 0u : 1u);
            mma_tf32(dg, ah, bl, id_g1, 1u);
            mma_tf32(dg, ah, bh, id_g1, 1u);
          }
          commit(&bar[b]);
        }
        __syncwarp();
        pend[b] = true;
      }
      // every MMA of the unit has landed in TMEM
#pragma unroll
      for (int b = 0; b < 2; ++b)
        if (pend[b]) {
          mbar_wait_parity(&bar[b], ph[b] & 1u);
          ++ph[b];
          pend[b] = false;
        }
      fence_after_sync();
      // ---- epilogue: warp w reads TMEM lanes 32*(w%4) .. +31
      const int q = wid & 3, half = wid >> 2;
      {  // D0: row m = 32q + lane (M=128: row m in lane m), columns [32 half, +32)
        const int m = 32 * q + lane;
#pragma unroll
        for (int c16 = 0; c16 < 2; ++c16) {
          float v[16];
          const int col = 32 * half + 16 * c16;
          ld_32x32b_x16(tm + (static_cast<uint32_t>(32 * q) << 16) + col, v);
          if (m < rows) {
            float* dst = D0 + static_cast<int64_t>(lo + m / P0) * S0 + (m % P0) * R1 + col;
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
      }
      {  // dG1 (M=64: row r in lane (r%16) + 32*(r/16)), columns [C1/2 * half, +C1/2)
        const int r = 16 * q + lane;
        float* dst = partials + static_cast<int64_t>(run) * S1 + static_cast<int64_t>(r) * C1;
#pragma unroll 1
        for (int c16 = 0; c16 < C1 / 32; ++c16) {
          float v[16];
          const int col = (C1 / 2) * half + 16 * c16;
          ld_32x32b_x16(tm + (static_cast<uint32_t>(32 * q) << 16) + 64 + col, v);
          if (lane < 16) {
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(dst + col + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
      }
      fence_before_sync();
      __syncthreads();  // TMEM and the A_G0 / stage buffers are reused by the next unit
      fence_after_sync();
      ++run;
      lo = hi;
    }
  }
  fence_before_sync();
  __syncthreads();
  if (wid == 0) tmem_dealloc(tm, H::TMEM_COLS);
}

}  // namespace tc
}  // namespace ttgpu
