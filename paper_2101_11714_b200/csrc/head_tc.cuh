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

__device__ __forceinline__ void mbar_init1(uint64_t* bar, uint32_t count = 1) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
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

template <int C1, int NT>
__global__ void __launch_bounds__(NT, 1) k_head_bwd_tc(
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
  if (tid == 0) {  // two MMA issuers (D0: thread 0, dG1: thread 32) commit to each buffer
    mbar_init1(&bar[0], 2);
    mbar_init1(&bar[1], 2);
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
      // run end: every warp reads the chunk's (<= 32) keys at once and ballots
      const uint32_t i1 = pair_key_u[lo] / m0;
      int hi;
      {
        const int pp = lo + lane;
        const bool diff = pp < p1 && pair_key_u[pp] / m0 != i1;
        const unsigned m = __ballot_sync(0xffffffffu, diff || pp >= p1);
        hi = lo + (m ? __ffs(m) - 1 : 32);
      }
      const int np = hi - lo;  // <= CH <= 32
      const int rows = P0 * np;
      const int ksteps_g1 = (rows + 7) / 8;
      const float* Sp = S + static_cast<int64_t>(lo) * W1;
      const float* G1i = G1 + static_cast<int64_t>(i1) * S1;
      // this thread's items of a C1 chunk: S (row, 4 columns) x NSI, G1 (r1, 4 columns) x NGI,
      // loaded into registers one chunk ahead of their smem stores
      constexpr int NSI = H::ROWS * (KC / 4) / NT, NGI = R1 * (KC / 4) / NT;
      float4 sreg[NSI], greg[NGI];
      auto load_chunk = [&](int kc) {
        const int c0 = kc * KC;
#pragma unroll
        for (int j = 0; j < NSI; ++j) {
          const int e = tid + NT * j, row = e / (KC / 4), q = e - row * (KC / 4);
          sreg[j] = row < rows
                        ? __ldg(reinterpret_cast<const float4*>(Sp + static_cast<int64_t>(row) * C1 + c0) + q)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < NGI; ++j) {
          const int e = tid + NT * j, r = e / (KC / 4), q = e - r * (KC / 4);
          greg[j] = __ldg(reinterpret_cast<const float4*>(G1i + static_cast<int64_t>(r) * C1 + c0) + q);
        }
      };
      load_chunk(0);
      // ---- A_G0 = G0[i0(p)]ᵀ stacked: (r1, k = 4p + a), zero for p >= np (loads batched)
      {
        constexpr int NAI = R1 * H::PAIRS / NT;
        float v[NAI][4];
#pragma unroll
        for (int j = 0; j < NAI; ++j) {
          const int e = tid + NT * j, p = e / R1, r = e - p * R1;
          if (p < np) {
            const uint32_t i0 = pair_key_u[lo + p] % m0;
            const float* g = G0 + static_cast<int64_t>(i0) * S0 + r;
#pragma unroll
            for (int a = 0; a < P0; ++a) v[j][a] = __ldg(g + a * R1);
          } else {
#pragma unroll
            for (int a = 0; a < P0; ++a) v[j][a] = 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < NAI; ++j) {
          const int e = tid + NT * j, p = e / R1, r = e - p * R1;
          float4 h4, l4;
          split_tf32(v[j][0], h4.x, l4.x);
          split_tf32(v[j][1], h4.y, l4.y);
          split_tf32(v[j][2], h4.z, l4.z);
          split_tf32(v[j][3], h4.w, l4.w);
          const uint32_t o = kmaj_off(r, P0 * p, H::LBO, H::SBO_KR);
          *reinterpret_cast<float4*>(AGh + o) = h4;
          *reinterpret_cast<float4*>(AGl + o) = l4;
        }
      }
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
#pragma unroll
        for (int j = 0; j < NSI; ++j) {  // S chunk: row = (p, a) = 4p + a
          const int e = tid + NT * j, row = e / (KC / 4), q = e - row * (KC / 4);
          float4 h4, l4;
          split_tf32(sreg[j].x, h4.x, l4.x);
          split_tf32(sreg[j].y, h4.y, l4.y);
          split_tf32(sreg[j].z, h4.z, l4.z);
          split_tf32(sreg[j].w, h4.w, l4.w);
          const uint32_t oa = kmaj_off(row, 4 * q, H::LBO, H::SBO_KC);
          *reinterpret_cast<float4*>(ASh + oa) = h4;
          *reinterpret_cast<float4*>(ASl + oa) = l4;
          // transposed copy: (n = c, k = row)
          const float hv[4] = {h4.x, h4.y, h4.z, h4.w}, lv[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            const uint32_t ob = kmaj_off(4 * q + jj, row, H::LBO, H::SBO_KR);
            *reinterpret_cast<float*>(BSh + ob) = hv[jj];
            *reinterpret_cast<float*>(BSl + ob) = lv[jj];
          }
        }
#pragma unroll
        for (int j = 0; j < NGI; ++j) {  // G1 chunk: (n = r1, k = c)
          const int e = tid + NT * j, r = e / (KC / 4), q = e - r * (KC / 4);
          float4 h4, l4;
          split_tf32(greg[j].x, h4.x, l4.x);
          split_tf32(greg[j].y, h4.y, l4.y);
          split_tf32(greg[j].z, h4.z, l4.z);
          split_tf32(greg[j].w, h4.w, l4.w);
          const uint32_t o = kmaj_off(r, 4 * q, H::LBO, H::SBO_KC);
          *reinterpret_cast<float4*>(BGh + o) = h4;
          *reinterpret_cast<float4*>(BGl + o) = l4;
        }
        if (kc + 1 < NKC) load_chunk(kc + 1);  // in flight during the MMAs of this chunk
        fence_smem_to_async();
        __syncthreads();
        // descriptors: start address field (bits 0..13, 16-byte units) advanced
        // from a per-operand base -- no carry: every operand lies inside the CTA's smem
        if (tid == 0) {
          fence_after_sync();
          // D0 (128 x 64) += S_chunk (128 x KC) · G1_chunkᵀ (KC x 64)
          const uint64_t ah0 = smem_desc(smem_addr(ASh), H::LBO, H::SBO_KC);
          const uint64_t al0 = smem_desc(smem_addr(ASl), H::LBO, H::SBO_KC);
          const uint64_t bh0 = smem_desc(smem_addr(BGh), H::LBO, H::SBO_KC);
          const uint64_t bl0 = smem_desc(smem_addr(BGl), H::LBO, H::SBO_KC);
#pragma unroll
          for (int ks = 0; ks < KC / 8; ++ks) {
            const uint64_t o = static_cast<uint64_t>(ks * 256 / 16);
            const uint32_t first = (kc == 0 && ks == 0) ? 0u : 1u;
            mma_tf32(tm, al0 + o, bh0 + o, id_d0, first);
            mma_tf32(tm, ah0 + o, bl0 + o, id_d0, 1u);
            mma_tf32(tm, ah0 + o, bh0 + o, id_d0, 1u);
          }
          commit(&bar[b]);
        } else if (tid == 32) {
          fence_after_sync();
          // dG1[:, c0:c0+KC] (64 x KC) = G0stackᵀ (64 x rows) · S_chunk (rows x KC)
          const uint32_t dg = tm + 64 + static_cast<uint32_t>(c0);
          const uint64_t ah0 = smem_desc(smem_addr(AGh), H::LBO, H::SBO_KR);
          const uint64_t al0 = smem_desc(smem_addr(AGl), H::LBO, H::SBO_KR);
          const uint64_t bh0 = smem_desc(smem_addr(BSh), H::LBO, H::SBO_KR);
          const uint64_t bl0 = smem_desc(smem_addr(BSl), H::LBO, H::SBO_KR);
          for (int ks = 0; ks < ksteps_g1; ++ks) {
            const uint64_t o = static_cast<uint64_t>(ks * 256 / 16);
            mma_tf32(dg, al0 + o, bh0 + o, id_g1, ks == 0 ? 0u : 1u);
            mma_tf32(dg, ah0 + o, bl0 + o, id_g1, 1u);
            mma_tf32(dg, ah0 + o, bh0 + o, id_g1, 1u);
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
      constexpr int NG = NT / 128;  // warp groups: columns split between them
      const int q = wid & 3, grp = wid >> 2;
      {  // D0: row m = 32q + lane (M=128: row m in lane m), columns [64/NG grp, +64/NG)
        const int m = 32 * q + lane;
#pragma unroll
        for (int c16 = 0; c16 < 4 / NG; ++c16) {
          float v[16];
          const int col = (64 / NG) * grp + 16 * c16;
          ld_32x32b_x16(tm + (static_cast<uint32_t>(32 * q) << 16) + col, v);
          if (m < rows) {
            float* dst = D0 + static_cast<int64_t>(lo + m / P0) * S0 + (m % P0) * R1 + col;
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          }
        }
      }
      {  // dG1 (M=64: row r in lane (r%16) + 32*(r/16)), columns [C1/NG grp, +C1/NG)
        const int r = 16 * q + lane;
        float* dst = partials + static_cast<int64_t>(run) * S1 + static_cast<int64_t>(r) * C1;
#pragma unroll 1
        for (int c16 = 0; c16 < C1 / (16 * NG); ++c16) {
          float v[16];
          const int col = (C1 / NG) * grp + 16 * c16;
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
