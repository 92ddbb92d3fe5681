// tcgen05 (5th-gen tensor core) building blocks for the error-compensated
// 3xTF32 contractions: TMEM allocation, UMMA shared-memory / instruction
// descriptors, kind::tf32 MMA issue, commit to an mbarrier, TMEM -> register
// loads.  sm_100a only (PTX ISA 8.6+).
//
// Operand layout used everywhere: SWIZZLE_NONE ("interleave") canonical UMMA
// layouts built by ordinary st.shared from registers (every operand here is
// gathered and split into hi/lo parts by threads, so no TMA tensor map is
// needed).  A "core matrix" is 8 rows x 16 bytes (4 tf32) stored as 128
// contiguous bytes:
//   K-major  (rows = M or N, 4 consecutive K per core row):
//     byte(r, k) = (r%8)*16 + (k%4)*4 + (r/8)*SBO + (k/4)*LBO
//   MN-major (core = 8 consecutive K rows of 4 consecutive M/N):
//     byte(r, k) = (r%4)*4 + (k%8)*16 + (r/4)*SBO + (k/8)*LBO
// (cute::UMMA::make_umma_desc, Major::K / Major::MN INTERLEAVE.)
//
// 3xTF32: x = hi + lo with hi = x with the low 13 mantissa bits cleared (what
// the tensor core reads of an fp32 operand) and lo = x - hi (exact in fp32);
// a*b ~= hi_a*hi_b + hi_a*lo_b + lo_a*hi_b, accumulated in fp32 in TMEM.
#pragma once

#include <cstdint>

namespace ttgpu {
namespace tc {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- TMEM allocation (one full warp executes these) ------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_addr(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// st.shared (generic proxy) -> visible to tcgen05.mma operand reads (async proxy)
__device__ __forceinline__ void fence_smem_to_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- descriptors -----------------------------------------------------------
// SWIZZLE_NONE shared-memory matrix descriptor (version 1 = sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  return d;                              // base offset 0, lbo mode 0, layout 0 (no swizzle)
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, dense.
// a_mn / b_mn: 1 = MN-major operand, 0 = K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)                                  // D format F32
         | (2u << 7)                                // A format TF32
         | (2u << 10)                               // B format TF32
         | (static_cast<uint32_t>(a_mn) << 15)      // A major
         | (static_cast<uint32_t>(b_mn) << 16)      // B major
         | (static_cast<uint32_t>(N >> 3) << 17)    // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);   // M / 16
}

// D[tmem] (+)= A[smem] * B[smem]; issued by ONE thread for the whole CTA.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Arrive (count 1) on an mbarrier when every MMA issued so far by this thread
// has completed (implies tcgen05.fence::before_thread_sync).
__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(mbar))
               : "memory");
}

// 32 lanes x 16 consecutive 32-bit columns: thread t of the warp gets lane
// (taddr.lane + t), columns taddr.col .. +15.  The warp may only address its
// own 32-lane quarter (warp_id % 4).
__device__ __forceinline__ void ld_32x32b_x16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// fp32 -> (hi, lo) with hi exactly representable in tf32 (low 13 bits clear).
__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  lo = x - hi;
}

// Byte offset of element (r, k) in a SWIZZLE_NONE K-major operand.
__host__ __device__ constexpr uint32_t kmaj_off(int r, int k, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint32_t>((r & 7) * 16 + (k & 3) * 4) + static_cast<uint32_t>(r >> 3) * sbo +
         static_cast<uint32_t>(k >> 2) * lbo;
}
// Byte offset of element (r, k) in a SWIZZLE_NONE MN-major operand.
__host__ __device__ constexpr uint32_t mnmaj_off(int r, int k, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint32_t>((r & 3) * 4 + (k & 7) * 16) + static_cast<uint32_t>(r >> 2) * sbo +
         static_cast<uint32_t>(k >> 3) * lbo;
}

}  // namespace tc
}  // namespace ttgpu
