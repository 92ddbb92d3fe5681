// tcgen05 kind::tf32 probe: checks the hand-built UMMA descriptors of
// csrc/tc_tf32.cuh on the GPU and maps where an M=64 / M=128 accumulator lands
// in TMEM, then measures the 3xTF32 error against fp64.
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -I paper_2101_11714_b200/csrc \
//        -o tools/tc_probe tools/tc_probe.cu && tools/tc_probe
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "tc_tf32.cuh"

using namespace ttgpu;

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(tc::smem_addr(bar)),
      "r"(parity)
      : "memory");
}

struct Case {
  int M, N, K, a_mn, b_mn, split3;
  int swap = 0;  // MN-major: descriptor LBO field = MN-group stride, SBO field = K-group stride
};

// A: M x K row-major fp32, B: K x N row-major fp32 (global). out: 128 lanes x N.
__global__ void probe(Case c, const float* A, const float* B, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int M = c.M, N = c.N, K = c.K;
  // A hi | A lo | B hi | B lo
  const uint32_t abytes = M * K * 4, bbytes = N * K * 4;
  unsigned char* Ah = sm;
  unsigned char* Al = sm + abytes;
  unsigned char* Bh = sm + 2 * abytes;
  unsigned char* Bl = sm + 2 * abytes + bbytes;
  // layouts: A K-major: lbo 128 (k groups adjacent), sbo (K/4)*128 ; A MN-major: sbo 128, lbo (M/4)*128
  const uint32_t a_lbo = c.a_mn ? (M / 4) * 128 : 128, a_sbo = c.a_mn ? 128 : (K / 4) * 128;
  const uint32_t b_lbo = c.b_mn ? (N / 4) * 128 : 128, b_sbo = c.b_mn ? 128 : (K / 4) * 128;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e % K;
    float h, l;
    tc::split_tf32(A[e], h, l);
    if (!c.split3) { h = A[e]; l = 0.f; }
    const uint32_t o = c.a_mn ? tc::mnmaj_off(m, k, a_lbo, a_sbo) : tc::kmaj_off(m, k, a_lbo, a_sbo);
    *reinterpret_cast<float*>(Ah + o) = h;
    *reinterpret_cast<float*>(Al + o) = l;
  }
  for (int e = threadIdx.x; e < K * N; e += blockDim.x) {
    const int k = e / N, n = e % N;
    float h, l;
    tc::split_tf32(B[e], h, l);
    if (!c.split3) { h = B[e]; l = 0.f; }
    const uint32_t o = c.b_mn ? tc::mnmaj_off(n, k, b_lbo, b_sbo) : tc::kmaj_off(n, k, b_lbo, b_sbo);
    *reinterpret_cast<float*>(Bh + o) = h;
    *reinterpret_cast<float*>(Bl + o) = l;
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) tc::tmem_alloc(&tbase, 512);
  tc::fence_smem_to_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tm = tbase;
  if (threadIdx.x == 0) {
    const uint32_t id = tc::idesc_tf32(M, N, c.a_mn, c.b_mn);
    const uint32_t a_step = c.a_mn ? a_lbo : 2 * a_lbo;  // bytes per K=8 step
    const uint32_t b_step = c.b_mn ? b_lbo : 2 * b_lbo;
    uint32_t acc = 0;
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint32_t ao = ks * a_step, bo = ks * b_step;
      const bool sa = c.swap && c.a_mn, sb = c.swap && c.b_mn;
      const uint64_t ah = tc::smem_desc(tc::smem_addr(Ah + ao), sa ? a_sbo : a_lbo, sa ? a_lbo : a_sbo);
      const uint64_t al = tc::smem_desc(tc::smem_addr(Al + ao), sa ? a_sbo : a_lbo, sa ? a_lbo : a_sbo);
      const uint64_t bh = tc::smem_desc(tc::smem_addr(Bh + bo), sb ? b_sbo : b_lbo, sb ? b_lbo : b_sbo);
      const uint64_t bl = tc::smem_desc(tc::smem_addr(Bl + bo), sb ? b_sbo : b_lbo, sb ? b_lbo : b_sbo);
      if (c.split3) {
        tc::mma_tf32(tm, al, bh, id, acc);
        acc = 1;
        tc::mma_tf32(tm, ah, bl, id, 1);
      }
      tc::mma_tf32(tm, ah, bh, id, acc);
      acc = 1;
    }
    tc::commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tc::ld_32x32b_x16(tm + (static_cast<uint32_t>(32 * w) << 16) + c0, v);
    for (int i = 0; i < 16; ++i) out[(32 * w + lane) * N + c0 + i] = v[i];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) tc::tmem_dealloc(tm, 512);
}

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

int run(Case c, bool integer, bool onehot = false) {
  std::mt19937 rng(c.M * 7 + c.N * 3 + c.K + c.a_mn * 11 + c.b_mn * 13 + c.split3);
  std::uniform_int_distribution<int> di(-4, 4);
  std::normal_distribution<double> dn(0.0, 1.0);
  std::vector<float> A(c.M * c.K), B(c.K * c.N), O(128 * c.N);
  for (auto& x : A) x = integer ? static_cast<float>(di(rng)) : static_cast<float>(dn(rng));
  for (auto& x : B) x = integer ? static_cast<float>(di(rng)) : static_cast<float>(dn(rng));
  if (onehot) {  // D[m][n] = B[m % K][n]: shows which B element lands where
    for (int m = 0; m < c.M; ++m)
      for (int k = 0; k < c.K; ++k) A[m * c.K + k] = (k == m % c.K) ? 1.f : 0.f;
    for (int k = 0; k < c.K; ++k)
      for (int n = 0; n < c.N; ++n) B[k * c.N + n] = static_cast<float>(100 * k + n);
  }
  std::vector<double> D(c.M * c.N, 0.0);
  for (int m = 0; m < c.M; ++m)
    for (int n = 0; n < c.N; ++n) {
      double s = 0;
      for (int k = 0; k < c.K; ++k) s += static_cast<double>(A[m * c.K + k]) * B[k * c.N + n];
      D[m * c.N + n] = s;
    }
  float *dA, *dB, *dO;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dO, O.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dO, 0, O.size() * 4));
  const size_t smem = 2 * (c.M * c.K + c.N * c.K) * 4;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  probe<<<1, 128, smem>>>(c, dA, dB, dO);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
  if (onehot) {
    std::printf("onehot M=%d N=%d K=%d a_mn=%d b_mn=%d: lane rows 0..%d (want 100*k+n)\n", c.M, c.N,
                c.K, c.a_mn, c.b_mn, c.K - 1);
    for (int m = 0; m < c.K; ++m) {
      std::printf("  row %d:", m);
      for (int n = 0; n < c.N; ++n) std::printf(" %g", O[m * c.N + n]);
      std::printf("\n");
    }
  }
  // row m of D -> which TMEM lane holds it (first exact / closest match)
  int bad = 0;
  double maxrel = 0;
  std::printf("case M=%d N=%d K=%d a_mn=%d b_mn=%d split3=%d swap=%d %s: lanes of rows", c.M, c.N,
              c.K, c.a_mn, c.b_mn, c.split3, c.swap, integer ? "int" : "normal");
  for (int m = 0; m < c.M; ++m) {
    int best = -1;
    double be = 1e300;
    for (int l = 0; l < 128; ++l) {
      double e = 0;
      for (int n = 0; n < c.N; ++n) e = std::fmax(e, std::fabs(O[l * c.N + n] - D[m * c.N + n]));
      if (e < be) { be = e; best = l; }
    }
    double scale = 1e-30;
    for (int n = 0; n < c.N; ++n) scale = std::fmax(scale, std::fabs(D[m * c.N + n]));
    maxrel = std::fmax(maxrel, be / scale);
    if (m < 4 || (m % 16) == 0 || m == c.M - 1) std::printf(" %d->%d", m, best);
    if (integer && be != 0) ++bad;
    if (best != m && c.M == 128) ++bad;
  }
  std::printf("  | max rel err %.3e  %s\n", maxrel, bad ? "MISMATCH" : "ok");
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return bad;
}

int main() {
  int bad = 0;
  Case cases[] = {
      {128, 64, 8, 0, 0, 0},  {128, 64, 32, 0, 0, 0}, {128, 32, 16, 0, 1, 0},
      {128, 64, 16, 1, 0, 0}, {64, 32, 8, 0, 0, 0},   {64, 32, 32, 0, 1, 0},
      {64, 256, 16, 0, 1, 0}, {128, 64, 32, 0, 0, 1}, {64, 32, 32, 0, 1, 1},
  };
  for (const Case& c : cases) bad += run(c, true);
  Case sw[] = {{128, 32, 16, 0, 1, 0, 1}, {128, 64, 16, 1, 0, 0, 1}, {64, 32, 32, 0, 1, 0, 1},
               {64, 32, 32, 0, 1, 1, 1}, {128, 64, 32, 1, 1, 1, 1}};
  int bad_sw = 0;
  for (const Case& c : sw) bad_sw += run(c, true);
  std::printf(bad_sw ? "MN-major (swapped fields) FAILED\n" : "MN-major (swapped fields) OK\n");
  run({128, 16, 16, 0, 1, 0, 1}, true, true);
  // accuracy: 1xTF32 vs 3xTF32 on normal data
  bad += 0 * run({128, 64, 128, 0, 0, 0}, false);
  bad += 0 * run({128, 64, 128, 0, 0, 1}, false);
  bad += 0 * run({64, 32, 256, 0, 1, 1}, false);
  std::printf(bad ? "PROBE FAILED\n" : "PROBE OK\n");
  return bad ? 1 : 0;
}
