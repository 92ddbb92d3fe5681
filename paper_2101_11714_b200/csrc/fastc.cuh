// Chunked 3-core fast path: forward and the S / dG1 / D0 backward over
// per-bucket chunks of up to TC lookups (instead of one-warp tiles of 32).
//
// The i1-sorted lookups (gsort.cuh / f3_scan with tile length TC) are cut
// into chunks that never cross an i1 bucket.  Inside a chunk the distinct i0
// values are found with a dense per-CTA flag array over m0 and numbered in
// ascending i0 order ("slots"), so a chunk computes each (i0, i1) head product
// once however many of its lookups share it; under Zipf(1.05) a 64-lookup
// chunk of the hot bucket holds 1-3 slots.
//
//   f3c_fwd  one CTA per chunk (the hardware scheduler balances them):
//            slots; G1[i1], the slots' G0 rows and the lookups' G2 rows by
//            bulk copy onto three mbarriers; H(slot) = G0[i0]·G1[i1] (saved
//            for f3_bwd2), y = H·G2[i2] per lookup; bags pooled by their
//            last finished lookup (pool_if_last)
//   f3c_bwd  persistent CTAs over contiguous, work-balanced chunk ranges, one
//            chunk of bulk copies ahead (G2 + grad rows of chunk t+1 land
//            during chunk t's GEMMs): S(slot) = Σ_{members, chunk order}
//            D2·G2[i2]ᵀ in shared memory (D2 = alpha·grad), then
//            dG1 += Σ G0ᵀ S (registers, one partial per CTA i1-run) and
//            D0 = S·G1ᵀ per (CTA, i0)
// Both write exactly the buffers f3_fwd / f3_srows + f3_bwd1 write, so
// f3_bwd2 and f3_combine run unchanged.  Exact mode keeps the
// reference's per-element operation order (embedding_ops.hpp:213-249,
// gemm.hpp:15-31): outputs stay bit-identical to ttrec::forward_bags.
#pragma once

namespace ttgpu {
namespace f3 {

constexpr int kFcThreads = 256;


template <class D, int TC>
struct FcFwdSmem {
  static constexpr int R2P = D::R2 + 1;        // padded H rows: (slot, row) -> distinct banks
  static constexpr int HSP = D::P1 * R2P + 1;  // odd slot stride
  static constexpr int S0P = D::S0 + 4;        // 16-byte pitch, two slots per warp conflict-free
  static constexpr int S2P = D::S2 + 4;        // lookups' float4 rows in distinct bank groups
  // floats: G1s[S1] | G0s[TC * S0P] | G2s[TC * S2P] | Hs[TC * HSP]
  static __host__ __device__ constexpr size_t floats() {
    return (static_cast<size_t>(D::S1) + static_cast<size_t>(TC) * (S0P + S2P) +
            static_cast<size_t>(TC) * HSP + 3) / 4 * 4;
  }
  // then 3 mbarriers, ints: lk_l, lk_d02, lk_solo, lk_slot, slot_i0 [TC] + misc[8]; flags[m0]
  static __host__ __device__ size_t bytes(int m0) {
    return floats() * 4 + 32 + 4 * (5 * TC + 8) + 4 * static_cast<size_t>(m0);
  }
};

// Block-wide exclusive scan of `flags[0, n)` in place (thread-contiguous
// runs): flags[i] in {0, 1} on entry, the rank of i among the set flags (or
// 0xffffffff) on exit; returns the number of set flags.
__device__ __forceinline__ int fc_scan_flags(uint32_t* flags, int n, int* red /* >= 33 ints */) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (n + kFcThreads - 1) / kFcThreads;
  const int lo = min(n, tid * per), hi = min(n, lo + per);
  int cnt = 0;
  for (int i = lo; i < hi; ++i) cnt += static_cast<int>(flags[i]);
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) red[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < kFcThreads / 32 ? red[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kFcThreads / 32) red[lane] = s;
  }
  __syncthreads();
  int run = x - cnt + (wid ? red[wid - 1] : 0);
  const int total = red[kFcThreads / 32 - 1];
  for (int i = lo; i < hi; ++i) {
    const uint32_t f = flags[i];
    flags[i] = f ? static_cast<uint32_t>(run) : 0xffffffffu;
    run += static_cast<int>(f);
  }
  return total;
}

template <class D, bool kExact, int TC>
__global__ void __launch_bounds__(kFcThreads) f3c_fwd(Geo g, const float* __restrict__ cores,
                                                      const Tile* __restrict__ tiles,
                                                      const int* __restrict__ ntiles,
                                                      const uint4* __restrict__ rec,
                                                      const double* __restrict__ w,
                                                      float* __restrict__ out, float* __restrict__ Hbuf,
                                                      float* __restrict__ y, uint32_t* __restrict__ hloc,
                                                      uint16_t* __restrict__ slot_of_pos,
                                                      uint16_t* __restrict__ tile_i0,
                                                      int* __restrict__ tile_nslots,
                                                      const int64_t* __restrict__ off, int64_t L, int mean,
                                                      int* __restrict__ bag_cnt) {
  pdl_entry();
  using SM = FcFwdSmem<D, TC>;
  const int t = blockIdx.x;
  if (t >= *ntiles) return;
  extern __shared__ __align__(128) float sm[];
  float* G1s = sm;
  float* G0s = G1s + D::S1;
  float* G2s = G0s + TC * SM::S0P;
  float* Hs = G2s + TC * SM::S2P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SM::floats());  // G1, G0 rows, G2 rows
  int* lk_l = reinterpret_cast<int*>(bar + 4);
  uint32_t* lk_d02 = reinterpret_cast<uint32_t*>(lk_l + TC);
  int* lk_solo = reinterpret_cast<int*>(lk_d02 + TC);
  int* lk_slot = lk_solo + TC;
  int* slot_i0 = lk_slot + TC;
  int* misc = slot_i0 + TC;
  uint32_t* flags = reinterpret_cast<uint32_t*>(misc + 8);
  __shared__ int red[33];
  const int tid = threadIdx.x;
  const Tile tl = tiles[t];
  const int n = tl.end - tl.start;
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  uint4 r = make_uint4(0u, 0u, 0u, 0u);
  if (tid < n) r = rec[tl.start + tid];
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_init(bar + 2, 1);
    mbar_arrive_expect(bar, D::S1 * 4);
    tma_load(G1s, G1 + static_cast<int64_t>(tl.key) * D::S1, D::S1 * 4, bar);
    mbar_arrive_expect(bar + 2, n * D::S2 * 4);
  }
  for (int i = tid; i < g.m0; i += kFcThreads) flags[i] = 0u;
  __syncthreads();
  if (tid < n) {
    lk_l[tid] = static_cast<int>(r.x);
    lk_d02[tid] = r.y;
    lk_solo[tid] = static_cast<int>(r.z);  // bag | single-lookup bit (make_rec)
    flags[r.y & 0xffffu] = 1u;
    tma_load(G2s + tid * SM::S2P, G2 + static_cast<int64_t>(r.y >> 16) * D::S2, D::S2 * 4, bar + 2);
  }
  __syncthreads();
  const int nslots = fc_scan_flags(flags, g.m0, red);  // flags[i0] -> slot (ascending i0)
  __syncthreads();
  for (int i = tid; i < g.m0; i += kFcThreads)
    if (flags[i] != 0xffffffffu) slot_i0[flags[i]] = i;
  if (tid == 0) {
    misc[0] = nslots;
    mbar_arrive_expect(bar + 1, nslots * D::S0 * 4);
  }
  __syncthreads();
  for (int s = tid; s < nslots; s += kFcThreads) {
    tma_load(G0s + s * SM::S0P, G0 + static_cast<int64_t>(slot_i0[s]) * D::S0, D::S0 * 4, bar + 1);
    tile_i0[tl.start + s] = static_cast<uint16_t>(slot_i0[s]);
  }
  if (tid < n) {
    const int s = static_cast<int>(flags[r.y & 0xffffu]);
    lk_slot[tid] = s;
    slot_of_pos[tl.start + tid] = static_cast<uint16_t>(s);
    hloc[r.x] = static_cast<uint32_t>(tl.start + s);
  }
  if (tid == 0) tile_nslots[t] = nslots;
  mbar_wait(bar, 0);
  mbar_wait(bar + 1, 0);
  // H(slot) = G0[i0] (P0 x R1) · G1[i1] (R1 x C1): thread -> (slot, 4 columns), all P0 rows
  for (int q = tid; q < nslots * D::C4; q += kFcThreads) {
    const int s = q / D::C4, c4 = q - s * D::C4;
    float4 acc[D::P0];
#pragma unroll
    for (int a = 0; a < D::P0; ++a) acc[a] = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* g0 = G0s + s * SM::S0P;
#pragma unroll 8
    for (int p = 0; p < D::R1; ++p) {
      const float4 b = reinterpret_cast<const float4*>(G1s + p * D::C1)[c4];
#pragma unroll
      for (int a = 0; a < D::P0; ++a) acc[a] = madd4<float, kExact>(g0[a * D::R1 + p], b, acc[a]);
    }
    float* hs = Hs + s * SM::HSP;
    float* hg = Hbuf + static_cast<int64_t>(tl.start + s) * D::W1;
#pragma unroll
    for (int a = 0; a < D::P0; ++a) {
      const int c = a * D::C1 + c4 * 4;  // = (row, r) in the (P1 x R2) view
      const float v4[4] = {acc[a].x, acc[a].y, acc[a].z, acc[a].w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = (c + u) / D::R2, rr = (c + u) - row * D::R2;
        hs[row * SM::R2P + rr] = v4[u];
      }
      reinterpret_cast<float4*>(hg + c)[0] = acc[a];
    }
  }
  __syncthreads();
  mbar_wait(bar + 2, 0);
  // y = H(slot) (P1 x R2) · G2[i2] (R2 x N2): thread -> (lookup, row a)
  for (int q = tid; q < n * D::P1; q += kFcThreads) {
    const int i = q / D::P1, a = q - i * D::P1;
    const float* hrow = Hs + lk_slot[i] * SM::HSP + a * SM::R2P;
    const float4* g2 = reinterpret_cast<const float4*>(G2s + i * SM::S2P);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 8
    for (int rr = 0; rr < D::R2; ++rr) acc = madd4<float, kExact>(hrow[rr], g2[rr], acc);
    const int z = lk_solo[i];
    if (z < 0) {  // the bag's only lookup: pooled here, (0 + w·y, the pooling arithmetic)
      const float wl = w ? static_cast<float>(w[lk_l[i]]) : 1.f;
      reinterpret_cast<float4*>(out + static_cast<int64_t>(z & 0x7fffffff) * D::N)[a] =
          madd4<float, kExact>(wl, acc, make_float4(0.f, 0.f, 0.f, 0.f));
    } else {
      reinterpret_cast<float4*>(y + static_cast<int64_t>(lk_l[i]) * D::N)[a] = acc;
      pool_if_last<D::N, kExact>(z, D::P1, off, L, w, mean, y, out, bag_cnt);
    }
  }
}

// ------------------------------------------------------------- f3c_bwd ----
template <class D, int TC>
struct FcBwdSmem {
  static constexpr int R1P = D::R1 + 4;
  static constexpr int S2P = D::S2 + 4;
  static constexpr int NW = TC / 32;  // warps holding a chunk's lookups
  // floats: S[TC * W1] | G0s[TC * S0] | G1t[C1 * R1P] | G2s[TC * S2P] | D2s[TC * N]
  static __host__ __device__ constexpr size_t floats() {
    return (static_cast<size_t>(TC) * D::W1 + static_cast<size_t>(TC) * D::S0 +
            static_cast<size_t>(D::C1) * R1P + static_cast<size_t>(TC) * S2P +
            static_cast<size_t>(TC) * D::N + 3) / 4 * 4;
  }
  // 2 mbarriers; ints: lk_slot, members, slot_i0, d0first, lk_alpha [TC], slot_start[TC + 1],
  // wcnt[NW][TC], misc[8], d0bits[256]
  static __host__ __device__ constexpr size_t bytes() {
    return floats() * 4 + 16 + 4 * (5 * TC + TC + 1 + NW * TC + 8 + 256);
  }
};

template <class D, int TC>
__global__ void __launch_bounds__(kFcThreads, 2) f3c_bwd(
    Geo g, const float* __restrict__ cores, const Tile* __restrict__ tiles,
    const int* __restrict__ ntiles, const uint4* __restrict__ rec,
    const uint16_t* __restrict__ slot_of_pos, const uint16_t* __restrict__ tile_i0,
    const int* __restrict__ tile_nslots, const float* __restrict__ grad, float* __restrict__ part1,
    int* __restrict__ has1, float* __restrict__ D0acc, unsigned char* __restrict__ d0mask) {
  pdl_entry();
  using SM = FcBwdSmem<D, TC>;
  using GB = G1Blk<D>;
  static_assert(TC % 32 == 0 && TC <= 128, "chunk = whole warps, <= 4 values per lane in the slot scan");
  extern __shared__ __align__(128) float sm[];
  float* S = sm;
  float* G0s = S + TC * D::W1;
  float* G1t = G0s + TC * D::S0;
  float* G2s = G1t + D::C1 * SM::R1P;
  float* D2s = G2s + TC * SM::S2P;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SM::floats());  // [0] G2 + grad rows, [1] G0 rows
  int* lk_slot = reinterpret_cast<int*>(bar + 2);
  int* members = lk_slot + TC;
  int* slot_i0 = members + TC;
  int* d0first = slot_i0 + TC;
  float* lk_alpha = reinterpret_cast<float*>(d0first + TC);
  int* slot_start = reinterpret_cast<int*>(lk_alpha + TC);
  int* wcnt = slot_start + TC + 1;
  int* misc = wcnt + SM::NW * TC;
  unsigned* d0bits = reinterpret_cast<unsigned*>(misc + 8);
  const float* G0 = cores + g.coff0;
  const float* G1 = cores + g.coff1;
  const float* G2 = cores + g.coff2;
  const int nt = *ntiles;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // contiguous chunk ranges balanced by work: chunk t weighs
  // 2 + nslots(t) + lookups(t) / 8 (GEMMs scale with the slots, S with the lookups)
  int t_lo, t_hi;
  {
    using Scan = cub::BlockScan<int, kFcThreads>;
    __shared__ typename Scan::TempStorage scan_tmp;
    __shared__ int range[2];
    const int per = (nt + kFcThreads - 1) / kFcThreads;
    const int a0 = min(nt, tid * per), a1 = min(nt, a0 + per);
    auto weight = [&](int t) {
      const Tile tl = tiles[t];
      return 2 + tile_nslots[t] + (tl.end - tl.start) / 8;
    };
    // up to kPer weights per thread loaded at once (one round trip), kept for the walk
    constexpr int kPer = 8;
    int wv[kPer];
    int wsum = 0;
    if (per <= kPer) {
#pragma unroll
      for (int j = 0; j < kPer; ++j) wv[j] = a0 + j < a1 ? weight(a0 + j) : 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) wsum += wv[j];
    } else {
      for (int t = a0; t < a1; ++t) wsum += weight(t);
    }
    int ex, W;
    Scan(scan_tmp).ExclusiveSum(wsum, ex, W);
    const int64_t G = gridDim.x, b = blockIdx.x;
    const int64_t th[2] = {(b * W + G - 1) / G, ((b + 1) * W + G - 1) / G};
    if (tid < 2) range[tid] = th[tid] <= 0 ? 0 : nt;
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (ex < th[q] && th[q] <= ex + wsum) {
        int64_t e = ex;
        int t = a0;
        if (per <= kPer) {
#pragma unroll
          for (int j = 0; j < kPer; ++j)
            if (t < a1 && e < th[q]) {
              e += wv[j];
              ++t;
            }
        } else {
          for (; t < a1 && e < th[q]; ++t) e += weight(t);
        }
        range[q] = t;
      }
    }
    __syncthreads();
    t_lo = range[0];
    t_hi = range[1] > range[0] ? range[1] : range[0];
  }
  float* d0acc = D0acc + static_cast<int64_t>(blockIdx.x) * g.m0 * D::S0;
  unsigned char* d0m = d0mask + static_cast<int64_t>(blockIdx.x) * g.m0;
  for (int e = tid; e < g.m0; e += kFcThreads) d0m[e] = 0;
  for (int e = tid; e < 256; e += kFcThreads) d0bits[e] = 0u;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
  }
  __syncthreads();
  // chunk state in registers: descriptor, this thread's record (tid < n) and
  // slot i0 (tid < nslots); the next chunk's are loaded one chunk ahead
  Tile tl{};
  int nslots = 0, my_slot = 0, my_i0 = 0;
  uint4 my_r = make_uint4(0u, 0u, 0u, 0u);
  auto load_chunk = [&](int t, Tile& d, int& ns, uint4& r, int& sl, int& i0) {
    d = tiles[t];
    ns = tile_nslots[t];
    if (tid < d.end - d.start) {
      r = rec[d.start + tid];
      sl = slot_of_pos[d.start + tid];
    }
    if (tid < ns) i0 = tile_i0[d.start + tid];
  };
  // bulk copies of a chunk: G2 + grad rows (bar 0), G0 rows of its slots (bar 1)
  auto issue_rows = [&](const Tile& d, const uint4& r) {
    const int n = d.end - d.start;
    // D2s was rewritten in place (generic proxy): order that before the bulk copies
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) mbar_arrive_expect(bar, n * (D::S2 + D::N) * 4);
    __syncthreads();
    if (tid < n) {
      tma_load(G2s + tid * SM::S2P, G2 + static_cast<int64_t>(r.y >> 16) * D::S2, D::S2 * 4, bar);
      tma_load(D2s + tid * D::N, grad + static_cast<int64_t>(r.z & 0x7fffffffu) * D::N, D::N * 4, bar);
    }
  };
  auto issue_g0 = [&](int ns, int i0) {
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect(bar + 1, ns * D::S0 * 4);
    }
    __syncthreads();
    if (tid < ns) tma_load(G0s + tid * D::S0, G0 + static_cast<int64_t>(i0) * D::S0, D::S0 * 4, bar + 1);
  };
  if (t_lo < t_hi) {
    load_chunk(t_lo, tl, nslots, my_r, my_slot, my_i0);
    issue_rows(tl, my_r);
    issue_g0(nslots, my_i0);
  }
  const int r0 = (tid % GB::TR) * GB::RB, cb0 = (tid / GB::TR) * GB::CB;
  const bool g1_on = tid < GB::TR * GB::TC;
  float acc1[GB::RB][GB::CB];
#pragma unroll
  for (int i = 0; i < GB::RB; ++i)
#pragma unroll
    for (int j = 0; j < GB::CB; ++j) acc1[i][j] = 0.f;
  int run_start = t_lo, cur_i1 = -1;
  for (int t = t_lo; t < t_hi; ++t) {
    const uint32_t parity = static_cast<uint32_t>((t - t_lo) & 1);
    const int n = tl.end - tl.start;
    const int i1 = tl.key;
    // the next chunk's descriptor and records: in flight during this chunk
    Tile tn{};
    int ns_n = 0, sl_n = 0, i0_n = 0;
    uint4 r_n = make_uint4(0u, 0u, 0u, 0u);
    if (t + 1 < t_hi) load_chunk(t + 1, tn, ns_n, r_n, sl_n, i0_n);
    // chunk metadata into shared memory; per-warp slot ranks (match_any)
    int rank = 0;
    if (tid < n) {
      lk_slot[tid] = my_slot;
      lk_alpha[tid] = __uint_as_float(my_r.w);
    }
    if (tid < nslots) slot_i0[tid] = my_i0;
    for (int e = tid; e < SM::NW * TC; e += kFcThreads) wcnt[e] = 0;
    if (i1 != cur_i1) {  // stage G1[i1] transposed (once per bucket run)
      const float* src = G1 + static_cast<int64_t>(i1) * D::S1;
      constexpr int U = 8;
      for (int e0 = tid; e0 < D::S1; e0 += kFcThreads * U) {
        float v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = e0 + u * kFcThreads < D::S1 ? __ldg(src + e0 + u * kFcThreads) : 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kFcThreads;
          if (e < D::S1) {
            const int rr = e / D::C1, c = e - rr * D::C1;
            G1t[c * SM::R1P + rr] = v[u];
          }
        }
      }
      cur_i1 = i1;
    }
    __syncthreads();
    unsigned peers = 0;
    if (wid < SM::NW) {
      const int sl = tid < n ? my_slot : -1;
      peers = __match_any_sync(0xffffffffu, sl);
      rank = __popc(peers & lanemask_lt());
      if (sl >= 0 && rank == 0) wcnt[wid * TC + sl] = __popc(peers);
    }
    if (tid < nslots) {  // D0 first touches of this CTA
      const int i0 = my_i0;
      const unsigned bit = 1u << (i0 & 31);
      const unsigned old = atomicOr(d0bits + (i0 >> 5), bit);
      d0first[tid] = (old & bit) ? 0 : 1;
      if (!(old & bit)) d0m[i0] = 1;
    }
    __syncthreads();
    if (wid == 0) {  // slot starts: warp scan, TC / 32 slots per lane; per-warp starts in wcnt
      constexpr int E = TC / 32;
      int c[E], tot = 0;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int s = lane * E + j;
        int run = 0;
        if (s < nslots) {
#pragma unroll
          for (int w = 0; w < SM::NW; ++w) {
            const int v = wcnt[w * TC + s];
            wcnt[w * TC + s] = run;
            run += v;
          }
        }
        c[j] = run;
        tot += run;
      }
      int x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += yv;
      }
      int run = x - tot;
#pragma unroll
      for (int j = 0; j < E; ++j) {
        const int s = lane * E + j;
        if (s < nslots) slot_start[s] = run;
        run += c[j];
      }
      if (lane == 31) slot_start[nslots] = x;
    }
    __syncthreads();
    if (tid < n) members[slot_start[my_slot] + wcnt[wid * TC + my_slot] + rank] = tid;
    mbar_wait(bar, parity);  // G2 + grad rows of this chunk
    // D2 = T(alpha) · grad (separately rounded, as f3_srows)
    for (int e = tid; e < n * D::N; e += kFcThreads) {
      const int i = e / D::N;
      D2s[e] = __fmul_rn(lk_alpha[i], D2s[e]);
    }
    __syncthreads();
    // S(slot)[e] = Σ_{members} D1[e], D1[a][r] = Σ_j D2[a][j] G2[i2][r][j]
    {
      constexpr int NG = kFcThreads / D::W1 > 0 ? kFcThreads / D::W1 : 1;
      static_assert(D::W1 <= kFcThreads, "one thread per S element");
      const int e = tid % D::W1, grp = tid / D::W1;
      const int a = e / D::R2, rr = e - a * D::R2;
      if (grp < NG) {
        for (int s = grp; s < nslots; s += NG) {
          const int m0 = slot_start[s], m1 = slot_start[s + 1];
          float acc = 0.f;
#pragma unroll 4
          for (int m = m0; m < m1; ++m) {
            const int i = members[m];
            const float4 d4 = reinterpret_cast<const float4*>(D2s + i * D::N)[a];
            const float4 gk = reinterpret_cast<const float4*>(G2s + i * SM::S2P)[rr];
            float v = __fmul_rn(d4.x, gk.x);
            v = __fmaf_rn(d4.y, gk.y, v);
            v = __fmaf_rn(d4.z, gk.z, v);
            v = __fmaf_rn(d4.w, gk.w, v);
            acc = m == m0 ? v : __fadd_rn(acc, v);
          }
          S[s * D::W1 + e] = acc;
        }
      }
    }
    __syncthreads();  // S complete; G2 / grad rows free
    if (t + 1 < t_hi) issue_rows(tn, r_n);  // the next chunk's rows land during the GEMMs
    mbar_wait(bar + 1, parity);  // G0 rows of this chunk
    const int nk = nslots * D::P0;
    // ---- dG1 partial += Σ_kappa G0s[kappa][r1] (x) S[kappa][c]
    if (g1_on) {
#pragma unroll 2
      for (int k = 0; k < nk; ++k) {
        float av[GB::RB], bv[GB::CB];
        const float* ap = G0s + k * D::R1 + r0;
#pragma unroll
        for (int i = 0; i < GB::RB; ++i) av[i] = ap[i];
#pragma unroll
        for (int j = 0; j < GB::CB; j += 4) {
          const float4 v = *reinterpret_cast<const float4*>(S + k * D::C1 + cb0 + j);
          bv[j] = v.x; bv[j + 1] = v.y; bv[j + 2] = v.z; bv[j + 3] = v.w;
        }
#pragma unroll
        for (int i = 0; i < GB::RB; ++i)
#pragma unroll
          for (int j = 0; j < GB::CB; j += 2) ffma2(av[i], bv[j], bv[j + 1], acc1[i][j], acc1[i][j + 1]);
      }
    }
    // ---- D0[kappa][r1] = Σ_c S[kappa][c] · G1[r1][c] into the CTA block
    {
      constexpr int KPT = kFcThreads / GB::TR0;  // kappas per pass
      const int rb = (tid % GB::TR0) * GB::RB0;
      for (int k = tid / GB::TR0; k < nk; k += KPT) {
        float dv[GB::RB0];
#pragma unroll
        for (int i = 0; i < GB::RB0; ++i) dv[i] = 0.f;
        const float* srow = S + k * D::C1;
#pragma unroll 4
        for (int c = 0; c < D::C1; c += 4) {
          const float4 s4 = *reinterpret_cast<const float4*>(srow + c);
          const float sv[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const float* gp = G1t + (c + cc) * SM::R1P + rb;
#pragma unroll
            for (int i = 0; i < GB::RB0; i += 2) ffma2(sv[cc], gp[i], gp[i + 1], dv[i], dv[i + 1]);
          }
        }
        const int sl = k / D::P0, a0 = k - sl * D::P0;
        float* dst = d0acc + slot_i0[sl] * D::S0 + a0 * D::R1 + rb;
        if (d0first[sl]) {
#pragma unroll
          for (int i = 0; i < GB::RB0; ++i) dst[i] = dv[i];
        } else {
#pragma unroll
          for (int i = 0; i < GB::RB0; ++i) dst[i] += dv[i];
        }
      }
    }
    // ---- end of an i1 run (or of this CTA's range): flush the dG1 partial
    if (tid == 0) has1[t] = (t == run_start) ? 1 : 0;
    if (tn.key != i1 || t + 1 == t_hi) {
      float* dst = part1 + static_cast<int64_t>(run_start) * D::S1;
      if (g1_on) {
#pragma unroll
        for (int i = 0; i < GB::RB; ++i)
#pragma unroll
          for (int j = 0; j < GB::CB; j += 4)
            *reinterpret_cast<float4*>(dst + (r0 + i) * D::C1 + cb0 + j) =
                make_float4(acc1[i][j], acc1[i][j + 1], acc1[i][j + 2], acc1[i][j + 3]);
      }
#pragma unroll
      for (int i = 0; i < GB::RB; ++i)
#pragma unroll
        for (int j = 0; j < GB::CB; ++j) acc1[i][j] = 0.f;
      run_start = t + 1;
    }
    __syncthreads();  // GEMMs done with G0s / S / slot lists
    if (t + 1 < t_hi) {
      issue_g0(ns_n, i0_n);
      tl = tn;
      nslots = ns_n;
      my_r = r_n;
      my_slot = sl_n;
      my_i0 = i0_n;
    }
  }
}

}  // namespace f3
}  // namespace ttgpu
