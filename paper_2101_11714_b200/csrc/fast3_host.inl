// Host launch code for the 3-core fast path (fast3.cuh).  Included by ttgpu.cu
// after the table/context definitions.
namespace ttgpu {

struct F3Bufs {
  DevBuf d0, d1, d2, hist1, hist2, perm1, perm2, rec1, solo, tiles1, tiles2, tile_base1, tile_base2, ntiles,
      Hbuf, y, hloc, slotpos, tile_i0, tile_nslots, part1, has1, part2, has2, D0acc, d0mask,
      group_base1, group_base2, gpart, gtouch, counters, tot, Sbuf, gs_hist, gs_tot, bag_cnt, b1plan,
      b1ulen, tile_one;
  f3::Geo geo{};
  int max_tiles1 = 0, max_tiles2 = 0;
  int kind = -1;  // instantiation index
  bool chunked = false;  // forward ran the chunked kernels (fastc.cuh); backward follows it
};

void f3_free(F3Bufs* f) { delete f; }

namespace {

// Launch of a fast-path kernel: plain, or with programmatic dependent launch
// (the kernels begin with f3::pdl_entry(), so both are correct).
template <typename... KArgs, typename... Args>
void f3_launch(int pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
               Args... args) {
  if (!pdl) {
    k<<<grid, block, smem, st>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}

constexpr int kF3MaxHist = 48 * 1024;  // histogram entries one f3_scan CTA stages (kScanKeys x NT)

// lookups per hist/scatter CTA: 512 * LPT, LPT in {1, 2, ..., 32}; 0 = infeasible.
// The smallest LPT (most CTAs) whose histogram still fits the 1-CTA scan.
int f3_lpt(int64_t L, int K) {
  for (int lpt = 1; lpt <= 32; lpt *= 2) {
    const int64_t nt = (L + 512 * lpt - 1) / (512 * lpt);
    if (nt * f3::kScanKeys <= kF3MaxHist && nt * K <= (int64_t{1} << 26)) return lpt;
  }
  return 0;
}

f3::Geo make_geo(const ttgpu_table* t) {
  f3::Geo g{};
  const DevPlan& P = t->dp;
  g.m0 = P.m[0];
  g.m1 = P.m[1];
  g.m2 = P.m[2];
  g.m12 = static_cast<uint32_t>(P.m[1]) * static_cast<uint32_t>(P.m[2]);
  g.num_rows = P.num_rows;
  g.coff0 = P.coff[0];
  g.coff1 = P.coff[1];
  g.coff2 = P.coff[2];
  return g;
}

template <int LPT>
void launch_hist(int grid, size_t smem, cudaStream_t st, const f3::Geo& g, const int64_t* idx,
                 int64_t L, int NT, const int64_t* off, int64_t B, const double* w, int pooling,
                 F3Bufs& f, int32_t* lk_bag, float* alpha, float* out, ttgpu_table* t) {
  f3_launch(t->pdl, f3::f3_hist<float, LPT>, dim3(grid), dim3(512), smem, st, 
      g, idx, L, NT, off, B, w, pooling, f.d0.as<uint16_t>(), f.d1.as<uint16_t>(),
      f.d2.as<uint16_t>(), lk_bag, alpha, f.hist1.as<uint32_t>(), f.hist2.as<uint32_t>(),
      f.tot.as<uint32_t>(), f.tot.as<uint32_t>() + g.m1, t->d_bad(), t->d_struct(),
      f.solo.as<int32_t>(), out, static_cast<int>(t->dp.N), f.bag_cnt.as<int>());
}

// Cooperative launch of the one-kernel sort (gsort.cuh): all CTAs co-resident.
void launch_gsort(const ttgpu_table* t, int G, size_t smem, const f3::GsortArgs& a) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(f3::kGsThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = t->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const int rounds = a.PW / 32;
  const bool cache = a.K3 > 0 || a.counts != nullptr;
  auto kern = rounds <= 1 ? (cache ? f3::f3_gsort<1, true> : f3::f3_gsort<1, false>)
            : rounds <= 2 ? (cache ? f3::f3_gsort<2, true> : f3::f3_gsort<2, false>)
            : rounds <= 4 ? (cache ? f3::f3_gsort<4, true> : f3::f3_gsort<4, false>)
                          : (cache ? f3::f3_gsort<8, true> : f3::f3_gsort<8, false>);
  CK(cudaLaunchKernelEx(&cfg, kern, a));
}

template <class K>
int grid_occ(K kern, int threads, size_t smem, int num_sms, int cap) {
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
  return std::max(1, std::min(cap, num_sms * std::max(occ, 1)));
}

constexpr int kChunk = 64;  // lookups per chunk of the chunked path (fastc.cuh)

// Cache mode of the fast path (lfu_cache_host.inl): the LFU cache is consulted
// inside f3_gsort; its hits leave the chain.
struct F3Cache {
  int K3 = 0;
  unsigned long long* counts = nullptr;
  const unsigned long long* hkeys = nullptr;
  const int* hvals = nullptr;
  int hshift = 63;
  unsigned long long hmask = 0;
  int active = 0;
  unsigned long long* hits = nullptr;
  unsigned long long* hits2 = nullptr;
  unsigned long long* accesses = nullptr;
  const int64_t* slot_rows = nullptr;
  int* lk_slot = nullptr;
  uint32_t* perm3 = nullptr;
  int* skey3 = nullptr;
  int* seg_lo3 = nullptr;
  int* seg_hi3 = nullptr;
  int* ncached = nullptr;
  const float* store = nullptr;
};

// Grid of the one-kernel sort for L lookups (0: infeasible): G CTAs, PW lookups per warp.
void gsort_grid(const ttgpu_table* t, const f3::Geo& g, int64_t L, int K3, int* GS, int* PW) {
  *GS = 0;
  *PW = 0;
  const size_t gs_smem = f3::gsort_smem_bytes(g.m1, g.m2, K3);
  if (!t->grid_sort || g.m1 + g.m2 > 4 * f3::kGsThreads || K3 > 8 * f3::kGsThreads ||
      gs_smem > 160 * 1024)
    return;
  const size_t gsm = std::max<size_t>(gs_smem, f3::gsort_smem_bytes(g.m1, g.m2));
  set_smem(f3::f3_gsort<1, false>, gsm);
  set_smem(f3::f3_gsort<2, false>, gsm);
  set_smem(f3::f3_gsort<4, false>, gsm);
  set_smem(f3::f3_gsort<8, false>, gsm);
  set_smem(f3::f3_gsort<1, true>, gsm);
  set_smem(f3::f3_gsort<2, true>, gsm);
  set_smem(f3::f3_gsort<4, true>, gsm);
  set_smem(f3::f3_gsort<8, true>, gsm);
  int occ = 0;  // the widest variant bounds the co-resident grid
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f3::f3_gsort<8, true>, f3::kGsThreads, gs_smem));
  const int64_t cap = std::min<int64_t>(32 * f3::kGsMaxGridChunks,
                                        static_cast<int64_t>(t->num_sms) * std::max(occ, 0));
  const int64_t per = 16 * 32;  // lookups per CTA round
  const int64_t rounds = (L + cap * per - 1) / std::max<int64_t>(1, cap * per);
  if (cap > 0 && rounds <= f3::kGsMaxRounds) {
    *PW = static_cast<int>(32 * std::max<int64_t>(1, rounds));
    *GS = static_cast<int>((L + 16 * *PW - 1) / (16 * *PW));
  }
}

template <class D>
struct F3Runner {
  static void forward(ttgpu_table* t, F3Bufs& f, const int64_t* idx, int64_t L, const int64_t* off,
                      int64_t B, const double* w, int pooling, float* out, bool exact,
                      int32_t* lk_bag, float* alpha, const F3Cache* cache = nullptr) {
    cudaStream_t st = t->stream;
    f3::Geo& g = f.geo;
    g = make_geo(t);
    const int Kmax = std::max(g.m1, g.m2);
    // one-kernel sort when the batch fits one co-resident grid (gsort.cuh)
    const int K3 = cache ? cache->K3 : 0;
    const size_t gs_smem = f3::gsort_smem_bytes(g.m1, g.m2, K3);
    int GS = 0, PW = 0;
    gsort_grid(t, g, L, K3, &GS, &PW);
    if (cache && !GS) fail(TTGPU_ERR_RUNTIME, "cache fast path needs the one-kernel sort");
    if (cache) f.chunked = false;
    const int lpt = f3_lpt(L, Kmax);
    if (lpt == 0) fail(TTGPU_ERR_RUNTIME, "batch too large for the fast path histogram");
    const int TL = 512 * lpt;
    const int NT = static_cast<int>((L + TL - 1) / TL);
    f.chunked = t->chunked && !cache;
    const int TT1 = f.chunked ? kChunk : D::TT;  // i1-bucket tile (chunk) length
    f.max_tiles1 = static_cast<int>((L + TT1 - 1) / TT1) + g.m1;
    f.max_tiles2 = static_cast<int>((L + D::TT2 - 1) / D::TT2) + g.m2;
    f.d0.ensure(2 * L);
    f.d1.ensure(2 * L);
    f.d2.ensure(2 * L);
    f.hist1.ensure(4 * static_cast<size_t>(g.m1) * NT);
    f.hist2.ensure(4 * static_cast<size_t>(g.m2) * NT);
    if (f.tot.cap < 4 * static_cast<size_t>(g.m1 + g.m2)) {  // kept zero between batches by f3_scatter
      f.tot.ensure(4 * static_cast<size_t>(g.m1 + g.m2));
      CK(cudaMemsetAsync(f.tot.p, 0, f.tot.cap, st));
    }
    f.perm1.ensure(4 * L);
    f.rec1.ensure(16 * L);
    f.solo.ensure(4 * L);
    f.perm2.ensure(4 * L);
    f.tiles1.ensure(sizeof(f3::Tile) * f.max_tiles1);
    f.tiles2.ensure(sizeof(f3::Tile) * f.max_tiles2);
    f.tile_base1.ensure(4 * (g.m1 + 1));
    f.tile_base2.ensure(4 * (g.m2 + 1));
    f.group_base1.ensure(4 * (g.m1 + 1));
    f.group_base2.ensure(4 * (g.m2 + 1));
    f.ntiles.ensure(16);
    f.Hbuf.ensure(4 * static_cast<size_t>(L) * D::W1);
    f.y.ensure(4 * static_cast<size_t>(L) * D::N);
    f.hloc.ensure(4 * L);
    f.slotpos.ensure(2 * L);
    f.tile_i0.ensure(2 * L);
    f.tile_nslots.ensure(4 * f.max_tiles1);
    f.tile_one.ensure(4 * f.max_tiles1);
    f.bag_cnt.ensure(4 * static_cast<size_t>(B));
    const int gb = std::max(NT, grid_for(B, 512, t->num_sms, 4));
    t->mark("fwd_begin");
    if (GS) {
      const int K = g.m1 + g.m2 + K3;  // key 3 = cache slots
      f.gs_hist.ensure(4 * static_cast<size_t>(K) * GS);
      f.gs_tot.ensure(4 * static_cast<size_t>(K));
      f3::GsortArgs a{};
      a.g = g;
      a.idx = idx;
      a.L = L;
      a.off = off;
      a.B = B;
      a.w = w;
      a.mean = pooling;
      a.PW = PW;
      a.TT1 = TT1;
      a.TT2 = D::TT2;
      a.inv_m12 = 1.0 / static_cast<double>(g.m12);
      a.inv_m2 = 1.0 / static_cast<double>(g.m2);
      a.d2 = f.d2.as<uint16_t>();
      a.lk_bag = lk_bag;
      a.alpha = alpha;
      a.solo = f.solo.as<int32_t>();
      a.hist = f.gs_hist.as<uint32_t>();
      a.tot = f.gs_tot.as<uint32_t>();
      a.perm1 = f.perm1.as<uint32_t>();
      a.perm2 = f.perm2.as<uint32_t>();
      a.rec1 = f.rec1.as<uint4>();
      a.tiles1 = f.tiles1.as<f3::Tile>();
      a.tiles2 = f.tiles2.as<f3::Tile>();
      a.tile_base1 = f.tile_base1.as<int32_t>();
      a.tile_base2 = f.tile_base2.as<int32_t>();
      a.group_base1 = f.group_base1.as<int32_t>();
      a.group_base2 = f.group_base2.as<int32_t>();
      a.ntiles = f.ntiles.as<int>();
      a.bad = t->d_bad();
      a.errs = t->d_struct();
      a.out = out;
      a.N = static_cast<int>(t->dp.N);
      a.bag_cnt = f.bag_cnt.as<int>();
      if (cache) {
        a.mean = 0;  // both partition parts are Sum-pooled (the Mean rescale is the combine's)
        a.pool_mean = pooling;
        a.parts = D::P1;
        a.K3 = cache->K3;
        a.counts = cache->counts;
        a.hkeys = cache->hkeys;
        a.hvals = cache->hvals;
        a.hshift = cache->hshift;
        a.hmask = cache->hmask;
        a.active = cache->active;
        a.hits = cache->hits;
        a.hits2 = cache->hits2;
        a.accesses = cache->accesses;
        a.lk_slot = cache->lk_slot;
        a.slot_rows = cache->slot_rows;
        a.perm3 = cache->perm3;
        a.skey3 = cache->skey3;
        a.seg_lo3 = cache->seg_lo3;
        a.seg_hi3 = cache->seg_hi3;
        a.ncached = cache->ncached;
        a.store = cache->store;
      }
      launch_gsort(t, GS, gs_smem, a);
      t->mark("gsort");
    } else {
      const size_t hs = 4 * static_cast<size_t>(g.m1 + g.m2);
      switch (lpt) {
        case 1: launch_hist<1>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
        case 2: launch_hist<2>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
        case 4: launch_hist<4>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
        case 8: launch_hist<8>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
        case 16: launch_hist<16>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
        default: launch_hist<32>(gb, hs, st, g, idx, L, NT, off, B, w, pooling, f, lk_bag, alpha, out, t); break;
      }
      t->mark("hist");
      {
        f3::ScanArgs a1{f.hist1.as<uint32_t>(), f.tot.as<uint32_t>(), f.tile_base1.as<int32_t>(),
                        f.group_base1.as<int32_t>(), f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(),
                        g.m1, TT1};
        f3::ScanArgs a2{f.hist2.as<uint32_t>(), f.tot.as<uint32_t>() + g.m1, f.tile_base2.as<int32_t>(),
                        f.group_base2.as<int32_t>(), f.tiles2.as<f3::Tile>(), f.ntiles.as<int>() + 1,
                        g.m2, D::TT2};
        const size_t n = static_cast<size_t>(f3::kScanKeys) * NT;
        const size_t sm = 4 * (n + n / 32 + 2);
        set_smem(f3::f3_scan, sm);
        const int nb1 = (g.m1 + f3::kScanKeys - 1) / f3::kScanKeys;
        const int nb2 = (g.m2 + f3::kScanKeys - 1) / f3::kScanKeys;
        f3_launch(t->pdl, f3::f3_scan, dim3(nb1 + nb2), dim3(f3::kScanThreads), sm, st, a1, a2, nb1, NT, L);
      }
      t->mark("scan");
      {
        const size_t sm = 4 * 8 * static_cast<size_t>(Kmax);
        set_smem(f3::f3_scatter, sm);
        f3_launch(t->pdl, f3::f3_scatter, dim3(NT), dim3(256), sm, st, g, f.d0.as<uint16_t>(), f.d1.as<uint16_t>(),
                                            f.d2.as<uint16_t>(), L, TL, NT, f.hist1.as<uint32_t>(),
                                            f.hist2.as<uint32_t>(), f.perm1.as<uint32_t>(),
                                            f.perm2.as<uint32_t>(), f.tot.as<uint32_t>(),
                                            f.solo.as<int32_t>(), f.rec1.as<uint4>(), lk_bag, alpha);
      }
      t->mark("scatter");
    }
    if (f.chunked) {
      const size_t sm = f3::FcFwdSmem<D, kChunk>::bytes(g.m0);
      auto kern = exact ? f3::f3c_fwd<D, true, kChunk> : f3::f3c_fwd<D, false, kChunk>;
      set_smem(kern, sm);
      f3_launch(t->pdl, kern, dim3(f.max_tiles1), dim3(f3::kFcThreads), sm, st, g, t->cores.as<float>(),
                f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(), f.rec1.as<uint4>(), w, out, f.Hbuf.as<float>(),
                f.y.as<float>(), f.hloc.as<uint32_t>(), f.slotpos.as<uint16_t>(), f.tile_i0.as<uint16_t>(),
                f.tile_nslots.as<int>(), off, L, pooling, f.bag_cnt.as<int>());
    } else {
      const size_t sm = f3::FwdSmem<D>::bytes(g.m0);
      auto kern = cache ? (exact ? f3::f3_fwd<D, true, true> : f3::f3_fwd<D, false, true>)
                        : (exact ? f3::f3_fwd<D, true> : f3::f3_fwd<D, false>);
      set_smem(kern, sm);
      const int grid = grid_occ(kern, f3::kThreads, sm, t->num_sms, f.max_tiles1);
      f3_launch(t->pdl, kern, dim3(grid), dim3(f3::kThreads), sm, st, g, t->cores.as<float>(), f.tiles1.as<f3::Tile>(),
                                           f.ntiles.as<int>(), f.rec1.as<uint4>(), w, out,
                                           f.Hbuf.as<float>(), f.y.as<float>(), f.hloc.as<uint32_t>(),
                                           f.slotpos.as<uint16_t>(), f.tile_i0.as<uint16_t>(),
                                           f.tile_nslots.as<int>(), f.tile_one.as<int>(), off, L, pooling,
                                           f.bag_cnt.as<int>(),
                                           cache ? cache->lk_slot : nullptr,
                                           cache ? cache->store : nullptr);
    }
    t->mark("f3_fwd");
    CK(cudaGetLastError());
  }

  static void backward(ttgpu_table* t, F3Bufs& f, const float* grad, int mode, float lr,
                       const int32_t* lk_bag, const float* alpha, int64_t L) {
    cudaStream_t st = t->stream;
    const f3::Geo& g = f.geo;
    const size_t sm1 = f.chunked ? f3::FcBwdSmem<D, kChunk>::bytes() : f3::Bwd1Smem<D>::bytes();
    auto k1 = f3::f3_bwd1<D>;
    auto kc = f3::f3c_bwd<D, kChunk>;
    int grid1;
    if (f.chunked) {
      set_smem(kc, sm1);
      grid1 = grid_occ(kc, f3::kFcThreads, sm1, t->num_sms, f.max_tiles1);
    } else {
      set_smem(k1, sm1);
      grid1 = grid_occ(k1, f3::kThreads, sm1, t->num_sms, f.max_tiles1);
      if (t->fuse_comb) {  // the cooperative variant must fit co-resident
        set_smem(f3::f3_bwd1_comb<D>, sm1);
        grid1 = std::min(grid1, grid_occ(f3::f3_bwd1_comb<D>, f3::kThreads, sm1, t->num_sms, f.max_tiles1));
      }
    }
    const int grid2 = grid_occ(f3::f3_bwd2<D>, 128, 0, t->num_sms, f.max_tiles2);
    f.part1.ensure(4 * static_cast<size_t>(f.max_tiles1) * f3::G1Blk<D>::KG * D::S1);
    f.has1.ensure(4 * static_cast<size_t>(f.max_tiles1));
    f.part2.ensure(4 * static_cast<size_t>(f.max_tiles2) * D::S2);
    f.has2.ensure(4 * static_cast<size_t>(f.max_tiles2));
    f.D0acc.ensure(4 * static_cast<size_t>(grid1) * g.m0 * D::S0);
    f.d0mask.ensure(static_cast<size_t>(grid1) * g.m0);
    f.Sbuf.ensure(4 * static_cast<size_t>(L) * D::W1);
    // combine arguments (f3_combine, or the combine phase of f3_bwd1_comb)
    constexpr int C1c = (D::S1 + 127) / 128, C2c = (D::S2 + 127) / 128, C0c = (D::S0 + 127) / 128;
    f3::CombineArgs A{};
    A.tile_base1 = f.tile_base1.as<int32_t>();
    A.tile_base2 = f.tile_base2.as<int32_t>();
    A.group_base1 = f.group_base1.as<int32_t>();
    A.group_base2 = f.group_base2.as<int32_t>();
    A.part1 = f.part1.as<float>();
    A.part2 = f.part2.as<float>();
    A.D0acc = f.D0acc.as<float>();
    A.has1 = f.has1.as<int>();
    A.has2 = f.has2.as<int>();
    A.d0mask = f.d0mask.as<unsigned char>();
    A.maxg1 = g.m1 + (f.max_tiles1 + f3::kGroup - 1) / f3::kGroup;
    A.maxg2 = g.m2 + (f.max_tiles2 + f3::kGroup - 1) / f3::kGroup;
    A.nbwd = grid1;
    const int ng0 = (grid1 + f3::kGroup0 - 1) / f3::kGroup0;
    const int tasks = A.maxg1 * C1c + A.maxg2 * C2c + g.m0 * ng0 * C0c;  // one warp each
    const int ncnt = g.m1 * C1c + g.m2 * C2c + g.m0 * C0c;
    if (f.counters.cap < 4 * static_cast<size_t>(ncnt)) {
      f.counters.ensure(4 * static_cast<size_t>(ncnt));
      CK(cudaMemsetAsync(f.counters.p, 0, f.counters.cap, st));
    }
    f.gpart.ensure(4 * 128 * static_cast<size_t>(tasks));
    f.gtouch.ensure(4 * static_cast<size_t>(tasks));
    A.gpart = f.gpart.as<float>();
    A.gtouch = f.gtouch.as<int>();
    A.counters = f.counters.as<int>();
    // bwd1 + combine in one cooperative launch when the bwd1 grid is co-resident
    const bool fuse_comb = !f.chunked && t->fuse_comb &&
                           4 * static_cast<size_t>(g.m1 + g.m2 + 2) <= sm1;
    int* b1plan_ptr = nullptr;  // f3_bwd1 ranges planned by f3_srows_bwd2 (fused path)
    uint8_t* b1ulen_ptr = nullptr;  // and its merge units
    t->mark("bwd_begin");
    if (f.chunked) {
      f3_launch(t->pdl, kc, dim3(grid1), dim3(f3::kFcThreads), sm1, st, g, t->cores.as<float>(),
                f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(), f.rec1.as<uint4>(), f.slotpos.as<uint16_t>(),
                f.tile_i0.as<uint16_t>(), f.tile_nslots.as<int>(), grad, f.part1.as<float>(),
                f.has1.as<int>(), f.D0acc.as<float>(), f.d0mask.as<unsigned char>());
      t->mark("f3c_bwd");
    } else if (t->fuse_sb) {
      // f3_srows and f3_bwd2 in one launch (they are independent)
      // the launch's first CTA plans f3_bwd1's tile ranges (unless the
      // cooperative bwd1+combine variant runs, which plans them itself)
      int* plan = nullptr;
      uint8_t* ulen = nullptr;
      if (!fuse_comb && t->plan_bwd1) {
        f.b1plan.ensure(4 * (static_cast<size_t>(grid1) + 1));
        plan = f.b1plan.as<int>();
        if (t->merge1) {
          f.b1ulen.ensure(static_cast<size_t>(f.max_tiles1) + 16);
          ulen = f.b1ulen.as<uint8_t>();
        }
      }
      f3::SrowsArgs sa{t->cores.as<float>(), g.coff2, f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(),
                       f.max_tiles1, f.perm1.as<uint32_t>(), f.d2.as<uint16_t>(),
                       f.slotpos.as<uint16_t>(), f.tile_nslots.as<int>(), f.Sbuf.as<float>(),
                       plan, grid1, f.rec1.as<uint4>(), ulen, f.tile_one.as<int>(),
                       t->b1tile, t->b1cont};
      b1plan_ptr = plan;
      b1ulen_ptr = ulen;
      f3::Bwd2Args ba{f.tiles2.as<f3::Tile>(), f.ntiles.as<int>() + 1, f.perm2.as<uint32_t>(),
                      f.hloc.as<uint32_t>(), f.Hbuf.as<float>(), f.part2.as<float>(), f.has2.as<int>()};
      // srows warps walk the tiles grid-stride: TTGPU_SROWS_CTAS_PER_SM virtual
      // CTAs per SM (0 = one warp per tile)
      static const int srows_per_sm = [] {
        const char* e = std::getenv("TTGPU_SROWS_CTAS_PER_SM");
        return e ? std::atoi(e) : 0;
      }();
      const int nbs_all = (f.max_tiles1 * 32 + 127) / 128;
      const int nbs = srows_per_sm > 0 ? std::min(nbs_all, t->num_sms * srows_per_sm) : nbs_all;
      f3_launch(t->pdl, f3::f3_srows_bwd2<D>, dim3(grid2 + nbs + (plan ? 1 : 0)), dim3(128), 0, st, g, sa,
                ba, grid2, nbs, lk_bag, alpha, grad);
      t->mark("f3_srows_bwd2");
    } else {
      f3_launch(t->pdl, f3::f3_srows<D>, dim3((f.max_tiles1 * 32 + 255) / 256), dim3(256), 0, st,
                t->cores.as<float>(), g.coff2, f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(), f.max_tiles1,
                f.perm1.as<uint32_t>(), f.d2.as<uint16_t>(), lk_bag, alpha, grad,
                f.slotpos.as<uint16_t>(), f.tile_nslots.as<int>(), f.Sbuf.as<float>());
      t->mark("f3_srows");
    }
    auto launch_bwd2 = [&] {
      f3_launch(t->pdl, f3::f3_bwd2<D>, dim3(grid2), dim3(128), 0, st, g, f.tiles2.as<f3::Tile>(),
                f.ntiles.as<int>() + 1, f.perm2.as<uint32_t>(), f.hloc.as<uint32_t>(), lk_bag, alpha, grad,
                f.Hbuf.as<float>(), f.part2.as<float>(), f.has2.as<int>());
      t->mark("f3_bwd2");
    };
    if (fuse_comb) {
      if (!t->fuse_sb) launch_bwd2();  // the combine phase reads its partials
      auto kf = f3::f3_bwd1_comb<D>;
      set_smem(kf, sm1);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(grid1);
      cfg.blockDim = dim3(f3::kThreads);
      cfg.dynamicSmemBytes = sm1;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeCooperative;
      at[0].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, kf, g, t->cores.as<float>(), static_cast<const f3::Tile*>(f.tiles1.as<f3::Tile>()),
                            static_cast<const int*>(f.ntiles.as<int>()), static_cast<const float*>(f.Sbuf.as<float>()),
                            static_cast<const uint16_t*>(f.tile_i0.as<uint16_t>()),
                            static_cast<const int*>(f.tile_nslots.as<int>()), f.part1.as<float>(),
                            f.has1.as<int>(), f.D0acc.as<float>(), f.d0mask.as<unsigned char>(),
                            t->grads.as<float>(), A, lr, mode, tasks));
      t->mark("f3_bwd1_comb");
      CK(cudaGetLastError());
      return;
    }
    if (!f.chunked) {
      f3_launch(t->pdl, k1, dim3(grid1), dim3(f3::kThreads), sm1, st, g, t->cores.as<float>(),
                f.tiles1.as<f3::Tile>(), f.ntiles.as<int>(), f.Sbuf.as<float>(), f.tile_i0.as<uint16_t>(),
                f.tile_nslots.as<int>(), f.part1.as<float>(), f.has1.as<int>(), f.D0acc.as<float>(),
                f.d0mask.as<unsigned char>(), static_cast<const int*>(b1plan_ptr),
                static_cast<const uint8_t*>(b1ulen_ptr));
      t->mark("f3_bwd1");
    }
    if (!t->fuse_sb || f.chunked) launch_bwd2();
    {
      auto ck = mode == 1 ? f3::f3_combine<D, 1> : f3::f3_combine<D, 0>;
      const size_t csm = 4 * static_cast<size_t>(g.m1 + 1 + g.m2 + 1);
      set_smem(ck, csm);
      f3_launch(t->pdl, ck, dim3((tasks * 32 + f3::kThreads - 1) / f3::kThreads), dim3(f3::kThreads), csm, st,
                g, t->cores.as<float>(), t->grads.as<float>(), A, lr);
    }
    t->mark("f3_combine");
    CK(cudaGetLastError());
  }
};

// instantiation table: (P0, R1, N1, R2, N2, TT)
using F3_R4 = f3::Dims<2, 4, 2, 4, 4, 32>;
using F3_R8 = f3::Dims<2, 8, 2, 8, 4, 32>;
using F3_R16 = f3::Dims<2, 16, 2, 16, 4, 32>;
using F3_R32 = f3::Dims<2, 32, 2, 32, 4, 32>;
using F3_R64 = f3::Dims<2, 64, 2, 64, 4, 32>;

template <class D>
bool dims_match(const DevPlan& P) {
  return P.n[0] == D::P0 && P.r[1] == D::R1 && P.n[1] == D::N1 && P.r[2] == D::R2 &&
         P.n[2] == D::N2 && P.r[3] == 1;
}

// Which fast-path instantiation serves this table (-1: generic path).
int f3_kind(const ttgpu_table* t) {
  const DevPlan& P = t->dp;
  if (t->dtype != TTGPU_F32 || P.d != 3) return -1;
  if (P.m[0] >= 65536 || P.m[1] >= 65536 || P.m[2] >= 65536) return -1;
  if (P.num_rows >= (1ll << 32) || static_cast<int64_t>(P.m[0]) * P.m[1] * P.m[2] >= (1ll << 32))
    return -1;
  if (std::max(P.m[1], P.m[2]) > 6144 || P.m[0] > 8192) return -1;
  if (dims_match<F3_R4>(P)) return 4;
  if (dims_match<F3_R8>(P)) return 0;
  if (dims_match<F3_R16>(P)) return 1;
  if (dims_match<F3_R32>(P)) return 2;
  if (dims_match<F3_R64>(P)) return 3;
  return -1;
}

bool f3_feasible(const ttgpu_table* t, int64_t L) {
  const f3::Geo g = make_geo(t);
  return L < (1ll << 31) && f3_lpt(L, std::max(g.m1, g.m2)) > 0;
}

void f3_forward(int kind, ttgpu_table* t, F3Bufs& f, const int64_t* idx, int64_t L,
                const int64_t* off, int64_t B, const double* w, int pooling, float* out, bool exact,
                int32_t* lk_bag, float* alpha, const F3Cache* cache = nullptr) {
  f.kind = kind;
  switch (kind) {
    case 0: F3Runner<F3_R8>::forward(t, f, idx, L, off, B, w, pooling, out, exact, lk_bag, alpha, cache); break;
    case 1: F3Runner<F3_R16>::forward(t, f, idx, L, off, B, w, pooling, out, exact, lk_bag, alpha, cache); break;
    case 2: F3Runner<F3_R32>::forward(t, f, idx, L, off, B, w, pooling, out, exact, lk_bag, alpha, cache); break;
    case 3: F3Runner<F3_R64>::forward(t, f, idx, L, off, B, w, pooling, out, exact, lk_bag, alpha, cache); break;
    case 4: F3Runner<F3_R4>::forward(t, f, idx, L, off, B, w, pooling, out, exact, lk_bag, alpha, cache); break;
    default: fail(TTGPU_ERR_RUNTIME, "bad fast-path kind");
  }
}

void f3_backward(ttgpu_table* t, F3Bufs& f, const float* grad, int mode, float lr,
                 const int32_t* lk_bag, const float* alpha, int64_t L) {
  switch (f.kind) {
    case 0: F3Runner<F3_R8>::backward(t, f, grad, mode, lr, lk_bag, alpha, L); break;
    case 1: F3Runner<F3_R16>::backward(t, f, grad, mode, lr, lk_bag, alpha, L); break;
    case 2: F3Runner<F3_R32>::backward(t, f, grad, mode, lr, lk_bag, alpha, L); break;
    case 3: F3Runner<F3_R64>::backward(t, f, grad, mode, lr, lk_bag, alpha, L); break;
    case 4: F3Runner<F3_R4>::backward(t, f, grad, mode, lr, lk_bag, alpha, L); break;
    default: fail(TTGPU_ERR_RUNTIME, "bad fast-path kind");
  }
}

}  // namespace
}  // namespace ttgpu
