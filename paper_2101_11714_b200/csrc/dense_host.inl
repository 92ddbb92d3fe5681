// Uncompressed embedding-bag tables on the GPU (the 19
// DLRM features of cfg5 that are not TT-compressed).  All tables of a group
// share one row store (row r of table t at global row base[t] + r), one batch
// structure (offsets) and one launch per phase:
//   forward   out[t][b] = Σ_{l in bag b} E_t[idx[t][l]]  -- lookup order, each
//             sum separately rounded (the reference's axpy with w = 1,
//             gemm.hpp:64-66; EmbeddingLayer's plain-table path)
//   backward  rows sorted by global row id (stable, CUB radix), per-row
//             gradient = Σ grad[t][bag(l)] over the row's lookups in lookup
//             order (chunk sums + fixed-order fold, the LFU slot kernels), then
//             row -= T(lr)·g fused (one replica) or written to a dense
//             gradient buffer for an allreduce followed by ttgpu_dense_apply_grad.
// Out-of-range indices are latched on the device and reported by
// ttgpu_dense_check with the reference's message shape.
namespace ttgpu {
namespace {

template <typename T>
__global__ void k_dense_fwd(const int64_t* __restrict__ base, const int64_t* __restrict__ rows,
                            const T* __restrict__ E, int N, const int64_t* __restrict__ idx,
                            int64_t L, const int64_t* __restrict__ off, int64_t B,
                            T* __restrict__ out, unsigned long long* __restrict__ bad) {
  // grid.y = table; threads over (bag, column quad): no 64-bit divisions, and
  // a bag's lookups are read once per 4 columns
  const int t = blockIdx.y;
  const int Q = (N + 3) / 4;
  const int64_t rt = rows[t], bt = base[t];
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < B * Q;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / Q;
    const int c0 = static_cast<int>(q - b * Q) * 4;
    int64_t lo = off[b], hi = off[b + 1];
    lo = lo < 0 ? 0 : lo;
    hi = hi > L ? L : hi;
    T acc[4] = {T(0), T(0), T(0), T(0)};
    for (int64_t l = lo; l < hi; ++l) {
      const int64_t r = idx[static_cast<int64_t>(t) * L + l];
      if (r < 0 || r >= rt) {
        if (c0 == 0) atomicMin(bad, static_cast<unsigned long long>(static_cast<int64_t>(t) * L + l));
        continue;
      }
      const T* row = E + (bt + r) * N + c0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u < N) acc[u] = lfu::add_rn(acc[u], row[u]);
    }
    T* o = out + (static_cast<int64_t>(t) * B + b) * N + c0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (c0 + u < N) o[u] = acc[u];
  }
}

// lookup -> bag (offsets are shared by every table of the group)
__global__ void k_dense_bags(const int64_t* __restrict__ off, int64_t B, int64_t L,
                             int32_t* __restrict__ lk_bag) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t lo = off[b], hi = off[b + 1];
    lo = lo < 0 ? 0 : lo;
    hi = hi > L ? L : hi;
    for (int64_t l = lo; l < hi; ++l) lk_bag[l] = static_cast<int32_t>(b);
  }
}

// sort keys: global row id; values: lookup position (t*L + l); bag' = t*B + bag
__global__ void k_dense_keys(int ntab, const int64_t* __restrict__ base,
                             const int64_t* __restrict__ rows, const int64_t* __restrict__ idx,
                             int64_t L, int64_t B, const int32_t* __restrict__ lk_bag,
                             int* __restrict__ key, int* __restrict__ pos,
                             int32_t* __restrict__ cbag) {
  const int64_t n = static_cast<int64_t>(ntab) * L;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(q / L);
    const int64_t l = q - static_cast<int64_t>(t) * L;
    int64_t r = idx[q];
    r = (r < 0 || r >= rows[t]) ? 0 : r;  // rejected by the forward's latch
    key[q] = static_cast<int>(base[t] + r);
    pos[q] = static_cast<int>(q);
    cbag[q] = static_cast<int32_t>(static_cast<int64_t>(t) * B + lk_bag[l]);
  }
}

template <typename T>
__global__ void k_dense_apply(int64_t n, const T* __restrict__ g, T* __restrict__ E, T lr) {
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x)
    E[q] = lfu::sub_rn(E[q], lfu::mul_rn(lr, g[q]));
}

}  // namespace
}  // namespace ttgpu

struct ttgpu_dense {
  int ntab = 0;
  int64_t N = 0;
  int dtype = TTGPU_F32;
  size_t esz = 4;
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  std::vector<int64_t> rows, base;
  int64_t total = 0;
  ttgpu::DevBuf E, d_rows, d_base, idx, off, lk_bag, key_in, key, pos_in, pos, cbag, seg_lo, seg_hi,
      part, sg, tmp, errs;
  int64_t L = 0, B = 0;
  bool valid = false;
};

namespace ttgpu {
namespace {
template <typename T>
void dense_backward(ttgpu_dense* d, const T* grad, int fused, double lr) {
  cudaStream_t st = d->stream;
  const int64_t n = static_cast<int64_t>(d->ntab) * d->L;
  const int N = static_cast<int>(d->N);
  d->seg_lo.ensure(4 * d->total);
  d->seg_hi.ensure(4 * d->total);
  d->sg.ensure(d->esz * d->total * d->N);
  CK(cudaMemsetAsync(d->seg_lo.p, 0xff, 4 * d->total, st));
  if (!fused) CK(cudaMemsetAsync(d->sg.p, 0, d->esz * d->total * d->N, st));
  if (n == 0) return;
  d->key_in.ensure(4 * n);
  d->key.ensure(4 * n);
  d->pos_in.ensure(4 * n);
  d->pos.ensure(4 * n);
  d->cbag.ensure(4 * n);
  d->part.ensure(d->esz * n * d->N);
  k_dense_keys<<<grid_for(n, kThreads, d->num_sms, 8), kThreads, 0, st>>>(
      d->ntab, d->d_base.as<int64_t>(), d->d_rows.as<int64_t>(), d->idx.as<int64_t>(), d->L, d->B,
      d->lk_bag.as<int32_t>(), d->key_in.as<int>(), d->pos_in.as<int>(), d->cbag.as<int32_t>());
  const int bits = bits_for(static_cast<uint64_t>(d->total));
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, d->key_in.as<int>(), d->key.as<int>(),
                                     d->pos_in.as<int>(), d->pos.as<int>(), static_cast<int>(n), 0,
                                     bits, st));
  d->tmp.ensure(tb);
  CK(cub::DeviceRadixSort::SortPairs(d->tmp.p, tb, d->key_in.as<int>(), d->key.as<int>(),
                                     d->pos_in.as<int>(), d->pos.as<int>(), static_cast<int>(n), 0,
                                     bits, st));
  lfu::k_segments<<<grid_for(n, kThreads, d->num_sms, 8), kThreads, 0, st>>>(
      d->key.as<int>(), n, d->seg_lo.as<int>(), d->seg_hi.as<int>());
  const int64_t chunks = (n + lfu::kSlotChunk - 1) / lfu::kSlotChunk;
  lfu::k_slot_chunks<T><<<grid_for(chunks * 32, kThreads, d->num_sms, 8), kThreads, 0, st>>>(
      n, N, d->key.as<int>(), d->pos.as<int>(), nullptr, d->cbag.as<int32_t>(), grad,
      d->seg_lo.as<int>(), d->seg_hi.as<int>(), d->part.as<T>(), d->sg.as<T>(), d->E.as<T>(), fused,
      static_cast<T>(lr));
  lfu::k_slot_fold_runs<T><<<grid_for(chunks * N * 32, kThreads, d->num_sms, 8), kThreads, 0, st>>>(
      n, N, d->key.as<int>(), d->seg_lo.as<int>(), d->seg_hi.as<int>(), d->part.as<T>(),
      d->sg.as<T>(), d->E.as<T>(), fused, static_cast<T>(lr));
  CK(cudaGetLastError());
}
}  // namespace
}  // namespace ttgpu

extern "C" {

int ttgpu_dense_create(int n_tables, const int64_t* rows, int64_t dim, int dtype, int device,
                       void* stream, ttgpu_dense** out) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(n_tables >= 1, cat("need at least one table, got ", n_tables));
    require_arg(dim >= 1, cat("emb_dim must be positive, got ", dim));
    require_arg(dim <= lfu::kSlotMaxN,
                cat("dense tables support emb_dim <= ", lfu::kSlotMaxN, ", got ", dim));
    require_arg(dtype == TTGPU_F32 || dtype == TTGPU_F64, "dtype must be TTGPU_F32 or TTGPU_F64");
    CK(cudaSetDevice(device));
    auto d = std::make_unique<ttgpu_dense>();
    d->ntab = n_tables;
    d->N = dim;
    d->dtype = dtype;
    d->esz = dtype == TTGPU_F64 ? 8 : 4;
    d->device = device;
    d->stream = static_cast<cudaStream_t>(stream);
    cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, device);
    int64_t acc = 0;
    for (int t = 0; t < n_tables; ++t) {
      require_arg(rows[t] >= 1, cat("table ", t, " needs at least one row"));
      d->rows.push_back(rows[t]);
      d->base.push_back(acc);
      acc += rows[t];
    }
    require_arg(acc < (int64_t{1} << 31), "dense tables: more than 2^31 rows in one group");
    d->total = acc;
    d->E.ensure(d->esz * acc * dim);
    CK(cudaMemsetAsync(d->E.p, 0, d->esz * acc * dim, d->stream));
    d->d_rows.ensure(8 * n_tables);
    d->d_base.ensure(8 * n_tables);
    CK(cudaMemcpy(d->d_rows.p, d->rows.data(), 8 * n_tables, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d->d_base.p, d->base.data(), 8 * n_tables, cudaMemcpyHostToDevice));
    d->errs.ensure(8);
    CK(cudaMemset(d->errs.p, 0xff, 8));
    CK(cudaStreamSynchronize(d->stream));
    *out = d.release();
  });
}

int ttgpu_dense_destroy(ttgpu_dense* d) {
  return guarded([&] {
    if (d) cudaStreamSynchronize(d->stream);
    delete d;
  });
}

int ttgpu_dense_set_stream(ttgpu_dense* d, void* stream) {
  return guarded([&] { d->stream = static_cast<cudaStream_t>(stream); });
}

// rows of table t as host (rows[t] x dim) arrays
int ttgpu_dense_set_table(ttgpu_dense* d, int t, const void* host) {
  return guarded([&] {
    require_arg(t >= 0 && t < d->ntab, cat("table ", t, " out of range"));
    CK(cudaMemcpyAsync(static_cast<char*>(d->E.p) + d->esz * d->base[t] * d->N, host,
                       d->esz * d->rows[t] * d->N, cudaMemcpyHostToDevice, d->stream));
    CK(cudaStreamSynchronize(d->stream));
  });
}

int ttgpu_dense_get_table(ttgpu_dense* d, int t, void* host) {
  return guarded([&] {
    require_arg(t >= 0 && t < d->ntab, cat("table ", t, " out of range"));
    CK(cudaMemcpyAsync(host, static_cast<char*>(d->E.p) + d->esz * d->base[t] * d->N,
                       d->esz * d->rows[t] * d->N, cudaMemcpyDeviceToHost, d->stream));
    CK(cudaStreamSynchronize(d->stream));
  });
}

// indices: n_tables x L (table-major), offsets: B + 1 shared by every table,
// out: n_tables x B x dim.  Asynchronous; the indices/offsets are kept (copied)
// for the backward.
int ttgpu_dense_forward_device(ttgpu_dense* d, const int64_t* d_idx, int64_t L,
                               const int64_t* d_off, int64_t B, void* d_out) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(L >= 0 && B >= 0, "negative batch size");
    cudaStream_t st = d->stream;
    const int64_t n = static_cast<int64_t>(d->ntab) * L;
    d->idx.ensure(8 * std::max<int64_t>(n, 1));
    d->off.ensure(8 * (B + 1));
    d->lk_bag.ensure(4 * std::max<int64_t>(L, 1));
    if (n) CK(cudaMemcpyAsync(d->idx.p, d_idx, 8 * n, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d->off.p, d_off, 8 * (B + 1), cudaMemcpyDeviceToDevice, st));
    d->L = L;
    d->B = B;
    d->valid = true;
    if (B == 0) return;
    const int64_t per_tab = B * ((d->N + 3) / 4);
    const dim3 grid(static_cast<unsigned>(
                        std::max<int64_t>(1, std::min<int64_t>((per_tab + kThreads - 1) / kThreads,
                                                               int64_t{d->num_sms} * 2))),
                    static_cast<unsigned>(d->ntab));
    if (d->dtype == TTGPU_F64)
      k_dense_fwd<double><<<grid, kThreads, 0, st>>>(
          d->d_base.as<int64_t>(), d->d_rows.as<int64_t>(), d->E.as<double>(),
          static_cast<int>(d->N), d->idx.as<int64_t>(), L, d->off.as<int64_t>(), B,
          static_cast<double*>(d_out), d->errs.as<unsigned long long>());
    else
      k_dense_fwd<float><<<grid, kThreads, 0, st>>>(
          d->d_base.as<int64_t>(), d->d_rows.as<int64_t>(), d->E.as<float>(),
          static_cast<int>(d->N), d->idx.as<int64_t>(), L, d->off.as<int64_t>(), B,
          static_cast<float*>(d_out), d->errs.as<unsigned long long>());
    k_dense_bags<<<grid_for(B, kThreads, d->num_sms, 8), kThreads, 0, st>>>(
        d->off.as<int64_t>(), B, L, d->lk_bag.as<int32_t>());
    CK(cudaGetLastError());
  });
}

// grad: n_tables x B x dim.  fused (1): rows -= lr * g in the reduction's
// epilogue; 0: the dense per-row gradient stays in the group's buffer
// (ttgpu_dense_grad_buffer) for an allreduce, then ttgpu_dense_apply_grad.
int ttgpu_dense_backward_device(ttgpu_dense* d, const void* d_grad, int fused, double lr) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(d->valid, "dense backward needs a forward first");
    if (d->dtype == TTGPU_F64)
      dense_backward<double>(d, static_cast<const double*>(d_grad), fused ? 1 : 0, lr);
    else
      dense_backward<float>(d, static_cast<const float*>(d_grad), fused ? 1 : 0, lr);
  });
}

int ttgpu_dense_grad_buffer(ttgpu_dense* d, void** ptr, int64_t* n_elems) {
  return guarded([&] {
    d->sg.ensure(d->esz * d->total * d->N);
    *ptr = d->sg.p;
    *n_elems = d->total * d->N;
  });
}

int ttgpu_dense_apply_grad(ttgpu_dense* d, double lr) {
  using namespace ttgpu;
  return guarded([&] {
    const int64_t n = d->total * d->N;
    if (d->dtype == TTGPU_F64)
      k_dense_apply<double><<<grid_for(n, kThreads, d->num_sms, 8), kThreads, 0, d->stream>>>(
          n, d->sg.as<double>(), d->E.as<double>(), lr);
    else
      k_dense_apply<float><<<grid_for(n, kThreads, d->num_sms, 8), kThreads, 0, d->stream>>>(
          n, d->sg.as<float>(), d->E.as<float>(), static_cast<float>(lr));
    CK(cudaGetLastError());
  });
}

// synchronises; reports an out-of-range index like index_batch.hpp:50-54
int ttgpu_dense_check(ttgpu_dense* d) {
  using namespace ttgpu;
  return guarded([&] {
    unsigned long long h = 0;
    CK(cudaStreamSynchronize(d->stream));
    CK(cudaMemcpy(&h, d->errs.p, 8, cudaMemcpyDeviceToHost));
    if (h == ULLONG_MAX) return;
    CK(cudaMemset(d->errs.p, 0xff, 8));
    const int64_t q = static_cast<int64_t>(h);
    const int t = static_cast<int>(d->L ? q / d->L : 0);
    int64_t r = 0;
    CK(cudaMemcpy(&r, d->idx.as<int64_t>() + q, 8, cudaMemcpyDeviceToHost));
    d->valid = false;
    throw std::out_of_range(cat("index ", r, " out of range [0, ", d->rows[t],
                                ") for dense table ", t));
  });
}

}  // extern "C"
