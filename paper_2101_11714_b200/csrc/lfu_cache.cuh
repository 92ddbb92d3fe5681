// LFU cache of hot uncompressed rows in front of a TT table -- device side.
//
// Reference: LfuCache<T> / FreqTable / CachePartition / combine_partition_outputs
// (proj/include/ttrec/lfu_cache.hpp:18-310, proj/src/lfu_cache.cpp:15-126) and
// the EmbeddingLayer composition (proj/include/ttrec/model.hpp:195-284).
//
// B200 layout:
//   * frequencies: one dense uint64 counter per table row (8 B/row: 81 MB for
//     the 10M-row Criteo table) -- one warp-aggregated atomicAdd per lookup
//     instead of a host hash-table probe.  Same counts as FreqTable.
//   * residency: an open-addressing hash table row -> slot (power-of-two
//     capacity >= 2x slots, Fibonacci hashing, linear probing, uint64 keys),
//     a few KB that stays L1/L2-resident; every lookup probes it before any
//     decompression ("consulted before decompression").
//   * store: capacity x emb_dim rows, slot i = i-th hottest row.
// Every reduction has a fixed order (stable partition, stable sort by slot,
// chunk partials folded in chunk order): results are bitwise reproducible.
#pragma once

#include <cstdint>

namespace ttgpu {
namespace lfu {

constexpr unsigned long long kEmptyKey = ~0ull;
constexpr unsigned long long kFib = 0x9E3779B97F4A7C15ull;
constexpr int kSlotChunk = 32;  // sorted cached lookups per slot-gradient chunk
constexpr int kSlotMaxN = 64;   // row width the slot-gradient kernels handle in registers

__device__ __forceinline__ int probe(const unsigned long long* __restrict__ keys,
                                     const int* __restrict__ vals, int shift,
                                     unsigned long long mask, unsigned long long key) {
  unsigned long long i = (key * kFib) >> shift;
  while (true) {
    const unsigned long long k = keys[i];
    if (k == key) return vals[i];
    if (k == kEmptyKey) return -1;
    i = (i + 1) & mask;
  }
}

__global__ void k_hash_insert(const int64_t* __restrict__ rows, int64_t n,
                              unsigned long long* __restrict__ keys, int* __restrict__ vals,
                              int shift, unsigned long long mask) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long key = static_cast<unsigned long long>(rows[i]);
    unsigned long long h = (key * kFib) >> shift;
    while (true) {
      const unsigned long long prev = atomicCAS(keys + h, kEmptyKey, key);
      if (prev == kEmptyKey || prev == key) {
        vals[h] = static_cast<int>(i);
        break;
      }
      h = (h + 1) & mask;
    }
  }
}

// record_and_partition, per lookup (lfu_cache.hpp:187-219): frequency += 1
// (warp-aggregated), probe the residency hash when Active, emit the slot (or
// -1) and the hit flag.  count_only: record() (frequencies only).
__global__ void k_partition(const int64_t* __restrict__ idx, int64_t L, int64_t key_space,
                            unsigned long long* __restrict__ counts,
                            const unsigned long long* __restrict__ hkeys,
                            const int* __restrict__ hvals, int hshift, unsigned long long hmask,
                            int active, int count_only, int* __restrict__ lk_slot,
                            int* __restrict__ flags, unsigned long long* __restrict__ bad,
                            unsigned long long* __restrict__ hits) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) - lane;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  unsigned my_hits = 0;
  for (int64_t base = warp0; base < L; base += wstride) {
    const int64_t l = base + lane;
    const bool in = l < L;
    const int64_t row = in ? idx[l] : -1;
    const bool valid = in && row >= 0 && row < key_space;
    if (in && !valid) atomicMin(bad, static_cast<unsigned long long>(l));
    const unsigned long long key = valid ? static_cast<unsigned long long>(row) : kEmptyKey;
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    if (valid && lane == __ffs(peers) - 1) atomicAdd(counts + row, static_cast<unsigned long long>(__popc(peers)));
    if (count_only) continue;
    const int slot = (valid && active) ? probe(hkeys, hvals, hshift, hmask, key) : -1;
    if (in) {
      lk_slot[l] = slot;
      flags[l] = slot >= 0 ? 1 : 0;
    }
    my_hits += __popc(__ballot_sync(0xffffffffu, slot >= 0));
  }
  if (!count_only && lane == 0 && my_hits) atomicAdd(hits, static_cast<unsigned long long>(my_hits));
  if (!count_only && blockIdx.x == 0 && threadIdx.x == 0) flags[L] = 0;
}

// Offsets structure check (index_batch.hpp:41-48), latched like the table's.
__global__ void k_check_offsets(const int64_t* __restrict__ off, int64_t B, int64_t L,
                                int* __restrict__ errs) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < B;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = off[b], e = off[b + 1];
    if (b == 0 && s != 0) atomicOr(errs, 1);
    if (e < s) atomicOr(errs, 2);
    if (b == B - 1 && e != L) atomicOr(errs, 4);
  }
}

// Stable split of the batch into the cached part (slot ids, original rows,
// weights, bag of each cached lookup) and the chain part (rows, weights);
// both keep every bag (CachePartition, lfu_cache.hpp:92-104).
__global__ void k_split(const int64_t* __restrict__ idx, int64_t L, const int64_t* __restrict__ off,
                        int64_t B, const double* __restrict__ w, const int* __restrict__ lk_slot,
                        const int* __restrict__ hpos, int64_t* __restrict__ c_idx,
                        int64_t* __restrict__ c_rows, double* __restrict__ c_w,
                        int32_t* __restrict__ c_bag, int64_t* __restrict__ c_off,
                        int64_t* __restrict__ t_idx, double* __restrict__ t_w,
                        int64_t* __restrict__ t_off) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t g0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  for (int64_t l = g0; l < L; l += stride) {
    const int h = hpos[l];
    const int s = lk_slot[l];
    if (s >= 0) {
      c_idx[h] = s;
      c_rows[h] = idx[l];
      if (w) c_w[h] = w[l];
      // bag of lookup l: last b with off[b] <= l (upper_bound - 1)
      int64_t lo = 0, hi = B;  // off[lo] <= l < off[hi]
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (off[mid] <= l) lo = mid; else hi = mid;
      }
      c_bag[h] = static_cast<int32_t>(lo);
    } else {
      const int64_t t = l - h;
      t_idx[t] = idx[l];
      if (w) t_w[t] = w[l];
    }
  }
  for (int64_t b = g0; b <= B; b += stride) {
    int64_t o = off[b];
    o = o < 0 ? 0 : (o > L ? L : o);
    const int64_t h = hpos[o];
    c_off[b] = h;
    t_off[b] = o - h;
  }
}

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <typename T>
__device__ __forceinline__ T sub_rn(T a, T b);
template <>
__device__ __forceinline__ float sub_rn<float>(float a, float b) { return __fsub_rn(a, b); }
template <>
__device__ __forceinline__ double sub_rn<double>(double a, double b) { return __dsub_rn(a, b); }

// EmbeddingLayer::forward with a cache (model.hpp:210-223): cached_out[b] =
// Σ T(w)·store[slot] in lookup order (axpy, gemm.hpp:64-66: product and sum
// separately rounded), out = cached_out + tt_out, then the original pooling's
// mean division (combine_partition_outputs, lfu_cache.hpp:106-126).
template <typename T>
__global__ void k_combine(int64_t B, int N, const int64_t* __restrict__ c_off,
                          const int64_t* __restrict__ c_idx, const double* __restrict__ c_w,
                          const T* __restrict__ store, const int64_t* __restrict__ t_off,
                          const T* __restrict__ tt_out, int mean, T* __restrict__ out) {
  const int64_t n = B * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / N;
    const int j = static_cast<int>(q - b * N);
    T c = T(0);
    for (int64_t t = c_off[b]; t < c_off[b + 1]; ++t) {
      const T a = c_w ? static_cast<T>(c_w[t]) : T(1);
      c = add_rn(c, mul_rn(a, store[c_idx[t] * N + j]));
    }
    T v = add_rn(c, tt_out[q]);
    if (mean) {
      const int64_t sz = (c_off[b + 1] - c_off[b]) + (t_off[b + 1] - t_off[b]);
      if (sz > 1) v = mul_rn(v, static_cast<T>(1.0 / static_cast<double>(sz)));
    }
    out[q] = v;
  }
}

// grad_eff for a Mean batch on the cache fast path: the original bag size from
// the batch's own offsets (model.hpp:242-252).
__global__ void k_grad_eff_off(int64_t B, int N, const int64_t* __restrict__ off,
                               const float* __restrict__ g, float* __restrict__ ge) {
  const int64_t n = B * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / N;
    const int64_t sz = off[b + 1] - off[b];
    float v = g[q];
    if (sz > 1) v = __fmul_rn(v, static_cast<float>(1.0 / static_cast<double>(sz)));
    ge[q] = v;
  }
}

// grad_eff for a Mean batch (model.hpp:242-252): the original bag size folded
// into the upstream gradient once, for both parts.
template <typename T>
__global__ void k_grad_eff(int64_t B, int N, const int64_t* __restrict__ c_off,
                           const int64_t* __restrict__ t_off, const T* __restrict__ g,
                           T* __restrict__ ge) {
  const int64_t n = B * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = q / N;
    const int64_t sz = (c_off[b + 1] - c_off[b]) + (t_off[b + 1] - t_off[b]);
    T v = g[q];
    if (sz > 1) v = mul_rn(v, static_cast<T>(1.0 / static_cast<double>(sz)));
    ge[q] = v;
  }
}

__global__ void k_fill_slot_keys(const int64_t* __restrict__ c_idx, int64_t n, int* __restrict__ key,
                                 int* __restrict__ pos) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    key[i] = static_cast<int>(c_idx[i]);
    pos[i] = static_cast<int>(i);
  }
}

// cached lookups sorted by slot (stable) -> per-slot segment [lo, hi)
__global__ void k_segments(const int* __restrict__ skey, int64_t n, int* __restrict__ seg_lo,
                           int* __restrict__ seg_hi) {
  for (int64_t p = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < n;
       p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = skey[p];
    if (p == 0 || skey[p - 1] != s) seg_lo[s] = static_cast<int>(p);
    if (p == n - 1 || skey[p + 1] != s) seg_hi[s] = static_cast<int>(p + 1);
  }
}

// Slot gradients (model.hpp:253-261: row_for(slot) += T(w)·grad_eff[bag] in
// lookup order).  One warp per chunk of kSlotChunk sorted cached lookups,
// lanes over columns: runs of one slot are summed in order; a slot wholly
// inside the chunk is final (written to the gradient, or -- fused -- applied:
// row -= T(lr)·g, lfu_cache.hpp:246-257), otherwise the run's partial is
// parked at its first position for k_slot_fold.
template <typename T>
__global__ void k_slot_chunks(int64_t n, int N, const int* __restrict__ skey,
                              const int* __restrict__ spos, const double* __restrict__ c_w,
                              const int32_t* __restrict__ c_bag, const T* __restrict__ ge,
                              const int* __restrict__ seg_lo, const int* __restrict__ seg_hi,
                              T* __restrict__ part, T* __restrict__ sg, T* __restrict__ store,
                              int fused, T lr, const int* __restrict__ dn = nullptr) {
  static_assert(kSlotChunk == 32, "one chunk position per lane");
  if (dn) n = *dn;  // device-side count (cache fast path: no host sync)
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (n + kSlotChunk - 1) / kSlotChunk;
  const int64_t warp = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t ch = warp; ch < nchunks; ch += nwarps) {
    const int64_t p0 = ch * kSlotChunk;
    const int m = static_cast<int>(p0 + kSlotChunk < n ? kSlotChunk : n - p0);
    // lane q holds position p0 + q's slot / weight / bag: one round trip for the chunk
    int my_s = -1, my_bag = 0;
    T my_a = T(0);
    // neighbours of the chunk: a run is final here iff it neither continues
    // from the previous chunk nor into the next one
    const int key_before = p0 > 0 ? skey[p0 - 1] : -1;
    const int key_after = p0 + m < n ? skey[p0 + m] : -1;
    if (lane < m) {
      my_s = skey[p0 + lane];
      const int pos = spos[p0 + lane];
      my_bag = c_bag[pos];
      my_a = c_w ? static_cast<T>(c_w[pos]) : T(1);
    }
    for (int j0 = 0; j0 < N; j0 += 32) {
      const int j = j0 + lane;
      // every position's value for this lane's column, loads issued together
      T v[kSlotChunk];
#pragma unroll
      for (int q = 0; q < kSlotChunk; ++q) {
        const int bag = __shfl_sync(0xffffffffu, my_bag, q);
        const T a = __shfl_sync(0xffffffffu, my_a, q);
        v[q] = (q < m && j < N) ? mul_rn(a, ge[static_cast<int64_t>(bag) * N + j]) : T(0);
      }
      T acc = T(0);
      int run = 0;
#pragma unroll
      for (int q = 0; q < kSlotChunk; ++q) {
        if (q >= m) break;
        const int s = __shfl_sync(0xffffffffu, my_s, q);
        const int prev = __shfl_sync(0xffffffffu, my_s, q > 0 ? q - 1 : 0);
        const int next = __shfl_sync(0xffffffffu, my_s, q + 1 < m ? q + 1 : q);
        const bool first = q == 0 || prev != s;
        if (first) run = q;
        acc = first ? v[q] : add_rn(acc, v[q]);
        if (q + 1 == m || next != s) {  // run ends
          const int64_t p = p0 + q;
          const bool whole = (run > 0 || key_before != s) && (q + 1 < m || key_after != s);
          if (j < N) {
            if (whole) {
              if (fused) {
                T* r = store + static_cast<int64_t>(s) * N + j;
                *r = sub_rn(*r, mul_rn(lr, acc));
              } else {
                sg[static_cast<int64_t>(s) * N + j] = acc;
              }
            } else {
              part[(p0 + run) * N + j] = acc;
            }
          }
          (void)p;
        }
      }
    }
  }
}


// Fold for the slots whose run spans chunk boundaries, found from the sorted
// keys themselves: boundary c (position c * kSlotChunk) starts a fold task iff
// the key there continues the previous chunk's last key and c is that key's
// FIRST crossed boundary.  One warp per boundary; a candidate warp folds all
// columns (lanes over the slot's chunk partials, fixed butterfly per column).
// Work scales with the number of chunks, not with the row count -- what the
// uncompressed tables (150k rows) need; the LFU cache uses it too.
template <typename T>
__global__ void k_slot_fold_runs(int64_t n, int N, const int* __restrict__ skey,
                                 const int* __restrict__ seg_lo, const int* __restrict__ seg_hi,
                                 const T* __restrict__ part, T* __restrict__ sg,
                                 T* __restrict__ store, int fused, T lr) {
  const int lane = threadIdx.x & 31;
  const int64_t nchunks = (n + kSlotChunk - 1) / kSlotChunk;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  // task = (boundary c, column j): a hot slot's columns fold in parallel
  for (int64_t task = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       task < (nchunks - 1) * N; task += nw) {
    const int64_t c = 1 + task / N;
    const int j = static_cast<int>(task - (c - 1) * N);
    const int64_t p = c * kSlotChunk;
    const int s = skey[p];
    if (skey[p - 1] != s) continue;
    const int lo = seg_lo[s], hi = seg_hi[s];
    if (lo / kSlotChunk != c - 1) continue;  // not the first boundary this slot crosses
    const int c_lo = lo / kSlotChunk, c_hi = (hi - 1) / kSlotChunk;
    {
      T acc = T(0);
      for (int cc = c_lo + lane; cc <= c_hi; cc += 32) {
        const int pp = cc == c_lo ? lo : cc * kSlotChunk;
        acc = add_rn(acc, part[static_cast<int64_t>(pp) * N + j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (lane == 0) {
        if (fused) {
          T* r = store + static_cast<int64_t>(s) * N + j;
          *r = sub_rn(*r, mul_rn(lr, acc));
        } else {
          sg[static_cast<int64_t>(s) * N + j] = acc;
        }
      }
    }
  }
}

// Slots whose sorted range spans chunks: add the chunk partials in order.
template <typename T>
__global__ void k_slot_fold(int64_t cap, int N, const int* __restrict__ seg_lo,
                            const int* __restrict__ seg_hi, const T* __restrict__ part,
                            T* __restrict__ sg, T* __restrict__ store, int fused, T lr) {
  // one warp per (slot, column): a hot slot's chunk partials (Zipf: the top
  // row's run spans hundreds of chunks) are summed lane-strided, then by a
  // fixed xor butterfly -- a fixed order for a given chunk count, so the
  // result is deterministic, and the chain is ~n/32 + 5 adds long
  const int lane = threadIdx.x & 31;
  const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t q = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
       q < cap * N; q += nw) {
    const int64_t s = q / N;
    const int j = static_cast<int>(q - s * N);
    const int lo = seg_lo[s], hi = seg_hi[s];
    if (lo < 0 || lo / kSlotChunk == (hi - 1) / kSlotChunk) continue;
    // partial rows: the run's first position, then every later chunk start
    const int c_lo = lo / kSlotChunk, c_hi = (hi - 1) / kSlotChunk;  // chunks c_lo..c_hi
    T acc = T(0);
    for (int c = c_lo + lane; c <= c_hi; c += 32) {
      const int p = c == c_lo ? lo : c * kSlotChunk;
      acc = add_rn(acc, part[static_cast<int64_t>(p) * N + j]);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = add_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) {
      if (fused) {
        T* r = store + s * N + j;
        *r = sub_rn(*r, mul_rn(lr, acc));
      } else {
        sg[q] = acc;
      }
    }
  }
}

// cached_sgd_update (lfu_cache.hpp:246-257) on the touched slots
template <typename T>
__global__ void k_slot_sgd(int64_t cap, int N, const int* __restrict__ seg_lo,
                           const T* __restrict__ sg, T* __restrict__ store, T lr) {
  const int64_t n = cap * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (seg_lo[q / N] < 0) continue;
    store[q] = sub_rn(store[q], mul_rn(lr, sg[q]));
  }
}

// caller-supplied SlotGradients (slots + rows): row -= T(lr)·g
template <typename T>
__global__ void k_rows_sgd(const int64_t* __restrict__ slots, int64_t n, int N,
                           const T* __restrict__ g, T* __restrict__ store, T lr) {
  const int64_t m = n * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < m;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = q / N;
    const int j = static_cast<int>(q - i * N);
    T* r = store + slots[i] * N + j;
    *r = sub_rn(*r, mul_rn(lr, g[q]));
  }
}

struct HasCount {
  const unsigned long long* c;
  __host__ __device__ bool operator()(const int64_t& r) const { return c[r] != 0ull; }
};

__global__ void k_gather_counts(const int64_t* __restrict__ rows, int64_t n,
                                const unsigned long long* __restrict__ counts,
                                unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = counts[rows[i]];
}

// admit (lfu_cache.hpp:266-296): row i of the new hot list keeps its trained
// value when it was resident, else takes the chain value (computed for the
// newly admitted rows only, compacted by an exclusive scan of `fresh`).
__global__ void k_admit_mark(const int64_t* __restrict__ rows, int64_t k,
                             const unsigned long long* __restrict__ okeys,
                             const int* __restrict__ ovals, int oshift, unsigned long long omask,
                             int have_old, int* __restrict__ old_slot, int* __restrict__ fresh) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = have_old ? probe(okeys, ovals, oshift, omask, static_cast<unsigned long long>(rows[i])) : -1;
    old_slot[i] = s;
    fresh[i] = s < 0 ? 1 : 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) fresh[k] = 0;
}

__global__ void k_admit_compact(const int64_t* __restrict__ rows, int64_t k,
                                const int* __restrict__ fresh, const int* __restrict__ fpos,
                                int64_t* __restrict__ new_rows) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (fresh[i]) new_rows[fpos[i]] = rows[i];
}

template <typename T>
__global__ void k_admit_fill(int64_t k, int64_t cap, int N, const int64_t* __restrict__ rows,
                             const int* __restrict__ old_slot, const int* __restrict__ fpos,
                             const T* __restrict__ chain, const T* __restrict__ old_store,
                             T* __restrict__ store, int64_t* __restrict__ slot_rows) {
  const int64_t n = cap * N;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = q / N;
    const int j = static_cast<int>(q - i * N);
    if (i >= k) {
      store[q] = T(0);
      if (j == 0) slot_rows[i] = -1;
      continue;
    }
    const int os = old_slot[i];
    store[q] = os >= 0 ? old_store[static_cast<int64_t>(os) * N + j]
                       : chain[static_cast<int64_t>(fpos[i]) * N + j];
    if (j == 0) slot_rows[i] = rows[i];
  }
}

// FreqTable::decay (lfu_cache.cpp:78-88): floor(count * factor)
__global__ void k_decay(unsigned long long* __restrict__ counts, int64_t n, double factor) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long c = counts[i];
    if (c) counts[i] = static_cast<unsigned long long>(floor(static_cast<double>(c) * factor));
  }
}

__global__ void k_count_nonzero(const unsigned long long* __restrict__ counts, int64_t n,
                                unsigned long long* __restrict__ out) {
  unsigned long long mine = 0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    mine += counts[i] != 0ull;
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, mine);
}

}  // namespace lfu
}  // namespace ttgpu
