// Fused cross-GPU gradient reduction + SGD over peer memory.
//
// The multi-GPU step is: per-rank backward_bags on its bag shard (dense core
// gradient in the table's buffer) -> allreduce(SUM) -> identical sgd_step on
// every replica (embedding_ops.hpp:355-376).  ttgpu_peer_reduce_sgd does the
// last two in ONE kernel, as a reduce-scatter + all-gather over NVLink:
//   rank q owns the shard [q*per, (q+1)*per) of the flat core vector; it reads
//   that shard of every rank's gradient buffer (16-byte P2P loads, all ranks'
//   loads in flight at once), sums them in rank order, applies
//   core -= T(lr) * g, and stores the new values into its own cores AND every
//   peer's cores (P2P stores through the CUDA IPC mappings).
// Each element is reduced by exactly one rank in a fixed order and the result
// is copied everywhere, so the replicas stay bitwise equal.  Per rank and call
// the NVLink traffic is 2 (W-1)/W of the core bytes (about 3.5 MB at W = 8 for
// the 1.98 MB cfg2 table) instead of (W-1) times them for all-to-all reads.
// No NCCL launch, no separate SGD kernel, no intermediate reduced buffer.
//
// Synchronisation, per call (epoch e = previous + 1, kept on the device so the
// kernel is CUDA-graph replayable):
//   start   CTA 0 of rank q writes ready[q] = e into every rank's flag block
//           (release, system scope); every CTA waits until its own block has
//           ready[r] >= e for all r (acquire) -- all gradients are final and
//           no rank still reads its cores for this step's backward;
//   body    the shard: reduce in rank order + SGD + push to every replica;
//   finish  every CTA fences its P2P stores (system scope); the last CTA to
//           finish writes done[q] = e everywhere, then waits for done[r] >= e
//           from all ranks -- every replica's cores are complete and no
//           rank's next backward can overwrite a gradient a peer still reads;
//           it commits e.
// Spins are bounded (~seconds): a missing peer latches an error that the next
// ttgpu_check() reports instead of hanging the GPU.
namespace ttgpu {
namespace {

constexpr int kMaxPeers = 8;
// flag block (uint32): [0, 8) ready epochs by rank, [8, 16) done epochs by rank,
// [16] committed epoch, [17] CTA arrival counter, [18] timeout flag
constexpr int kFlagWords = 64;

template <typename T>
struct PeerPtrs {
  const T* grads[kMaxPeers];
  T* cores[kMaxPeers];
  unsigned* flags[kMaxPeers];
};

template <typename T> struct Vec;
template <> struct Vec<float> { using V = float4; static constexpr int n = 4; };
template <> struct Vec<double> { using V = double2; static constexpr int n = 2; };

__device__ __forceinline__ void vadd(float4& a, const float4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}
__device__ __forceinline__ void vadd(double2& a, const double2& b) {
  a.x += b.x; a.y += b.y;
}
__device__ __forceinline__ float4 vsgd(float4 c, float4 g, float step) {
  return make_float4(__fadd_rn(c.x, -__fmul_rn(step, g.x)), __fadd_rn(c.y, -__fmul_rn(step, g.y)),
                     __fadd_rn(c.z, -__fmul_rn(step, g.z)), __fadd_rn(c.w, -__fmul_rn(step, g.w)));
}
__device__ __forceinline__ double2 vsgd(double2 c, double2 g, double step) {
  return make_double2(__dadd_rn(c.x, -__dmul_rn(step, g.x)), __dadd_rn(c.y, -__dmul_rn(step, g.y)));
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// wait until every rank's word at `slot` reached `epoch`; false on timeout
__device__ __forceinline__ bool wait_all(const unsigned* own, int slot0, int world, unsigned epoch) {
  for (int r = 0; r < world; ++r) {
    long long spins = 0;
    while (static_cast<int>(ld_acquire_sys(own + slot0 + r) - epoch) < 0) {
      __nanosleep(64);
      if (++spins > (1ll << 26)) return false;
    }
  }
  return true;
}

// shard of rank q: [q * per, min(n, (q + 1) * per)), per a multiple of 4 elements
__host__ __device__ inline int64_t peer_shard(int64_t n, int world) {
  return ((n + world - 1) / world + 3) / 4 * 4;
}

template <typename T>
__global__ void __launch_bounds__(256) k_peer_reduce_sgd(PeerPtrs<T> pp, int world, int rank, int64_t n,
                                                         T step, unsigned* own) {
  using V = typename Vec<T>::V;
  constexpr int NV = Vec<T>::n;
  __shared__ unsigned epoch_s;
  __shared__ int ok_s;
  if (threadIdx.x == 0) {
    const unsigned epoch = *reinterpret_cast<volatile unsigned*>(own + 16) + 1u;
    epoch_s = epoch;
    if (blockIdx.x == 0) {
      __threadfence_system();  // this rank's gradient (previous kernels) before the flag
      for (int r = 0; r < world; ++r) st_release_sys(pp.flags[r] + rank, epoch);
    }
    const bool ok = wait_all(own, 0, world, epoch);
    if (!ok) atomicExch(own + 18, 1u);
    ok_s = ok;
  }
  __syncthreads();
  const unsigned epoch = epoch_s;
  if (ok_s) {
    const int64_t per = peer_shard(n, world);
    const int64_t lo = rank * per, hi = lo + per < n ? lo + per : n;
    for (int64_t e = lo + (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) * NV; e < hi;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x * NV) {
      V g[kMaxPeers];
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r)  // every rank's load in flight
        if (r < world) g[r] = __ldcg(reinterpret_cast<const V*>(pp.grads[r] + e));
      V sum = g[0];
#pragma unroll
      for (int r = 1; r < kMaxPeers; ++r)
        if (r < world) vadd(sum, g[r]);  // rank order everywhere
      const V c = vsgd(*reinterpret_cast<const V*>(pp.cores[rank] + e), sum, step);
#pragma unroll
      for (int r = 0; r < kMaxPeers; ++r)
        if (r < world) __stcg(reinterpret_cast<V*>(pp.cores[r] + e), c);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();  // this CTA's P2P core stores before it counts as done
    const unsigned prev = atomicAdd(own + 17, 1u);
    if (prev == gridDim.x - 1) {  // last CTA of this rank
      own[17] = 0u;
      __threadfence_system();
      for (int r = 0; r < world; ++r) st_release_sys(pp.flags[r] + 8 + rank, epoch);
      if (!wait_all(own, 8, world, epoch)) atomicExch(own + 18, 1u);
      *reinterpret_cast<volatile unsigned*>(own + 16) = epoch;
    }
  }
}

}  // namespace
}  // namespace ttgpu

struct ttgpu_peers {
  int world = 0, rank = 0;
  std::vector<void*> grads, cores, flags;  // per rank (own entries are the table's buffers)
  std::vector<void*> opened;        // IPC mappings to close
  ~ttgpu_peers() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
  }
};

namespace ttgpu {
namespace {
unsigned* peer_flags(ttgpu_table* t) {
  if (!t->peer_flag_buf.p) {
    t->peer_flag_buf.ensure(sizeof(unsigned) * kFlagWords);
    CK(cudaMemset(t->peer_flag_buf.p, 0, sizeof(unsigned) * kFlagWords));
  }
  return t->peer_flag_buf.as<unsigned>();
}
}  // namespace
}  // namespace ttgpu

extern "C" {

int ttgpu_peer_flags_ptr(ttgpu_table* t, void** out) {
  return guarded([&] { *out = ttgpu::peer_flags(t); });
}

int ttgpu_peer_export(ttgpu_table* t, void* grad_handle, void* core_handle, void* flags_handle) {
  return guarded([&] {
    ttgpu::peer_flags(t);
    CK(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(grad_handle), t->grads.p));
    CK(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(core_handle), t->cores.p));
    CK(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(flags_handle), t->peer_flag_buf.p));
  });
}

static void attach_common(ttgpu_table* t, int world, int rank) {
  require_arg(world >= 1 && world <= ttgpu::kMaxPeers,
              cat("peer reduce supports 1..", ttgpu::kMaxPeers, " ranks, got ", world));
  require_arg(rank >= 0 && rank < world, cat("rank ", rank, " outside world ", world));
  require_arg(t->dtype == TTGPU_F32 || t->dtype == TTGPU_F64, "bad dtype");
  delete t->peers;
  t->peers = new ttgpu_peers;
  t->peers->world = world;
  t->peers->rank = rank;
  t->peers->grads.assign(world, nullptr);
  t->peers->cores.assign(world, nullptr);
  t->peers->flags.assign(world, nullptr);
}

int ttgpu_peer_attach(ttgpu_table* t, int world, int rank, const void* grad_handles,
                      const void* core_handles, const void* flags_handles) {
  return guarded([&] {
    attach_common(t, world, rank);
    const auto* gh = static_cast<const cudaIpcMemHandle_t*>(grad_handles);
    const auto* ch = static_cast<const cudaIpcMemHandle_t*>(core_handles);
    const auto* fh = static_cast<const cudaIpcMemHandle_t*>(flags_handles);
    for (int r = 0; r < world; ++r) {
      if (r == rank) {
        t->peers->grads[r] = t->grads.p;
        t->peers->cores[r] = t->cores.p;
        t->peers->flags[r] = ttgpu::peer_flags(t);
        continue;
      }
      void* g = nullptr;
      void* c = nullptr;
      void* f = nullptr;
      CK(cudaIpcOpenMemHandle(&g, gh[r], cudaIpcMemLazyEnablePeerAccess));
      t->peers->opened.push_back(g);
      CK(cudaIpcOpenMemHandle(&c, ch[r], cudaIpcMemLazyEnablePeerAccess));
      t->peers->opened.push_back(c);
      CK(cudaIpcOpenMemHandle(&f, fh[r], cudaIpcMemLazyEnablePeerAccess));
      t->peers->opened.push_back(f);
      t->peers->grads[r] = g;
      t->peers->cores[r] = c;
      t->peers->flags[r] = f;
    }
  });
}

int ttgpu_peer_attach_ptrs(ttgpu_table* t, int world, int rank, void* const* grad_ptrs,
                           void* const* core_ptrs, void* const* flag_ptrs) {
  return guarded([&] {
    attach_common(t, world, rank);
    for (int r = 0; r < world; ++r) {
      t->peers->grads[r] = r == rank ? t->grads.p : grad_ptrs[r];
      t->peers->cores[r] = r == rank ? t->cores.p : core_ptrs[r];
      t->peers->flags[r] = r == rank ? static_cast<void*>(ttgpu::peer_flags(t)) : flag_ptrs[r];
      require_arg(t->peers->grads[r] && t->peers->cores[r] && t->peers->flags[r],
                  cat("missing buffers of rank ", r));
    }
  });
}

int ttgpu_peer_reduce_sgd(ttgpu_table* t, double lr) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(t->peers != nullptr, "peer reduce needs ttgpu_peer_attach first");
    const ttgpu_peers& P = *t->peers;
    // at most half the SMs: two ranks sharing one GPU (tests) must be co-resident
    const int64_t n = t->total;
    const int64_t shard = peer_shard(n, P.world);
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>((shard + 1023) / 1024, std::max(1, t->num_sms / 2))));
    if (t->dtype == TTGPU_F64) {
      PeerPtrs<double> pp{};
      for (int r = 0; r < P.world; ++r) {
        pp.grads[r] = static_cast<const double*>(P.grads[r]);
        pp.cores[r] = static_cast<double*>(P.cores[r]);
        pp.flags[r] = static_cast<unsigned*>(P.flags[r]);
      }
      k_peer_reduce_sgd<double><<<grid, 256, 0, t->stream>>>(pp, P.world, P.rank, n, lr, peer_flags(t));
    } else {
      PeerPtrs<float> pp{};
      for (int r = 0; r < P.world; ++r) {
        pp.grads[r] = static_cast<const float*>(P.grads[r]);
        pp.cores[r] = static_cast<float*>(P.cores[r]);
        pp.flags[r] = static_cast<unsigned*>(P.flags[r]);
      }
      k_peer_reduce_sgd<float><<<grid, 256, 0, t->stream>>>(pp, P.world, P.rank, n,
                                                             static_cast<float>(lr), peer_flags(t));
    }
    CK(cudaGetLastError());
    ++t->generation;
  });
}

// 1 if a peer reduce timed out waiting for a rank (flag cleared on read)
int ttgpu_peer_status(ttgpu_table* t, int* timed_out) {
  return guarded([&] {
    unsigned v = 0;
    CK(cudaStreamSynchronize(t->stream));
    CK(cudaMemcpy(&v, ttgpu::peer_flags(t) + 18, sizeof(v), cudaMemcpyDeviceToHost));
    if (v) CK(cudaMemset(ttgpu::peer_flags(t) + 18, 0, sizeof(v)));
    *timed_out = v ? 1 : 0;
  });
}

}  // extern "C"
