// Device index-stream producer: Zipf(s) / uniform row
// indices drawn on the GPU for throughput runs, so large batches (cfg3: 2M
// lookups per step) are not bound by host generation.
//
// Same distribution as the reference's ZipfianSampler (data.cpp:8-33): the
// CDF is built on the host with the reference's exact loop (acc += (r+1)^-s,
// normalised, last entry forced to 1.0 -- the same code ttgpu_zipf_batch uses
// and that tests pin byte-for-byte against the reference stream), uploaded
// once, and inverted with upper_bound on the device.  The uniform variates
// come from a counter-based SplitMix64 stream (element i of a draw uses
// counter + i), NOT from the reference's mt19937_64: device streams are for
// throughput only; parity runs keep host-generated inputs (§8(c)).
namespace ttgpu {
namespace {

__device__ __forceinline__ uint64_t d_splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// one draw per element; exponent 0 (uniform) skips the CDF: floor(u64 * n / 2^64)
__global__ void k_sample_rows(const double* __restrict__ cdf, int64_t population, uint64_t key,
                              uint64_t counter, int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t h = d_splitmix(key + (counter + static_cast<uint64_t>(i)) * 0xD1B54A32D192ED03ull);
    int64_t r;
    if (cdf == nullptr) {
      r = static_cast<int64_t>(__umul64hi(h, static_cast<uint64_t>(population)));
    } else {
      const double u = static_cast<double>(h >> 11) * 0x1.0p-53;  // [0, 1)
      int64_t lo = 0, hi = population;                            // upper_bound(cdf, u)
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(cdf + mid) <= u) lo = mid + 1; else hi = mid;
      }
      r = lo < population ? lo : population - 1;
    }
    out[i] = r;
  }
}

__global__ void k_bag_offsets(int64_t bags, int64_t pf, int64_t* __restrict__ off) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b <= bags;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x)
    off[b] = b * pf;
}

}  // namespace
}  // namespace ttgpu

struct ttgpu_sampler {
  int64_t population = 0;
  double exponent = 0;
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  ttgpu::DevBuf cdf;  // empty for exponent 0
  bool uniform = true;
};

extern "C" {

int ttgpu_sampler_create(int64_t population, double exponent, int device, void* stream,
                         ttgpu_sampler** out) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(population >= 1, cat("population must be positive, got ", population));
    require_arg(exponent >= 0, cat("exponent must be non-negative, got ", exponent));
    CK(cudaSetDevice(device));
    auto s = std::make_unique<ttgpu_sampler>();
    s->population = population;
    s->exponent = exponent;
    s->device = device;
    s->stream = static_cast<cudaStream_t>(stream);
    cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, device);
    s->uniform = exponent == 0.0;
    if (!s->uniform) {
      std::vector<double> cdf(population);  // ZipfianSampler::ZipfianSampler (data.cpp:8-20)
      double acc = 0.0;
      for (int64_t r = 0; r < population; ++r) {
        acc += std::pow(static_cast<double>(r + 1), -exponent);
        cdf[r] = acc;
      }
      const double inv = 1.0 / acc;
      for (double& c : cdf) c *= inv;
      cdf.back() = 1.0;
      s->cdf.ensure(sizeof(double) * population);
      CK(cudaMemcpyAsync(s->cdf.p, cdf.data(), sizeof(double) * population,
                         cudaMemcpyHostToDevice, s->stream));
      CK(cudaStreamSynchronize(s->stream));
    }
    *out = s.release();
  });
}

int ttgpu_sampler_destroy(ttgpu_sampler* s) {
  return guarded([&] {
    if (s) cudaStreamSynchronize(s->stream);
    delete s;
  });
}

int ttgpu_sampler_set_stream(ttgpu_sampler* s, void* stream) {
  return guarded([&] { s->stream = static_cast<cudaStream_t>(stream); });
}

int ttgpu_sampler_draw_device(ttgpu_sampler* s, uint64_t seed, uint64_t counter, int64_t n,
                              int64_t* d_out) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(n >= 0, "negative draw count");
    if (n == 0) return;
    const int grid = grid_for(n, 256, s->num_sms, 8);
    k_sample_rows<<<grid, 256, 0, s->stream>>>(s->uniform ? nullptr : s->cdf.as<double>(),
                                               s->population, splitmix(seed), counter, n, d_out);
    CK(cudaGetLastError());
  });
}

int ttgpu_bag_offsets_device(int64_t bags, int64_t pooling_factor, int64_t* d_offsets,
                             void* stream) {
  using namespace ttgpu;
  return guarded([&] {
    require_arg(bags >= 0, "num_bags must be non-negative");
    require_arg(pooling_factor >= 1, cat("pooling_factor must be >= 1, got ", pooling_factor));
    k_bag_offsets<<<grid_for(bags + 1, 256, 148, 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        bags, pooling_factor, d_offsets);
    CK(cudaGetLastError());
  });
}

}  // extern "C"
