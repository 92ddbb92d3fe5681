// ttrec_gpu_override.hpp -- route the reference's own operator names to the GPU.
//
// Explicit specialisations of ttrec::forward_bags / backward_bags / sgd_step /
// lookup_row (embedding_ops.hpp:120-376) for float and double that forward to
// ttrec::gpu:: (include/ttrec_gpu.hpp).  Force-included ahead of an unchanged
// reference translation unit (`-include ttrec_gpu_override.hpp`), every call
// that names those operators -- `forward_bags(t, batch)` in the reference's
// tests, model.hpp's EmbeddingLayer, LfuCache::admit's lookup_row -- runs on
// the GPU through the C ABI; ttrec::ref:: (the serial oracle) stays on the CPU.
#pragma once

#include "ttrec/embedding_ops.hpp"
#include "ttrec_gpu.hpp"

namespace ttrec {

#define TTREC_GPU_OVERRIDE(T)                                                               \
  template <>                                                                               \
  inline ForwardResult<T> forward_bags<T>(const TtTable<T>& table, const IndexBatch& batch, \
                                          index_t micro_batch, bool save_intermediates) {   \
    return gpu::forward_bags<T>(table, batch, micro_batch, save_intermediates);             \
  }                                                                                         \
  template <>                                                                               \
  inline CoreGradients<T> backward_bags<T>(const TtTable<T>& table, const IndexBatch& batch,  \
                                           const ForwardContext<T>& ctx,                    \
                                           std::span<const T> grad_output) {                \
    return gpu::backward_bags<T>(table, batch, ctx, grad_output);                           \
  }                                                                                         \
  template <>                                                                               \
  inline void sgd_step<T>(TtTable<T>& table, const CoreGradients<T>& grads, double lr) {    \
    gpu::sgd_step<T>(table, grads, lr);                                                     \
  }                                                                                         \
  template <>                                                                               \
  inline void lookup_row<T>(const TtTable<T>& table, index_t row, std::span<T> out) {       \
    gpu::lookup_row<T>(table, row, out);                                                    \
  }                                                                                         \
  template <>                                                                               \
  inline std::vector<T> lookup_row<T>(const TtTable<T>& table, index_t row) {               \
    return gpu::lookup_row<T>(table, row);                                                  \
  }

TTREC_GPU_OVERRIDE(float)
TTREC_GPU_OVERRIDE(double)
#undef TTREC_GPU_OVERRIDE

}  // namespace ttrec
