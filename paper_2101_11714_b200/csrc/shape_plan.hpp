// Host-side shape planning for TT-compressed tables.
//
// Mirrors the reference's ShapePlan / plan_shapes contract
// (/root/reference/proj/include/ttrec/shape_plan.hpp:19-67,
//  src/shape_plan.cpp:98-198): same factor choices, rank clipping,
// parameter counts, memory-reduction rounding and error types, so that a
// plan built here is interchangeable with one built by the reference.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace ttgpu {

using index_t = std::int64_t;

inline constexpr int kMinTtDim = 2;
inline constexpr int kMaxTtDim = 8;

struct ShapePlan {
  index_t num_rows = 0;
  index_t emb_dim = 0;
  int tt_dim = 0;
  std::vector<index_t> row_factors;  // m_k
  std::vector<index_t> col_factors;  // n_k
  std::vector<index_t> ranks;        // R_0..R_d, R_0 = R_d = 1

  index_t padded_rows() const;
  index_t core_size(int k) const;        // R_{k-1} m_k n_k R_k
  index_t slice_size(int k) const;       // R_{k-1} n_k R_k
  index_t parameter_count() const;
  index_t memory_reduction() const;
  void validate() const;                 // throws std::invalid_argument
};

ShapePlan plan_shapes(index_t num_rows, index_t emb_dim, int tt_dim, index_t rank,
                      const index_t* row_factors /*nullable*/,
                      const index_t* col_factors /*nullable*/);

std::vector<index_t> decompose_index(index_t flat, const index_t* radices, int n);
index_t recompose_index(const index_t* digits, const index_t* radices, int n);

}  // namespace ttgpu
