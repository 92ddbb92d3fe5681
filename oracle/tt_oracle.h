/* TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TT-EmbeddingBag path.
 *
 * A plain-C restatement of the reference's serial algorithm
 * (/root/reference/proj/include/ttrec/embedding_ops.hpp ref::forward_bags
 * :382-423, ref::backward_bags :426-490, sgd_step :361-376, lookup_row
 * :120-152, tt_table.hpp decompose_row :71-78).  Only tests/, smoke() and
 * bench.py's cpu_baseline leg may load it; the product path never does.
 *
 * Pinned against the reference itself: tests/test_oracle.py checks this
 * library bit-for-bit against oracle/_ref/libttref.so (the reference compiled
 * from its own sources) and against the committed fixtures in tests/golden/.
 *
 * A "plan" is passed as (d, num_rows, emb_dim, row_factors[d],
 * col_factors[d], ranks[d+1]); cores[k] points at core k in the reference
 * physical layout (m_k, R_{k-1}, n_k, R_k) row-major.
 */
#ifndef TT_ORACLE_H
#define TT_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mixed-radix digits of a flat row, most-significant first. */
void tto_decompose_row(int64_t flat, int d, const int64_t* row_factors, int64_t* digits);

/* Returns 0 ok, 2 invalid batch structure, 3 index out of range (first bad lookup in *bad). */
int tto_validate(int64_t num_rows, const int64_t* idx, int64_t L, const int64_t* off,
                 int64_t B, int64_t* bad);

int tto_forward_f32(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                    const int64_t* rk, const float* const* cores, const int64_t* idx, int64_t L,
                    const int64_t* off, int64_t B, const double* w, int pooling, float* out);
int tto_forward_f64(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                    const int64_t* rk, const double* const* cores, const int64_t* idx, int64_t L,
                    const int64_t* off, int64_t B, const double* w, int pooling, double* out);

/* grads[k] is zero-filled by the callee and receives the dense core-k gradient. */
int tto_backward_f32(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                     const int64_t* rk, const float* const* cores, const int64_t* idx,
                     int64_t L, const int64_t* off, int64_t B, const double* w, int pooling,
                     const float* grad_out, float* const* grads);
int tto_backward_f64(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                     const int64_t* rk, const double* const* cores, const int64_t* idx,
                     int64_t L, const int64_t* off, int64_t B, const double* w, int pooling,
                     const double* grad_out, double* const* grads);

void tto_sgd_f32(int d, const int64_t* rf, const int64_t* cf, const int64_t* rk, float* const* cores,
                 const float* const* grads, double lr);
void tto_sgd_f64(int d, const int64_t* rf, const int64_t* cf, const int64_t* rk, double* const* cores,
                 const double* const* grads, double lr);

int tto_lookup_row_f32(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                       const int64_t* rk, const float* const* cores, int64_t row, float* out);
int tto_lookup_row_f64(int d, int64_t num_rows, int64_t emb, const int64_t* rf, const int64_t* cf,
                       const int64_t* rk, const double* const* cores, int64_t row, double* out);

/* Multi-threaded (OpenMP over bag ranges, per-worker dense grads merged in
 * worker order -- embedding_ops.hpp:187-191,280-287,355-357) fp32 step used as
 * the "port" CPU baseline when oracle/_ref is unavailable.  Returns seconds. */
double tto_time_step_f32(int d, int64_t num_rows, int64_t emb, const int64_t* rf,
                         const int64_t* cf, const int64_t* rk, float* const* cores,
                         const int64_t* idx, int64_t L, const int64_t* off, int64_t B,
                         const float* grad_out, double lr, int threads);

#ifdef __cplusplus
}
#endif
#endif
