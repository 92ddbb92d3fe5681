/*
 * ttgpu.h -- C ABI of the B200-native TT-EmbeddingBag (libttgpu.so).
 *
 * Drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/ttrec/embedding_ops.hpp).  The reference has
 * no C ABI (header-only C++ templates over TtTable<T> + IndexBatch); each
 * entry point below names the reference interface it replaces.  Plain
 * pointers and sizes only -- no torch or C++ types cross this boundary.
 *
 * Conventions
 *  - Status codes mirror the reference's exception types:
 *      TTGPU_OK 0, TTGPU_ERR_RUNTIME 1 (std::runtime_error),
 *      TTGPU_ERR_INVALID_ARGUMENT 2 (std::invalid_argument),
 *      TTGPU_ERR_OUT_OF_RANGE 3 (std::out_of_range).
 *    ttgpu_last_error() returns the thread-local message, worded like the
 *    reference's (table names, "stale", ...), so a C++ or Python wrapper can
 *    re-throw the same type with the same text.
 *  - Core layout is the reference's physical layout (tt_table.hpp:19-22):
 *    core k is (m_k, R_{k-1}, n_k, R_k) row-major, byte-identical to
 *    TtTable<T>::core(k).
 *  - "host" entry points take host pointers, copy in/out and synchronise
 *    before returning (value semantics, like the reference).  "_device"
 *    entry points take device pointers and are asynchronous on the table's
 *    stream (graph-capturable); data-dependent validation errors (index out
 *    of range, malformed offsets) are latched on the device and reported by
 *    the next ttgpu_check() / host call.
 *  - dtype: TTGPU_F32 or TTGPU_F64 (the reference instantiates float and
 *    double, common.hpp:13-15).  pooling: TTGPU_SUM / TTGPU_MEAN
 *    (index_batch.hpp:10).
 */
#ifndef TTGPU_H
#define TTGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TTGPU_OK = 0, TTGPU_ERR_RUNTIME = 1, TTGPU_ERR_INVALID_ARGUMENT = 2,
       TTGPU_ERR_OUT_OF_RANGE = 3 };
enum { TTGPU_F32 = 0, TTGPU_F64 = 1 };
enum { TTGPU_SUM = 0, TTGPU_MEAN = 1 };

typedef struct ttgpu_table ttgpu_table; /* TtTable<T> resident on one GPU */
typedef struct ttgpu_ctx ttgpu_ctx;     /* ForwardContext<T> (embedding_ops.hpp:101-110) */
typedef struct ttgpu_cache ttgpu_cache; /* LfuCache<T> (lfu_cache.hpp:134-310) */

const char* ttgpu_last_error(void);
int ttgpu_abi_version(void);

/* ---- shape planning: shape_plan.hpp:19-67 / src/shape_plan.cpp -------- */
/* plan_shapes (shape_plan.hpp:56-58).  rf_in / cf_in may be NULL (auto). */
int ttgpu_plan_shapes(int64_t num_rows, int64_t emb_dim, int tt_dim, int64_t rank,
                      const int64_t* rf_in, const int64_t* cf_in, int64_t* rf_out,
                      int64_t* cf_out, int64_t* ranks_out);
/* ShapePlan::validate / padded_rows / parameter_count / memory_reduction (:28-43) */
int ttgpu_plan_info(int64_t num_rows, int64_t emb_dim, int tt_dim, const int64_t* rf,
                    const int64_t* cf, const int64_t* ranks, int64_t* padded_rows,
                    int64_t* parameter_count, int64_t* memory_reduction);
/* decompose_index / recompose_index (shape_plan.hpp:60-66) */
int ttgpu_decompose_index(int64_t flat, const int64_t* radices, int n, int64_t* digits);
int ttgpu_recompose_index(const int64_t* digits, const int64_t* radices, int n, int64_t* flat);

/* ---- tables: TtTable<T> (tt_table.hpp:23-102) -------------------------- */
/* TtTable(ShapePlan, name) (tt_table.hpp:25-33); cores zero-initialised.
 * stream: a cudaStream_t (NULL = legacy default stream). */
int ttgpu_create(int64_t num_rows, int64_t emb_dim, int tt_dim, const int64_t* row_factors,
                 const int64_t* col_factors, const int64_t* ranks, int dtype, const char* name,
                 int device, void* stream, ttgpu_table** out);
int ttgpu_destroy(ttgpu_table* t);
int ttgpu_set_stream(ttgpu_table* t, void* stream);
int ttgpu_core_size(const ttgpu_table* t, int k, int64_t* n);
/* TtTable::core(k) read / write as raw bytes (tt_table.hpp:43-44).  A write
 * bumps the mutation counter (tt_table.hpp:82-85) like init / sgd_step. */
int ttgpu_get_core(ttgpu_table* t, int k, void* host_dst);
/* copy of core k's slice of the table's dense gradient buffer (the last
 * non-fused backward's CoreGradients::core(k)) */
int ttgpu_get_grad(ttgpu_table* t, int k, void* host_dst);
int ttgpu_set_core(ttgpu_table* t, int k, const void* host_src);
int ttgpu_core_device_ptr(ttgpu_table* t, int k, void** dptr);
int ttgpu_mark_mutated(ttgpu_table* t);                        /* tt_table.hpp:85 */
/* on (default): forward products and sums separately rounded in the
 * reference's loop order -> forward_bags / lookup_row bit-identical to the
 * reference (gemm.hpp:15-31, embedding_ops.hpp:232-249).  off: FFMA. */
int ttgpu_set_exact_forward(ttgpu_table* t, int on);
/* 3-core float tables with a compiled shape use the specialised fast path
 * (kind >= 0); on=1 forces the generic pipeline instead (used by tests to
 * cross-check the two implementations). */
/* Backward contractions on the tcgen05 tensor cores (error-compensated
 * 3xTF32, fp32 accumulation) where the shape allows it (1 = default) or on the
 * FP32 FFMA path (0).  Forward results never depend on it; gradients differ
 * within the 1e-4 tolerance.  No reference counterpart (the reference is CPU
 * only, embedding_ops.hpp:335-347). */
int ttgpu_set_tensor_path(ttgpu_table* t, int on);
/* Fast path: sort the batch with the one-kernel cooperative sort (gsort.cuh) (1 = default,
 * used when the batch fits one co-resident grid) or with the three-kernel
 * histogram / scan / scatter sort (0).  Results never depend on it. */
int ttgpu_set_grid_sort(ttgpu_table* t, int on);
/* Fast path: chunked kernels (1: per-bucket chunks of 64 lookups, CTA-wide
 * i0 dedup, fused S / dG1 / D0 backward; fastc.cuh) or the one-warp
 * 32-lookup tile kernels (0 = default; measured faster at cfg2).  Forward
 * outputs are bit-identical either way; gradients agree within 1e-4. */
int ttgpu_set_chunked(ttgpu_table* t, int on);
int ttgpu_set_generic_path(ttgpu_table* t, int on);
/* d == 3 wide-row tables (cfg3's shape class: fp32, n0·n1 = 16, R2 = 64,
 * n2 = 4): warp-per-chunk tail kernels with register-resident operands
 * (1 = default, wide3.cuh) or the shared-memory staged kernels (0).  Forward
 * outputs are bit-identical either way; gradients agree within 1e-4. */
int ttgpu_set_wide3(ttgpu_table* t, int on);
int ttgpu_fast_path_kind(const ttgpu_table* t, int* kind);
int ttgpu_mutation_counter(const ttgpu_table* t, uint64_t* out); /* tt_table.hpp:84 */

/* ---- forward_bags (embedding_ops.hpp:159-253) ---------------------------- */
int ttgpu_ctx_create(ttgpu_table* t, ttgpu_ctx** out);
int ttgpu_ctx_destroy(ttgpu_ctx* c);
/* Host pointers; out is (B x emb_dim) row-major.  weights may be NULL (all
 * ones, index_batch.hpp:24).  micro_batch must be >= 1 (:165) but does not
 * change results (:155-158).  save keeps the per-lookup chain partials for
 * backward (:181-185); backward results are identical either way. */
int ttgpu_forward(ttgpu_table* t, const int64_t* indices, int64_t L, const int64_t* offsets,
                  int64_t B, const double* weights, int pooling, int64_t micro_batch, int save,
                  void* out, ttgpu_ctx* ctx);
int ttgpu_forward_device(ttgpu_table* t, const int64_t* d_indices, int64_t L,
                         const int64_t* d_offsets, int64_t B, const double* d_weights,
                         int pooling, int save, void* d_out, ttgpu_ctx* ctx);

/* ---- backward_bags (embedding_ops.hpp:260-358) --------------------------- */
/* Checks the reference's contract (:264-274): context table identity,
 * L/B match, stale mutation snapshot, grad size == B*emb_dim.  Writes the
 * dense CoreGradients into the table's gradient buffer; grads_out (host
 * pointers, one per core, each core_size elements) may be NULL. */
int ttgpu_backward(ttgpu_table* t, ttgpu_ctx* ctx, int64_t L, int64_t B, const void* grad_out,
                   int64_t grad_len, void* const* grads_out);
/* device variant; the dense gradient stays in the table's gradient buffer
 * (ttgpu_grad_device_ptr), e.g. for an NCCL allreduce before ttgpu_apply_grad */
int ttgpu_backward_device(ttgpu_table* t, ttgpu_ctx* ctx, const void* d_grad_out);
int ttgpu_grad_device_ptr(ttgpu_table* t, int k, void** dptr);

/* ---- sgd_step (embedding_ops.hpp:361-376) -------------------------------- */
/* sgd_step(table, grads, lr) with caller gradients (host, one per core) */
int ttgpu_sgd_step(ttgpu_table* t, const void* const* host_grads, double lr);
/* host variant of the fused call: copies grad_out in, synchronises */
int ttgpu_backward_sgd(ttgpu_table* t, ttgpu_ctx* ctx, int64_t L, int64_t B, const void* grad_out,
                       int64_t grad_len, double lr);
/* the whole dense gradient buffer (all cores, aligned offsets, padding zero) */
int ttgpu_grad_buffer(ttgpu_table* t, void** dptr, int64_t* n_elems);
/* core -= lr * (table gradient buffer); async */
int ttgpu_apply_grad(ttgpu_table* t, double lr);
/* fused backward_bags + sgd_step: gradients are reduced per touched core
 * slice and applied in the reduction epilogue (no dense gradient); async */
int ttgpu_backward_sgd_device(ttgpu_table* t, ttgpu_ctx* ctx, const void* d_grad_out,
                              double lr);

/* ---- lookup_row (embedding_ops.hpp:120-152) ------------------------------ */
int ttgpu_lookup_row(ttgpu_table* t, int64_t row, void* host_out);
int ttgpu_lookup_rows_device(ttgpu_table* t, const int64_t* d_rows, int64_t n, void* d_out);

/* ---- CUDA graphs: capture any sequence of _device calls on the table's
 * (non-default) stream, then replay it with one launch ------------------- */
int ttgpu_graph_begin(ttgpu_table* t);
int ttgpu_graph_end(ttgpu_table* t, int* kernel_nodes, int* total_nodes);
int ttgpu_graph_launch(ttgpu_table* t);

/* ---- synchronisation / deferred device errors ----------------------------- */
int ttgpu_sync(ttgpu_table* t);
int ttgpu_check(ttgpu_table* t); /* sync + report latched validation errors */

/* ---- instrumentation (no reference counterpart; diagnostics only) ------- */
/* on: record CUDA events between pipeline phases on the table's stream;
 * read: per-phase milliseconds since the last read ("decode;sort_pairs;...").
 * Marks recorded while a graph is being captured (profile on before
 * ttgpu_graph_begin) become event nodes of that graph: read after each
 * ttgpu_graph_launch gives that launch's per-kernel times. */
int ttgpu_profile(ttgpu_table* t, int on);
int ttgpu_profile_read(ttgpu_table* t, char* names, int64_t names_len, float* ms, int max_phases,
                       int* n_out);

/* ---- LFU cache of hot uncompressed rows (lfu_cache.hpp:18-310,
 * lfu_cache.cpp:15-126) and the cached EmbeddingLayer (model.hpp:195-284).
 * Frequencies are dense per-row counters over [0, key_space) (the table's
 * row count); a small GPU hash table (row -> slot) is probed for every lookup
 * before any decompression.  Host entry points synchronise; the _device
 * layer calls run on the table's stream (one host sync per forward reads the
 * size of the chain part). --------------------------------------------- */
int ttgpu_cache_create(int64_t capacity, int64_t emb_dim, int64_t refresh_period,
                       int64_t key_space, int dtype, int device, void* stream, ttgpu_cache** out);
int ttgpu_cache_destroy(ttgpu_cache* c);
int ttgpu_cache_set_stream(ttgpu_cache* c, void* stream);
/* Fast path (default on): for fp32 3-core tables with a compiled fast-path
 * shape, the cached forward consults the cache inside the fast-path sort
 * (record + probe + slot counting sort in one kernel, no host sync, CUDA-graph
 * capturable).  enable = 0 forces the partition path (record_and_partition +
 * forward_bags(part.tt) + combine, lfu_cache.hpp:187-219 / model.hpp:210-223). */
int ttgpu_cache_set_fast(ttgpu_cache* c, int enable);
/* sizes of the last cached forward's partition (syncs on the fast path), its
 * bag count, whether it had weights and its original pooling (any may be NULL) */
int ttgpu_cache_last_counts(ttgpu_cache* c, int64_t* n_cached, int64_t* n_tt, int64_t* bags,
                            int* has_weights, int* pooling);
int64_t ttgpu_cache_default_capacity(int64_t table_rows);              /* :146-148 */
/* state() / resident_count() / active_accesses() / active_hits() (:150-160, 259-264) */
int ttgpu_cache_info(ttgpu_cache* c, int* active, int64_t* resident, uint64_t* accesses,
                     uint64_t* hits);
int ttgpu_cache_record(ttgpu_cache* c, const int64_t* indices, int64_t L);   /* record (:180-183) */
/* record_and_partition (:187-219): sizes of the two parts; fetch them with
 * ttgpu_cache_last_partition (any output may be NULL; weights only if given) */
int ttgpu_cache_record_and_partition(ttgpu_cache* c, const int64_t* indices, int64_t L,
                                     const int64_t* offsets, int64_t B, const double* weights,
                                     int pooling, int64_t* n_cached, int64_t* n_tt);
/* After a fast-path cached forward (ttgpu_cache_set_fast) the partition is rebuilt
 * from the per-lookup slots and the forward's own index / offset / weight arrays:
 * for ttgpu_cache_forward_device those device arrays must still be alive. */
int ttgpu_cache_last_partition(ttgpu_cache* c, int64_t* cached_slots, int64_t* cached_rows,
                               int64_t* cached_offsets, double* cached_weights, int64_t* tt_indices,
                               int64_t* tt_offsets, double* tt_weights);
int ttgpu_cache_warmup_finalize(ttgpu_cache* c, ttgpu_table* t);           /* :223-229 */
int ttgpu_cache_refresh(ttgpu_cache* c, ttgpu_table* t, double* drift);     /* :233-243 */
int ttgpu_hot_set_drift(const int64_t* prev, int64_t n_prev, const int64_t* cur, int64_t n_cur,
                        int64_t k, double* out);                            /* lfu_cache.cpp:113-126 */
int ttgpu_cache_hot_rows(ttgpu_cache* c, int64_t* out, int64_t max, int64_t* n); /* :166-174 */
int ttgpu_cache_slot_rows(ttgpu_cache* c, int64_t* out);   /* row_at(slot) for every slot */
int ttgpu_cache_slot_of(ttgpu_cache* c, int64_t row, int64_t* slot);        /* :160-163 */
int ttgpu_cache_get_rows(ttgpu_cache* c, void* host_out);  /* row_values, capacity x emb_dim */
int ttgpu_cache_set_row(ttgpu_cache* c, int64_t slot, const void* host_in);
int ttgpu_cache_store_device_ptr(ttgpu_cache* c, void** ptr);
int ttgpu_cache_counts_device_ptr(ttgpu_cache* c, void** ptr, int64_t* n); /* for allreduce */
/* FreqTable (lfu_cache.hpp:18-50): count / size / decay / clear / top_k */
int ttgpu_cache_freq_count(ttgpu_cache* c, int64_t key, uint64_t* out);
int ttgpu_cache_freq_size(ttgpu_cache* c, int64_t* out);
int ttgpu_cache_freq_decay(ttgpu_cache* c, double factor);
int ttgpu_cache_freq_clear(ttgpu_cache* c);
int ttgpu_cache_top_k(ttgpu_cache* c, ttgpu_table* t, int64_t k, int64_t* rows, uint64_t* counts,
                      int64_t* n);
/* cached EmbeddingLayer::forward (model.hpp:210-223): partition, cached pooling,
 * forward_bags on the chain part, combine_partition_outputs */
int ttgpu_cache_forward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const int64_t* indices,
                        int64_t L, const int64_t* offsets, int64_t B, const double* weights,
                        int pooling, int save, void* out);
int ttgpu_cache_forward_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx,
                               const int64_t* d_indices, int64_t L, const int64_t* d_offsets,
                               int64_t B, const double* d_weights, int pooling, int save,
                               void* d_out);
/* EmbeddingLayer::backward (model.hpp:237-262): chain gradients -> the table's
 * gradient buffer, slot gradients -> the cache; EmbeddingLayer::step (:265-284) */
int ttgpu_cache_backward(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx, const void* grad_out,
                         int64_t grad_len);
int ttgpu_cache_backward_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx,
                                const void* d_grad_out);
int ttgpu_cache_step(ttgpu_cache* c, ttgpu_table* t, double lr);
/* fused backward + step: SGD applied in both reductions' epilogues (async) */
int ttgpu_cache_backward_step_device(ttgpu_cache* c, ttgpu_table* t, ttgpu_ctx* ctx,
                                     const void* d_grad_out, double lr);
int ttgpu_cache_slot_grads(ttgpu_cache* c, void* host_grads, uint8_t* touched);
/* cached_sgd_update(SlotGradients, lr) with caller rows (:246-257) */
int ttgpu_cache_sgd_update(ttgpu_cache* c, const int64_t* slots, int64_t n, const void* rows,
                           double lr);

/* ---- EmbeddingStats (embedding_stats.hpp:12-23) -------------------------- */
void ttgpu_stats_reset(void);
uint64_t ttgpu_stats_rows(void);            /* tt_rows_computed */
uint64_t ttgpu_stats_peak_workspace(void);  /* peak_workspace_bytes (device) */
void ttgpu_stats_add_rows(uint64_t n);

/* ---- synthetic index streams (data.hpp:11-37), host ---------------------- */
/* ZipfianSampler(population, s) + generate_zipfian_batch with Rng(seed):
 * same CDF-inversion algorithm and mt19937_64 stream as the reference, so
 * the bytes match data.cpp:8-47 on the same libstdc++. */
int ttgpu_zipf_batch(int64_t population, double exponent, uint64_t seed, int64_t bags,
                     int64_t pooling_factor, int64_t* indices, int64_t* offsets);
/* Rng(seed).uniform_int(0, rows) x n (rng.hpp:47-51) */
int ttgpu_uniform_indices(int64_t rows, uint64_t seed, int64_t n, int64_t* indices);
/* Rng::derive(seed, stream).uniform_int(0, rows) x n (rng.hpp:25-29,47-51) */
int ttgpu_derived_uniform_indices(int64_t rows, uint64_t seed, uint64_t stream, int64_t n,
                                  int64_t* out);
/* init_tt_cores(table, InitSpec::sampled_gaussian(), seed) (initializer.hpp:143-154) */
int ttgpu_init_sampled_gaussian(ttgpu_table* t, uint64_t seed);

/* ---- fused cross-GPU gradient reduction + SGD over peer memory (§8(e)) ----
 * Replaces allreduce(SUM) of the dense core gradients + sgd_step on every
 * replica (embedding_ops.hpp:355-376) with ONE kernel per rank, a
 * reduce-scatter + all-gather over NVLink: rank q reduces its 1/W shard of
 * every rank's gradient buffer in rank order, applies core -= lr * g and
 * stores the result into every replica's cores (CUDA IPC mappings), so the
 * replicas stay bitwise equal.
 * Usage: after ttgpu_backward_device on each rank's bag shard,
 * ttgpu_peer_reduce_sgd(t, lr) on every rank (asynchronous, graph-capturable).
 * Handles are cudaIpcMemHandle_t (64 bytes) per rank, exchanged by the caller
 * (e.g. an all_gather over torch.distributed). */
int ttgpu_peer_export(ttgpu_table* t, void* grad_handle, void* core_handle, void* flags_handle);
int ttgpu_peer_attach(ttgpu_table* t, int world, int rank, const void* grad_handles,
                      const void* core_handles, const void* flags_handles);
/* peers addressable from this process (one process driving several GPUs with
 * P2P enabled, or several ranks' tables on one GPU in tests) */
int ttgpu_peer_attach_ptrs(ttgpu_table* t, int world, int rank, void* const* grad_ptrs,
                           void* const* core_ptrs, void* const* flag_ptrs);
int ttgpu_peer_flags_ptr(ttgpu_table* t, void** out);
int ttgpu_peer_reduce_sgd(ttgpu_table* t, double lr);
/* synchronises; timed_out = 1 if a reduce gave up waiting for a rank */
int ttgpu_peer_status(ttgpu_table* t, int* timed_out);

/* ---- uncompressed embedding-bag tables (the DLRM
 * features that are not TT-compressed).  A group of tables shares one row
 * store and one bag structure: indices n_tables x L (table-major), offsets
 * B + 1, outputs / gradients n_tables x B x dim.  Forward sums in lookup
 * order (separately rounded); backward = stable sort by row + fixed-order
 * segmented sums, fused with row -= lr * g (fused = 1) or into a dense gradient
 * buffer for an allreduce (fused = 0, then ttgpu_dense_apply_grad). */
typedef struct ttgpu_dense ttgpu_dense;
int ttgpu_dense_create(int n_tables, const int64_t* rows, int64_t dim, int dtype, int device,
                       void* stream, ttgpu_dense** out);
int ttgpu_dense_destroy(ttgpu_dense* d);
int ttgpu_dense_set_stream(ttgpu_dense* d, void* stream);
int ttgpu_dense_set_table(ttgpu_dense* d, int t, const void* host);
int ttgpu_dense_get_table(ttgpu_dense* d, int t, void* host);
int ttgpu_dense_forward_device(ttgpu_dense* d, const int64_t* d_idx, int64_t L,
                               const int64_t* d_off, int64_t B, void* d_out);
int ttgpu_dense_backward_device(ttgpu_dense* d, const void* d_grad, int fused, double lr);
int ttgpu_dense_grad_buffer(ttgpu_dense* d, void** ptr, int64_t* n_elems);
int ttgpu_dense_apply_grad(ttgpu_dense* d, double lr);
int ttgpu_dense_check(ttgpu_dense* d);

/* ---- device index streams -------------------------
 * ZipfianSampler(population, s) (data.hpp:16-28, data.cpp:8-33) resident on
 * the GPU: the CDF is built on the host with the reference's loop and
 * inverted on the device (upper_bound); s = 0 is uniform.  Variates come from
 * a counter-based SplitMix64 stream -- element i of a draw uses counter + i,
 * so a stream splits across calls and ranks deterministically.  Same
 * distribution as the reference, not the same bytes (its mt19937_64 stream
 * is reproduced on the host by ttgpu_zipf_batch for parity runs). */
typedef struct ttgpu_sampler ttgpu_sampler;
int ttgpu_sampler_create(int64_t population, double exponent, int device, void* stream,
                         ttgpu_sampler** out);
int ttgpu_sampler_destroy(ttgpu_sampler* s);
int ttgpu_sampler_set_stream(ttgpu_sampler* s, void* stream);
int ttgpu_sampler_draw_device(ttgpu_sampler* s, uint64_t seed, uint64_t counter, int64_t n,
                              int64_t* d_out);
/* offsets of num_bags fixed-size bags: off[b] = b * pooling_factor (b <= bags) */
int ttgpu_bag_offsets_device(int64_t bags, int64_t pooling_factor, int64_t* d_offsets,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TTGPU_H */
