/*
 * glint_b200.h -- C ABI of the B200 (sm_100a) layer-wise GNN inference kernels.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `glint` (arXiv 2211.15082, "DGI").  The reference has no FFI of its own: its
 * boundary is the Python module API in pkg/src/glint/kernels.py and the
 * engine in pkg/src/glint/executor.py.  Each entry point below names the
 * reference interface it replaces (file:line relative to the reference's
 * pkg/src/glint/).  INTEGRATION.md shows the ctypes binding a glint maintainer
 * would add.
 *
 * Conventions
 *   - Every pointer argument is caller-allocated DEVICE memory unless the
 *     comment says "host".  The library never allocates or frees caller
 *     memory; scratch space is passed in as an explicit workspace whose size
 *     the matching *_workspace_bytes() query returns.
 *   - Every launching call takes a stream (a cudaStream_t; NULL = legacy
 *     default stream) and is asynchronous: no hidden host synchronisation.
 *   - Return value: 0 on success, a negative GLINT_E* code on failure; the
 *     message is available from glint_last_error() (thread-local).
 *     GLINT_EINVAL maps to Python ValueError (the reference kernels raise
 *     ValueError on shape mismatch, kernels.py:99-105,129-130,180-181);
 *     GLINT_ECUDA maps to glint.errors.InternalError (errors.py:37-38).
 *   - Matrices are row-major fp32 with an explicit leading dimension (row
 *     pitch, in elements).  When ld % 4 == 0 and the base is 16-byte aligned
 *     the kernels use 128-bit loads; otherwise a scalar path runs.
 *   - Node ids in adjacency `indices` are int32 on device (111M-node graphs
 *     fit); offsets (`indptr`) and row-id lists are int64, as in the reference
 *     (storage.py:47-48).
 */
#ifndef GLINT_B200_H
#define GLINT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* glint_stream_t; /* cudaStream_t */

#define GLINT_OK 0
#define GLINT_EINVAL (-1)
#define GLINT_ECUDA (-2)
#define GLINT_EUNSUPPORTED (-3)

/* Elementwise kinds (kernels.py:25 ELEMENTWISE_KINDS order). */
#define GLINT_EW_RELU 0
#define GLINT_EW_LEAKY_RELU 1
#define GLINT_EW_ADD 2
#define GLINT_EW_NORM 3
#define GLINT_EW_DROPOUT_IDENTITY 4

/* Epilogue activations fused into glint_linear_f32. */
#define GLINT_ACT_NONE 0
#define GLINT_ACT_RELU 1
#define GLINT_ACT_LEAKY_RELU 2

/* GEMM precisions. */
#define GLINT_PREC_FP32 0   /* CUDA-core fp32 FMA chain, fixed k order */
#define GLINT_PREC_3XTF32 1 /* tcgen05 kind::tf32, split operands (big+small), 3 MMAs */

/* ------------------------------------------------------------------ misc */
const char* glint_last_error(void);
int glint_abi_version(void);

/* Process-wide tuning knobs.  0 selects the measured default everywhere.
 * Performance knobs never change results (every setting is byte-checked
 * against the default in tests/test_kernels_gpu.py); the two DIAGNOSTIC
 * settings marked below produce wrong numbers on purpose and exist only for
 * tools/sweep_kernels.py. */
#define GLINT_TUNE_MEAN_VARIANT 0 /* K1 regular-row variant: 0 default (cp.async ring),
                                     1-6 register-staged, 7-15 other ring shapes */
#define GLINT_TUNE_GEMM_PROF 1    /* K2: 1 phase-cycle counters (v1); DIAGNOSTIC 2 MMA
                                     issue only, 3 no lo pass (v2) */
#define GLINT_TUNE_HUB_INLINE 2   /* hub-row path.  K1: 0 auto (ring CTAs < 2^19 rows,
                                     else register CTAs), 1 register CTAs, 2 LDGSTS
                                     ring 32 cols, 3 TMA ring 32 cols, 4 LDGSTS ring
                                     64 cols, 5 one-warp cp.async units.  K4: 0 TMA
                                     ring 128 cols, 1 register CTAs, 2 LDGSTS ring
                                     128 cols, 4 TMA ring 64 cols */
#define GLINT_TUNE_GAT_VARIANT 3  /* K4 regular-row variant (0 default; 5-8 cp.async
                                     ring; two-phase path 1-3) */
#define GLINT_TUNE_GEMM_V1 4      /* 1: K2 uses the v1 single-accumulator kernel */
#define GLINT_TUNE_GEMM_RAWHI 5   /* v1 only: the unmasked fp32 word as the tf32 "hi"
                                     operand (the truncation probe) */
#define GLINT_TUNE_HUB_CTAS_PER_SM 6 /* K1 register hub kernel: k > 0 caps it at k CTAs
                                        per SM (persistent) */
#define GLINT_TUNE_GEMM_WIDE 7    /* K2: N in (128, 256] 0 = 128 x N tiles, 2 = 256 x
                                     N/2; N <= 128: 3 = 128-row tiles */
#define GLINT_TUNE_HUB_AFTER 8    /* hub-row kernels: 0 concurrent (side stream), 1 after
                                     the regular rows on the caller's stream */
#define GLINT_TUNE_GEMM_V3 9     /* K2/K3: 0 v3 (tensor-map TMA, CTA pairs) where the
                                     shape allows, 1 the v2 kernel */
#define GLINT_TUNE_GEMM_PF 10    /* v3 K2: L2 prefetch of A, tiles ahead (0 default = 1,
                                     -1 off) */
#define GLINT_TUNE_L2_HINT 11    /* K1 regular rows: L2 policy per gathered row from the
                                     hot bit of its id (glint_hot_annotate): 0 none,
                                     1 hot evict_last + cold evict_first, 2 hot
                                     evict_last only, 3 all evict_first */
#define GLINT_TUNE_FUSED_VARIANT 12 /* K7 gather warps x ring depth: 0 26x8 (26x6,
                                       16x8 when shared memory is short), 1 24x8,
                                       2 20x10, 3 16x12 */
#define GLINT_TUNE_FUSED_PROF 13  /* K7: 1 phase-cycle counters (glint_debug_counters 1) */
#define GLINT_TUNE_GAT_L2 14      /* K4 cp.async ring L2 policy: 0 (default) source scores
                                     evict_last + Z rows evict_first, 1 none (results
                                     never change) */
#define GLINT_TUNE_SAMPLE_SORT 15 /* glint_sample_neighbors: 0 warp top-k selection for
                                     fanout <= 32, 1 the segmented-sort pipeline (same draws) */
#define GLINT_TUNE_GAT_PROJ 16   /* glint_gat_project_f32: 0 scores in the GEMM epilogue,
                                     1 GEMM + glint_gat_scores_f32, 2 the latter for K < 192 */
#define GLINT_TUNE_PACK24_LOOP 17 /* e2e CSR packing on host threads: 0 eight ids per
                                      three 64-bit stores, 1 the per-id loop (A/B) */
#define GLINT_TUNE_GAT_PEAK_FIRST 18 /* K4 ring rows: 0 (default) the first ring slots of
                                        Z rows are issued before the per-head peak pass,
                                        1 peak pass first (A/B; results never change) */
#define GLINT_TUNE_FUSED_PIPE 19  /* K7 gather warps: 0 (default) the next row claimed and
                                      its indptr, first ids and self row loaded while the
                                      current row's edges fly, 1 one row at a time (A/B;
                                      results never change) */
#define GLINT_TUNE_GAT_EPI 20     /* fused GAT score epilogue (K3): 0 (default) each
                                      16-column half-chunk lies in one head (head pitch
                                      % 16 == 0), a_src / a_dst as 128-bit loads, 32-column
                                      chunks on v3 and v3 for every K; 1 the per-column head
                                      walk in 16-column chunks, v2 for K < 192 (the earlier
                                      default); 3 as 0 with 16-column chunks (A/B; results
                                      never change); DIAGNOSTIC 2 no score math */
#define GLINT_TUNE_COUNT 21
int glint_set_tuning(int key, int value);
int glint_get_tuning(int key);
/* Copy (host_out, n <= 8) and optionally reset the phase-cycle counters of
 * kernel family `which` (0 = tcgen05 GEMM, 1 = K7 fused conv). */
int glint_debug_counters(int which, uint64_t* host_out, int n, int reset);
/* host pointers; fills the properties of `device` */
int glint_device_info(int device, int* sm_count, int* cc_major, int* cc_minor,
                      size_t* free_bytes, size_t* total_bytes);

/* ----------------------------------------------------- K1 mean aggregation
 * Replaces kernels.py:122-135 agg_mean (and _segment_sum kernels.py:110-115).
 * For output row r (0 <= r < n_rows):
 *   rid  = row_ids ? row_ids[r] : row_base + r            (CSR row)
 *   map(u) = col_map ? col_map[u] : u                      (row of h)
 *   self = self_rows ? self_rows[r] : map(rid)
 *   out[r, c] = ((0 + h[map(u_0), c]) + h[map(u_1), c] + ... + h[self, c])
 *               / (float)(deg + 1)
 * with u_k = indices[indptr[rid] + k] in STORED order and IEEE fp32 adds /
 * division -- byte-identical to the reference's np.add.at accumulation.
 * `schedule` (nullable) is a processing order of the n_rows output rows as
 * produced by glint_degree_schedule; its first n_hub entries are hub rows
 * processed cooperatively by a whole CTA (columns split across threads, so
 * the per-column summation order is unchanged).  Without a schedule rows run
 * in natural order and n_hub must be 0.
 * Optional epilogue (bias nullable, act = GLINT_ACT_*):
 *   out = act(mean + bias[c]) -- used when a ConvMean is reassociated as
 *   mean(h W^T) + b for layers that narrow the width (same math as
 *   model_ir.py:336-338 up to fp32 rounding); bias=NULL, act=NONE is the
 *   plain agg_mean. */
int glint_spmm_mean_f32(int64_t n_rows, int32_t dim, const int64_t* indptr,
                        const int32_t* indices, const int64_t* row_ids,
                        int64_t row_base, const int64_t* self_rows,
                        const int32_t* col_map, const float* h, int64_t ld_h,
                        float* out, int64_t ld_out, const int32_t* schedule,
                        int64_t n_hub, const float* bias, int32_t act,
                        glint_stream_t stream);

/* Degree-bucketed longest-first schedule over n_rows output rows (CSR rows
 * as for glint_spmm_mean_f32).  Writes a permutation of [0, n_rows) to
 * schedule_out: rows bucketed by floor(log2(deg+1)) in descending bucket
 * order; *n_hub_out (device int64) = number of leading rows whose
 * deg + 1 >= hub_min_degree (hub_min_degree must be a power of two, or 0
 * to disable the hub path). */
size_t glint_degree_schedule_workspace_bytes(void);
int glint_degree_schedule(int64_t n_rows, const int64_t* indptr,
                          const int64_t* row_ids, int64_t row_base,
                          int64_t hub_min_degree, int32_t* schedule_out,
                          int64_t* n_hub_out, void* workspace,
                          size_t workspace_bytes, glint_stream_t stream);

/* ----------------------------------------------- RCMK on the device
 * Building blocks of reorder.rcmk for a DeviceGraph (reference reorder.py:
 * 72-123), over the symmetrised adjacency (ptr int64 [n+1], adj int32, every
 * row distinct neighbours without self loops, ordered by (degree, id)).
 * components: comp_out[v] = the minimum id of v's connected component.
 * starts: start_key[c] = min over members v of component c of
 *   (degree(v) << 32 | v); untouched entries are UINT64_MAX.
 * expand: for i < n_front and every neighbour u of frontier[i] with
 *   level[u] < 0: best[u] = min(best[u], i). */
int glint_rcmk_components(int64_t n, const int64_t* ptr, const int32_t* adj,
                          int32_t* comp_out, glint_stream_t stream);
int glint_rcmk_starts(int64_t n, const int64_t* ptr, const int32_t* comp,
                      uint64_t* start_key, glint_stream_t stream);
int glint_rcmk_expand(int64_t n_front, const int32_t* frontier, const int64_t* ptr,
                      const int32_t* adj, const int32_t* level, int64_t* best,
                      glint_stream_t stream);

/* ------------------------------------------------------ K2 dense transform
 * Replaces kernels.py:95-107 linear (einsum "ij,kj->ik" + bias), with an
 * optional fused activation (elementwise ReLU/LeakyReLU, kernels.py:206-215).
 *   C[i, n] = act( sum_k A[a_row(i), k] * W[n, k] + bias[n] )
 * a_rows (nullable) gathers A rows.  Each output row depends only on its own
 * A row (row/batch invariant, kernels.py:1-14). */
int glint_linear_f32(int64_t M, int32_t N, int32_t K, const float* A,
                     int64_t lda, const int64_t* a_rows, const float* W,
                     int64_t ldw, const float* bias, int32_t act, float* C,
                     int64_t ldc, int32_t precision, glint_stream_t stream);

/* ----------------------------------------- K7 fused aggregate -> transform
 * Replaces model_ir.py:336-338 (ConvMean: agg_mean kernels.py:122-135, then
 * linear kernels.py:95-107) for an aggregate-first layer in ONE kernel:
 *   out[r, n] = act( sum_k mean_r[k] * W[n, k] + bias[n] )
 * where mean_r is exactly glint_spmm_mean_f32's row r (same add chain, same
 * division; row addressing, self_rows and col_map as there) and the transform
 * is glint_linear_f32's 3xTF32 product order.  The B x dim_in aggregate
 * never reaches HBM.  `schedule` (nullable) is glint_degree_schedule's order
 * over all n_rows rows (no hub split: rows are taken dynamically by warps).
 * Shapes: glint_conv_mean_supported(dim_in, dim_out) (dim_in <= 128, a
 * multiple of 4, dim_out <= 256); ld_h, ld_out multiples of 4 with 16-byte
 * aligned h / out; otherwise GLINT_EUNSUPPORTED (the caller runs K1 + K2).
 * max_ctas > 0 caps the persistent grid (default 0: one CTA per SM, each
 * holding a whole SM): leaving a few SMs free lets concurrent work on other
 * streams (the batch planner's counting kernels) run beside it.
 * Workspace: glint_conv_mean_workspace_bytes (the pre-split W panel and a
 * tile counter). */
size_t glint_conv_mean_workspace_bytes(int32_t dim_in, int32_t dim_out);
int glint_conv_mean_supported(int32_t dim_in, int32_t dim_out);
int glint_conv_mean_f32(int64_t n_rows, int32_t dim_in, int32_t dim_out,
                        const int64_t* indptr, const int32_t* indices,
                        const int64_t* row_ids, int64_t row_base,
                        const int64_t* self_rows, const int32_t* col_map,
                        const float* h, int64_t ld_h, const float* W, int64_t ldw,
                        const float* bias, int32_t act, float* out, int64_t ld_out,
                        const int32_t* schedule, int32_t max_ctas, void* workspace,
                        size_t workspace_bytes, glint_stream_t stream);

/* -------------------------------------------------------- K3/K4 attention
 * Replaces kernels.py:170-203 agg_attn.  The projection z_h = linear(h, W_h)
 * for all heads is one glint_linear_f32 into a head-padded Z
 * (Z[:, h*ldh + j], ldh >= head_dim), then: */
/* s_src[i,h] = z_h[i] . attn[h, :dh]; s_dst[i,h] = z_h[i] . attn[h, dh:]
 * (einsum "ij,j->i", kernels.py:188-189). */
int glint_gat_scores_f32(int64_t M, int32_t heads, int32_t head_dim,
                         int32_t head_pitch, const float* Z, int64_t ldz,
                         const float* attn, float* s_src, float* s_dst,
                         glint_stream_t stream);
/* Fused per-layer GAT projection (kernels.py:185-189 for all heads at once):
 * Z = A W_pad^T with W_pad = [heads * head_pitch, K] (zero pad rows per head),
 * and s_src / s_dst as glint_gat_scores_f32, computed in the GEMM epilogue
 * while the Z tile is in registers (3xTF32 path; other precisions / shapes
 * run glint_linear_f32 + glint_gat_scores_f32).  Scores are one sequential
 * fmaf chain over j per (row, head). */
int glint_gat_project_f32(int64_t M, int32_t heads, int32_t head_dim,
                          int32_t head_pitch, int32_t K, const float* A,
                          int64_t lda, const int64_t* a_rows, const float* W_pad,
                          int64_t ldw, const float* attn, float* Z, int64_t ldz,
                          float* s_src, float* s_dst, int32_t precision,
                          glint_stream_t stream);
/* Edge softmax + weighted sum over N(v) u {v} per head (kernels.py:190-202):
 * logit = LeakyReLU_slope(s_src[u,h] + s_dst[v,h]); peak = max(self, edges);
 * w = exp(logit - peak); out[r, h*head_dim + j] =
 *   (sum_e w_e * z_h[u_e, j] (stored order) + w_self * z_h[v, j]) /
 *   (sum_e w_e + w_self).  Row addressing as glint_spmm_mean_f32; the
 * self row of Z / s_* is `self`, the source rows map(u).  act (GLINT_ACT_*)
 * is applied to each output element (the model's following ReLU fused into
 * the epilogue; GLINT_ACT_NONE = the reference op alone). */
int glint_gat_aggregate_f32(int64_t n_rows, int32_t heads, int32_t head_dim,
                            int32_t head_pitch, const int64_t* indptr,
                            const int32_t* indices, const int64_t* row_ids,
                            int64_t row_base, const int64_t* self_rows,
                            const int32_t* col_map, const float* Z, int64_t ldz,
                            const float* s_src, const float* s_dst, float slope,
                            float* out, int64_t ld_out, const int32_t* schedule,
                            int64_t n_hub, int32_t act, glint_stream_t stream);
/* The same result in two phases for the regular rows: an edge-softmax pass
 * (SDDMM) writes every edge's H weights to the workspace, then a weighted
 * SpMM streams them beside the Z rows (the K1 ring kernels) -- same weights,
 * same accumulation order, same bytes.  Every regular row's edges must lie in
 * [edge_base, edge_base + edge_span) of indptr; workspace from
 * glint_gat_aggregate_workspace_bytes (NULL workspace = one-phase kernel). */
size_t glint_gat_aggregate_workspace_bytes(int64_t n_rows, int64_t edge_span, int32_t heads);
int glint_gat_aggregate_ws_f32(int64_t n_rows, int32_t heads, int32_t head_dim,
                               int32_t head_pitch, const int64_t* indptr,
                               const int32_t* indices, const int64_t* row_ids,
                               int64_t row_base, const int64_t* self_rows,
                               const int32_t* col_map, const float* Z, int64_t ldz,
                               const float* s_src, const float* s_dst, float slope,
                               float* out, int64_t ld_out, const int32_t* schedule,
                               int64_t n_hub, int32_t act, int64_t edge_base,
                               int64_t edge_span, void* workspace, size_t workspace_bytes,
                               glint_stream_t stream);

/* --------------------------------------------------- K5 per-row operators
 * Replaces kernels.py:206-231 elementwise.  inputs / ld_inputs / input_rows
 * are HOST arrays of n_inputs entries (device pointers inside); input_rows[k]
 * (nullable) gathers rows of operand k (the executor's target restriction,
 * executor.py:358-368).  Add sums operands sequentially in order. */
int glint_elementwise_f32(int32_t kind, int64_t n_rows, int32_t dim,
                          int32_t n_inputs, const float* const* inputs,
                          const int64_t* ld_inputs,
                          const int64_t* const* input_rows, float* out,
                          int64_t ld_out, glint_stream_t stream);

/* Row copy with optional gather/scatter: dst[dst_row(i), :dim] =
 * src[src_row(i), :dim].  Serves EmbeddingStore.gather/scatter
 * (storage.py:224-246), concat (kernels.py:234-239, dst column offset via
 * the dst pointer) and apply_order's feature permutation (reorder.py:175-180). */
int glint_copy_rows_f32(int64_t n_rows, int32_t dim, const float* src,
                        int64_t ld_src, const int64_t* src_rows, float* dst,
                        int64_t ld_dst, const int64_t* dst_rows,
                        glint_stream_t stream);

/* ------------------------------------------------ K6 integer set machinery
 * Sorted id sets over [0, num_nodes) as a bitmap plus per-word rank prefix.
 * Replaces the np.unique / np.searchsorted pairs of build_batch_csc
 * (kernels.py:71-77), trivial_batch_csc (kernels.py:80-88), _expand
 * (executor.py:118-121) and _StoreEntry.locate (executor.py:270-276). */
size_t glint_idset_workspace_bytes(int64_t num_nodes);
int glint_idset_clear(void* ws, int64_t num_nodes, glint_stream_t stream);
/* add ids[0..n) (ids == NULL: add the range [base, base+n)) */
int glint_idset_add_ids(void* ws, int64_t num_nodes, const int64_t* ids,
                        int64_t base, int64_t n, glint_stream_t stream);
/* add the in-neighbours of targets (targets == NULL: rows [base, base+n)) */
int glint_idset_add_neighbors(void* ws, int64_t num_nodes, const int64_t* indptr,
                              const int32_t* indices, const int64_t* targets,
                              int64_t base, int64_t n, glint_stream_t stream);
/* rank prefix; *count_out (device int64) = |set| */
int glint_idset_finalize(void* ws, int64_t num_nodes, int64_t* count_out,
                         glint_stream_t stream);
/* ascending members -> ids_out[0..|set|) (after finalize) */
int glint_idset_extract(const void* ws, int64_t num_nodes, int64_t* ids_out,
                        glint_stream_t stream);
/* pos[i] = rank of ids[i] in the set, -1 when absent (after finalize).
 * Either output may be NULL. */
int glint_idset_lookup(const void* ws, int64_t num_nodes, const int64_t* ids,
                       const int32_t* ids32, int64_t n, int64_t* pos64,
                       int32_t* pos32, glint_stream_t stream);
/* dense id -> rank map over all nodes: map[u] = rank or -1 */
int glint_idset_rank_map(const void* ws, int64_t num_nodes, int32_t* map_out,
                         glint_stream_t stream);

/* Exclusive prefix of in-degrees over a target list: out[0] = 0,
 * out[j+1] = out[j] + deg(target_j).  Replaces storage.py:159-165
 * prefix_for_targets and the local indptr of gather_slices
 * (kernels.py:56-68).  targets == NULL: rows [base, base+n). */
size_t glint_scan_workspace_bytes(int64_t n);
int glint_degree_prefix(const int64_t* indptr, const int64_t* targets,
                        int64_t base, int64_t n, int64_t* out, void* ws,
                        size_t ws_bytes, glint_stream_t stream);
/* Exclusive prefix of hub flags [deg(t)+1 >= min_degp1] over the same target
 * addressing (sizes the hub path of a batch without a host pass over N). */
int glint_hub_prefix(const int64_t* indptr, const int64_t* targets, int64_t base,
                     int64_t n, int64_t min_degp1, int64_t* out, void* ws,
                     size_t ws_bytes, glint_stream_t stream);
/* Concatenated in-neighbour slices (kernels.py:56-68 gather_slices):
 * srcs[local_indptr[j] + k] = indices[indptr[t_j] + k]; either output may
 * be NULL; local positions through an idset when pos_ws != NULL
 * (local_srcs of build_batch_csc). */
int glint_gather_slices(const int64_t* indptr, const int32_t* indices,
                        const int64_t* targets, int64_t base, int64_t n,
                        const int64_t* local_indptr, int64_t* srcs64,
                        int32_t* srcs32, const void* pos_ws, int64_t num_nodes,
                        int64_t* local64, int32_t* local32,
                        glint_stream_t stream);

/* ------------------------------------------------------ graph utilities */
/* apply_order relabel (reorder.py:149-181): new row j = old row perm[j],
 * slice mapped elementwise through inv, stored order preserved. */
int glint_relabel_csc(int64_t num_nodes, const int64_t* old_indptr,
                      const int32_t* old_indices, const int64_t* perm,
                      const int64_t* inv, const int64_t* new_indptr,
                      int32_t* new_indices, glint_stream_t stream);
/* int64 -> int32 id narrowing with range check; *bad_out (device int64)
 * receives the count of ids outside [0, limit). */
int glint_narrow_ids(int64_t n, const int64_t* src, int32_t* dst,
                     int64_t limit, int64_t* bad_out, glint_stream_t stream);

/* ---------------------------------------------------- neighbour sampling
 * Replaces executor.py:74-115 sample_neighbors on the device.  For selected
 * node i (id nodes[i], or i when nodes is NULL): its in-edge slots s get
 * prio = mix(base ^ mix(v*M1) ^ s), base = mix(mix(seed) ^ mix(layer*M2))
 * (splitmix64), it keeps its min(fanout, deg) smallest priorities (ties by
 * slot) and writes the kept source ids ascending to
 * out_indices[out_off[i] .. out_off[i+1]).  local_off[i] = sum of deg over
 * selected nodes before i (n_sel+1 entries, e_sel = local_off[n_sel]).
 * All arrays device memory.  fanout <= 32 runs one warp per node (top-k by
 * warp bitonic merges) and needs neither local_off nor a workspace (both may
 * be NULL); larger fanouts segment-sort every slot and need local_off and
 * glint_sample_workspace_bytes of scratch. */
size_t glint_sample_workspace_bytes(int64_t n_sel, int64_t e_sel, int64_t e_out);
int glint_sample_neighbors(const int64_t* indptr, const int32_t* indices,
                           const int64_t* nodes, int64_t n_sel,
                           const int64_t* local_off, int64_t e_sel,
                           const int64_t* out_off, int64_t e_out, int32_t fanout,
                           int64_t seed, int32_t layer, int32_t* out_indices,
                           void* workspace, size_t workspace_bytes,
                           glint_stream_t stream);

/* Host-side (pure C++, host pointers): reverse Cuthill-McKee order with the
 * reference's tie rules (reorder.py:55-123). perm_out[new] = old. */
int glint_rcmk_host(int64_t num_nodes, const int64_t* indptr,
                    const int64_t* indices, int64_t* perm_out);
/* Asynchronous CSR upload with host narrowing (upload.cu): a native thread
 * narrows the int64 ids of edge chunk k = [chunk_edges[k], chunk_edges[k+1])
 * on `threads` CPU threads into stage_pinned (caller's pinned int32 buffer),
 * queues the H2D copy into dst_dev on copy_stream and records chunk k's event.
 * glint_upload_wait blocks until chunk k is queued, then makes `stream` wait
 * for it; glint_upload_query returns 1 once it has landed; glint_upload_finish
 * joins the thread and frees the handle. */
int glint_upload_start(const int64_t* src_host, int32_t* dst_dev, int32_t* stage_pinned,
                       const int64_t* chunk_edges, int32_t n_chunks, int32_t threads,
                       glint_stream_t copy_stream, void** handle_out);
/* The same with id_bytes = 3 (node ids < 2^24): ids cross PCIe as 24-bit
 * little-endian triples (stage_pinned: 3 bytes per edge) into dev_stage
 * (device, 3 bytes per edge), and a kernel on copy_stream unpacks each chunk
 * into dst_dev before its event -- 25% fewer bytes on the e2e path's floor.
 * id_bytes = 4 is glint_upload_start (stage_pinned is int32, dev_stage unused).
 * An id outside [0, 2^24) fails the chunk with GLINT_EINVAL. */
int glint_upload_start_packed(const int64_t* src_host, int32_t* dst_dev, uint8_t* stage_pinned,
                              uint8_t* dev_stage, int32_t id_bytes, const int64_t* chunk_edges,
                              int32_t n_chunks, int32_t threads, glint_stream_t copy_stream,
                              void** handle_out);
int glint_upload_wait(void* handle, int32_t chunk, glint_stream_t stream);
/* Row-pitched async copy, any direction (cudaMemcpy2DAsync with
 * cudaMemcpyDefault): `rows` rows of row_bytes, pitches in bytes.  Used by the
 * e2e output sink (pitched device store -> dense pinned host rows; reference
 * run_inference returns the output as a host array, executor.py:481-543). */
int glint_copy_rows_async(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                          int64_t row_bytes, int64_t rows, glint_stream_t stream);
int glint_upload_query(void* handle, int32_t chunk);
int glint_upload_finish(void* handle);
/* Pageable host -> device copy of `bytes` through the library's pinned
 * staging on `threads` CPU threads (each thread double-buffers its slice);
 * returns once every byte has landed.  run_inference uses it for numpy
 * feature matrices (reference API: storage.py / executor.py:481-543 take
 * host arrays), which a plain pageable cudaMemcpy moves at ~10 GB/s. */
int glint_h2d_pageable(void* dst_dev, const void* src_host, int64_t bytes, int32_t threads,
                       glint_stream_t stream);
/* Host int64 -> int32 narrowing on `threads` CPU threads (host pointers);
 * returns the number of ids outside int32 (the e2e upload narrows CSR chunks
 * on the host so they cross PCIe at half the bytes). */
int64_t glint_narrow_ids_host(const int64_t* src, int32_t* dst, int64_t n, int32_t threads);
/* The same order from a symmetrised adjacency whose rows are already
 * deduplicated, free of self loops and ordered by (degree, id) -- built on the
 * device by reorder._sorted_adjacency_device -- so the host pass is linear
 * (components, then BFS).  Host pointers. */
int glint_rcmk_sorted_host(int64_t num_nodes, const int64_t* ptr,
                           const int32_t* adj, int64_t* perm_out);

#ifdef __cplusplus
}
#endif
#endif /* GLINT_B200_H */
