/*
 * gnnc.h — C ABI of the B200 (sm_100a) GCN/GAT composition kernels.
 *
 * The reference (gnncompose 0.1.0, Python) has no native ABI: its operator
 * boundary is the set of Python functions in gnncompose/sparse.py plus
 * gat.atten_calc, and the `spmm_fn=` plug-in hook on the layer functions
 * (gcn.py:125-161, gat.py:121-153).  Every entry point below replaces one of
 * those calls (cited per function); the Python mirror in
 * paper_2306_15155_b200/ binds them through ctypes.
 *
 * Conventions (all entry points):
 *   - extern "C", plain pointers and sizes, int return: 0 = ok, < 0 = error
 *     (gc_last_error() holds a message; Python maps GC_ERR_SHAPE to
 *     ShapeError, GC_ERR_VALUE to ValueError, the rest to RuntimeError).
 *   - Data pointers are DEVICE pointers unless the parameter name ends in
 *     `_host`.  CSR indices are int32 (row_ptr[n_rows+1], col_idx[nnz]),
 *     values and dense operands are float32, dense matrices are row-major
 *     with an explicit leading dimension (in elements).
 *   - `stream` is a cudaStream_t passed as void*; work is stream-ordered,
 *     the library never synchronises and never allocates device memory:
 *     the caller owns every buffer, including workspaces.
 *   - Validation happens before any launch; no partial work on error.
 *   - Results are deterministic (no floating-point atomics): each output
 *     element has one fixed accumulation order.
 */
#ifndef GNNC_H_
#define GNNC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNNC_ABI_VERSION 2

#if defined(__GNUC__)
#define GNNC_API __attribute__((visibility("default")))
#else
#define GNNC_API
#endif

/* status codes */
#define GC_OK 0
#define GC_ERR_SHAPE (-1)       /* operand dimensions do not conform  -> ShapeError */
#define GC_ERR_VALUE (-2)       /* bad scalar argument / flag         -> ValueError */
#define GC_ERR_CUDA (-3)        /* launch or device error             -> RuntimeError */
#define GC_ERR_UNSUPPORTED (-4) /* combination not implemented        -> RuntimeError */
#define GC_ERR_WORKSPACE (-5)   /* workspace missing or too small     -> RuntimeError */

/* epilogue / mode flags */
#define GC_RELU (1u << 0)       /* out = max(out, 0) (gcn.py:115-116, gat.py:117-118) */
#define GC_ACCUMULATE (1u << 1) /* out += result instead of out = result */
#define GC_HUB_TAGGED (1u << 2) /* col_idx entries carry a hub tag in bit 31 (gc_tag_hub_columns):
                                   tagged rows of B are gathered with L1::evict_last, the rest
                                   with L1::no_allocate (SpMM / GAT aggregation only) */
#define GC_SPMM_SHRINK(s) ((uint32_t)(s) << 8) /* SpMM/GAT lane-group variant s in {0,1,2}:
                                                 (K/4 >> s) lanes per row, each owning 4<<s
                                                 columns; more rows per warp for short rows */
#define GC_SPMM_SHRINK_MASK (3u << 8)
#define GC_SPMM_B_F16 (1u << 10) /* gc_spmm_f32: B holds fp16 rows (ldb in elements; K % 4 == 0,
                                  * ldb % 4 == 0, 8-byte aligned), see gc_pack_rows_f16 */
#define GC_SPMM_SIG_CHUNKS(c) ((uint32_t)((c) - 1) << 12) /* fp16 rows (GC_SPMM_B_F16): c >= 1
                                   scales per row (d_col / sigma is n x c, one per 256-column
                                   chunk; K = 256 c), as gc_gemm_f16rows_f32 emits for N > 256;
                                   SpMM and GAT reassoc aggregation only */
#define GC_SPMM_SIG_MASK (15u << 12)
#define GC_HUB_SIG_CHUNKS(c) ((int32_t)((c) - 1) << 8) /* gc_hub_pack_f16rows fmt: c scales
                                   per row (256-column chunks) */
#define GC_GEMM_TF32 (1u << 4)  /* tcgen05.mma kind::tf32, TMEM accumulators, TMA operands */
#define GC_GEMM_FP32 (1u << 5)  /* exact fp32 CUDA-core path (rtol 1e-4 parity mode) */
#define GC_GEMM_TF32X3 (1u << 7) /* 3xTF32 on tcgen05: hi·hi + hi·lo + lo·hi, fp32-class (1e-4) */
#define GC_HUB_A_BITS (1u << 6) /* gc_hub_stair_gemm: A_steps are bitmaps (see there) */

/* SpMM work decomposition */
#define GC_SPMM_ROW 1       /* one lane-group per CSR row                          */
#define GC_SPMM_NNZ_SPLIT 2 /* plan-driven: heavy rows split into fixed-size edge
                               chunks, partial sums combined in a fixed order     */

/* ---- library state ---------------------------------------------------- */
GNNC_API int gc_abi_version(void);
GNNC_API const char *gc_last_error(void);      /* message of the last error on this thread */
GNNC_API uint64_t gc_launch_count(void);       /* kernels launched by this library so far   */
GNNC_API int gc_device_sm_count(int device);   /* multiprocessor count of `device`          */

/* ---- SpMM ---------------------------------------------------------------
 * C[i,:] (=|+=) epi( d_row[i] * sum_{p in row i} w_p * B[col_idx[p],:] )
 *   w_p = (values ? values[p] : 1) * (d_col ? d_col[col_idx[p]] : 1)
 * Replaces: sparse.spmm (sparse.py:240-247 -> _spmm_kernel 196-205) when
 *   values != NULL; sparse.spmm_unweighted (sparse.py:250-264 -> 208-219)
 *   when values == NULL (the values array is then never read); and the
 *   dynamic-normalisation sequence scale_rows -> spmm -> scale_rows of
 *   gcn.gcn_layer_dynamic (gcn.py:137-155) when d_col/d_row are given.
 * Edges of a row are accumulated in ascending storage order (sequential
 *   FMA), so values == NULL is bit-identical to all-ones values.
 * `items`/`split_rows` come from gc_spmm_plan_* (GC_SPMM_NNZ_SPLIT only);
 *   that mode needs n_slots*K floats of `workspace`.                      */
GNNC_API int gc_spmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *values,
                const float *d_row, const float *d_col, const float *B, int64_t ldb,
                int64_t n_rows, int64_t n_cols, int64_t K, float *C, int64_t ldc,
                uint32_t flags, int algo, const int32_t *items, int64_t n_items,
                const int32_t *split_rows, int64_t n_split_rows, void *workspace,
                size_t ws_bytes, void *stream);

/* Aggregate-first layer with the narrow update fused into the SpMM epilogue
 * (replaces `gemm(spmm(a, h), w)` of reference gcn.py:119-122 /
 * gcn.py:131-134 for small k2): C = epi(D_row A D_col B) W with W row-major
 * K1 x K2, K1 % 4 == 0, K1 <= 256, K2 <= 32, B 16-byte aligned (ldb % 4 ==
 * 0); flags: GC_RELU.  The n x K1 aggregate stays in registers; it is the
 * SpMM's own sum (same edge order), the product with W an fp32 dot. */
GNNC_API int gc_spmm_gemm_f32(const int32_t *row_ptr, const int32_t *col_idx,
                              const float *values, const float *d_row, const float *d_col,
                              const float *B, int64_t ldb, int64_t n_rows, int64_t n_cols,
                              int64_t K1, const float *W, int64_t K2, float *C, int64_t ldc,
                              uint32_t flags, void *stream);

/* Host-side planner for GC_SPMM_NNZ_SPLIT (one pass over a host copy of
 * row_ptr).  Rows with more than `chunk` edges become ceil(deg/chunk)
 * items whose partial sums land in consecutive workspace slots; every other
 * row is one item writing C directly.  items: int32[4*n_items] =
 * {row, begin, end, slot|-1}; split_rows: int32[4*n_split_rows] =
 * {row, first_slot, n_slots, 0}.  With GC_PLAN_LENGTH_CLASSES the items are
 * stably ordered by floor(log2(length)), longest class first: lane groups
 * sharing a warp get similar trip counts and the longest items start first
 * (the order of work only; every output keeps its fixed accumulation order).
 * gc_spmm_default_chunk: chunk that bounds the longest item to ~2x the mean
 * work of one resident lane group for this K on `sm_count` SMs. */
#define GC_PLAN_LENGTH_CLASSES 1u
GNNC_API int32_t gc_spmm_default_chunk(int64_t n_rows, int64_t nnz, int64_t K, int sm_count);
GNNC_API int gc_spmm_plan_count(const int32_t *row_ptr_host, int64_t n_rows, int32_t chunk,
                       int64_t *n_items, int64_t *n_slots, int64_t *n_split_rows);
GNNC_API int gc_spmm_plan_fill(const int32_t *row_ptr_host, int64_t n_rows, int32_t chunk,
                      uint32_t plan_flags, int32_t *items_host, int32_t *split_rows_host);

/* Fused GAT aggregation: for each row i
 *   C[i,:] = epi( sum_p alpha_p * B[col_idx[p],:] ),
 *   alpha_p = exp(e_p - max_row) / sum_row,  e_p = LeakyReLU(s[i] + t[col_idx[p]])
 * i.e. gat.py:72-95 (_edge_scores_softmax) followed by the aggregation
 * spmm(alpha, B) of gat_layer_reuse/recompute (gat.py:121-145), computed with
 * an online softmax so alpha is never materialised.  Rows without edges give 0.
 * Same plan/workspace protocol as gc_spmm_f32; NNZ_SPLIT needs
 * n_slots*(4*K + 8) + 8 bytes of workspace (partial rows, then 8-byte aligned
 * (max, sum) pairs).  GC_SPMM_B_F16: B holds fp16 rows (gc_pack_rows_f16) and
 * sigma their row scales (NULL otherwise); sigma_j scales row j in the
 * aggregation, not the softmax. */
GNNC_API int gc_gat_aggregate_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *s,
                                  const float *t, float slope, const float *B, int64_t ldb,
                                  const float *sigma, int64_t n_rows, int64_t n_cols, int64_t K,
                                  float *C, int64_t ldc,
                                  uint32_t flags, int algo, const int32_t *items, int64_t n_items,
                                  const int32_t *split_rows, int64_t n_split_rows, void *workspace,
                                  size_t ws_bytes, void *stream);

/* Half-width gather operand of the TF32 numerics class: per row j, with
 * Y[j,:] = fp32(d[j] * X[j,:]) (Y = X when d is NULL),
 *   Xh[j,:] = fp16_rn(Y[j,:] * 2^-e_j)  (max |.| in [2^14, 2^15)),
 *   sigma[j] = 2^e_j  (a power of two: d folds into the rows),
 * so sigma[j] * Xh[j,:] = d[j] * X[j,:] to fp16's 11 significant bits (the
 * input rounding TF32 applies).  gc_spmm_f32 with GC_SPMM_B_F16 and
 * d_col = sigma then gathers 2 bytes per feature instead of 4, and weighs
 * unit-valued edges in fp16 exactly (sigma in fp16 range). */
GNNC_API int gc_pack_rows_f16(const float *X, int64_t ldx, int64_t n_rows, int64_t K,
                              const float *d, void *Xh, int64_t ldh, float *sigma, void *stream);
/* The same with n_proj <= 16 row projections computed from the fp32 rows in
 * the same pass (the GAT node scores s, t = X a_src, X a_dst of gat.py:110-111,
 * replacing gc_node_proj_f32 when the rows are packed anyway):
 * proj_out[p * n_rows + r] = X[r,:] . P[p,:] (P: n_proj x K, 16-byte
 * aligned; K % 4 == 0). */
GNNC_API int gc_pack_rows_f16_proj(const float *X, int64_t ldx, int64_t n_rows, int64_t K,
                                   const float *d, void *Xh, int64_t ldh, float *sigma,
                                   const float *P, int32_t n_proj, float *proj_out, void *stream);

/* col_tagged[p] = col_idx[p] | (hot[col_idx[p]] ? 1<<31 : 0): a copy of the
 * pattern whose hub columns (hot: uint8 per column) are tagged for
 * GC_HUB_TAGGED launches.  The untagged col_idx stays valid for every other
 * kernel. */
GNNC_API int gc_tag_hub_columns(const int32_t *col_idx, int64_t nnz, const uint8_t *hot,
                                int32_t *col_tagged, void *stream);

/* Fused GAT aggregation with the attention as an SDDMM over edges (SURVEY.md
 * §8(a) A17 fused with N1): e_p = LeakyReLU(a_src.B[i,:] + a_dst.B[j,:]),
 * alpha = row softmax, C[i,:] = epi(sum_p alpha_p B[j,:]).  Each gathered row
 * B[j,:] feeds both its score and the aggregation (one gather per edge); the
 * reuse composition (B = HW, gat.py:121-129).  The source term a_src.B_i
 * reads row i of B_self (ld_self), or of B when B_self is NULL (square
 * pattern); a rank's row block of a partitioned graph passes its own rows of
 * HW as B_self and the gathered HW as B.  Needs K % 4 == 0, K <= 1024,
 * 16-byte aligned B/B_self/C/a_src/a_dst (else GC_ERR_UNSUPPORTED).
 * Plan/workspace protocol as gc_gat_aggregate_f32.  GC_SPMM_B_F16: B holds
 * fp16 rows with row scales sigma (the score uses sigma_j * a_dst.Bh[j,:]);
 * B_self must then be the fp32 source rows. */
GNNC_API int gc_gat_sddmm_aggregate_f32(const int32_t *row_ptr, const int32_t *col_idx,
                                        const float *a_src, const float *a_dst, float slope,
                                        const float *B, int64_t ldb, const float *B_self,
                                        int64_t ld_self, const float *sigma, int64_t n_rows,
                                        int64_t K,
                                        float *C, int64_t ldc, uint32_t flags, int algo,
                                        const int32_t *items, int64_t n_items,
                                        const int32_t *split_rows, int64_t n_split_rows,
                                        void *workspace, size_t ws_bytes, void *stream);

/* ---- SDDMM --------------------------------------------------------------
 * out[p] = (a_vals ? a_vals[p] : 1) * sum_t B[i,t] * Cm[col_idx[p],t]
 * Replaces sparse.sddmm (sparse.py:267-282 -> _sddmm_kernel 222-232).
 * The output shares row_ptr/col_idx with the input (pattern bit-identical). */
GNNC_API int gc_sddmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *a_vals,
                 const float *B, int64_t ldb, const float *Cm, int64_t ldc, int64_t n_rows,
                 int64_t n_cols, int64_t k, float *out_vals, void *stream);

/* k = 1 special case used for the normalised adjacency:
 * out[p] = (a_vals ? a_vals[p] : 1) * (d[i] * d[col_idx[p]])
 * Replaces gcn.precompute_normalized (gcn.py:103-112). */
GNNC_API int gc_sddmm_norm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *a_vals,
                      const float *d, int64_t n_rows, int64_t nnz, float *out_vals, void *stream);

/* ---- dense --------------------------------------------------------------
 * C = epi( diag(row_scale) * A * W ), A: M x K (lda), W: K x N (ldw),
 * C: M x N (ldc).  Replaces sparse.gemm (sparse.py:285-291).
 * GC_GEMM_TF32: tcgen05/TMEM/TMA kernel, needs lda % 4 == 0 and 16-byte
 *   aligned A, plus workspace >= gc_gemm_workspace_bytes(K, N) for the
 *   transposed (K-major) W.  GC_GEMM_FP32: exact fp32 FMA on CUDA cores.  */
GNNC_API size_t gc_gemm_workspace_bytes(int64_t K, int64_t N);
GNNC_API int gc_gemm_f32(const float *A, int64_t lda, const float *W, int64_t ldw, int64_t M,
                int64_t K, int64_t N, float *C, int64_t ldc, const float *row_scale,
                uint32_t flags, void *workspace, size_t ws_bytes, void *stream);

/* C[i,:] = epi( d[i] * B[i,:] ).  Replaces sparse.scale_rows
 * (sparse.py:294-300); with d == NULL and GC_RELU it is the ReLU of
 * gcn.py:115-116 / gat.py:117-118. */
GNNC_API int gc_scale_rows_f32(const float *d, const float *B, int64_t ldb, int64_t n_rows, int64_t K,
                      float *C, int64_t ldc, uint32_t flags, void *stream);

/* ---- GAT attention -------------------------------------------------------
 * Node projections (the reassociated attention of gat.py:110-111):
 *   s[h*n + i] = sum_c X[i, h*head_stride + c] * a_src[h*k2 + c],  likewise t/a_dst,
 * for heads h = 0..heads-1 (heads = 1 is the reference's single head).
 * X = HW with head_stride = k2 is the reference's form; X = H with
 * head_stride = 0 and a = W_h a_h (k1-vectors) gives the same s, t without
 * forming HW (used by the recompute composition). */
GNNC_API int gc_node_proj_f32(const float *X, int64_t ld, int64_t n_rows, int64_t k2, int32_t heads,
                     int64_t head_stride, const float *a_src, const float *a_dst, float *s,
                     float *t, void *stream);

/* Fused LeakyReLU + edge softmax over each CSR row (gat.py:72-95):
 *   e = s[h,i] + t[h,j]; e = e < 0 ? e * slope : e;
 *   alpha[h*nnz + p] = exp(e - max_row) / sum_row
 * Rows without edges produce nothing.  Requires a square pattern.
 * heavy_rows (optional, device int32[n_heavy]): the rows longer than
 * gc_edge_softmax_heavy_threshold(n_rows, nnz) — each gets a whole CTA
 * instead of a lane group, so power-law hub rows do not serialise the launch.
 * NULL: every row goes to a lane group (same results). */
GNNC_API int gc_edge_softmax_heavy_threshold(int64_t n_rows, int64_t nnz);
GNNC_API int gc_edge_softmax_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *s,
                        const float *t, int32_t heads, float slope, int64_t n_rows,
                        int64_t nnz, const int32_t *heavy_rows, int64_t n_heavy,
                        float *alpha, void *stream);

/* Attention as an SDDMM over edges: per edge
 *   e = a_src[h]·HW[i, h] + a_dst[h]·HW[j, h]   (k2-wide dot products),
 * then the same LeakyReLU + edge softmax as gc_edge_softmax_f32 (same
 * heavy_rows convention).  The a_dst·HW_j term is gathered per edge
 * (edge-parallel, uniform chunks); the a_src·HW_i term is one dot per node
 * over row i of HW_self (ld_self; NULL: HW itself, a square pattern — a
 * rank's row block passes its own HW rows), staged in the caller-owned
 * s_work[heads * n_rows]. */
GNNC_API int gc_attn_sddmm_f32(const int32_t *row_ptr, const int32_t *col_idx, const float *HW,
                      int64_t ld, const float *HW_self, int64_t ld_self, int64_t k2,
                      int32_t heads, const float *a_src,
                      const float *a_dst, float slope, int64_t n_rows, int64_t nnz,
                      const int32_t *heavy_rows, int64_t n_heavy, float *s_work,
                      float *alpha, void *stream);

/* ---- hybrid aggregation: dense blocks on tcgen05 ------
 * For a unit-valued pattern Ã and D = diag(d), the aggregation
 *   C = D Ã D X   (both GCN compositions: dynamic directly, precompute as Ñ = DÃD)
 * is split into dense 0/1 blocks of Ã (degree-sorted corners, or all rows x
 * the T most-referenced "hub" columns) and the remaining edges.  The dense
 * part is a tensor-core product  C_dense = D · A_dense · (D X)[hub_cols]
 * over terms of (D X)[hub_cols]:
 *   GC_HUB_BF16X3: hi/mid/lo bf16 terms — an exact fp32 split;
 *   GC_HUB_F16X2:  hi/lo fp16 terms of s·D·X, s = 2^(13 - floor(log2 max|D X|))
 *                  — 22 significant bits above 2^-10·max, absolute error
 *                  <= 2^-23·max|D X| per element; 2/3 of the MMAs.
 *   GC_HUB_F16:    the hi fp16 term alone — 11 significant bits, the same
 *                  input rounding as a TF32 GEMM (for the 1e-2 parity mode
 *                  the TF32 update already runs in); 1/3 of the MMAs.
 *   GC_HUB_F16_MN: GC_HUB_F16 packed MN-major: Bt is fp16[T][Kp], the
 *                  gathered rows as they are (no transpose); requires
 *                  gc_hub_f16_mn_supported(K) (CTA pairs, K > 64) and
 *                  16-bit A blocks.
 * The 0/1 blocks are bf16 (BF16X3) or fp16 (F16X2, F16) — exact either way.  The
 * remaining edges are the ordinary SpMM launched with GC_ACCUMULATE on top.
 *
 * gc_hub_terms_rows(K): rows per term of the packed operand (K rounded up to
 *   the kernel's N tile); the packed operand is {terms * rows * T} 16-bit
 *   elements (terms = 3 for BF16X3, 2 for F16X2, 1 for F16).
 * gc_hub_pack: Bt[q][f][t] = term_q(X[hub_cols[t], f] * d_col[hub_cols[t]])
 *   (d_col may be NULL), zero for f >= K; T % 64 == 0.  F16X2 / F16 also need
 *   scale_ws (float[2], caller-owned): the max and 1/s for the GEMM.
 * gc_hub_gemm: C[i, f] = d_row[i] * sum_t A_hub[i, t] * (sum_q B_q)[f, t]
 *   (d_row may be NULL; flags: GC_RELU, GC_ACCUMULATE — C = relu?(C + ...)).
 *   A_hub row-major [n_rows x lda], T % 64 == 0, 16-byte aligned operands.
 *   CTA pairs (tcgen05.mma.cta_group::2) when K > 16.                      */
#define GC_HUB_BF16X3 0
#define GC_HUB_F16X2 1
#define GC_HUB_F16 2
#define GC_HUB_F16_MN 3
GNNC_API int64_t gc_hub_terms_rows(int64_t K);
GNNC_API int gc_hub_pack(const float *X, int64_t ldx, int64_t K, const int32_t *hub_cols,
                int64_t T, const float *d_col, int32_t fmt, void *Bt, float *scale_ws,
                void *stream);
/* The TF32 GEMM with the TF32 class's gather operand as output: per row of
 * C = diag(row_scale) A W, Xh[row,:] = fp16_rn(C[row,:] * 2^-e) (max in
 * [2^14, 2^15); ldh = N rounded up to 8, pad zeroed) and sigma[row] = 2^e —
 * what gc_pack_rows_f16 makes of C, without writing C.  N <= 256: the whole
 * row in one TMEM tile (two passes over it in the epilogue), one scale per
 * row; N a multiple of 256: one scale per row and 256-column chunk, sigma
 * is M x (N/256) (consumers pass GC_SPMM_SIG_CHUNKS / GC_HUB_SIG_CHUNKS);
 * workspace as gc_gemm_f32. */
GNNC_API int gc_gemm_f16rows_f32(const float *A, int64_t lda, const float *W, int64_t ldw,
                                 int64_t M, int64_t K, int64_t N, const float *row_scale,
                                 void *Xh, int64_t ldh, float *sigma, void *workspace,
                                 size_t ws_bytes, void *stream);

/* gc_hub_pack from the fp16 gather operand (gc_pack_rows_f16): x_j =
 * sigma_j * Xh[j,:] (ldh in elements); one-term formats GC_HUB_F16 /
 * GC_HUB_F16_MN only (the TF32 class).  Lets the dense part and the tail of
 * the split read one operand. */
GNNC_API int gc_hub_pack_f16rows(const void *Xh, int64_t ldh, const float *sigma, int64_t K,
                                 const int32_t *hub_cols, int64_t T, const float *d_col,
                                 int32_t fmt, void *Bt, float *scale_ws, void *stream);
GNNC_API int gc_hub_gemm(const void *A_hub, int64_t lda, int64_t n_rows, int64_t T,
                const void *Bt, int64_t K, int32_t fmt, const float *scale_ws, float *C,
                int64_t ldc, const float *d_row, uint32_t flags, void *stream);

/* Staircase of dense blocks (degree-rank order).  Step s (0 <= s < n_steps
 * <= 16) is A_steps[s]: row-major [step_rows[s] x step_width[s]], the 0/1
 * adjacency of the step_rows[s] highest-degree rows (rank order) against the
 * hub columns at positions [step_c0[s], step_c0[s] + step_width[s]) of the
 * packed operand Bt (gc_hub_pack over T hub columns in rank order).  Rows
 * shrink and column ranges are consecutive across steps.  Rank row r of the
 * result goes to C row row_map[r] (NULL: r):
 *   C[row_map[r], f] = d_row[row_map[r]] * sum_{s: r < rows[s]} A_s[r, :] · B[.., c0_s ..]
 * One CTA-pair tcgen05 launch; flags GC_RELU / GC_ACCUMULATE.  Requires
 * gc_hub_stair_supported(K).  Optional static schedule (device int32):
 * n_clusters CTA pairs, pair c runs work items items[cluster_start[c] ..
 * cluster_start[c+1]), item = {tile, first k-block, end k-block (-1: to the
 * end), workspace slot (-1: write C)}, tile = m_pair * n_tiles + n_tile
 * (m_pair: 256 rank-ordered rows, n_tile: gc_hub_stair_pair_bn(K) columns);
 * NULL: round-robin whole tiles.  Split-K: items with a slot write their
 * (row-scaled) partial tile to workspace[slot][256][pair_bn]; fixups
 * {tile, first slot, slot count, 0} then add the partials to C in slot
 * order (deterministic; no GC_RELU with split items).
 * GC_HUB_A_BITS: A_steps[s] is instead a bitmap of uint64 words, word
 * (k, r) at index k * rpad_s + r (rpad_s = step_rows[s] rounded up to 256,
 * padding rows zero), bit j = A_s[r, 64k + j]; converter warps expand each
 * 128 x 64 tile into the 16-bit operand in shared memory (16x fewer A bytes). */
/* C[rows[i], :K] = 0 for i < n_rows (the rows outside every staircase step,
 * zeroed before the tail accumulates).                                    */
GNNC_API int gc_zero_rows(float *C, int64_t ldc, const int32_t *rows, int64_t n_rows, int64_t K,
                void *stream);
GNNC_API int gc_hub_stair_supported(int64_t K);
GNNC_API int gc_hub_f16_mn_supported(int64_t K);
GNNC_API int gc_hub_stair_pair_bn(int64_t K);
GNNC_API int gc_hub_stair_gemm(const void *const *A_steps, const int64_t *step_rows,
                const int64_t *step_c0, const int64_t *step_width, int32_t n_steps,
                const int32_t *row_map, const int32_t *items, const int32_t *cluster_start,
                int32_t n_clusters, float *workspace, const int32_t *fixups, int32_t n_fixups,
                const void *Bt, int64_t T, int64_t K, int32_t fmt, const float *scale_ws,
                float *C, int64_t ldc, const float *d_row, uint32_t flags, void *stream);

/* ---- multi-GPU row partition -----------------
 * nnz-balanced contiguous row blocks over a HOST copy of row_ptr (int64):
 *   bounds[0] = 0, bounds[P] = n, bounds[p] = first r with row_ptr[r] >=
 *   ceil(p*nnz/P).  Bit-exact with the oracle restatement.              */
GNNC_API int gc_partition_rows(const int64_t *row_ptr_host, int64_t n_rows, int32_t parts,
                      int64_t *bounds_host);

#ifdef __cplusplus
}
#endif
#endif /* GNNC_H_ */
