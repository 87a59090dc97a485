/*
 * graphmill_b200.h — C-ABI of the B200-native message-passing hot path.
 *
 * Drop-in boundary for the reference engine `graphmill` (/root/reference/proj).
 * Every entry point names the reference interface it replaces (file:line,
 * relative to /root/reference/proj). Conventions:
 *   - plain pointers and sizes only; array arguments are DEVICE pointers unless
 *     the parameter name ends in `_host`;
 *   - the caller owns every buffer (the library never allocates or frees caller
 *     memory); scratch comes from caller-supplied workspace with a size query;
 *   - every call is stream-ordered on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and reentrant; no exceptions cross the ABI: a call returns
 *     a gm_status and gm_last_error() holds a thread-local message shaped like
 *     the reference's exception text (e.g. "EdgeIndex: src index 7 at position
 *     3 outside [0, 5)", edge_index.cpp:19-25);
 *   - indices on the device are int32 for col/perm/argmax (all configured
 *     graphs have N, E < 2^31; checked) and int64 for rowptr, matching the
 *     reference's int64 `Index` (tensor.hpp:23) at the boundary arrays keys/values.
 */
#ifndef GRAPHMILL_B200_H
#define GRAPHMILL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GM_API __attribute__((visibility("default")))

typedef void* gm_stream_t; /* cudaStream_t */

typedef enum gm_status {
  GM_OK = 0,
  GM_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  GM_ERR_OUT_OF_RANGE = 2,     /* reference: std::out_of_range */
  GM_ERR_CUDA = 3,
  GM_ERR_UNSUPPORTED = 4,
  GM_ERR_LOGIC = 5,            /* reference: std::logic_error */
  GM_ERR_RUNTIME = 6,          /* reference: std::runtime_error (dataset IO) */
  GM_ERR_NCCL = 7
} gm_status;

typedef enum gm_dtype { GM_F32 = 0, GM_F64 = 1, GM_BF16 = 2 } gm_dtype;

/* aggregate.hpp:13 AggKind subset on the hot path. */
typedef enum gm_reduce { GM_SUM = 0, GM_MEAN = 1, GM_MAX = 2, GM_MIN = 3 } gm_reduce;

/* Thread-local message of the last failing call on this thread. */
GM_API const char* gm_last_error(void);
GM_API const char* gm_version(void);
/* 1 if this build's kernels can run on the current device (sm_100). */
GM_API int gm_device_supported(void);

/* ------------------------------------------------------------------------ */
/* Graph structure (L1): edge_index.hpp:22-29 CsrView, edge_index.cpp:45-62  */
/* ------------------------------------------------------------------------ */

/* Device CSR/CSC view. rowptr[num_rows+1] (int64), col[nnz] and perm[nnz]
 * (int32, compressed position -> COO position). Same meaning as CsrView. */
typedef struct gm_csr {
  int64_t num_rows;
  int64_t num_cols;
  int64_t nnz;
  const int64_t* rowptr;
  const int32_t* col;
  const int32_t* perm;
} gm_csr;

/* Replaces edge_index.cpp:19-25 check_bounds / tensor.hpp:489-495
 * check_index_range: first position i with ids[i] outside [0, bound).
 * Returns GM_ERR_OUT_OF_RANGE with message "<prefix> index X at position i
 * outside [0, bound)". Synchronizes `stream` (the result decides control flow).
 * workspace >= 64 bytes of device memory. */
GM_API gm_status gm_check_index_bounds(const int64_t* ids, int64_t len, int64_t bound,
                                       const char* prefix, void* workspace, gm_stream_t stream);

/* Replaces edge_index.cpp:28-32 first_unsorted (claim verification,
 * edge_index.cpp:88-95): writes the first position violating non-decreasing
 * order, or -1, to *pos_host. Synchronizes. workspace >= 64 bytes. */
GM_API gm_status gm_first_unsorted(const int64_t* keys, int64_t len, int64_t* pos_host,
                                   void* workspace, gm_stream_t stream);

/* Replaces the is_undirected claim check (edge_index.cpp:98-118): writes the
 * first COO position i whose pair multiplicity count(src[i], dst[i]) differs
 * from count(dst[i], src[i]), or -1 if the edge multiset is symmetric, to
 * *pos_host (radix sort of the pair keys + per-position binary searches).
 * n = num_src_nodes = num_dst_nodes. Synchronizes. */
GM_API size_t gm_first_asymmetric_workspace(int64_t len);
GM_API gm_status gm_first_asymmetric(const int64_t* src, const int64_t* dst, int64_t len, int64_t n,
                                     int64_t* pos_host, void* workspace, size_t workspace_bytes,
                                     gm_stream_t stream);

/* Occurrence counts of ids in [0, n) into deg[n] (int32); ids outside are
 * skipped (message_passing.hpp:76-78 spmm-mean degree; 441-443 full-array
 * degrees of gcn_norm). */
GM_API gm_status gm_degree(const int64_t* ids, int64_t len, int64_t n, int32_t* deg,
                           gm_stream_t stream);

/* Replaces build_compressed (edge_index.hpp:120-121, edge_index.cpp:45-62):
 * stable counting sort of (keys, values) into a CSR. Bit-exact: within each
 * row entries are in ascending COO position; perm[k] = COO position;
 * col[k] = values[perm[k]]. keys must lie in [0, num_rows) (check first with
 * gm_check_index_bounds, as EdgeIndex's constructor does). */
GM_API size_t gm_build_compressed_workspace(int64_t num_edges, int64_t num_rows);
GM_API gm_status gm_build_compressed(const int64_t* keys, const int64_t* values,
                                     int64_t num_edges, int64_t num_rows, int64_t* rowptr,
                                     int32_t* col, int32_t* perm, void* workspace,
                                     size_t workspace_bytes, gm_stream_t stream);

/* out[k] = in[perm[k]] for nnz elements of dtype: edge values in COO order ->
 * compressed order (the `w[perm[k]]` lookup of message_passing.hpp:68, done
 * once and cached instead of per edge). A raw element move: GM_F64 also moves
 * int64 index arrays (EdgeIndex::sort_by's new src/dst, edge_index.cpp:152-160). */
GM_API gm_status gm_permute_edge_values(gm_dtype dtype, const void* in, const int32_t* perm,
                                        int64_t nnz, void* out, gm_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Aggregation (L2/L3): spmm, the max path and GCN norm                      */
/* ------------------------------------------------------------------------ */

/* Scheduling metadata for gm_spmm, computed once per CSR (cache it next to
 * the CSR like EdgeIndex caches its CsrView, edge_index.hpp:94-103):
 * destination rows are split into nnz-balanced windows of ~window_edges edges
 * (win_row[num_windows+1]) for the warp-per-row kernel, and rows longer than
 * heavy_threshold go to a CTA-per-row pipelined kernel, longest first
 * (heavy_rows[num_heavy]). Pure scheduling: results do not depend on it. */
#define GM_PLAN_CLASSES 128
typedef struct gm_spmm_plan {
  int64_t num_windows;
  int64_t window_edges;
  int64_t num_heavy;
  int64_t heavy_threshold;
  const int32_t* win_row;
  const int32_t* heavy_rows;
  /* The same windows split around heavy rows: (first_row, end_row) pairs of
   * heavy-free row runs, streamed edge-contiguously by the flat kernel. */
  int64_t num_light_windows;
  const int32_t* light_windows;
  /* L2 residency hint (B200: 126 MB L2). Per compressed entry, the hotness
   * class of its source row: floor(4*log2(1 + G)), G = number of source rows
   * with a strictly larger out-degree. Gathers of rows whose class fits the
   * l2_hot_bytes budget use an L2 evict_last policy, all others evict_first,
   * so power-law hub rows stay L2-resident for the whole sweep. The caller
   * may change l2_hot_bytes between calls (0 disables the hint). */
  const uint8_t* src_class;
  int64_t l2_hot_bytes;
  /* hot_edge_frac[c]: share of the entries whose source class is < c. gm_spmm
   * applies the hint only when the rows that fit l2_hot_bytes serve at least
   * 15% of the gathers (the per-entry class read and policy select cost more
   * than they save on flat degree distributions, e.g. papers100M-shaped). */
  float hot_edge_frac[GM_PLAN_CLASSES];
} gm_spmm_plan;

GM_API size_t gm_spmm_plan_bytes(int64_t num_rows, int64_t num_cols, int64_t nnz);
/* Builds the plan into `buffer` (device, gm_spmm_plan_bytes) and fills
 * *plan_host. On entry plan_host->heavy_threshold may raise the hub-row
 * threshold above the default 1024 (0 = default; rows >= 1 KB wide do best
 * with 4096) and plan_host->window_edges may fix the window size (0 = auto:
 * 1024 entries, halved down to 256 until there are >= 8 waves of warps; rows
 * >= 1 KB wide do best with 256). Synchronizes once (reads the heavy-row count). */
GM_API gm_status gm_spmm_plan_build(const gm_csr* csr, void* buffer, size_t buffer_bytes,
                                    gm_spmm_plan* plan_host, gm_stream_t stream);

/* GCN degree normalisation fused into the SpMM (message_passing.hpp:437-463,
 * 490-495): per edge (s -> v) the scale is 1 / sqrt(float(deg_src[s]) *
 * float(deg_dst[v])), exactly as gcn_norm forms it (no rsqrt products). With
 * self_loops != 0 every row v gets a final term for the self loop (v, v),
 * which with_self_loops appends after all edges (edge_index.cpp:218-231) and
 * therefore comes last in CSC order. deg arrays are the effective degrees
 * (square: din+1 from the FULL dst array; bipartite: dout/din clamped >= 1),
 * see gm_gcn_degrees.
 * Layer epilogue, fused into the same store (no separate elementwise kernel):
 * bias (NULL or [f] of the accumulation type: float for F32/BF16, double for
 * F64) is added after the row's last term — layer_update's add(agg, bias),
 * message_passing.hpp:578 — and relu != 0 then applies the model's
 * inter-layer relu (message_passing.hpp:637, tensor.hpp:393-396:
 * v > 0 ? v : 0), both in the accumulation type before the final narrowing. */
typedef struct gm_gcn_norm {
  const int32_t* deg_src;
  const int32_t* deg_dst;
  int self_loops;
  const void* bias;
  int relu;
} gm_gcn_norm;

/* Effective GCN degrees (message_passing.hpp:441-460): square != 0 ->
 * deg_src = deg_dst = din + 1 (both arrays of length n_dst, may alias);
 * else deg_src = max(dout, 1) [n_src], deg_dst = max(din, 1) [n_dst].
 * full_src/full_dst: the base index's FULL arrays (trimmed views normalise
 * like the untrimmed graph). */
GM_API gm_status gm_gcn_degrees(const int64_t* full_src, const int64_t* full_dst, int64_t len,
                                int64_t n_src, int64_t n_dst, int square, int32_t* deg_src,
                                int32_t* deg_dst, gm_stream_t stream);

/* Replaces spmm (message_passing.hpp:92-169 forward, spmm_forward 47-85) and
 * the max/min path (message_passing.hpp:508-514 = dst_grouped_order 190-214 +
 * gather_rows tensor.hpp:499-530 + aggregate aggregate.hpp:197-215), fused:
 *   out[v] = reduce_{k in row v of csr} scale_k * x[col[k]]
 * csr: the destination grouping (EdgeIndex::transpose_view()).
 * x: [csr->num_cols, f] row-major of dtype. out: [csr->num_rows, f].
 * edge_weight: NULL or per-edge scale in COMPRESSED order (gm_permute_edge_values).
 * gcn: NULL or fused GCN norm (exclusive with edge_weight).
 * reduce: SUM, MEAN (sum * (1/deg), deg = row length; message_passing.hpp:76-84),
 *   MAX/MIN (first element initialises, then strict >/<; empty rows 0).
 * arg_out: NULL or 16-byte aligned int32 [num_rows, f]: COO edge id (perm[k]) of the first
 *   attaining edge, -1 for empty rows (MAX/MIN only; the reference keeps this
 *   only inside its backward closure, aggregate.hpp:295-308). Requires perm.
 * Accumulation is fp32 for F32/BF16 (BF16 in, BF16 out, RNE) and fp64 for F64,
 * sequential per output element in compressed order with no FMA contraction,
 * i.e. bit-identical to the reference for F32/F64. */
GM_API gm_status gm_spmm(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype,
                         const void* x, int64_t f, const void* edge_weight,
                         const gm_gcn_norm* gcn, gm_reduce reduce, void* out, int32_t* arg_out,
                         gm_stream_t stream);

/* Backward of spmm (message_passing.hpp:119-166). With g the gradient of the
 * output [n_dst, f]:
 *   scaled_g = mean ? g / S(max(deg_dst, 1)) : g           gm_scale_rows_div (:128-132)
 *   dx = gm_spmm(CSR by source, scaled_g, w in CSR order)   transposed product (:133-155)
 *   dw[i] = sum_j scaled_g[dst[i]][j] * x[src[i]][j]       gm_edge_dot (:156-165)
 * f32/f64, bit-identical to the reference's closure (sequential order, no FMA). */
GM_API gm_status gm_scale_rows_div(gm_dtype dtype, const void* in, int64_t rows, int64_t f,
                                   const int32_t* deg, void* out, gm_stream_t stream);
GM_API gm_status gm_edge_dot(gm_dtype dtype, const int64_t* src, const int64_t* dst, int64_t num_edges,
                             const void* a_by_dst, const void* b_by_src, int64_t f, void* out,
                             gm_stream_t stream);

/* dw in destination-grouped order (same result as gm_edge_dot, bit-identical):
 * entry k of the CSC view pairs a_by_dst[entry_rows[k]] with b_by_src[col[k]]
 * and writes out[perm[k]] (COO order). Consecutive entries share the
 * destination row, so its gradient row is fetched once per row run instead of
 * once per edge. entry_rows: gm_csr_entry_rows of the same view (int32 per
 * entry, indexed from the view's first entry); cache it beside the view.
 * plan (optional, gm_spmm_plan_build of the same view): its source hotness
 * classes give the source-row gathers gm_spmm's L2 residency policy. */
GM_API gm_status gm_csr_entry_rows(const gm_csr* csr, int32_t* rows_out, gm_stream_t stream);
GM_API gm_status gm_edge_dot_csc(gm_dtype dtype, const gm_csr* csc, const gm_spmm_plan* plan,
                                 const int32_t* entry_rows, const void* a_by_dst, const void* b_by_src, int64_t f,
                                 void* out, gm_stream_t stream);

/* Backward of the max/min aggregation path (message_passing.hpp:508-514):
 * the argpos scatter of aggregate's closure (aggregate.hpp:295-308) followed by
 * the gather_rows adjoint (tensor.hpp:510-524), fused and without atomics.
 * gm_source_view builds, once per graph, the "source view" of a CSC: per
 * source node its entries in ascending CSC position (rowptr[n_src+1], col =
 * destination node, eid = COO edge id) — a stable counting sort of the CSC
 * sequence by source. Then
 *   dx[s][j] = sum over the view's row s, in order, of g[v][j] where
 *              arg[v][j] == eid  (arg: gm_spmm's MAX/MIN arg_out)
 * accumulated sequentially from +0 — bit-identical to the reference tape
 * (the non-winning positions it adds are exact zeros). plan: gm_spmm_plan_build
 * of the source view (hub sources take a column-parallel kernel). f32/f64;
 * dx [n_src, f] is fully written. */
GM_API size_t gm_source_view_workspace(int64_t nnz, int64_t n_src);
GM_API gm_status gm_source_view(const gm_csr* csc, int64_t n_src, int64_t* rowptr, int32_t* col, int32_t* eid,
                                void* workspace, size_t workspace_bytes, gm_stream_t stream);
GM_API gm_status gm_spmm_max_backward(const gm_csr* source_view, const gm_spmm_plan* plan, gm_dtype dtype,
                                      const int32_t* arg, const void* g, int64_t f, void* dx, gm_stream_t stream);

/* Heterogeneous combine (hetero.hpp:338-343 InterCombine::sum, then
 * layer_update hetero.hpp:362 / message_passing.hpp:579-580 for SAGE):
 *   out = ((((parts[0] + parts[1]) + ...) + self_term) + bias)   fp32, in this
 * order; parts are the per-edge-type results for one destination node type in
 * sorted canonical edge-type order (host array of <= 8 device pointers, each
 * [rows, f]); self_term [rows, f] and bias [f] may be NULL. */
GM_API gm_status gm_hetero_combine(const float* const* parts, int32_t n_parts, const float* self_term,
                                   const float* bias, int64_t rows, int64_t f, float* out,
                                   gm_stream_t stream);

/* ------------------------------------------------------------------------ */
/* segment_matmul (L4): hetero.hpp:134-157 grouped_matmul                    */
/* ------------------------------------------------------------------------ */

/* out[ptr[g]:ptr[g+1], :] = x[ptr[g]:ptr[g+1], :] @ w[g] for g < groups.
 * x: [ptr_host[groups], k] row-major BF16; w: [groups, k, n] row-major BF16
 * (the reference's stacked W[G,F,F'] layout); out: [rows, n] of out_dtype
 * (GM_BF16 or GM_F32). tcgen05 (UMMA) tensor cores, fp32 accumulation in
 * TMEM, TMA-fed. ptr_host is a HOST array of groups+1 non-decreasing offsets
 * (ptr_host[0] = 0). Empty groups produce no rows (0 x n, hetero.hpp:131).
 * Any K, N >= 1 and groups <= 128: K % 64 == 0 and N % 16 == 0 run in place
 * (16-byte aligned x/out); other shapes run zero-padded through the
 * workspace. N > 256 is tiled in 256-wide column tiles.
 * workspace: gm_segment_matmul_workspace(rows = ptr_host[groups], ...) bytes
 * (K-major W^T copy, plus padded x / out for odd shapes). */
GM_API size_t gm_segment_matmul_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n);
GM_API gm_status gm_segment_matmul(const void* x, const int64_t* ptr_host, int64_t groups,
                                   int64_t k, int64_t n, const void* w, gm_dtype out_dtype,
                                   void* out, void* workspace, size_t workspace_bytes,
                                   gm_stream_t stream);

/* Pre-packed weights (serving: pack once, reuse every call): the K-major,
 * zero-padded W^T that gm_segment_matmul otherwise rebuilds per call.
 * packed: gm_segment_matmul_packed_w_bytes(groups, k, n) device bytes. */
GM_API size_t gm_segment_matmul_packed_w_bytes(int64_t groups, int64_t k, int64_t n);
GM_API gm_status gm_segment_matmul_pack_w(const void* w, int64_t groups, int64_t k, int64_t n, void* packed,
                                          gm_stream_t stream);
GM_API size_t gm_segment_matmul_packed_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n);
GM_API gm_status gm_segment_matmul_packed(const void* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                          int64_t n, const void* packed_w, gm_dtype out_dtype, void* out,
                                          void* workspace, size_t workspace_bytes, gm_stream_t stream);
/* fp32 activations x bf16 pre-packed weights, fp32 out: x is read once as fp32
 * by the GEMM kernel and rounded to bf16 (RNE) in shared memory — the same
 * operands as casting x to bf16 first, without the separate cast pass.
 * Requires k % 4 == 0 and x 16-byte aligned; workspace as
 * gm_segment_matmul_packed_workspace. */
GM_API gm_status gm_segment_matmul_packed_xf32(const float* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                               int64_t n, const void* packed_w, float* out, void* workspace,
                                               size_t workspace_bytes, gm_stream_t stream);

/* fp32 grouped_matmul (hetero.hpp:134-157 with S = float) at fp32 accuracy on
 * the tcgen05 tensor pipe: each fp32 operand is split into three bf16 pieces
 * (hi, mid, lo; residual <= 2^-27 |v|) and fp32 TMEM accumulators collect the
 * six products hi*hi + hi*mid + mid*hi + hi*lo + lo*hi + mid*mid down to 2^-18
 * scale: |out - x W| <= 1e-5 * sum_k |x_ik||W_kj| (the north_star fp32 GEMM
 * bar). When k % 4 == 0 and x is 16-byte aligned the split of x happens inside
 * the GEMM kernel (x read once); otherwise x is split into a staged piece
 * matrix first. x [rows, k], w [groups, k, n], out [rows, n], all f32
 * row-major; the workspace size covers either route. */
GM_API size_t gm_segment_matmul_f32_workspace(int64_t rows, int64_t groups, int64_t k, int64_t n);
GM_API gm_status gm_segment_matmul_f32(const float* x, const int64_t* ptr_host, int64_t groups, int64_t k,
                                       int64_t n, const float* w, float* out, void* workspace, size_t workspace_bytes,
                                       gm_stream_t stream);

/* grouped_matmul over SEPARATE per-group tensors — the reference's
 * grouped_matmul(vector<Tensor> inputs, Tensor W[G,F,F']) (hetero.hpp:134-157):
 * out_host[g] = x_host[g] @ w[g] for groups of rows_host[g] rows (host arrays
 * of device pointers). Operands (x_dtype, w_dtype): (F32, F32) fp32-accurate
 * split route, out F32; (F32, BF16) x rounded to bf16 inside the kernel, out
 * F32; (BF16, BF16) out BF16 or F32. With <= 8 groups, n % 16 == 0, x f32
 * k % 4 == 0 / x bf16 k % 64 == 0 and 16-byte aligned pointers, one kernel
 * reads and writes every group in place through per-group TMA maps (no
 * concatenation); otherwise the groups are gathered into the workspace and
 * scattered back (stream-ordered copies). */
GM_API size_t gm_grouped_matmul_workspace(const int64_t* rows_host, int64_t groups, int64_t k, int64_t n,
                                          gm_dtype x_dtype, gm_dtype w_dtype, gm_dtype out_dtype);
GM_API gm_status gm_grouped_matmul(const void* const* x_host, const int64_t* rows_host, int64_t groups, int64_t k,
                                   int64_t n, const void* w, gm_dtype x_dtype, gm_dtype w_dtype,
                                   void* const* out_host, gm_dtype out_dtype, void* workspace, size_t workspace_bytes,
                                   gm_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU partitioning (north_star: dst-row partition + source all-gather) */
/* ------------------------------------------------------------------------ */

/* nnz-balanced contiguous destination-row cuts: cuts_host[p] = first row r
 * with rowptr[r] >= p * nnz / parts (cuts_host[0] = 0, cuts_host[parts] =
 * num_rows). rowptr_host is a HOST copy of the CSR row pointer. */
GM_API gm_status gm_partition_rows_by_nnz(const int64_t* rowptr_host, int64_t num_rows,
                                          int32_t parts, int64_t* cuts_host);

/* Stable split of a (row-slice) CSR into num_blocks source blocks, for the
 * exchange-overlapped multi-GPU aggregation ("local CSR per GPU
 * is 2-D blocked by source shard"): entry k of row r moves to block
 * b = src_block[col[k]] with column src_col[col[k]] (e.g. the row inside the
 * peer shard / exchange chunk that will hold that source) and keeps perm[k].
 * Inside each (block, row) entries keep their compressed order, so each
 * block is itself a valid compressed view of the same rows.
 * Outputs: rowptr_out [num_blocks][num_rows+1] (block b's view is
 * {rowptr_out + b*(num_rows+1), col_out, perm_out}, offsets into the shared
 * col_out/perm_out arrays of csr->nnz entries). src_block/src_col are device
 * arrays of csr->num_cols entries; src_block values in [0, num_blocks). */
GM_API size_t gm_csr_split_blocks_workspace(int64_t num_rows, int32_t num_blocks);
GM_API gm_status gm_csr_split_blocks(const gm_csr* csr, const int32_t* src_block, const int32_t* src_col,
                                     int32_t num_blocks, int64_t* rowptr_out, int32_t* col_out,
                                     int32_t* perm_out, void* workspace, size_t workspace_bytes,
                                     gm_stream_t stream);

/* Halo exchange helpers (SURVEY.md §8e "halo-only variant"): mark[c] = 1 for
 * every column c referenced by the CSR's rows (num_cols bytes, zeroed first);
 * out[i] = x[idx[i]] row gather (the per-peer send pack, f elements of dtype). */
GM_API gm_status gm_mark_columns(const gm_csr* csr, uint8_t* mark, gm_stream_t stream);
GM_API gm_status gm_gather_rows(gm_dtype dtype, const void* x, int64_t f, const int32_t* idx, int64_t n, void* out,
                                gm_stream_t stream);

/* Continue an aggregation over another block of the same destination rows
 * (gm_csr_split_blocks): every row starts from the current out (and, for
 * MAX/MIN, arg_out) contents and accumulates this block's entries in
 * compressed order. MAX/MIN break ties on the smaller COO id (arg_out
 * required), so the value and argmax equal the single-pass result exactly for
 * NaN-free inputs whatever the block order; SUM continues the running sum (one
 * re-association per block boundary: within the fp32 tolerance, not
 * bit-identical). reduce = MEAN finalises: sum, then * (1 / mean_deg[row])
 * with mean_deg the FULL row degrees (earlier blocks run as SUM). F32/F64 for
 * SUM/MEAN (BF16 would round between blocks); any dtype for MAX/MIN. */
GM_API gm_status gm_spmm_accumulate(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype,
                                    const void* x, int64_t f, const void* edge_weight, gm_reduce reduce,
                                    const int32_t* mean_deg, void* out, int32_t* arg_out,
                                    gm_stream_t stream);

/* Epilogue extras of gm_spmm_ex (either part may be unused):
 *  - fp32 carry for bf16 sums continued across source blocks (multi-GPU
 *    overlap): carry_mode GM_CARRY_START starts the rows at 0 and stores fp32
 *    rows to `carry`; GM_CARRY_CONTINUE seeds each row from `carry` and stores
 *    it back; GM_CARRY_FINISH seeds from `carry` and stores the row rounded
 *    (RNE) to `out` — one rounding per row, as on one GPU. bf16 sum/mean only.
 *  - push: every finished output row is also stored, as `out` holds it, into
 *    up to GM_MAX_PUSH peer buffers at global row push_row0 + local row (the
 *    peers' [num_global_rows, f] input of the next layer, mapped into this
 *    process: CUDA IPC / VMM over NVLink). push_mask[r] bit q selects peer q
 *    for local row r (NULL: every peer). The caller orders the peers' later
 *    reads after this call (e.g. a collective on `stream`). push_mask bit j
 *    refers to push_dst[j]. Unweighted layers (sum / mean / max / min: the
 *    values are pushed, arg_out stays local). */
#define GM_MAX_PUSH 8
typedef enum { GM_CARRY_NONE = 0, GM_CARRY_START = 1, GM_CARRY_CONTINUE = 2, GM_CARRY_FINISH = 3 } gm_carry_mode;
typedef struct gm_spmm_epilogue {
  float* carry;
  int32_t carry_mode;
  int32_t n_push;
  void* push_dst[GM_MAX_PUSH];
  int64_t push_row0;
  const uint32_t* push_mask;
} gm_spmm_epilogue;
/* gm_spmm (accumulate = 0) / gm_spmm_accumulate (accumulate = 1: every row
 * continues from out / arg_out, or from the carry for CONTINUE / FINISH) with
 * an epilogue (NULL: none). */
GM_API gm_status gm_spmm_ex(const gm_csr* csr, const gm_spmm_plan* plan, gm_dtype dtype, const void* x, int64_t f,
                            const void* edge_weight, gm_reduce reduce, int32_t accumulate, const int32_t* mean_deg,
                            const gm_spmm_epilogue* epilogue, void* out, int32_t* arg_out, gm_stream_t stream);

/* Peer memory for the push epilogue: export a device pointer (CUDA IPC handle
 * of its allocation + the pointer's offset, gm_ipc_handle_bytes() bytes), open
 * a peer's export (NVLink P2P mapping; *base_out is what gm_ipc_close_handle
 * takes). */
GM_API size_t gm_ipc_handle_bytes(void);
GM_API gm_status gm_ipc_get_handle(const void* dev_ptr, void* handle_out);
GM_API gm_status gm_ipc_open_handle(const void* handle, void** dev_ptr_out, void** base_out);
GM_API gm_status gm_ipc_close_handle(void* base);

/* Multi-GPU SpMM over NCCL (north_star: dst-row partition + source exchange).
 * ncclComm_t is NCCL's own handle (struct ncclComm*); the library resolves
 * NCCL at run time (dlopen libnccl.so.2). Hosts without their own NCCL
 * bootstrap can use gm_nccl_unique_id (128 bytes, to broadcast out of band)
 * and gm_nccl_comm_init. */
typedef struct ncclComm* ncclComm_t;
GM_API gm_status gm_nccl_unique_id(void* id_out);
GM_API gm_status gm_nccl_comm_init(int32_t world, const void* id, int32_t rank, ncclComm_t* comm);
GM_API gm_status gm_nccl_comm_destroy(ncclComm_t comm);

typedef enum gm_dist_mode {
  GM_DIST_EXACT = 0,   /* one all-gather, one gm_spmm: bit-identical to one GPU */
  GM_DIST_BLOCKED = 1, /* `chunks` all-gathers overlapped with source-blocked aggregation */
  GM_DIST_HALO = 2     /* ncclSend/Recv of the referenced remote rows only, overlapped */
} gm_dist_mode;

/* One rank's view of the partitioned SpMM. X is row-sharded: rank q owns
 * shard rows [q * shard_rows, (q+1) * shard_rows) (last padded).
 *  EXACT:   blocks[0] = this rank's destination rows with GLOBAL source ids
 *           (the gathered X is [world * shard_rows, f]);
 *  BLOCKED: blocks[0..chunks] from gm_csr_split_blocks: block 0 = sources in
 *           the own shard (column = row inside x_shard, which is padded to
 *           chunks * chunk_rows rows), block 1+c = sources of exchange chunk c
 *           (column = q * chunk_rows + row inside the chunk);
 *  HALO:    blocks[0] = own shard, blocks[1] = halo rows (column = position in
 *           the receive buffer: peers in rank order, each ascending);
 *           halo_send_idx = rows of my shard each peer needs (peers in rank
 *           order), per-peer HOST counts of what I send / receive.
 * plans: gm_spmm_plan_build of each block. mean_deg: FULL row degrees (MEAN). */
typedef struct gm_dist_layout {
  int32_t rank;
  int32_t world;
  gm_dist_mode mode;
  int32_t chunks;
  int64_t shard_rows;
  int64_t chunk_rows;
  const gm_csr* blocks;
  const gm_spmm_plan* plans;
  const int32_t* mean_deg;
  const int32_t* halo_send_idx;
  const int64_t* halo_send_counts_host;
  const int64_t* halo_recv_counts_host;
} gm_dist_layout;

/* The exchange runs on comm_stream (gated on `stream` having reached the
 * call), aggregation on `stream`, each block waiting (device-side event) for
 * only the chunk it reads. Numerics: EXACT bit-identical to gm_spmm on the
 * full graph; BLOCKED/HALO: max/min + argmax bit-identical (NaN-free), sums
 * continued across blocks (fp32 tolerance; bf16 sum/mean refused — use EXACT).
 * workspace: gm_dist_spmm_workspace bytes (receive buffers); keep it alive
 * until `stream` has passed the call. */
GM_API size_t gm_dist_spmm_workspace(const gm_dist_layout* layout, gm_dtype dtype, int64_t f);
GM_API gm_status gm_dist_spmm(const gm_dist_layout* layout, gm_dtype dtype, const void* x_shard, int64_t f,
                              gm_reduce reduce, void* out, int32_t* arg_out, void* workspace,
                              size_t workspace_bytes, ncclComm_t comm, gm_stream_t comm_stream,
                              gm_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Dataset ingestion (L5): dataset_io.hpp:14-20 layout, load_dataset          */
/* (dataset_io.cpp:295-341) — straight to the device                          */
/* ------------------------------------------------------------------------ */

/* Reads a whole file (e.g. node_<type>.f32.bin, *.time.i64.bin) into device
 * memory dst. The file must hold exactly expected_bytes (else
 * GM_ERR_RUNTIME "dataset: <path> holds X bytes, manifest requires Y", the
 * reference's MappedFile check, dataset_io.cpp:107-119). staging: PINNED host
 * buffer, used as two halves so file reads overlap the host->device copies.
 * Synchronizes `stream` before returning. */
GM_API gm_status gm_read_file_to_device(const char* path, int64_t expected_bytes, void* dst, void* staging,
                                        size_t staging_bytes, gm_stream_t stream);

/* Reads edge_<src>__<rel>__<dst>.u64.bin (edge_count interleaved little-endian
 * (src, dst) u64 pairs) into device int64 src[edge_count], dst[edge_count]
 * (dataset_io.cpp:317-326; bounds are then checked by EdgeIndex, as in the
 * reference). workspace: DEVICE bytes >= gm_read_edge_pairs_workspace(staging_bytes).
 * Synchronizes. */
GM_API size_t gm_read_edge_pairs_workspace(size_t staging_bytes);
GM_API gm_status gm_read_edge_pairs_to_device(const char* path, int64_t edge_count, int64_t* src, int64_t* dst,
                                              void* staging, size_t staging_bytes, void* workspace,
                                              size_t workspace_bytes, gm_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Synthetic inputs (bench/test infrastructure; bit-identical host & device) */
/* ------------------------------------------------------------------------ */

/* kind 0 = uniform, 1 = power-law (Chung-Lu alpha = 0.5, permuted ids).
 * Generates edges [first, first+count) of the stream keyed by seed. */
GM_API gm_status gm_synth_edges(int kind, uint64_t seed, int64_t first, int64_t count,
                                int64_t n_src, int64_t n_dst, int64_t* src, int64_t* dst,
                                gm_stream_t stream);
GM_API void gm_synth_edges_host(int kind, uint64_t seed, int64_t first, int64_t count,
                                int64_t n_src, int64_t n_dst, int64_t* src, int64_t* dst);
/* Rows [first_row, first_row+rows) of an f-wide feature matrix, U[-1,1),
 * written as dtype (BF16 = RNE of the fp32 value). quantize: see synth.h. */
GM_API gm_status gm_synth_features(uint64_t seed, int64_t first_row, int64_t rows, int64_t f,
                                   int quantize, gm_dtype dtype, void* x, gm_stream_t stream);
GM_API void gm_synth_features_host(uint64_t seed, int64_t first_row, int64_t rows, int64_t f,
                                   int quantize, gm_dtype dtype, void* x);
/* Edge weights U[0.5, 1.5) for edges [first, first+count). */
GM_API gm_status gm_synth_weights(uint64_t seed, int64_t first, int64_t count, gm_dtype dtype,
                                  void* w, gm_stream_t stream);
GM_API void gm_synth_weights_host(uint64_t seed, int64_t first, int64_t count, gm_dtype dtype,
                                  void* w);

#ifdef __cplusplus
}
#endif
#endif /* GRAPHMILL_B200_H */
