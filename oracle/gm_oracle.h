/*
 * gm_oracle.h — CPU restatement of the reference's hot path (TEST
 * INFRASTRUCTURE ONLY).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker. The product path
 * (paper_2507_16991_b200/) never links or calls it.
 *
 * Parity pinning: every function here is checked bit-for-bit against the
 * reference itself compiled in place (oracle/_ref/libgraphmill_ref.so, built by
 * oracle/Makefile from /root/reference/proj) and against committed golden
 * fixtures generated from it (tests/golden/, tests/make_golden.py).
 *
 * All pointers are host pointers; all indices are int64 like the reference's
 * `Index` (tensor.hpp:23). Built with -ffp-contract=off so no FMA contraction
 * changes the rounding of `o[j] += w * x[j]`.
 */
#ifndef GM_ORACLE_H
#define GM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* edge_index.cpp:45-62 build_compressed: stable counting sort by `keys`. */
void or_build_compressed(const int64_t* keys, const int64_t* values, int64_t num_edges,
                         int64_t num_rows, int64_t* rowptr, int64_t* col, int64_t* perm);

/* message_passing.hpp:47-85 spmm_forward over a destination grouping
 * (rowptr/col/perm of transpose_view()). w_coo may be NULL (COO order, looked
 * up through perm, :68). mean != 0 scales by S(1)/S(deg) (:76-84), deg = row
 * length. Only rows listed in `rows` (NULL = all n_rows) are written, into
 * out[i*f] for the i-th listed row — the row-subset oracle for full-scale
 * sampled parity (per-row results are independent). */
void or_spmm_f32(const int64_t* rowptr, const int64_t* col, const int64_t* perm, int64_t n_rows,
                 const float* x, int64_t f, const float* w_coo, int mean, const int64_t* rows,
                 int64_t n_list, float* out);
void or_spmm_f64(const int64_t* rowptr, const int64_t* col, const int64_t* perm, int64_t n_rows,
                 const double* x, int64_t f, const double* w_coo, int mean, const int64_t* rows,
                 int64_t n_list, double* out);

/* message_passing.hpp:51-59 undirected + weights: COO sweep. */
void or_spmm_coo_f32(const int64_t* src, const int64_t* dst, int64_t num_edges, int64_t n_dst,
                     const float* x, int64_t f, const float* w, int mean, float* out);
void or_spmm_coo_f64(const int64_t* src, const int64_t* dst, int64_t num_edges, int64_t n_dst,
                     const double* x, int64_t f, const double* w, int mean, double* out);

/* Max/min path: dst_grouped_order (message_passing.hpp:190-214) + gather_rows
 * (tensor.hpp:499-530) + aggregate(max|min) (aggregate.hpp:197-215). First
 * element initialises, then strict `>` (`<` for min); empty rows give 0 and
 * arg -1. arg is the COO edge id of the first attaining edge (grouped
 * position mapped through perm). w_coo != NULL composes row_scale first
 * (tensor.hpp:553-588): value = x * w. Row-subset semantics as or_spmm_*. */
void or_spmm_max_f32(const int64_t* rowptr, const int64_t* col, const int64_t* perm,
                     int64_t n_rows, const float* x, int64_t f, const float* w_coo, int is_min,
                     const int64_t* rows, int64_t n_list, float* out, int64_t* arg);
void or_spmm_max_f64(const int64_t* rowptr, const int64_t* col, const int64_t* perm,
                     int64_t n_rows, const double* x, int64_t f, const double* w_coo, int is_min,
                     const int64_t* rows, int64_t n_list, double* out, int64_t* arg);

/* message_passing.hpp:437-463 gcn_norm. base_full_{src,dst}: the base index's
 * FULL arrays (lengths base_len). g_{src,dst}: the (self-loop augmented) graph
 * the norm is for. square != 0: din+1 both ends; else dout/din clamped >= 1. */
/* Backward of the max/min path (aggregate.hpp:295-308 + gather_rows adjoint
 * tensor.hpp:510-524): dx[n_src, f] from the CSC, the COO-id argmax and g. */
void or_spmm_max_backward_f32(const int64_t* rowptr, const int64_t* col, const int64_t* perm, int64_t n_rows,
                              const int64_t* arg, const float* g, int64_t f, int64_t n_src, float* dx);
void or_spmm_max_backward_f64(const int64_t* rowptr, const int64_t* col, const int64_t* perm, int64_t n_rows,
                              const int64_t* arg, const double* g, int64_t f, int64_t n_src, double* dx);
void or_gcn_norm_f32(const int64_t* base_full_src, const int64_t* base_full_dst, int64_t base_len,
                     int64_t n_src, int64_t n_dst, const int64_t* g_src, const int64_t* g_dst,
                     int64_t g_len, int square, float* norm);
void or_gcn_norm_f64(const int64_t* base_full_src, const int64_t* base_full_dst, int64_t base_len,
                     int64_t n_src, int64_t n_dst, const int64_t* g_src, const int64_t* g_dst,
                     int64_t g_len, int square, double* norm);

/* message_passing.hpp:119-166 spmm backward. csr_* : the CSR by SOURCE
 * (EdgeIndex::to_csr(), :143). g: grad of out [n_dst, f]. deg_dst != NULL
 * selects mean (scaled_g = g / S(max(deg, 1)), :128-132). w_coo may be NULL.
 * dx [n_src, f] (:133-155); dw [E] if w_coo && dw (:156-165, sequential in j,
 * over the COO arrays src/dst). */
void or_spmm_backward_f32(const int64_t* csr_rowptr, const int64_t* csr_col, const int64_t* csr_perm,
                          int64_t n_src, const int64_t* src, const int64_t* dst, int64_t num_edges,
                          const float* g, const float* x, int64_t f, const float* w_coo,
                          const int64_t* deg_dst, float* dx, float* dw);
void or_spmm_backward_f64(const int64_t* csr_rowptr, const int64_t* csr_col, const int64_t* csr_perm,
                          int64_t n_src, const int64_t* src, const int64_t* dst, int64_t num_edges,
                          const double* g, const double* x, int64_t f, const double* w_coo,
                          const int64_t* deg_dst, double* dx, double* dw);

/* Occurrence counts of ids in [0, n) (message_passing.hpp:76-78, 441-443). */
void or_degree(const int64_t* ids, int64_t len, int64_t n, int64_t* deg);

/* hetero.hpp:134-157 grouped_matmul in concatenated (segment) form:
 * out[ptr[g]:ptr[g+1]] = x[ptr[g]:ptr[g+1]] @ w[g], w is [G, K, N] row-major.
 * Plain ascending-k loop (Eigen's rounding is unpinned). */
void or_segment_matmul_f64(const double* x, const int64_t* ptr, int64_t groups, int64_t k,
                           int64_t n, const double* w, double* out);
void or_segment_matmul_f32(const float* x, const int64_t* ptr, int64_t groups, int64_t k,
                           int64_t n, const float* w, float* out);

#ifdef __cplusplus
}
#endif
#endif
