/*
 * ifmm_b200.h -- C ABI of the B200-native IFMM factorize+solve engine.
 *
 * Plain pointers and sizes only (no torch types).  Every entry point maps
 * onto one function of the reference Python package
 * (/root/reference/pkg/src/ifmm); the mapping is given per function as
 * `file:line`.  Status codes: 0 ok, 1 ValueError, 2 SingularPivotError,
 * 3 CUDA error, 4 out of device memory, 5 AssertionError (broken invariant).
 * `ifmm_last_error()` returns the message of the last failure on the
 * calling thread.  There is no CPU fallback: without a CUDA device every
 * compute entry point fails with status 3.
 */
#ifndef IFMM_B200_H
#define IFMM_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library / context ------------------------------------------------ */
int ifmm_abi_version(void);
const char* ifmm_last_error(void);
/* Device arena + stream.  arena_bytes == 0 -> 90% of free device memory. */
void* ifmm_ctx_create(int device, unsigned long long arena_bytes);
void ifmm_ctx_destroy(void* ctx);
/* Bytes of the arena in use / high-water mark. */
int ifmm_ctx_memory(void* ctx, unsigned long long* in_use, unsigned long long* peak);

/* ---- tree + topology:  tree.py:107-239 ---------------------------------
 * The octree itself (depth rule, Morton keys, stable sort; tree.py:107-196)
 * is built host-side in the Python mirror; this call receives it and
 * computes compute_topology (tree.py:205-239) natively.
 *   points: N x 3 Morton-sorted, perm: points[i] = original[perm[i]];
 *   per cluster: level, parent (-1 root),
 *   start, stop, cell (3 ints), center (3), half_width; children CSR.  */
void* ifmm_tree_create(void* ctx, int n_points, const double* points, const int* perm, int depth,
                       int n_clusters, const int* level, const int* parent,
                       const int* start, const int* stop, const long long* cell,
                       const double* center, const double* half_width,
                       const int* child_ptr, const int* child_idx);
void ifmm_tree_destroy(void* tree);
int ifmm_tree_topology_sizes(void* tree, long long* n_nbr, long long* n_int);
int ifmm_tree_topology(void* tree, long long* nbr_ptr, int* nbr_idx,
                       long long* int_ptr, int* int_idx);

/* ---- H2 operators:  h2.py:104-182 (chebyshev_operators) --------------
 * kernel_kind: 1 exp(-r), 2 inverse multiquadric 1/sqrt(r^2+p0^2),
 * 3 benchmark kernel (kernels.py:42-56, d = p0), 4 zero.              */
void* ifmm_h2_build(void* tree, int kernel_kind, double p0, int n_cheb, double epsilon);
/* Same with a second kernel parameter.  kernel_kind 5: Rotne-Prager-Yamakawa
 * mobility (kernels.py:59-91, block_dim 3: three unknowns per point,
 * point-major), p0 = particle radius a, p1 = 1 / (6 pi eta a).  Vectors of
 * an operator built on a block_dim-3 kernel have 3 * n_points entries.      */
void* ifmm_h2_build_k(void* tree, int kernel_kind, double p0, double p1, int n_cheb,
                      double epsilon);
void ifmm_h2_destroy(void* h2);
int ifmm_h2_ranks(void* h2, int* ranks_out /* n_clusters, -1 if none */);
/* initialize_weights, rigorous mode (h2.py:185-231). */
int ifmm_h2_weights(void* h2);
/* initialize_weights(mode="sampled") (h2.py:197-225, _sampled_gram h2.py:250-262):
 * sample_ptr (n_clusters + 1 offsets) / sample_idx hold, per cluster, the
 * sorted row sample of its basis the caller drew (the reference's
 * rng.choice stream); clusters with an empty interaction list have none.   */
int ifmm_h2_weights_sampled(void* h2, const long long* sample_ptr, const int* sample_idx);
/* Host copy of one stored block for inspection (tests / views):
 * which: 0 leaf_u[i], 1 leaf_v[i], 2 transfer_u[i], 3 transfer_vt[i],
 *        4 coupling[(i,j)], 5 near[(i,j)], 6 sigma_u[i], 7 sigma_v[i].
 * With out == NULL only the shape is returned.                          */
int ifmm_h2_block(void* h2, int which, int i, int j, double* out, int* rows, int* cols);
/* h2_matvec (krylov.py:119-159), x/y in ORIGINAL point order, host or
 * device pointers (on_device = 1).                                       */
int ifmm_h2_matvec(void* h2, const double* x, double* y, int on_device);

/* ---- extended graph:  graph.py:219-229 / sigma0 graph.py:232-241 ------ */
/* consume != 0 moves the operator blocks into the graph instead of copying
 * them (halves peak memory; the operators are unusable afterwards). */
void* ifmm_graph_build(void* h2, int consume);
void ifmm_graph_destroy(void* graph);
int ifmm_graph_info(void* graph, long long* dim, long long* n_nodes, long long* n_edges);
/* randomized_svd(start_rank=1, max_rank=1) of the extended matrix with the
 * caller-supplied Gaussian sketch omega (dim x width, row-major), exactly
 * the draw of graph.py:235-240 / lowrank.py:100-113.                      */
int ifmm_graph_sigma0(void* graph, const double* omega, int width, int power_iters,
                      double* sigma0_out);

/* Read-only graph view (graph.py:30-216).  nodes: size / kind (0 x, 1 z,
 * 2 y) / owning cluster per node (n_nodes entries); cluster_nodes: the x, z,
 * y node of every cluster (-1 if none); edges: the (target, source) keys,
 * sorted, and the peak edge count; block: one edge block (row-major, r x c;
 * r = -1 if absent; out NULL queries the shape).                           */
int ifmm_graph_nodes(void* graph, int* size, int* kind, int* owner);
int ifmm_graph_cluster_nodes(void* graph, int* nx, int* nz, int* ny);
int ifmm_graph_edges(void* graph, int* target, int* source, long long* peak_edges);
int ifmm_graph_block(void* graph, int target, int source, double* out, int* r, int* c);
/* ExtendedGraph.copy (graph.py:190-216): deep device copy.                */
void* ifmm_graph_copy(void* graph);
/* ExtendedGraph.apply / apply_transpose (graph.py:157-170): out = E in or
 * E^T in over the full node vector (length dim, node order).              */
int ifmm_graph_apply(void* graph, const double* in, double* out, int transpose, int on_device);

/* ---- factorize:  factor.py:176-230 --------------------------------------
 * Consumes (mutates) the graph like the reference.  flags bit0: strict
 * (one pair per wave) pair order; bit1: exact SVD for every fill; bit2:
 * Morton cluster order (one cluster per wave).  Without a normal source the
 * rSVD sketches come from a counter-based device generator.                */
void* ifmm_factorize(void* graph, double epsilon, double sigma0, int flags);
/* The reference's factorize rng, np.random.Generator(PCG64(seed))
 * (factor.py:188), as a stream of standard normal deviates supplied by the
 * host: op 0 writes the next n deviates to out; op 1 saves the stream state
 * in slot n; op 2 restores slot n.  Returns 0 on success.                  */
typedef int (*ifmm_normal_source)(void* user, int op, long long n, double* out);
/* factorize drawing every Gaussian the reference draws (rSVD sketches,
 * lowrank.py:108; _extend_update, factor.py:350) from `src` in the
 * reference's order; implies Morton cluster order (flags bit2).           */
void* ifmm_factorize_rng(void* graph, double epsilon, double sigma0, int flags,
                         ifmm_normal_source src, void* user);
/* The same with the stream generated natively: numpy's PCG64 state as
 * {state_hi, state_lo, inc_hi, inc_lo} (np.random.PCG64(seed).state), its
 * standard normals from numpy's own ziggurat (libnpyrandom) -- bitwise
 * Generator(PCG64(seed)).standard_normal.                                 */
void* ifmm_factorize_pcg64(void* graph, double epsilon, double sigma0, int flags,
                           const unsigned long long* pcg_state);
/* n standard normals of that stream from a given state (host; tests).     */
int ifmm_pcg64_normals(const unsigned long long* pcg_state, long long n, double* out);
void ifmm_factor_destroy(void* factor);
/* Scalar stats: out[0..] = peak_edges, n_clusters, max_basis_rank,
 * max_fill_rank, forced_rank_truncations, n_levels, n_events_elim,
 * n_events_rebase, n_events_merge, n_top, top_dim.                       */
int ifmm_factor_stats(void* factor, long long* out, int n_out);
/* Per level (elimination order L..2): level, compressed_pairs, added,
 * dropped_pairs, sum_ranks, max_rank, n_ranks, forced.  8 per level.      */
int ifmm_factor_level_stats(void* factor, long long* out, int n_levels);
/* Ranks list of one level (n_ranks entries). */
int ifmm_factor_level_ranks(void* factor, int level_index, int* out);
/* Timings (seconds; factor.py:71-72 buckets, device time between bucket
 * switches on the engine stream): lu_and_triangular_solves, matmul_updates,
 * lowrank_approximations, operator_transfer, then total (host wall),
 * gemm_flops (count), all_flops (count), rSVD rounds, rSVD re-draws.       */
int ifmm_factor_timings(void* factor, double* out, int n_out);
/* Event log (factor.py:80, IFMMFactorization.events) as flat int64 records:
 *   elim   0, nx, nz, ny, size_x, size_z, n_src, n_tgt, src nodes, tgt nodes
 *   rebase 1, ny
 *   merge  2, px, n_parts, (child y node, size) pairs
 * Returns the record length; writes only when out has room (cap).       */
long long ifmm_factor_events(void* factor, long long* out, long long cap);
/* top_nodes / top_sizes / init_sizes / leaf_slices (factor.py:77-92);
 * sizes[0..2] = n_top, n_init, n_leaves.  Any array may be NULL.         */
int ifmm_factor_layout(void* factor, int* sizes, int* top_nodes, int* top_sizes, int* init_sizes,
                       int* leaf_nodes, int* leaf_start, int* leaf_stop);
/* FillinStats.compress_time per level (device s in lowrank_approximations). */
int ifmm_factor_level_times(void* factor, double* out, int n_levels);
/* IFMMFactorization.solve (factor.py:99-157): b, x length N (original
 * order), host or device pointers.                                         */
int ifmm_solve(void* factor, const double* b, double* x, int on_device);

/* Morton-range partitioned h2_matvec, one rank's share (no reference
 * counterpart: krylov.py:119-159 is single-process).  Device pointers in tree
 * order; the rank owns points [p_lo, p_hi) (whole leaves).  phase 0 writes the
 * partial multipoles of every cluster meeting the range into yv (length
 * ifmm_h2_multipole_size, zero-initialised by the caller, summed over ranks
 * by the caller); phase 1 reads the summed yv and the full xs (halo) and
 * writes the rows [p_lo, p_hi) of ys. */
int ifmm_h2_multipole_size(void* h2, long long* out);
int ifmm_h2_matvec_part(void* h2, const double* xs, double* ys, double* yv, int phase,
                        long long p_lo, long long p_hi);

/* ---- exact dense matvec:  dense.py:23-32 / experiments.py:157-162 ------
 * y = A x, A_ij = K(|p_i - p_j|) evaluated on the fly (no storage), points
 * and vectors in the same (any) order.  Used for the residual criterion. */
int ifmm_exact_matvec(void* ctx, int kernel_kind, double p0, int n, const double* points,
                      const double* x, double* y, int on_device);
int ifmm_exact_matvec_k(void* ctx, int kernel_kind, double p0, double p1, int n,
                        const double* points, const double* x, double* y, int on_device);

/* ---- GMRES Arnoldi on the device:  krylov.py:32-116 -------------------
 * Device pointers on the context's stream; V holds the Krylov vectors as
 * rows (row stride ldv >= n).  The Givens rotations and the triangular solve
 * stay with the caller (host scalars).
 *   ifmm_krylov_mgs: modified Gram-Schmidt of w against V[0..k1) in order
 *     (krylov.py:73-75: h_i = <V_i, w>; w -= h_i V_i), then h[k1] = ||w||
 *     (krylov.py:76).  h is a HOST array of k1+1 doubles; synchronizes.
 *   ifmm_krylov_div: out = w / hs (krylov.py:104, the next basis vector).
 *   ifmm_krylov_combine: u = sum_{i<k} y_i V_i in basis order
 *     (krylov.py:113); y is a HOST array of k doubles.               */
int ifmm_krylov_mgs(void* ctx, const double* V, long long ldv, int k1, long long n, double* w,
                    double* h);
int ifmm_krylov_div(void* ctx, const double* w, long long n, double hs, double* out);
int ifmm_krylov_combine(void* ctx, const double* V, long long ldv, int k, const double* y,
                        long long n, double* u);

/* ---- device micro-kernel entry points (tests and benchmarks) ---------- */
/* C[M,N] = alpha*op(A)op(B) + beta*C on device pointers (row-major). */
int ifmm_dev_gemm(void* ctx, int M, int N, int K, const double* A, int lda, int ta,
                  const double* B, int ldb, int tb, double* C, int ldc, double alpha,
                  double beta);
/* Truncated SVD (absolute threshold) of a row-major m x n device matrix. */
int ifmm_dev_svd(void* ctx, int m, int n, const double* A, double thr, double* U,
                 double* S, double* V, int* rank);
/* LU with partial pivoting + solve of nrhs right-hand sides (device). */
int ifmm_dev_lu_solve(void* ctx, int n, double* A, int* piv, double* X, int nrhs);
/* weighted_basis_union (lowrank.py:166-199) on device pointers. */
/* Orthonormal basis of a tall row-major n x w device matrix Y into Q
 * (n x w row-major): np.linalg.qr(Y)[0] (lowrank.py:74-76).               */
int ifmm_dev_orth(void* ctx, int n, int w, const double* Y, double* Q);
int ifmm_dev_union(void* ctx, int m, int k_old, int k_f, const double* B, const double* w,
                   const double* F, const double* wf, double thr, int min_rank,
                   double* NB, double* NW, double* OM, double* FM, int* rank);
int ifmm_dev_sync(void* ctx);
/* Diagnostics: clock64 cycles of `reps` CTA Jacobi SVDs of an s x s device
 * matrix (col-major) in shared memory; out[0] = cycles, out[1] = sweeps. */
int ifmm_dev_jacobi_bench(void* ctx, int s, const double* A, int reps, int threads,
                          unsigned long long* out);
/* Device timing on the engine stream: record event `slot` (0..63); elapsed
 * milliseconds between two recorded slots (waits for the second). */
int ifmm_ctx_event(void* ctx, int slot);
int ifmm_ctx_elapsed(void* ctx, int a, int b, double* ms);
/* Number of engine kernel launches issued on the context so far. */
long long ifmm_ctx_launches(void* ctx);
/* Per-category kernel timing (categories: gemm, copy, svd, union, lu,
 * lusolve, spmv, solve, other).  Reads the accumulated totals (seconds,
 * algorithmic work = flops or bytes, launch count); enable >= 0 also resets
 * and switches timing on (1) or off (0). */
int ifmm_ktime(void* ctx, int enable, double* time_s, double* work, long long* count, int n);
/* Diagnostics: union-kernel cycle counters (48 entries: [0..12] all unions --
 * ACA, CholeskyQR, core, Jacobi, output, steps, count, sum m, sum C, smem
 * count, sweeps, core sweeps, core cycles, [13] Householder fallbacks;
 * [16..24] the first nine for 256 < m <= 600, [25..33] for m > 600);
 * reset != 0 clears. */
int ifmm_union_profile(unsigned long long* out, int reset);
/* diagnostics: 16 phase counters of union_post_kernel (union_post.cu) */
int ifmm_union_post_profile(unsigned long long* out, int reset);
/* Dense kernel matrix out (m x n row-major) = K(|P_i - Q_j|) evaluated on
 * the device (dense.py:23-32, dense_matrix).  P (m x 3), Q (n x 3).       */
int ifmm_kernel_matrix(void* ctx, int kernel_kind, double p0, int m, const double* P, int n,
                       const double* Q, double* out, int on_device);
/* block_dim-3 kernels (kind 5): out is (3 m) x (3 n). */
int ifmm_kernel_matrix_k(void* ctx, int kernel_kind, double p0, double p1, int m, const double* P,
                         int n, const double* Q, double* out, int on_device);
/* block_diag_preconditioner (krylov.py:172-196): LU of the diagonal blocks
 * of A (n x n, ld lda; last block shorter) on the device; apply solves them
 * blockwise.  A singular block fails with status 2.                       */
void* ifmm_blockdiag_create(void* ctx, const double* A, int n, int lda, int block_size,
                            int on_device);
int ifmm_blockdiag_apply(void* bd, const double* v, double* out, int on_device);
void ifmm_blockdiag_destroy(void* bd);
/* Diagnostics: phase times (s) of the last factorize when IFMM_PROFILE=1. */
int ifmm_profile(double* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* IFMM_B200_H */
