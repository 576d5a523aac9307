/*
 * hssmf_b200.h — C-ABI of the B200-native numeric factorization and solve of
 * the HSS-compressed multifrontal sparse LU (arXiv 1502.07405 reference,
 * /root/reference/proj). Plain pointers and sizes only; no torch or CUDA types.
 *
 * Drop-in boundary: every entry point below replaces one reference interface,
 * cited as file:line under proj/include/hssmf (or proj/src). The C++ wrappers
 * in include/hssmf_b200/hssmf.hpp rebuild the reference's value types and
 * exception classes on top of these calls.
 *
 * Conventions
 *  - matrices are square CSR with sorted, duplicate-free rows, int32 indices
 *    (SparseMatrix<T>, sparse_matrix.hpp:14-47);
 *  - dense blocks are column-major with an explicit leading dimension
 *    (DenseMatrix<T>, dense_matrix.hpp:17-35);
 *  - every call returns an hssmf_code; failing calls fill *st (may be NULL).
 */
#ifndef HSSMF_B200_H
#define HSSMF_B200_H

#ifdef __cplusplus
extern "C" {
#endif

/* error codes; the C++ wrapper maps them to the reference's exception types
 * (errors.hpp:10-54): SHAPE -> IoError, NOT_FACTORED -> SolverError,
 * SINGULAR -> SingularMatrixError(front, column), RANK -> HssRankExceeded */
typedef enum {
  HSSMF_OK = 0,
  HSSMF_ERR_SHAPE = 1,
  HSSMF_ERR_NOT_FACTORED = 2,
  HSSMF_ERR_SINGULAR = 3,
  HSSMF_ERR_CUDA = 4,
  HSSMF_ERR_NCCL = 5,
  HSSMF_ERR_RANK = 6,
  HSSMF_ERR_OTHER = 7,
  HSSMF_ERR_DIVERGENCE = 8, /* KrylovDivergenceError (krylov.hpp) */
  HSSMF_ERR_STRUCTURAL = 9   /* StructuralSingularError (errors.hpp:32-35) */
} hssmf_code;

typedef struct {
  int code;
  int front;   /* failing front (postorder id) or -1 */
  int column;  /* zero-pivot column within that front's F11 or -1 */
  char msg[512];
} hssmf_status;

/* SolverOptions, numeric subset (solver_options.hpp:28-45). eps is the
 * relative ID tolerance; the absolute floor is derived per sampling round as
 * eps * max(|S_r|, |S_c|) exactly like hss_compress.hpp:335-338. */
typedef struct {
  int ls;        /* switch level: fronts with level < ls may use HSS */
  double eps;    /* relative compression tolerance */
  int leaf;      /* HSS leaf size */
  int d0, dd, p; /* initial sample columns, increment, oversampling */
  int min_hss;   /* minimum front dimension for HSS */
  int max_rank;  /* rank guard, 0 -> min(n/2, 5000) */
  int mode;      /* 0 auto, 1 mf (pure multifrontal), 2 mf-hss */
} hssmf_options;

typedef struct hssmf_csr hssmf_csr;
typedef struct hssmf_tree hssmf_tree;
typedef struct hssmf_factors hssmf_factors;
typedef struct hssmf_hss hssmf_hss;

/* ---- host analysis (integer outputs bit-exact with the reference) ---- */

/* generate_grid_problem (grid_problems.hpp:65-117); kind 0 p2d 1 p3d 2 c2d 3 c3d;
 * dims/ndims receive the GridGeometry (grid_problems.hpp:34-41) */
int hssmf_csr_grid(int kind, int k, double nu, hssmf_csr** out, int* dims, int* ndims,
                   hssmf_status* st);
/* BASELINE config 4: h^2-scaled -lap(u) + beta.grad(u), beta = scale*(1,.5,.25)/h,
 * upwind coefficients by the reference rule detail::upwind (grid_problems.hpp:57-61) */
int hssmf_csr_convdiff3d(int k, double scale, hssmf_csr** out, hssmf_status* st);
/* SparseMatrix(n, ptr, ind, val) (sparse_matrix.hpp:18-22) */
int hssmf_csr_create(int n, const int* ptr, const int* ind, const double* val,
                     hssmf_csr** out, hssmf_status* st);
/* SparseMatrix::permuted (sparse_matrix.hpp:95-102), perm[old] = new */
int hssmf_csr_permuted(const hssmf_csr* a, const int* perm, hssmf_csr** out, hssmf_status* st);
void hssmf_csr_info(const hssmf_csr* a, int* n, long long* nnz);
void hssmf_csr_get(const hssmf_csr* a, int* ptr, int* ind, double* val);
/* y = A x (SparseMatrix::matvec N, sparse_matrix.hpp:70-86), deterministic row order */
void hssmf_csr_matvec(const hssmf_csr* a, const double* x, double* y);
void hssmf_csr_free(hssmf_csr* a);

/* read_matrix_market (matrix_market.cpp:10-65): coordinate real|integer,
 * general|symmetric (lower triangle mirrored), duplicates summed as in
 * SparseMatrix::from_triplets; malformed input -> HSSMF_ERR_SHAPE (IoError) */
int hssmf_csr_read_mm(const char* path, hssmf_csr** out, hssmf_status* st);
/* write_matrix_market (matrix_market.cpp:67-77): general, %.17g values */
int hssmf_csr_write_mm(const hssmf_csr* a, const char* path, hssmf_status* st);
/* equilibrate_and_permute (scaling.hpp:40-139): *out = Dr A Dc Qc with the
 * ScalingState dr, dc (n doubles each), qc (n ints) and the sweep count;
 * structurally singular input -> HSSMF_ERR_STRUCTURAL. A x = b is solved as
 * (*out) xs = Dr b, x[qc[j]] = dc[qc[j]] xs[j]. */
int hssmf_equilibrate(const hssmf_csr* a, hssmf_csr** out, double* dr, double* dc, int* qc,
                      int* sweeps, hssmf_status* st);

/* nested_dissection_geometric (ordering.cpp:213-222) followed by
 * EliminationTree::from_separators (elimination_tree.cpp:10-26); perm[old]=new */
int hssmf_nd_geometric(const int* dims, int ndims, int leaf, int* perm, hssmf_tree** out,
                       hssmf_status* st);
/* nested_dissection_graph (ordering.cpp:224-236) of the structurally
 * symmetrized adjacency of a (SparseMatrix::symmetric_graph,
 * sparse_matrix.hpp:127-145), then EliminationTree::from_separators; fronts
 * may have one child or an empty separator; perm[old] = new */
int hssmf_nd_graph(const hssmf_csr* a, int leaf, int* perm, hssmf_tree** out, hssmf_status* st);
/* reorder_tree_separators (separator_reorder.cpp:119-135) on the adjacency of
 * a (already in the tree ordering): every front with selected[i] != 0 gets HSS
 * separator clusters of at most b vertices (FrontNode::sep_clusters), used by
 * front_cluster_tree (multifrontal.hpp:318-326) when it is compressed;
 * perm[old] = new relabels inside those separators. As with the reference the
 * caller then permutes a (hssmf_csr_permuted) and re-runs hssmf_symbolic. */
int hssmf_reorder_separators(hssmf_tree* t, const hssmf_csr* a, const char* selected, int b,
                             int* perm, hssmf_status* st);
/* a front's separator cluster tree (postorder, root last); returns the node
 * count (0: none, -1: bad front), arrays may be NULL */
int hssmf_tree_sep_clusters(const hssmf_tree* t, int front, int* begin, int* end, int* child0,
                            int* child1, int* parent);
/* sets a front's separator clusters (the drop-in path for trees reordered by
 * the reference's own reorder_tree_separators) */
int hssmf_tree_set_sep_clusters(hssmf_tree* t, int front, int nnodes, const int* begin,
                                const int* end, const int* child0, const int* child1,
                                hssmf_status* st);
/* EliminationTree with explicit nodes (upd sets optional: upd_ptr may be NULL) */
int hssmf_tree_create(int n, int nnodes, const int* sep_begin, const int* sep_end,
                      const int* child0, const int* child1, const int* parent,
                      const int* upd_ptr, const int* upd_ind, hssmf_tree** out,
                      hssmf_status* st);
/* symbolic_factorization(A, t) (elimination_tree.hpp:67-73) */
int hssmf_symbolic(const hssmf_csr* a, hssmf_tree* t, hssmf_status* st);
void hssmf_tree_info(const hssmf_tree* t, int* n, int* nnodes, long long* upd_total);
void hssmf_tree_get(const hssmf_tree* t, int* sep_begin, int* sep_end, int* child0,
                    int* child1, int* parent, int* level, int* upd_ptr, int* upd_ind);
void hssmf_tree_free(hssmf_tree* t);
/* front_cluster_tree (multifrontal.hpp:318-326) via ClusterTree::balanced/join
 * (cluster_tree.hpp:38-61); returns the node count, arrays may be NULL */
int hssmf_front_cluster_tree(int ns, int nu, int leaf, int* begin, int* end, int* child0,
                             int* child1, int* parent);

/* ---- numeric factorization / solve on a B200 ---- */

/* analysis upload + static schedule + numeric factorization:
 * mf_factor(a, t, opts) (multifrontal.hpp:473-503). a must carry the tree's
 * ordering. device: CUDA ordinal. */
int hssmf_factor(int device, const hssmf_csr* a, const hssmf_tree* t, const hssmf_options* o,
                 hssmf_factors** out, hssmf_status* st);
/* numeric re-factorization with new values on the same pattern; val is host
 * (on_device = 0) or device memory, nnz entries in the CSR order of a */
int hssmf_refactor(hssmf_factors* f, const double* val, int on_device, hssmf_status* st);
/* mf_solve(m, b) (multifrontal.hpp:612-622): b is n x nrhs column-major with
 * leading dimension ldb, in the tree ordering, solved in place; host or device */
int hssmf_solve(hssmf_factors* f, double* b, int ldb, int nrhs, int on_device,
                hssmf_status* st);
/* ---- multi-GPU subtree partition (no reference counterpart:
 * the reference is single-node OpenMP, multifrontal.hpp:398-503 is the
 * sequential schedule these phases reproduce) ----
 * analysis with an ownership mask (one char per front): only owned fronts are
 * factored / solved by this handle; the update blocks and forward
 * contributions of their non-owned children are imported between phases. */
int hssmf_analyze_owned(int device, const hssmf_csr* a, const hssmf_tree* t,
                        const hssmf_options* o, const char* owned, hssmf_factors** out,
                        hssmf_status* st);
int hssmf_nlevels(const hssmf_factors* f);
/* factor the owned fronts of tree levels lo..hi (deepest first); the phase
 * with hi = nlevels-1 starts a new factorization, the one with lo = 0 ends it */
int hssmf_factor_levels(hssmf_factors* f, int lo, int hi, hssmf_status* st);
/* update block of a front (nu x nu, ld nu): what factor_front passes to the
 * parent (multifrontal.hpp:340-344 dense cb, :369-376 HSS Schur operator) */
int hssmf_update_export(const hssmf_factors* f, int front, double* dst, int on_device,
                        hssmf_status* st);
int hssmf_update_import(hssmf_factors* f, int front, const double* src, int on_device,
                        hssmf_status* st);
/* forward-sweep contribution of a front (nu x nrhs, ld nu, device memory):
 * the bupd mf_forward passes up (multifrontal.hpp:545-560) */
int hssmf_bupd_export(const hssmf_factors* f, int front, double* dst, int nrhs,
                      hssmf_status* st);
int hssmf_bupd_import(hssmf_factors* f, int front, const double* src, int nrhs,
                      hssmf_status* st);
/* one sweep of the solve over levels lo..hi on device x (n x nrhs, ld ldx):
 * forward = 1 (deepest first) or backward = 0 (root first) */
int hssmf_solve_levels(hssmf_factors* f, double* x, int ldx, int nrhs, int lo, int hi,
                       int forward, hssmf_status* st);

/* ---- preconditioned iterative solves (krylov.hpp:93-232) ----
 * gmres(A, M^-1 = mf_solve(m), b, restart, rtol, atol, maxit) and
 * iterative_refinement(A, M^-1, b, rtol, atol, maxit), run on the device:
 * A is applied by a CSR SpMV kernel, M^-1 by the factors' solve, the Krylov
 * basis lives in HBM. m = NULL: identity preconditioner (device 0).
 * b, x: host vectors of length n (x = the solution, zero initial guess);
 * history (optional, history_cap entries) receives the residual norms. */
typedef struct {
  int iterations;
  double rel_resid, abs_resid;
  int converged, stagnated;
  int history_len;
} hssmf_krylov_report;
int hssmf_gmres(const hssmf_csr* a, hssmf_factors* m, const double* b, double* x, int restart,
                double rtol, double atol, int maxit, hssmf_krylov_report* rep, double* history,
                int history_cap, hssmf_status* st);
int hssmf_refine(const hssmf_csr* a, hssmf_factors* m, const double* b, double* x, double rtol,
                 double atol, int maxit, hssmf_krylov_report* rep, double* history,
                 int history_cap, hssmf_status* st);

/* MfFactors::{front_stats, hss_fronts, fallbacks, max_front_rank, factor_nnz()}
 * (multifrontal.hpp:454-468); type 0 dense 1 hss 2 hss_dense */
void hssmf_factor_summary(const hssmf_factors* f, int* nnodes, int* hss_fronts,
                          int* fallbacks, int* max_rank, long long* factor_nnz);
void hssmf_front_stats(const hssmf_factors* f, int* level, int* dim, int* sep, int* rank,
                       long long* flops, int* type);
/* per HSS-tree node u/v ranks of one front (hss_matrix.hpp:210-216) and the
 * adaptive sampling stats (HssCompressStats, hss_compress.hpp:34-37);
 * returns the node count (0 for a dense front); arrays may be NULL */
int hssmf_front_hss(const hssmf_factors* f, int front, int* u_rank, int* v_rank, int* rounds,
                    int* d_final);
/* device time of the last factor / solve (CUDA events on the engine stream) */
void hssmf_timing(const hssmf_factors* f, double* factor_ms, double* solve_ms);
/* per-kernel-class profile (events around each launch when enabled) */
void hssmf_set_profile(hssmf_factors* f, int on);
int hssmf_kernel_stats(const hssmf_factors* f, int max, char* names /* max*32 */,
                       int* launches, double* ms, double* flops, double* bytes);
void hssmf_reset_kernel_stats(hssmf_factors* f);
long long hssmf_device_bytes(const hssmf_factors* f);
void hssmf_factors_free(hssmf_factors* f);

/* ---- standalone dense HSS (BASELINE config 2) ---- */
/* hss_compress(A, ClusterTree::balanced(n, leaf), HssOptions) + ulv_factor
 * (hss_compress.hpp:373-383, hss_ulv.hpp:284-319); a is n x n, lda >= n */
int hssmf_hss_dense(int device, const double* a, int lda, int n, int leaf, double eps, int d0,
                    int dd, int p, int max_rank, int on_device, hssmf_hss** out,
                    hssmf_status* st);
/* hss_compress(A, tree, HssOptions) + ulv_factor for any postorder cluster
 * tree over [0, n) (ClusterTree, cluster_tree.hpp:12-97: nodes root last,
 * children split the parent's [begin, end)); seeds = row index
 * (hss_compress.hpp:380-381) */
int hssmf_hss_dense_tree(int device, const double* a, int lda, int n, int nnodes,
                         const int* begin, const int* end, const int* child0, const int* child1,
                         double eps, int d0, int dd, int p, int max_rank, int on_device,
                         hssmf_hss** out, hssmf_status* st);
int hssmf_hss_info(const hssmf_hss* h, int* u_rank, int* v_rank, int* rounds, int* d_final,
                   double* compress_ms, double* ulv_ms);
/* HssMatrix::matvec (hss_matrix.hpp:234-249, mv_up/mv_down :349-413):
 * y = op(A_hss) x on the subtree of cluster node `root` (-1: whole matrix),
 * op 'N', 'T' or 'C' (= 'T' for real data); x is nrows x nc with nrows the
 * node's size (else HSSMF_ERR_SHAPE, the reference's IoError) */
int hssmf_hss_matvec(hssmf_hss* h, char op, int root, const double* x, int ldx, int nrows,
                     int nc, double* y, int ldy, int on_device, hssmf_status* st);
/* HssMatrix::extract (hss_matrix.hpp:261-280, ex_up/ex_down :425-506):
 * out (ni x nj, ld ni) = A_hss(rows, cols) for index lists in any order (the
 * reference requires sorted lists); out-of-range indices ->
 * HSSMF_ERR_SHAPE. leaf_visits (optional) = leaves the pruned traversal read */
int hssmf_hss_extract(hssmf_hss* h, const int* rows, int ni, const int* cols, int nj,
                      double* out, int on_device, long long* leaf_visits, hssmf_status* st);
/* UlvFactors::solve (hss_ulv.hpp:150-176) */
int hssmf_hss_solve(hssmf_hss* h, double* b, int ldb, int nrhs, int on_device,
                    hssmf_status* st);
void hssmf_hss_free(hssmf_hss* h);

/* ---- kernel-level entry points used by the parity tests ---- */
/* SeededRowSampler values R(l, c), c in [c0, c1) for global rows grow[l]
 * (random_sampler.hpp:19-68) computed by the device generator; out is
 * nrows x (c1-c0) column-major, host memory */
int hssmf_dev_random_rows(int device, int nrows, const long long* grow, int c0, int c1,
                          double* out, hssmf_status* st);
/* C = alpha op(A) op(B) + beta C on the device DMMA GEMM, host buffers */
int hssmf_dev_gemm(int device, char ta, char tb, int m, int n, int k, double alpha,
                   const double* a, int lda, const double* b, int ldb, double beta, double* c,
                   int ldc, hssmf_status* st);
/* interpolative_decomposition (rrqr.hpp:175-194) on the device CPQR: y is m x n;
 * perm (n), rank, certified, coeffs (rank x (n-rank), ld rank) */
int hssmf_dev_id(int device, const double* y, int m, int n, double eps, int max_rank,
                 double abs_tol, int* perm, int* rank, int* certified, double* coeffs,
                 hssmf_status* st);
/* the Gram route of the same ID (no reference counterpart: a BLAS3 restatement
 * of rrqr_tolerance, rrqr.hpp:32-151, used by the HSS path for eps >= 5e-5):
 * pivoted Cholesky of Y^T Y with the CPQR stop rules; r receives R = L^T
 * (rank x n, column j = position j) */
int hssmf_dev_gram_id(int device, const double* y, int m, int n, double eps, int max_rank,
                      double abs_tol, int* perm, int* rank, int* certified, double* r,
                      hssmf_status* st);
/* lu_partial_pivot (lu.hpp:80-85) on the device panel kernels; a is m x n (m>=n) */
int hssmf_dev_lu(int device, double* a, int m, int n, int* piv, hssmf_status* st);

/* measurement (no reference counterpart): per-kernel device-time probes used
 * by bench.py's roofline entries. While enabled, every launch of the probed
 * kernels is bracketed by CUDA events on its stream; read returns, per kind
 * (0 = DMMA grouped GEMM, 1 = Gram-ID cluster panel, 2 = Gram-ID trailing
 * SYRK), the launch count, summed device ms and algorithmic flops / bytes,
 * and resets them. */
typedef struct {
  long long launches;
  double ms, flops, bytes;
} hssmf_probe_stat;
int hssmf_probe_enable(int on, hssmf_status* st);
int hssmf_probe_read(hssmf_probe_stat* out /* [3] */, hssmf_status* st);

/* measurement: average device time (ms) of `iters` m x n x k DGEMMs (NN) on
 * the DMMA kernel, device-resident operands; used for the FP64 roofline */
int hssmf_bench_gemm(int device, int m, int n, int k, int iters, double* ms, hssmf_status* st);
/* Timing of the Gram-route ID kernels (no reference counterpart; measurement
   only): ntask tasks of an n x n Gram matrix of rank min(n, d). */
int hssmf_bench_gram(int device, int n, int d, int ntask, int iters, double* ms, int* steps,
                     hssmf_status* st);

/* number of kernel launches this library has issued (process-wide) */
long long hssmf_launch_count(void);

const char* hssmf_version(void);

/* ---- multi-GPU subtree partition ----
 * One process per GPU. The elimination tree's 2^L subtrees at level
 * L = log2(nranks) are factored independently (rank r owns the r-th); a front
 * above level L belongs to the owner of its child0 subtree. Update blocks
 * (factor), bupd (forward solve) and x(upd) (backward solve) cross ranks
 * along tree edges only, through the caller's point-to-point transport
 * (include/hssmf_b200/mgpu_nccl.hpp: ncclSend / ncclRecv over NVLink). Every
 * rank calls the same entry points with the same matrix and tree. */
typedef struct hssmf_transport {
  void* ctx;
  /* blocking: dev_buf (count doubles of device memory) may be reused on return */
  int (*send)(void* ctx, const double* dev_buf, long long count, int peer);
  /* blocking: the data has landed in dev_buf on return */
  int (*recv)(void* ctx, double* dev_buf, long long count, int peer);
} hssmf_transport;
/* owner rank per front (nnodes) and the number of cross-rank tree edges */
int hssmf_mgpu_partition(const hssmf_tree* t, int nranks, int* owner, int* nedges,
                         hssmf_status* st);
/* this rank's share of mf_factor (multifrontal.hpp:473-503) */
int hssmf_mgpu_factor(int device, const hssmf_csr* a, const hssmf_tree* t,
                      const hssmf_options* o, int rank, int nranks, const hssmf_transport* tr,
                      hssmf_factors** out, hssmf_status* st);
/* this rank's share of mf_solve (multifrontal.hpp:612-622) on a device x
 * (n x nrhs, ld ldx) holding b on entry; on return x is correct on the
 * separators of the fronts this rank owns */
int hssmf_mgpu_solve(hssmf_factors* f, const hssmf_transport* tr, double* x, int ldx, int nrhs,
                     hssmf_status* st);
/* all nranks ranks in this process on one device (in-process mailbox): the
 * partitioned factor + solve of the device block x (n x nrhs, ld n), b on
 * entry, the assembled solution on return */
int hssmf_mgpu_local(int device, const hssmf_csr* a, const hssmf_tree* t, const hssmf_options* o,
                     int nranks, double* x, int nrhs, hssmf_status* st);

#ifdef __cplusplus
}
#endif

#endif
