// ORACLE — test infrastructure only. Not part of the product.
//
// extern "C" shim over the UNMODIFIED reference headers and sources under
// /root/reference/proj (compiled in place by oracle/Makefile; nothing is
// copied into this repository). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load the resulting
// oracle/_ref/libhssmf_ref.so.
//
// One semantics-preserving shim is applied, as an explicit specialization
// (declared before multifrontal.hpp instantiates its caller), never as an
// edit of the reference source:
//
//   LowRankSchur<double>::extract  (reference hss_ulv.hpp:46-60)
//
// The reference's element oracle forwards skeleton index lists stored in
// pivot order (hss_compress.hpp:277-282) through front_elements
// (multifrontal.hpp:245-262) into HssMatrix::extract, whose window splits
// (hss_matrix.hpp:438-442, 471-473) require ascending indices. Unsorted
// requests read out of bounds and segfault under -DNDEBUG.
// The specialization sorts the request, runs the reference's own extract on
// the sorted lists and scatters the block back, so the documented contract
// out(ii,jj) = S(i[ii], j[jj]) holds for any order.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "ref_shim.hpp"
  // namespace hssmf

#include "hssmf/counters.hpp"
#include "hssmf/elimination_tree.hpp"
#include "hssmf/grid_problems.hpp"
#include "hssmf/hss_compress.hpp"
#include "hssmf/multifrontal.hpp"
#include "hssmf/ordering.hpp"
#include "hssmf/random_sampler.hpp"
#include "hssmf/rrqr.hpp"
#include "hssmf/separator_reorder.hpp"
#include "hssmf/matrix_market.hpp"
#include "hssmf/scaling.hpp"
#include "hssmf/lu.hpp"
#include "hssmf/solver_options.hpp"
#include "hssmf/sparse_matrix.hpp"
#include "hssmf/task_parallel.hpp"
#include "hssmf/stats.hpp"

using namespace hssmf;

namespace {

  struct Ordered {
    SparseMatrix<double> a;  // permuted into tree order
    EliminationTree t;
    std::vector<int> perm;   // perm[old] = new
  };

  struct Factored {
    MfFactors<double> m;
    double t_factor = 0;
  };

  struct DenseHss {
    HssMatrix<double> h;
    UlvFactors<double> ulv;
    HssCompressStats st;
    double t_compress = 0, t_ulv = 0;
  };

  thread_local std::string g_err;

  double now() {
    using namespace std::chrono;
    return duration<double>(steady_clock::now().time_since_epoch()).count();
  }

  GridKind kind_of(int k) {
    switch (k) {
      case 0: return GridKind::P2D;
      case 1: return GridKind::P3D;
      case 2: return GridKind::C2D;
      default: return GridKind::C3D;
    }
  }

  SparseMatrix<double> csr_copy(int n, const int* ptr, const int* ind, const double* val) {
    std::vector<int> p(ptr, ptr + n + 1), i(ind, ind + ptr[n]);
    std::vector<double> v(val, val + ptr[n]);
    return SparseMatrix<double>(n, std::move(p), std::move(i), std::move(v));
  }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int t) { params::set_threads(t); }
int ref_num_threads() { return params::num_threads(); }
long long ref_flops() { return counters::get_flops(); }
void ref_reset_counters() { counters::reset(); }

double ref_sampler_value(long long row, long long col) {
  return SeededRowSampler::value(row, col);
}

// R(l, c) for a list of global rows, columns [c0, c1) (build_random_block /
// grow_random, multifrontal.hpp:126-135, hss_compress.hpp:72-82)
void ref_random_rows(int nrows, const long long* grow, int c0, int c1, double* out) {
  DenseMatrix<double> r(nrows, c1);
  for (int l = 0; l < nrows; l++) SeededRowSampler::fill_row(r, l, grow[l], c0, c1);
  for (int c = c0; c < c1; c++)
    for (int l = 0; l < nrows; l++) out[l + (std::size_t)(c - c0) * nrows] = r(l, c);
}

// ---- grid problems (grid_problems.hpp:65-117) ------------------------------
void* ref_grid(int kind, int k, double nu) {
  return new GridProblem<double>(generate_grid_problem<double>(kind_of(kind), k, nu));
}
void ref_grid_free(void* h) { delete static_cast<GridProblem<double>*>(h); }
int ref_grid_n(void* h) { return static_cast<GridProblem<double>*>(h)->A.size(); }
long long ref_grid_nnz(void* h) { return static_cast<GridProblem<double>*>(h)->A.nnz(); }
void ref_grid_csr(void* h, int* ptr, int* ind, double* val) {
  const auto& a = static_cast<GridProblem<double>*>(h)->A;
  std::copy(a.ptr().begin(), a.ptr().end(), ptr);
  std::copy(a.ind().begin(), a.ind().end(), ind);
  std::copy(a.val().begin(), a.val().end(), val);
}

// ---- canonical pipeline (tests/support/problems.hpp:20-30) -----------------
void* ref_ordered_grid(int kind, int k, double nu, int nd_leaf) {
  auto g = generate_grid_problem<double>(kind_of(kind), k, nu);
  auto* o = new Ordered;
  Permutation perm;
  auto st = nested_dissection_geometric(g.geom, nd_leaf, perm);
  o->a = g.A.permuted(perm.perm);
  o->t = EliminationTree::from_separators(st, o->a.size());
  symbolic_factorization(o->a, o->t);
  o->t.compute_levels();
  o->perm = perm.perm;
  return o;
}

// geometric ND + symbolic for an arbitrary CSR on a grid geometry (used for
// the convection-diffusion config that is not a reference generator)
void* ref_ordered_csr_geom(int n, const int* ptr, const int* ind, const double* val,
                           int dx, int dy, int dz, int ndims, int nd_leaf) {
  GridGeometry g;
  g.dims = {dx, dy, dz};
  g.ndims = ndims;
  auto a = csr_copy(n, ptr, ind, val);
  auto* o = new Ordered;
  Permutation perm;
  auto st = nested_dissection_geometric(g, nd_leaf, perm);
  o->a = a.permuted(perm.perm);
  o->t = EliminationTree::from_separators(st, o->a.size());
  symbolic_factorization(o->a, o->t);
  o->t.compute_levels();
  o->perm = perm.perm;
  return o;
}

// an already-ordered matrix plus an explicit tree (upd sets given)
void* ref_ordered_from_arrays(int n, const int* ptr, const int* ind, const double* val,
                              int nnodes, const int* sep_begin, const int* sep_end,
                              const int* child0, const int* child1, const int* parent,
                              const int* upd_ptr, const int* upd_ind) {
  auto* o = new Ordered;
  o->a = csr_copy(n, ptr, ind, val);
  o->t.n = n;
  o->t.nodes.resize(nnodes);
  for (int i = 0; i < nnodes; i++) {
    auto& f = o->t.nodes[i];
    f.sep_begin = sep_begin[i];
    f.sep_end = sep_end[i];
    f.child0 = child0[i];
    f.child1 = child1[i];
    f.parent = parent[i];
    f.upd.assign(upd_ind + upd_ptr[i], upd_ind + upd_ptr[i + 1]);
  }
  o->t.compute_levels();
  o->perm.resize(n);
  std::iota(o->perm.begin(), o->perm.end(), 0);
  return o;
}

// graph pipeline: nested_dissection_graph (ordering.cpp:224-236) + symbolic;
// reorder_b > 0: reorder_tree_separators (separator_reorder.cpp:119-135) of the
// selected fronts (selected == NULL: every front with a separator), then the
// relabeled matrix and its symbolic analysis
void* ref_ordered_graph(int n, const int* ptr, const int* ind, const double* val, int nd_leaf,
                        int reorder_b, const char* selected) {
  auto a = csr_copy(n, ptr, ind, val);
  std::vector<int> gptr, gind;
  a.symmetric_graph(gptr, gind);
  Permutation perm;
  auto st = nested_dissection_graph(n, gptr, gind, nd_leaf, perm);
  auto* o = new Ordered;
  o->a = a.permuted(perm.perm);
  o->t = EliminationTree::from_separators(st, n);
  symbolic_factorization(o->a, o->t);
  o->perm = perm.perm;
  if (reorder_b > 0) {
    std::vector<char> sel(o->t.size());
    for (int i = 0; i < o->t.size(); i++)
      sel[i] = selected ? selected[i] : (o->t.node(i).sep_size() > 0);
    std::vector<int> pptr, pind;
    o->a.symmetric_graph(pptr, pind);
    auto r = reorder_tree_separators(o->t, sel, pptr, pind, reorder_b);
    o->a = o->a.permuted(r.perm);
    for (int i = 0; i < n; i++) o->perm[i] = r.perm[o->perm[i]];
    symbolic_factorization(o->a, o->t);
  }
  o->t.compute_levels();
  return o;
}

int ref_ordered_sep_clusters(void* h, int front, int* begin, int* end, int* c0, int* c1,
                             int* parent) {
  const auto& c = static_cast<Ordered*>(h)->t.node(front).sep_clusters;
  for (int i = 0; i < c.size(); i++) {
    const auto& x = c.node(i);
    if (begin) begin[i] = x.begin;
    if (end) end[i] = x.end;
    if (c0) c0[i] = x.child0;
    if (c1) c1[i] = x.child1;
    if (parent) parent[i] = x.parent;
  }
  return c.size();
}

// equilibrate_and_permute (scaling.hpp:40-139); the output keeps a's row
// pointers. returns 0, or 9 when structurally singular (message in
// ref_last_error)
int ref_equilibrate(int n, const int* ptr, const int* ind, const double* val, int* oind,
                    double* oval, double* dr, double* dc, int* qc, int* sweeps) {
  auto a = csr_copy(n, ptr, ind, val);
  ScalingState<double> st;
  try {
    auto s = equilibrate_and_permute(a, st);
    std::copy(s.ind().begin(), s.ind().end(), oind);
    std::copy(s.val().begin(), s.val().end(), oval);
  } catch (const StructuralSingularError& e) {
    g_err = e.what();
    return 9;
  }
  std::copy(st.dr.begin(), st.dr.end(), dr);
  std::copy(st.dc.begin(), st.dc.end(), dc);
  std::copy(st.qc.begin(), st.qc.end(), qc);
  *sweeps = st.sweeps;
  return 0;
}

// read_matrix_market (matrix_market.cpp:10-65): sizes when ptr is NULL;
// returns 0, or 1 on IoError
int ref_read_mm(const char* path, int* n, long long* nnz, int* ptr, int* ind, double* val) {
  try {
    auto a = read_matrix_market(path);
    *n = a.size();
    *nnz = a.nnz();
    if (ptr) {
      std::copy(a.ptr().begin(), a.ptr().end(), ptr);
      std::copy(a.ind().begin(), a.ind().end(), ind);
      std::copy(a.val().begin(), a.val().end(), val);
    }
  } catch (const IoError& e) {
    g_err = e.what();
    return 1;
  }
  return 0;
}

void ref_ordered_free(void* h) { delete static_cast<Ordered*>(h); }
int ref_ordered_n(void* h) { return static_cast<Ordered*>(h)->a.size(); }
long long ref_ordered_nnz(void* h) { return static_cast<Ordered*>(h)->a.nnz(); }
void ref_ordered_csr(void* h, int* ptr, int* ind, double* val) {
  const auto& a = static_cast<Ordered*>(h)->a;
  std::copy(a.ptr().begin(), a.ptr().end(), ptr);
  std::copy(a.ind().begin(), a.ind().end(), ind);
  std::copy(a.val().begin(), a.val().end(), val);
}
void ref_ordered_perm(void* h, int* perm) {
  const auto& p = static_cast<Ordered*>(h)->perm;
  std::copy(p.begin(), p.end(), perm);
}
int ref_ordered_nnodes(void* h) { return static_cast<Ordered*>(h)->t.size(); }
long long ref_ordered_upd_total(void* h) {
  long long s = 0;
  for (const auto& f : static_cast<Ordered*>(h)->t.nodes) s += f.upd_size();
  return s;
}
void ref_ordered_tree(void* h, int* sep_begin, int* sep_end, int* child0, int* child1,
                      int* parent, int* level, int* upd_ptr, int* upd_ind) {
  const auto& t = static_cast<Ordered*>(h)->t;
  long long off = 0;
  for (int i = 0; i < t.size(); i++) {
    const auto& f = t.node(i);
    sep_begin[i] = f.sep_begin;
    sep_end[i] = f.sep_end;
    child0[i] = f.child0;
    child1[i] = f.child1;
    parent[i] = f.parent;
    level[i] = f.level;
    upd_ptr[i] = (int)off;
    for (int g : f.upd) upd_ind[off++] = g;
  }
  upd_ptr[t.size()] = (int)off;
}

// ---- numeric factorization (multifrontal.hpp:473-503) ----------------------
// opts: ls, leaf, d0, dd, p, min_hss, max_rank, mode(0 auto,1 mf,2 mf-hss)
void* ref_factor(void* oh, const int* iopts, double eps, int* status, int* sfront,
                 int* scol) {
  auto* o = static_cast<Ordered*>(oh);
  SolverOptions so;
  so.ls = iopts[0];
  so.leaf = iopts[1];
  so.d0 = iopts[2];
  so.dd = iopts[3];
  so.p = iopts[4];
  so.min_hss = iopts[5];
  so.max_rank = iopts[6];
  so.mode = iopts[7] == 1 ? SolverMode::MF : iopts[7] == 2 ? SolverMode::MFHSS
                                                           : SolverMode::Auto;
  so.eps = eps;
  *status = 0;
  *sfront = -1;
  *scol = -1;
  try {
    auto* f = new Factored;
    const double t0 = now();
    f->m = mf_factor(o->a, o->t, so);
    f->t_factor = now() - t0;
    return f;
  } catch (const SingularMatrixError& e) {
    g_err = e.what();
    *status = 3;
    *scol = e.column();
    std::string w = e.what();
    auto p = w.find("front ");
    if (p != std::string::npos) *sfront = std::atoi(w.c_str() + p + 6);
  } catch (const IoError& e) {
    g_err = e.what();
    *status = 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = 2;
  }
  return nullptr;
}
void ref_factor_free(void* h) { delete static_cast<Factored*>(h); }
double ref_factor_seconds(void* h) { return static_cast<Factored*>(h)->t_factor; }
void ref_factor_summary(void* h, int* hss_fronts, int* fallbacks, int* max_rank,
                        long long* factor_nnz) {
  const auto& m = static_cast<Factored*>(h)->m;
  *hss_fronts = m.hss_fronts;
  *fallbacks = m.fallbacks;
  *max_rank = m.max_front_rank;
  *factor_nnz = m.factor_nnz();
}
// type: 0 dense, 1 hss, 2 hss_dense
void ref_front_stats(void* h, int* level, int* dim, int* sep, int* rank,
                     long long* flops, int* type) {
  const auto& m = static_cast<Factored*>(h)->m;
  for (std::size_t i = 0; i < m.front_stats.size(); i++) {
    const auto& s = m.front_stats[i];
    level[i] = s.level;
    dim[i] = s.dim;
    sep[i] = s.sep;
    rank[i] = s.rank;
    flops[i] = s.flops;
    type[i] = s.type == "hss" ? 1 : s.type == "hss_dense" ? 2 : 0;
  }
}
// per HSS-tree node of one front: u/v ranks (hss_matrix.hpp:210-216), plus
// compression stats (rounds, d_final); returns the node count (0 if dense)
int ref_front_hss(void* h, int front, int* u_rank, int* v_rank, int* rounds,
                  int* d_final) {
  const auto& fr = static_cast<Factored*>(h)->m.fronts[front];
  if (!fr.hss) return 0;
  const int nn = fr.h.tree().size();
  if (u_rank)
    for (int i = 0; i < nn; i++) {
      u_rank[i] = fr.h.node(i).u.rank();
      v_rank[i] = fr.h.node(i).v.rank();
    }
  if (rounds) *rounds = fr.cst.rounds;
  if (d_final) *d_final = fr.cst.d_final;
  return nn;
}
// b (n x nrhs, column-major, tree order) solved in place
double ref_solve(void* h, double* b, int nrhs) {
  auto& m = static_cast<Factored*>(h)->m;
  DenseMatrixWrapper<double> w(m.tree.n, nrhs, b, m.tree.n);
  const double t0 = now();
  mf_solve(m, w);
  return now() - t0;
}

// ---- standalone dense HSS (hss_compress.hpp:373-383, hss_ulv.hpp:284-319)
void* ref_hss_dense(const double* a, int n, int leaf, double eps, int d0, int dd, int p,
                    int max_rank, int* status) {
  *status = 0;
  try {
    DenseMatrix<double> A(n, n, a, n);
    HssOptions ho;
    ho.eps = eps;
    ho.d0 = d0;
    ho.dd = dd;
    ho.p = p;
    ho.max_rank = max_rank;
    auto* d = new DenseHss;
    double t0 = now();
    d->h = hss_compress(A, ClusterTree::balanced(n, leaf), ho, &d->st);
    double t1 = now();
    d->ulv = ulv_factor(d->h);
    d->t_compress = t1 - t0;
    d->t_ulv = now() - t1;
    return d;
  } catch (const HssRankExceeded& e) {
    g_err = e.what();
    *status = 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    *status = 2;
  }
  return nullptr;
}
void ref_hss_free(void* h) { delete static_cast<DenseHss*>(h); }
int ref_hss_info(void* h, int* u_rank, int* v_rank, int* rounds, int* d_final,
                 double* t_compress, double* t_ulv) {
  auto* d = static_cast<DenseHss*>(h);
  const int nn = d->h.tree().size();
  if (u_rank)
    for (int i = 0; i < nn; i++) {
      u_rank[i] = d->h.node(i).u.rank();
      v_rank[i] = d->h.node(i).v.rank();
    }
  *rounds = d->st.rounds;
  *d_final = d->st.d_final;
  *t_compress = d->t_compress;
  *t_ulv = d->t_ulv;
  return nn;
}
double ref_hss_solve(void* h, double* b, int nrhs) {
  auto* d = static_cast<DenseHss*>(h);
  DenseMatrixWrapper<double> w(d->h.rows(), nrhs, b, d->h.rows());
  const double t0 = now();
  d->ulv.solve(w);
  return now() - t0;
}
void ref_hss_matvec(void* h, const double* x, double* y, int nrhs) {
  auto* d = static_cast<DenseHss*>(h);
  const int n = d->h.rows();
  DenseMatrix<double> X(n, nrhs, x, n), Y(n, nrhs);
  d->h.matvec(Trans::N, X, Y);
  for (int c = 0; c < nrhs; c++)
    std::copy(Y.ptr(0, c), Y.ptr(0, c) + n, y + (std::size_t)c * n);
}

// ---- dense kernels pinned by the reference's unit tests ------------------
// lu_partial_pivot (lu.hpp:80-85): a overwritten by [L\U], piv (size
// min(m,n)); returns -1 or the singular column
int ref_lu(double* a, int m, int n, int* piv) {
  DenseMatrixWrapper<double> w(m, n, a, m);
  std::vector<int> p;
  try {
    lu_partial_pivot(w, p);
  } catch (const SingularMatrixError& e) {
    return e.column();
  }
  std::copy(p.begin(), p.end(), piv);
  return -1;
}
// interpolative_decomposition (rrqr.hpp:175-194); coeffs is rank x (n-rank)
void ref_id(const double* y, int m, int n, double eps, int max_rank, double abs_tol,
            int* perm, int* rank, int* certified, double* coeffs) {
  DenseMatrix<double> Y(m, n, y, m);
  auto id = interpolative_decomposition(Y, eps, max_rank, abs_tol);
  std::copy(id.perm.begin(), id.perm.end(), perm);
  *rank = id.rank;
  *certified = id.certified ? 1 : 0;
  for (std::size_t j = 0; j < id.coeffs.cols(); j++)
    for (std::size_t i = 0; i < id.coeffs.rows(); i++)
      coeffs[i + j * id.coeffs.rows()] = id.coeffs(i, j);
}
// ClusterTree::balanced / join (cluster_tree.hpp:38-61); returns node count
int ref_cluster_front(int ns, int nu, int leaf, int* begin, int* end, int* c0, int* c1,
                      int* parent) {
  ClusterTree sep = ClusterTree::balanced(ns, leaf);
  ClusterTree t = nu ? ClusterTree::join(sep, ClusterTree::balanced(nu, leaf)) : sep;
  if (begin)
    for (int i = 0; i < t.size(); i++) {
      begin[i] = t.node(i).begin;
      end[i] = t.node(i).end;
      c0[i] = t.node(i).child0;
      c1[i] = t.node(i).child1;
      parent[i] = t.node(i).parent;
    }
  return t.size();
}

// stats_to_json / stats_csv_header / stats_csv_row (src/stats.cpp:37-123) of
// a RunStats given field by field: ints = {n, nnz, ls, leaf, d0, dd, p,
// min_hss, max_rank, threads, restart, maxit, nd_leaf, factor_flops,
// solve_flops, factor_nnz, factor_nnz_bytes, peak_bytes, max_rank_obs, fronts,
// hss_fronts, hss_fallbacks, tree_depth, iterations, converged}; reals = {eps,
// rtol, atol, t_analysis, t_factor, t_solve, t_total, relres, absres};
// per-front rows pf = {id, level, dim, sep, rank, flops} x npf. Returns the
// bytes needed (json + csv header + csv row, NUL-separated).
long long ref_stats(const char* source, int strategy_graph, const char* mode, const long long* in,
                    const double* re, const char* method, const char* error, int npf,
                    const long long* pf, const char* const* pf_type, int include_pf, char* out,
                    long long cap) {
  RunStats s;
  s.source = source;
  s.opts.strategy = strategy_graph ? OrderingStrategy::Graph : OrderingStrategy::Geometric;
  s.opts.mode = parse_solver_mode(mode);
  s.n = (int)in[0];
  s.nnz = in[1];
  s.opts.ls = (int)in[2];
  s.opts.leaf = (int)in[3];
  s.opts.d0 = (int)in[4];
  s.opts.dd = (int)in[5];
  s.opts.p = (int)in[6];
  s.opts.min_hss = (int)in[7];
  s.opts.max_rank = (int)in[8];
  s.opts.threads = (int)in[9];
  s.opts.restart = (int)in[10];
  s.opts.maxit = (int)in[11];
  s.opts.nd_leaf = (int)in[12];
  s.factor_flops = in[13];
  s.solve_flops = in[14];
  s.factor_nnz = in[15];
  s.factor_nnz_bytes = in[16];
  s.peak_bytes = in[17];
  s.max_rank = (int)in[18];
  s.fronts = (int)in[19];
  s.hss_fronts = (int)in[20];
  s.hss_fallbacks = (int)in[21];
  s.tree_depth = (int)in[22];
  s.iterations = (int)in[23];
  s.converged = in[24] != 0;
  s.opts.eps = re[0];
  s.opts.rtol = re[1];
  s.opts.atol = re[2];
  s.t_analysis = re[3];
  s.t_factor = re[4];
  s.t_solve = re[5];
  s.t_total = re[6];
  s.relres = re[7];
  s.absres = re[8];
  s.method = method;
  s.error = error;
  for (int q = 0; q < npf; q++) {
    FrontStat f;
    f.id = (int)pf[6 * q];
    f.level = (int)pf[6 * q + 1];
    f.dim = (int)pf[6 * q + 2];
    f.sep = (int)pf[6 * q + 3];
    f.rank = (int)pf[6 * q + 4];
    f.flops = pf[6 * q + 5];
    f.type = pf_type[q];
    s.per_front.push_back(f);
  }
  std::string all = stats_to_json(s, include_pf != 0);
  all.push_back('\0');
  all += stats_csv_header();
  all.push_back('\0');
  all += stats_csv_row(s);
  all.push_back('\0');
  if ((long long)all.size() <= cap) std::memcpy(out, all.data(), all.size());
  return (long long)all.size();
}

}  // extern "C"
