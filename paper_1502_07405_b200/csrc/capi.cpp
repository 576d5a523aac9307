// extern "C" boundary (include/hssmf_b200.h) over the host analysis and the
// device engine. Exceptions never cross the ABI: they become hssmf_codes.
#include "../../include/hssmf_b200.h"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "engine.hpp"
#include "mgpu.hpp"
#include "hss.hpp"
#include "hss_dense.hpp"
#include "host/analysis.hpp"
#include "kernels_test.hpp"
#include "krylov.hpp"
#include "staging.cuh"

using namespace hssmf_b200;

namespace hssmf_b200 {
  std::atomic<long long>& launch_counter() {
    static std::atomic<long long> c{0};
    return c;
  }
  SyncClock& sync_clock() {
    static thread_local SyncClock c;
    return c;
  }
  void stream_sync(cudaStream_t s) {
    auto& c = sync_clock();
    const auto a = std::chrono::steady_clock::now();
    HSSMF_CUDA(cudaStreamSynchronize(s));
    c.wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count();
    c.n++;
    if (Staging* st = current_staging(s)) st->complete();
  }
}  // namespace hssmf_b200

struct hssmf_csr { Csr a; };
struct hssmf_tree { Etree t; };
struct hssmf_factors {
  std::unique_ptr<Engine> e;
  // multi-GPU rank handle (hssmf_mgpu_factor): the partition and the tree
  std::shared_ptr<MgpuPlan> plan;
  std::shared_ptr<Etree> tree;
  int rank = 0;
};
struct hssmf_hss { std::unique_ptr<DenseHss> h; };

namespace {
  int fail(hssmf_status* st, int code, const std::string& msg, int front = -1, int col = -1) {
    if (st) {
      st->code = code;
      st->front = front;
      st->column = col;
      std::snprintf(st->msg, sizeof(st->msg), "%s", msg.c_str());
    }
    return code;
  }
  int ok(hssmf_status* st) {
    if (st) {
      st->code = HSSMF_OK;
      st->front = st->column = -1;
      st->msg[0] = 0;
    }
    return HSSMF_OK;
  }
  template<typename F> int guard(hssmf_status* st, F&& f) {
    try {
      f();
      return ok(st);
    } catch (const SolverFailure& e) {
      return fail(st, e.code, e.what(), e.front, e.column);
    } catch (const HssSingular& e) {
      return fail(st, HSSMF_ERR_SINGULAR, e.what(), -1, e.column);
    } catch (const HssRankError& e) {
      return fail(st, HSSMF_ERR_RANK, e.what(), e.node, -1);
    } catch (const KrylovDivergence& e) {
      return fail(st, HSSMF_ERR_DIVERGENCE, e.what());
    } catch (const CudaError& e) {
      return fail(st, HSSMF_ERR_CUDA, e.what());
    } catch (const std::invalid_argument& e) {  // malformed input (IoError)
      return fail(st, HSSMF_ERR_SHAPE, e.what());
    } catch (const std::exception& e) {
      return fail(st, HSSMF_ERR_OTHER, e.what());
    }
  }
  Options to_opts(const hssmf_options* o) {
    Options r;
    if (!o) return r;
    r.ls = o->ls;
    r.eps = o->eps;
    r.leaf = o->leaf;
    r.d0 = o->d0;
    r.dd = o->dd;
    r.p = o->p;
    r.min_hss = o->min_hss;
    r.max_rank = o->max_rank;
    r.mode = o->mode;
    return r;
  }
}  // namespace

namespace {
  template<typename Run>
  int krylov_call(const hssmf_csr* a, hssmf_factors* m, const double* b, double* x,
                  hssmf_krylov_report* rep, double* history, int history_cap, hssmf_status* st,
                  Run&& run) {
    return guard(st, [&] {
      const Csr& A = a->a;
      if (m && (!m->e || !m->e->factored()))
        throw SolverFailure(2, -1, -1, "krylov: factors not factored");
      if (m && m->e->n() != A.n) throw SolverFailure(1, -1, -1, "krylov: size mismatch");
      if (m) HSSMF_CUDA(cudaSetDevice(m->e->device()));
      const int n = A.n;
      struct Buf {
        void* p = nullptr;
        explicit Buf(size_t b) { HSSMF_CUDA(cudaMalloc(&p, b ? b : 8)); }
        ~Buf() { cudaFree(p); }
      } dptr((n + 1) * 4), dind(A.ind.size() * 4), dval(A.val.size() * 8), db(n * 8), dx(n * 8);
      HSSMF_CUDA(cudaMemcpy(dptr.p, A.ptr.data(), (n + 1) * 4, cudaMemcpyHostToDevice));
      HSSMF_CUDA(cudaMemcpy(dind.p, A.ind.data(), A.ind.size() * 4, cudaMemcpyHostToDevice));
      HSSMF_CUDA(cudaMemcpy(dval.p, A.val.data(), A.val.size() * 8, cudaMemcpyHostToDevice));
      HSSMF_CUDA(cudaMemcpy(db.p, b, (size_t)n * 8, cudaMemcpyHostToDevice));
      CsrDevView v{n, (const int*)dptr.p, (const int*)dind.p, (const double*)dval.p};
      KrylovReport r = run(v, m ? m->e.get() : nullptr, (const double*)db.p, (double*)dx.p);
      HSSMF_CUDA(cudaMemcpy(x, dx.p, (size_t)n * 8, cudaMemcpyDeviceToHost));
      if (rep) {
        rep->iterations = r.iterations;
        rep->rel_resid = r.rel_resid;
        rep->abs_resid = r.abs_resid;
        rep->converged = r.converged;
        rep->stagnated = r.stagnated;
        rep->history_len = (int)r.history.size();
      }
      if (history)
        for (int i = 0; i < std::min(history_cap, (int)r.history.size()); i++) history[i] = r.history[i];
    });
  }
}  // namespace

extern "C" {

long long hssmf_launch_count(void) { return launch_counter().load(); }

const char* hssmf_version(void) { return "hssmf_b200 0.1 (sm_100a)"; }

int hssmf_csr_grid(int kind, int k, double nu, hssmf_csr** out, int* dims, int* ndims,
                   hssmf_status* st) {
  return guard(st, [&] {
    auto* c = new hssmf_csr;
    Geometry g;
    c->a = grid_problem(kind, k, nu, g);
    if (dims) for (int i = 0; i < 3; i++) dims[i] = g.dims[i];
    if (ndims) *ndims = g.ndims;
    *out = c;
  });
}

int hssmf_csr_convdiff3d(int k, double scale, hssmf_csr** out, hssmf_status* st) {
  return guard(st, [&] {
    auto* c = new hssmf_csr;
    Geometry g;
    c->a = convdiff3d_const(k, scale, g);
    *out = c;
  });
}

int hssmf_csr_create(int n, const int* ptr, const int* ind, const double* val,
                     hssmf_csr** out, hssmf_status* st) {
  return guard(st, [&] {
    if (n < 0) throw SolverFailure(1, -1, -1, "csr: negative size");
    auto* c = new hssmf_csr;
    c->a.n = n;
    c->a.ptr.assign(ptr, ptr + n + 1);
    c->a.ind.assign(ind, ind + ptr[n]);
    c->a.val.assign(val, val + ptr[n]);
    *out = c;
  });
}

int hssmf_csr_permuted(const hssmf_csr* a, const int* perm, hssmf_csr** out,
                       hssmf_status* st) {
  return guard(st, [&] {
    auto* c = new hssmf_csr;
    c->a = a->a.permuted(std::vector<int>(perm, perm + a->a.n));
    *out = c;
  });
}

void hssmf_csr_info(const hssmf_csr* a, int* n, long long* nnz) {
  *n = a->a.n;
  *nnz = a->a.nnz();
}

void hssmf_csr_get(const hssmf_csr* a, int* ptr, int* ind, double* val) {
  std::memcpy(ptr, a->a.ptr.data(), (a->a.n + 1) * sizeof(int));
  std::memcpy(ind, a->a.ind.data(), a->a.ind.size() * sizeof(int));
  std::memcpy(val, a->a.val.data(), a->a.val.size() * sizeof(double));
}

void hssmf_csr_matvec(const hssmf_csr* a, const double* x, double* y) {
  const auto& A = a->a;
  for (int i = 0; i < A.n; i++) {
    double s = 0;
    for (int k = A.ptr[i]; k < A.ptr[i + 1]; k++) s += A.val[k] * x[A.ind[k]];
    y[i] = s;
  }
}

void hssmf_csr_free(hssmf_csr* a) { delete a; }

int hssmf_nd_geometric(const int* dims, int ndims, int leaf, int* perm, hssmf_tree** out,
                       hssmf_status* st) {
  return guard(st, [&] {
    Geometry g;
    g.dims = {dims[0], dims[1], dims[2]};
    g.ndims = ndims;
    std::vector<int> p;
    auto* t = new hssmf_tree;
    t->t = nested_dissection_geometric(g, leaf, p);
    std::memcpy(perm, p.data(), p.size() * sizeof(int));
    *out = t;
  });
}

int hssmf_tree_create(int n, int nnodes, const int* sep_begin, const int* sep_end,
                      const int* child0, const int* child1, const int* parent,
                      const int* upd_ptr, const int* upd_ind, hssmf_tree** out,
                      hssmf_status* st) {
  return guard(st, [&] {
    auto* t = new hssmf_tree;
    t->t.n = n;
    t->t.nodes.resize(nnodes);
    for (int i = 0; i < nnodes; i++) {
      auto& f = t->t.nodes[i];
      f.sep_begin = sep_begin[i];
      f.sep_end = sep_end[i];
      f.child0 = child0[i];
      f.child1 = child1[i];
      f.parent = parent[i];
      if (upd_ptr) f.upd.assign(upd_ind + upd_ptr[i], upd_ind + upd_ptr[i + 1]);
    }
    t->t.compute_levels();
    *out = t;
  });
}

int hssmf_symbolic(const hssmf_csr* a, hssmf_tree* t, hssmf_status* st) {
  return guard(st, [&] {
    if (a->a.n != t->t.n) throw SolverFailure(1, -1, -1, "symbolic: size mismatch");
    symbolic_factorization(a->a, t->t);
    t->t.compute_levels();
  });
}

int hssmf_csr_read_mm(const char* path, hssmf_csr** out, hssmf_status* st) {
  return guard(st, [&] {
    auto* c = new hssmf_csr;
    try {
      c->a = read_matrix_market(path);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int hssmf_csr_write_mm(const hssmf_csr* a, const char* path, hssmf_status* st) {
  return guard(st, [&] { write_matrix_market(a->a, path); });
}

int hssmf_equilibrate(const hssmf_csr* a, hssmf_csr** out, double* dr, double* dc, int* qc,
                      int* sweeps, hssmf_status* st) {
  return guard(st, [&] {
    Scaling sc;
    Csr s = equilibrate_and_permute(a->a, sc);
    auto* c = new hssmf_csr;
    c->a = std::move(s);
    const size_t n = (size_t)a->a.n;
    if (n) {
      std::memcpy(dr, sc.dr.data(), n * sizeof(double));
      std::memcpy(dc, sc.dc.data(), n * sizeof(double));
      std::memcpy(qc, sc.qc.data(), n * sizeof(int));
    }
    *sweeps = sc.sweeps;
    *out = c;
  });
}

int hssmf_nd_graph(const hssmf_csr* a, int leaf, int* perm, hssmf_tree** out, hssmf_status* st) {
  return guard(st, [&] {
    std::vector<int> gptr, gind, p;
    a->a.symmetric_graph(gptr, gind);
    auto* t = new hssmf_tree;
    t->t = nested_dissection_graph(a->a.n, gptr, gind, leaf, p);
    if (a->a.n) std::memcpy(perm, p.data(), p.size() * sizeof(int));
    *out = t;
  });
}

int hssmf_reorder_separators(hssmf_tree* t, const hssmf_csr* a, const char* selected, int b,
                             int* perm, hssmf_status* st) {
  return guard(st, [&] {
    if (a->a.n != t->t.n) throw SolverFailure(1, -1, -1, "reorder: size mismatch");
    std::vector<int> gptr, gind;
    a->a.symmetric_graph(gptr, gind);
    std::vector<char> sel(selected, selected + t->t.nodes.size());
    const auto p = reorder_tree_separators(t->t, sel, gptr, gind, b);
    if (t->t.n) std::memcpy(perm, p.data(), p.size() * sizeof(int));
  });
}

int hssmf_tree_sep_clusters(const hssmf_tree* t, int front, int* begin, int* end, int* child0,
                            int* child1, int* parent) {
  if (front < 0 || front >= (int)t->t.nodes.size()) return -1;
  const auto& c = t->t.nodes[front].sep_clusters.nodes;
  for (size_t i = 0; i < c.size(); i++) {
    if (begin) begin[i] = c[i].begin;
    if (end) end[i] = c[i].end;
    if (child0) child0[i] = c[i].child0;
    if (child1) child1[i] = c[i].child1;
    if (parent) parent[i] = c[i].parent;
  }
  return (int)c.size();
}

int hssmf_tree_set_sep_clusters(hssmf_tree* t, int front, int nnodes, const int* begin,
                                const int* end, const int* child0, const int* child1,
                                hssmf_status* st) {
  return guard(st, [&] {
    if (front < 0 || front >= (int)t->t.nodes.size())
      throw SolverFailure(1, -1, -1, "sep clusters: front out of range");
    ClusterTree c;
    c.nodes.resize(nnodes);
    for (int i = 0; i < nnodes; i++) c.nodes[i] = {begin[i], end[i], child0[i], child1[i], -1};
    for (int i = 0; i < nnodes; i++) {
      if (child0[i] >= i || child1[i] >= i || (child0[i] < 0) != (child1[i] < 0))
        throw SolverFailure(1, -1, -1, "sep clusters: not a postorder binary tree");
      if (child0[i] >= 0) c.nodes[child0[i]].parent = c.nodes[child1[i]].parent = i;
    }
    t->t.nodes[front].sep_clusters = std::move(c);
  });
}

void hssmf_tree_info(const hssmf_tree* t, int* n, int* nnodes, long long* upd_total) {
  *n = t->t.n;
  *nnodes = (int)t->t.nodes.size();
  long long s = 0;
  for (const auto& f : t->t.nodes) s += f.nu();
  *upd_total = s;
}

void hssmf_tree_get(const hssmf_tree* t, int* sep_begin, int* sep_end, int* child0,
                    int* child1, int* parent, int* level, int* upd_ptr, int* upd_ind) {
  long long off = 0;
  for (size_t i = 0; i < t->t.nodes.size(); i++) {
    const auto& f = t->t.nodes[i];
    sep_begin[i] = f.sep_begin;
    sep_end[i] = f.sep_end;
    child0[i] = f.child0;
    child1[i] = f.child1;
    parent[i] = f.parent;
    level[i] = f.level;
    upd_ptr[i] = (int)off;
    for (int g : f.upd) upd_ind[off++] = g;
  }
  upd_ptr[t->t.nodes.size()] = (int)off;
}

void hssmf_tree_free(hssmf_tree* t) { delete t; }

int hssmf_front_cluster_tree(int ns, int nu, int leaf, int* begin, int* end, int* child0,
                             int* child1, int* parent) {
  auto c = front_cluster_tree(ns, nu, leaf);
  if (begin)
    for (size_t i = 0; i < c.nodes.size(); i++) {
      begin[i] = c.nodes[i].begin;
      end[i] = c.nodes[i].end;
      child0[i] = c.nodes[i].child0;
      child1[i] = c.nodes[i].child1;
      parent[i] = c.nodes[i].parent;
    }
  return (int)c.nodes.size();
}

int hssmf_factor(int device, const hssmf_csr* a, const hssmf_tree* t, const hssmf_options* o,
                 hssmf_factors** out, hssmf_status* st) {
  *out = nullptr;
  auto f = std::make_unique<hssmf_factors>();
  const int rc = guard(st, [&] {
    f->e = std::make_unique<Engine>(device);
    f->e->analyze(a->a, t->t, to_opts(o));
    f->e->factor();
  });
  if (rc == HSSMF_OK) *out = f.release();
  return rc;
}

int hssmf_analyze_owned(int device, const hssmf_csr* a, const hssmf_tree* t,
                        const hssmf_options* o, const char* owned, hssmf_factors** out,
                        hssmf_status* st) {
  *out = nullptr;
  auto f = std::make_unique<hssmf_factors>();
  const int rc = guard(st, [&] {
    f->e = std::make_unique<Engine>(device);
    f->e->analyze(a->a, t->t, to_opts(o), owned);
  });
  if (rc == HSSMF_OK) *out = f.release();
  return rc;
}

int hssmf_nlevels(const hssmf_factors* f) { return f->e->nlevels(); }

int hssmf_factor_levels(hssmf_factors* f, int lo, int hi, hssmf_status* st) {
  return guard(st, [&] { f->e->factor_levels(lo, hi); });
}

int hssmf_update_export(const hssmf_factors* f, int front, double* dst, int on_device,
                        hssmf_status* st) {
  return guard(st, [&] { f->e->export_update(front, dst, on_device != 0); });
}

int hssmf_update_import(hssmf_factors* f, int front, const double* src, int on_device,
                        hssmf_status* st) {
  return guard(st, [&] { f->e->import_update(front, src, on_device != 0); });
}

int hssmf_bupd_export(const hssmf_factors* f, int front, double* dst, int nrhs,
                      hssmf_status* st) {
  return guard(st, [&] { f->e->export_bupd(front, dst, nrhs); });
}

int hssmf_bupd_import(hssmf_factors* f, int front, const double* src, int nrhs,
                      hssmf_status* st) {
  return guard(st, [&] { f->e->import_bupd(front, src, nrhs); });
}

int hssmf_solve_levels(hssmf_factors* f, double* x, int ldx, int nrhs, int lo, int hi,
                       int forward, hssmf_status* st) {
  return guard(st, [&] {
    if (ldx < f->e->n()) throw SolverFailure(1, -1, -1, "mf solve: rhs rows mismatch");
    f->e->solve_levels(x, ldx, nrhs, lo, hi, forward != 0);
  });
}

int hssmf_gmres(const hssmf_csr* a, hssmf_factors* m, const double* b, double* x, int restart,
                double rtol, double atol, int maxit, hssmf_krylov_report* rep, double* history,
                int history_cap, hssmf_status* st) {
  return krylov_call(a, m, b, x, rep, history, history_cap, st,
                     [&](const CsrDevView& v, Engine* e, const double* db, double* dx) {
                       return krylov_gmres(v, e, db, dx, restart, rtol, atol, maxit, nullptr);
                     });
}

int hssmf_refine(const hssmf_csr* a, hssmf_factors* m, const double* b, double* x, double rtol,
                 double atol, int maxit, hssmf_krylov_report* rep, double* history,
                 int history_cap, hssmf_status* st) {
  return krylov_call(a, m, b, x, rep, history, history_cap, st,
                     [&](const CsrDevView& v, Engine* e, const double* db, double* dx) {
                       return krylov_refine(v, e, db, dx, rtol, atol, maxit, nullptr);
                     });
}

int hssmf_refactor(hssmf_factors* f, const double* val, int on_device, hssmf_status* st) {
  return guard(st, [&] {
    if (val) f->e->set_values(val, on_device != 0);
    f->e->factor();
  });
}

int hssmf_solve(hssmf_factors* f, double* b, int ldb, int nrhs, int on_device,
                hssmf_status* st) {
  return guard(st, [&] {
    if (!f || !f->e || !f->e->factored())
      throw SolverFailure(2, -1, -1, "mf solve: not factored");
    if (ldb < f->e->n()) throw SolverFailure(1, -1, -1, "mf solve: rhs rows mismatch");
    f->e->solve(b, ldb, nrhs, on_device != 0);
  });
}

void hssmf_factor_summary(const hssmf_factors* f, int* nnodes, int* hss_fronts,
                          int* fallbacks, int* max_rank, long long* factor_nnz) {
  *nnodes = (int)f->e->stats().size();
  *hss_fronts = f->e->hss_fronts();
  *fallbacks = f->e->fallbacks();
  *max_rank = f->e->max_front_rank();
  *factor_nnz = f->e->factor_nnz();
}

void hssmf_front_stats(const hssmf_factors* f, int* level, int* dim, int* sep, int* rank,
                       long long* flops, int* type) {
  const auto& s = f->e->stats();
  for (size_t i = 0; i < s.size(); i++) {
    level[i] = s[i].level;
    dim[i] = s[i].dim;
    sep[i] = s[i].sep;
    rank[i] = s[i].rank;
    flops[i] = s[i].flops;
    type[i] = s[i].type;
  }
}

int hssmf_front_hss(const hssmf_factors* f, int front, int* u_rank, int* v_rank, int* rounds,
                    int* d_final) {
  std::vector<int> u, v;
  int r = 0, d = 0;
  if (!f->e->front_hss(front, u, v, r, d)) return 0;
  if (u_rank)
    for (size_t i = 0; i < u.size(); i++) {
      u_rank[i] = u[i];
      v_rank[i] = v[i];
    }
  if (rounds) *rounds = r;
  if (d_final) *d_final = d;
  return (int)u.size();
}

void hssmf_timing(const hssmf_factors* f, double* factor_ms, double* solve_ms) {
  *factor_ms = f->e->factor_ms();
  *solve_ms = f->e->solve_ms();
}

void hssmf_set_profile(hssmf_factors* f, int on) { f->e->set_profile(on != 0); }

int hssmf_kernel_stats(const hssmf_factors* f, int max, char* names, int* launches, double* ms,
                       double* flops, double* bytes) {
  auto ks = f->e->kernel_stats();
  const int n = (int)ks.size() < max ? (int)ks.size() : max;
  for (int i = 0; i < n; i++) {
    std::snprintf(names + 32 * i, 32, "%s", ks[i].name.c_str());
    launches[i] = ks[i].launches;
    ms[i] = ks[i].ms;
    flops[i] = ks[i].flops;
    bytes[i] = ks[i].bytes;
  }
  return n;
}

void hssmf_reset_kernel_stats(hssmf_factors* f) { f->e->reset_kernel_stats(); }
long long hssmf_device_bytes(const hssmf_factors* f) { return (long long)f->e->device_bytes(); }
void hssmf_factors_free(hssmf_factors* f) { delete f; }

int hssmf_hss_dense(int device, const double* a, int lda, int n, int leaf, double eps, int d0,
                    int dd, int p, int max_rank, int on_device, hssmf_hss** out,
                    hssmf_status* st) {
  *out = nullptr;
  auto h = std::make_unique<hssmf_hss>();
  const int rc = guard(st, [&] {
    h->h = std::make_unique<DenseHss>(device);
    h->h->run(a, lda, n, leaf, eps, d0, dd, p, max_rank, on_device != 0);
  });
  if (rc == HSSMF_OK) *out = h.release();
  return rc;
}

int hssmf_hss_dense_tree(int device, const double* a, int lda, int n, int nnodes,
                         const int* begin, const int* end, const int* child0, const int* child1,
                         double eps, int d0, int dd, int p, int max_rank, int on_device,
                         hssmf_hss** out, hssmf_status* st) {
  *out = nullptr;
  auto h = std::make_unique<hssmf_hss>();
  const int rc = guard(st, [&] {
    h->h = std::make_unique<DenseHss>(device);
    h->h->run_tree(a, lda, n, nnodes, begin, end, child0, child1, eps, d0, dd, p, max_rank,
                   on_device != 0);
  });
  if (rc == HSSMF_OK) *out = h.release();
  return rc;
}

int hssmf_hss_matvec(hssmf_hss* h, char op, int root, const double* x, int ldx, int nrows,
                     int nc, double* y, int ldy, int on_device, hssmf_status* st) {
  return guard(st, [&] {
    if (op != 'N' && op != 'T' && op != 'C') throw std::invalid_argument("hss matvec: op must be N, T or C");
    if (nrows != h->h->node_size(root))
      throw std::invalid_argument("hss matvec: x rows do not match the cluster node");
    if (ldx < nrows || ldy < nrows) throw std::invalid_argument("hss matvec: leading dimension");
    h->h->matvec(op == 'N' ? 'N' : 'T', root, x, ldx, nc, y, ldy, on_device != 0);
  });
}

int hssmf_hss_extract(hssmf_hss* h, const int* rows, int ni, const int* cols, int nj,
                      double* out, int on_device, long long* leaf_visits, hssmf_status* st) {
  return guard(st, [&] {
    const long long v = h->h->extract(rows, ni, cols, nj, out, on_device != 0);
    if (leaf_visits) *leaf_visits = v;
  });
}

int hssmf_hss_info(const hssmf_hss* h, int* u_rank, int* v_rank, int* rounds, int* d_final,
                   double* compress_ms, double* ulv_ms) {
  std::vector<int> u, v;
  h->h->ranks(u, v);
  if (u_rank)
    for (size_t i = 0; i < u.size(); i++) {
      u_rank[i] = u[i];
      v_rank[i] = v[i];
    }
  if (rounds) *rounds = h->h->rounds();
  if (d_final) *d_final = h->h->d_final();
  if (compress_ms) *compress_ms = h->h->compress_ms();
  if (ulv_ms) *ulv_ms = h->h->ulv_ms();
  return (int)u.size();
}

int hssmf_hss_solve(hssmf_hss* h, double* b, int ldb, int nrhs, int on_device,
                    hssmf_status* st) {
  return guard(st, [&] { h->h->solve(b, ldb, nrhs, on_device != 0); });
}

void hssmf_hss_free(hssmf_hss* h) { delete h; }

int hssmf_dev_random_rows(int device, int nrows, const long long* grow, int c0, int c1,
                          double* out, hssmf_status* st) {
  return guard(st, [&] { test_random_rows(device, nrows, grow, c0, c1, out); });
}

int hssmf_dev_gemm(int device, char ta, char tb, int m, int n, int k, double alpha,
                   const double* a, int lda, const double* b, int ldb, double beta, double* c,
                   int ldc, hssmf_status* st) {
  return guard(st, [&] { test_gemm(device, ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc); });
}

int hssmf_dev_id(int device, const double* y, int m, int n, double eps, int max_rank,
                 double abs_tol, int* perm, int* rank, int* certified, double* coeffs,
                 hssmf_status* st) {
  return guard(st, [&] {
    test_id(device, y, m, n, eps, max_rank, abs_tol, perm, rank, certified, coeffs);
  });
}

int hssmf_dev_gram_id(int device, const double* y, int m, int n, double eps, int max_rank,
                      double abs_tol, int* perm, int* rank, int* certified, double* r,
                      hssmf_status* st) {
  return guard(st, [&] {
    test_gram_id(device, y, m, n, eps, max_rank, abs_tol, perm, rank, certified, r);
  });
}

int hssmf_probe_enable(int on, hssmf_status* st) {
  return guard(st, [&] { probe_enable(on != 0); });
}

int hssmf_probe_read(hssmf_probe_stat* out, hssmf_status* st) {
  return guard(st, [&] {
    ProbeStat p[PROBE_KINDS];
    probe_read(p);
    for (int k = 0; k < PROBE_KINDS; k++) out[k] = {p[k].launches, p[k].ms, p[k].flops, p[k].bytes};
  });
}

int hssmf_bench_gemm(int device, int m, int n, int k, int iters, double* ms, hssmf_status* st) {
  return guard(st, [&] { *ms = bench_gemm(device, m, n, k, iters); });
}

int hssmf_bench_gram(int device, int n, int d, int ntask, int iters, double* ms, int* steps,
                     hssmf_status* st) {
  return guard(st, [&] { *ms = bench_gram(device, n, d, ntask, iters, steps); });
}

int hssmf_dev_lu(int device, double* a, int m, int n, int* piv, hssmf_status* st) {
  return guard(st, [&] { test_lu(device, a, m, n, piv); });
}

}  // extern "C"

/* ---- multi-GPU subtree partition (mgpu.cu) ---- */
namespace {
  struct CallbackTransport : MgpuTransport {
    const hssmf_transport* cb;
    explicit CallbackTransport(const hssmf_transport* c) : cb(c) {}
    void send(const double* buf, long long count, int dst, int) override {
      if (cb->send(cb->ctx, buf, count, dst) != 0)
        throw SolverFailure(HSSMF_ERR_NCCL, -1, -1, "mgpu transport: send to rank " + std::to_string(dst) + " failed");
    }
    void recv(double* buf, long long count, int src, int) override {
      if (cb->recv(cb->ctx, buf, count, src) != 0)
        throw SolverFailure(HSSMF_ERR_NCCL, -1, -1, "mgpu transport: recv from rank " + std::to_string(src) + " failed");
    }
  };
  std::vector<char> owned_mask(const MgpuPlan& P, int rank) {
    std::vector<char> m(P.owner.size());
    for (size_t i = 0; i < m.size(); i++) m[i] = P.owner[i] == rank;
    return m;
  }
}  // namespace

int hssmf_mgpu_partition(const hssmf_tree* t, int nranks, int* owner, int* nedges,
                         hssmf_status* st) {
  return guard(st, [&] {
    const MgpuPlan P = mgpu_partition(t->t, nranks);
    if (owner) std::copy(P.owner.begin(), P.owner.end(), owner);
    if (nedges) *nedges = (int)P.edges.size();
  });
}

int hssmf_mgpu_factor(int device, const hssmf_csr* a, const hssmf_tree* t,
                      const hssmf_options* o, int rank, int nranks, const hssmf_transport* tr,
                      hssmf_factors** out, hssmf_status* st) {
  *out = nullptr;
  auto f = std::make_unique<hssmf_factors>();
  const int rc = guard(st, [&] {
    if (!tr || !tr->send || !tr->recv) throw std::invalid_argument("mgpu factor: no transport");
    if (rank < 0 || rank >= nranks) throw std::invalid_argument("mgpu factor: bad rank");
    f->plan = std::make_shared<MgpuPlan>(mgpu_partition(t->t, nranks));
    f->tree = std::make_shared<Etree>(t->t);
    f->rank = rank;
    const auto mask = owned_mask(*f->plan, rank);
    f->e = std::make_unique<Engine>(device);
    HSSMF_CUDA(cudaSetDevice(device));
    f->e->analyze(a->a, t->t, to_opts(o), mask.data());
    std::map<int, Engine*> eng{{rank, f->e.get()}};
    CallbackTransport ct(tr);
    mgpu_factor(*f->plan, eng, ct);
  });
  if (rc == HSSMF_OK) *out = f.release();
  return rc;
}

int hssmf_mgpu_solve(hssmf_factors* f, const hssmf_transport* tr, double* x, int ldx, int nrhs,
                     hssmf_status* st) {
  return guard(st, [&] {
    if (!f->plan) throw std::invalid_argument("mgpu solve: factors were not made by hssmf_mgpu_factor");
    std::map<int, Engine*> eng{{f->rank, f->e.get()}};
    std::map<int, double*> xs{{f->rank, x}};
    CallbackTransport ct(tr);
    mgpu_solve(*f->plan, *f->tree, eng, xs, ldx, nrhs, ct);
  });
}

int hssmf_mgpu_local(int device, const hssmf_csr* a, const hssmf_tree* t, const hssmf_options* o,
                     int nranks, double* x, int nrhs, hssmf_status* st) {
  return guard(st, [&] {
    HSSMF_CUDA(cudaSetDevice(device));
    const MgpuPlan P = mgpu_partition(t->t, nranks);
    const Options opts = to_opts(o);
    std::vector<std::unique_ptr<Engine>> es;
    std::map<int, Engine*> eng;
    for (int r = 0; r < nranks; r++) {
      const auto mask = owned_mask(P, r);
      es.push_back(std::make_unique<Engine>(device));
      es.back()->analyze(a->a, t->t, opts, mask.data());
      eng[r] = es.back().get();
    }
    LocalTransport lt;
    mgpu_factor(P, eng, lt);
    const int n = t->t.n;
    // every rank solves its own copy of b; the solution is assembled from the
    // separators each rank owns
    std::vector<double*> xr(nranks, nullptr);
    std::map<int, double*> xs;
    for (int r = 0; r < nranks; r++) {
      HSSMF_CUDA(cudaMalloc(&xr[r], (size_t)n * nrhs * sizeof(double) + 8));
      HSSMF_CUDA(cudaMemcpy(xr[r], x, (size_t)n * nrhs * sizeof(double), cudaMemcpyDeviceToDevice));
      xs[r] = xr[r];
    }
    mgpu_solve(P, t->t, eng, xs, n, nrhs, lt);
    for (size_t i = 0; i < t->t.nodes.size(); i++) {
      const auto& fn = t->t.nodes[i];
      if (!fn.ns()) continue;
      HSSMF_CUDA(cudaMemcpy2D(x + fn.sep_begin, (size_t)n * sizeof(double),
                              xr[P.owner[i]] + fn.sep_begin, (size_t)n * sizeof(double),
                              (size_t)fn.ns() * sizeof(double), nrhs, cudaMemcpyDeviceToDevice));
    }
    for (auto p : xr) cudaFree(p);
  });
}
