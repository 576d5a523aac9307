// hssmf_b200/hssmf.hpp — header-only C++ drop-in over the C-ABI (hssmf_b200.h).
//
// A program written against the reference (proj/include/hssmf) keeps its
// types — SparseMatrix<double>, EliminationTree, SolverOptions,
// DenseMatrix<double> — and swaps the two calls of the hot path:
//
//     auto m = hssmf::mf_factor(a, t, opts);      // multifrontal.hpp:473-503
//     hssmf::mf_solve(m, b);                      // multifrontal.hpp:612-622
//   becomes
//     auto m = hssmf_b200::mf_factor(a, t, opts); // sm_100a kernels on a B200
//     hssmf_b200::mf_solve(m, b);
//
// The functions are templates over the reference types (duck-typed: only the
// members the reference exposes are used), so this header does not depend on
// the reference sources. Define HSSMF_B200_REFERENCE_ERRORS after including
// the reference's "hssmf/errors.hpp" to receive the reference's own exception
// types (IoError, SolverError, SingularMatrixError(column), HssRankExceeded);
// otherwise same-named classes in namespace hssmf_b200 are thrown.
#ifndef HSSMF_B200_HSSMF_HPP
#define HSSMF_B200_HSSMF_HPP

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hssmf_b200.h"

namespace hssmf_b200 {

#ifdef HSSMF_B200_REFERENCE_ERRORS
  using SolverError = ::hssmf::SolverError;
  using IoError = ::hssmf::IoError;
  using SingularMatrixError = ::hssmf::SingularMatrixError;
  using KrylovDivergenceError = ::hssmf::KrylovDivergenceError;
#else
  struct SolverError : std::runtime_error {
    explicit SolverError(const std::string& m) : std::runtime_error(m) {}
  };
  struct IoError : SolverError {
    explicit IoError(const std::string& m) : SolverError(m) {}
  };
  struct SingularMatrixError : SolverError {
    SingularMatrixError(const std::string& where, int col)
        : SolverError(where), column_(col) {}
    int column() const { return column_; }

   private:
    int column_;
  };
  struct KrylovDivergenceError : SolverError {
    explicit KrylovDivergenceError(const std::string& m) : SolverError(m) {}
  };
#endif

  namespace detail {
    [[noreturn]] inline void raise(int rc, const hssmf_status& st) {
      const std::string m(st.msg);
      switch (rc) {
        case HSSMF_ERR_SHAPE: throw IoError(m);
#ifdef HSSMF_B200_REFERENCE_ERRORS
        case HSSMF_ERR_SINGULAR: throw SingularMatrixError("front " + std::to_string(st.front), st.column);
#else
        case HSSMF_ERR_SINGULAR: throw SingularMatrixError(m, st.column);
#endif
        case HSSMF_ERR_DIVERGENCE: throw KrylovDivergenceError(m);
        default: throw SolverError(m);
      }
    }
    inline void check(int rc, const hssmf_status& st) {
      if (rc != HSSMF_OK) raise(rc, st);
    }
  }  // namespace detail

  // FrontStat (reference stats.hpp:11-19)
  struct FrontStat {
    int id = 0, level = 0, dim = 0, sep = 0, rank = 0;
    long long flops = 0;
    std::string type;
  };

  // MfFactors (reference multifrontal.hpp:454-468); move-only, device-resident
  class MfFactors {
   public:
    MfFactors() = default;
    MfFactors(const MfFactors&) = delete;
    MfFactors& operator=(const MfFactors&) = delete;
    MfFactors(MfFactors&& o) noexcept { *this = std::move(o); }
    MfFactors& operator=(MfFactors&& o) noexcept {
      if (this != &o) {
        reset();
        h_ = o.h_;
        n_ = o.n_;
        front_stats = std::move(o.front_stats);
        factored = o.factored;
        hss_fronts = o.hss_fronts;
        fallbacks = o.fallbacks;
        max_front_rank = o.max_front_rank;
        nnz_ = o.nnz_;
        o.h_ = nullptr;
        o.factored = false;
      }
      return *this;
    }
    ~MfFactors() { reset(); }

    std::vector<FrontStat> front_stats;
    bool factored = false;
    int hss_fronts = 0, fallbacks = 0, max_front_rank = 0;
    std::int64_t factor_nnz() const { return nnz_; }
    int n() const { return n_; }
    hssmf_factors* handle() const { return h_; }

    void adopt(hssmf_factors* h, int n) {
      reset();
      h_ = h;
      n_ = n;
      int nn = 0;
      long long nz = 0;
      hssmf_factor_summary(h, &nn, &hss_fronts, &fallbacks, &max_front_rank, &nz);
      nnz_ = nz;
      std::vector<int> lv(nn), dim(nn), sep(nn), rk(nn), ty(nn);
      std::vector<long long> fl(nn);
      hssmf_front_stats(h, lv.data(), dim.data(), sep.data(), rk.data(), fl.data(), ty.data());
      static const char* names[3] = {"dense", "hss", "hss_dense"};
      front_stats.resize(nn);
      for (int i = 0; i < nn; i++)
        front_stats[i] = {i, lv[i], dim[i], sep[i], rk[i], fl[i], names[ty[i]]};
      factored = true;
    }

   private:
    void reset() {
      if (h_) hssmf_factors_free(h_);
      h_ = nullptr;
      factored = false;
    }
    hssmf_factors* h_ = nullptr;
    int n_ = 0;
    std::int64_t nnz_ = 0;
  };

  namespace detail {
    // C-ABI copies of a reference-typed matrix and tree (RAII)
    struct Inputs {
      hssmf_csr* c = nullptr;
      hssmf_tree* tr = nullptr;
      Inputs() = default;
      Inputs(const Inputs&) = delete;
      Inputs& operator=(const Inputs&) = delete;
      ~Inputs() {
        if (tr) hssmf_tree_free(tr);
        if (c) hssmf_csr_free(c);
      }
    };
    template<class Sparse, class Tree>
    void make_inputs(const Sparse& a, const Tree& t, Inputs& in) {
      hssmf_status st{};
      if (a.size() != t.n) throw IoError("mf factor: matrix and tree sizes differ");
      check(hssmf_csr_create(a.size(), a.ptr().data(), a.ind().data(), a.val().data(), &in.c, &st), st);
      const int nn = static_cast<int>(t.nodes.size());
      std::vector<int> sb(nn), se(nn), c0(nn), c1(nn), pa(nn), up(nn + 1, 0), ui;
      for (int i = 0; i < nn; i++) {
        const auto& f = t.nodes[i];
        sb[i] = f.sep_begin;
        se[i] = f.sep_end;
        c0[i] = f.child0;
        c1[i] = f.child1;
        pa[i] = f.parent;
        ui.insert(ui.end(), f.upd.begin(), f.upd.end());
        up[i + 1] = static_cast<int>(ui.size());
      }
      check(hssmf_tree_create(t.n, nn, sb.data(), se.data(), c0.data(), c1.data(), pa.data(),
                              up.data(), ui.data(), &in.tr, &st), st);
      // separator clusters from the reference's reorder_tree_separators
      // (FrontNode::sep_clusters) travel with the tree
      for (int i = 0; i < nn; i++) {
        const auto& sc = t.nodes[i].sep_clusters;
        if (sc.empty()) continue;
        const int cn = sc.size();
        std::vector<int> cb(cn), ce(cn), cc0(cn), cc1(cn);
        for (int k = 0; k < cn; k++) {
          cb[k] = sc.node(k).begin;
          ce[k] = sc.node(k).end;
          cc0[k] = sc.node(k).child0;
          cc1[k] = sc.node(k).child1;
        }
        check(hssmf_tree_set_sep_clusters(in.tr, i, cn, cb.data(), ce.data(), cc0.data(),
                                          cc1.data(), &st), st);
      }
    }
    template<class Opts> hssmf_options options(const Opts& opts) {
      return hssmf_options{opts.ls, opts.eps, opts.leaf, opts.d0, opts.dd, opts.p, opts.min_hss,
                           opts.max_rank, static_cast<int>(opts.mode)};
    }
  }  // namespace detail

  // mf_factor(a, t, opts) (reference multifrontal.hpp:473-503). `a` must carry
  // the tree's ordering (SparseMatrix::permuted), `t` the symbolic upd sets.
  template<class Sparse, class Tree, class Opts>
  MfFactors mf_factor(const Sparse& a, const Tree& t, const Opts& opts, int device = 0) {
    detail::Inputs in;
    detail::make_inputs(a, t, in);
    hssmf_options o = detail::options(opts);
    hssmf_status st{};
    hssmf_factors* h = nullptr;
    detail::check(hssmf_factor(device, in.c, in.tr, &o, &h, &st), st);
    MfFactors m;
    m.adopt(h, a.size());
    return m;
  }

  // mf_solve(m, b) in place (reference multifrontal.hpp:612-622); b is a
  // column-major dense matrix (rows() x cols(), ld(), data())
  template<class Dense>
  void mf_solve(MfFactors& m, Dense& b) {
    if (!m.factored || !m.handle()) throw SolverError("mf solve: not factored");
    if (static_cast<int>(b.rows()) != m.n()) throw IoError("mf solve: rhs rows mismatch");
    hssmf_status st{};
    detail::check(hssmf_solve(m.handle(), b.data(), static_cast<int>(b.ld()),
                              static_cast<int>(b.cols()), 0, &st),
                  st);
  }

  template<class Dense>
  Dense mf_solve_new(MfFactors& m, const Dense& b) {
    Dense x(b);
    mf_solve(m, x);
    return x;
  }

  // SolveReport (reference krylov.hpp:22-29)
  struct SolveReport {
    int iterations = 0;
    double rel_resid = 0, abs_resid = 0;
    bool converged = false, stagnated = false;
    std::vector<double> history;
  };

  namespace detail {
    template<class Sparse>
    hssmf_csr* upload_csr(const Sparse& a) {
      hssmf_status st{};
      hssmf_csr* c = nullptr;
      check(hssmf_csr_create(a.size(), a.ptr().data(), a.ind().data(), a.val().data(), &c, &st), st);
      return c;
    }
    template<class Call>
    std::pair<std::vector<double>, SolveReport> krylov(int n, int maxit, Call&& call) {
      std::vector<double> x(n), hist(maxit + 2);
      hssmf_krylov_report r{};
      hssmf_status st{};
      const int rc = call(x.data(), &r, hist.data(), static_cast<int>(hist.size()), &st);
      check(rc, st);
      SolveReport rep;
      rep.iterations = r.iterations;
      rep.rel_resid = r.rel_resid;
      rep.abs_resid = r.abs_resid;
      rep.converged = r.converged != 0;
      rep.stagnated = r.stagnated != 0;
      rep.history.assign(hist.begin(), hist.begin() + std::min<int>(r.history_len, hist.size()));
      return {std::move(x), std::move(rep)};
    }
  }  // namespace detail

  // gmres(A, M^-1 = mf_solve(m), b, restart, rtol, atol, maxit) (reference
  // krylov.hpp:93-184 with apply_a = a.matvec and apply_m_inv = the mf_op
  // closure of test_krylov.cpp:26-32), run on the device
  template<class Sparse>
  std::pair<std::vector<double>, SolveReport> gmres(const Sparse& a, MfFactors& m,
                                                    const std::vector<double>& b,
                                                    int restart = 30, double rtol = 1e-6,
                                                    double atol = 1e-10, int maxit = 500) {
    if (restart < 1) throw IoError("gmres: restart must be >= 1");
    hssmf_csr* c = detail::upload_csr(a);
    try {
      auto out = detail::krylov(a.size(), maxit, [&](double* x, hssmf_krylov_report* r, double* h,
                                                     int cap, hssmf_status* st) {
        return hssmf_gmres(c, m.handle(), b.data(), x, restart, rtol, atol, maxit, r, h, cap, st);
      });
      hssmf_csr_free(c);
      return out;
    } catch (...) {
      hssmf_csr_free(c);
      throw;
    }
  }

  // iterative_refinement (reference krylov.hpp:189-229)
  template<class Sparse>
  std::pair<std::vector<double>, SolveReport> iterative_refinement(
      const Sparse& a, MfFactors& m, const std::vector<double>& b, double rtol = 1e-6,
      double atol = 1e-10, int maxit = 500) {
    hssmf_csr* c = detail::upload_csr(a);
    try {
      auto out = detail::krylov(a.size(), maxit, [&](double* x, hssmf_krylov_report* r, double* h,
                                                     int cap, hssmf_status* st) {
        return hssmf_refine(c, m.handle(), b.data(), x, rtol, atol, maxit, r, h, cap, st);
      });
      hssmf_csr_free(c);
      return out;
    } catch (...) {
      hssmf_csr_free(c);
      throw;
    }
  }

}  // namespace hssmf_b200

#endif
