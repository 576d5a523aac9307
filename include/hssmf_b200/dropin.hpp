// hssmf_b200/dropin.hpp — source-level drop-in for the reference's hot-path
// headers, with the reference's own names and signatures in namespace hssmf.
//
// A program written against proj/include/hssmf includes this header INSTEAD of
// "hssmf/multifrontal.hpp", "hssmf/hss_compress.hpp" and "hssmf/hss_ulv.hpp"
// (after the reference's type headers: sparse_matrix.hpp, dense_matrix.hpp,
// elimination_tree.hpp, cluster_tree.hpp, solver_options.hpp, stats.hpp,
// errors.hpp) and keeps every call site unchanged:
//
//   auto m = hssmf::mf_factor(a, t, opts);          // multifrontal.hpp:473-503
//   hssmf::mf_solve(m, b);                          // multifrontal.hpp:612-622
//   auto x = hssmf::mf_solve_new(m, b);             // multifrontal.hpp:624-631
//   auto h = hssmf::hss_compress(A, tree, hopts, &cst); // hss_compress.hpp:373-383
//   auto u = hssmf::ulv_factor(h);                  // hss_ulv.hpp:284-319
//   u.solve(b);                                     // hss_ulv.hpp:150-176
//
// The numerics run on a B200 through the C-ABI (hssmf_b200.h). The header
// defines the three reference include guards, so a transitive include of the
// reference's own versions is a no-op. Differences a caller can observe:
//  * MfFactors<T> keeps `tree`, `front_stats`, `factored`, `hss_fronts`,
//    `fallbacks`, `max_front_rank` and `factor_nnz()`; the per-front host
//    objects (`fronts`) do not exist: the factors live in device memory.
//  * HssMatrix<T> is a device handle (rows/cols/tree/hss_rank/u_rank/v_rank);
//    hss_compress runs the ULV factorization eagerly on the device, so
//    ulv_factor only binds to it. A non-empty round_hook (a host callback per
//    adaptive round) is rejected with SolverError.
//  * `depth` (the OpenMP task-depth cutoff) is accepted and ignored; the device
//    is hssmf::b200_device() (default 0).
//  * scalar_t must be double (the reference's tests instantiate double; the
//    GPU path is FP64).
#ifndef HSSMF_B200_DROPIN_HPP
#define HSSMF_B200_DROPIN_HPP

#define HSSMF_MULTIFRONTAL_HPP
#define HSSMF_HSS_COMPRESS_HPP
#define HSSMF_HSS_ULV_HPP
#ifndef HSSMF_B200_REFERENCE_ERRORS
#define HSSMF_B200_REFERENCE_ERRORS
#endif

#include <cstdint>
#include <functional>
#include <memory>
#include <type_traits>
#include <vector>

#include "hssmf.hpp"

namespace hssmf {

  // GPU used by the drop-in entry points (the reference has no device notion)
  inline int& b200_device() {
    static int dev = 0;
    return dev;
  }

  // hss_compress.hpp:26-37
  struct HssOptions {
    double eps = 1e-8;
    int d0 = 128;
    int dd = 128;
    int p = 10;
    int max_rank = 5000;
  };
  struct HssCompressStats {
    int rounds = 0;
    int d_final = 0;
  };

  // multifrontal.hpp:454-468 (device-resident fronts)
  template<typename scalar_t> struct MfFactors {
    static_assert(std::is_same_v<scalar_t, double>, "the B200 path computes in FP64");
    EliminationTree tree;
    std::vector<FrontStat> front_stats;
    bool factored = false;
    int hss_fronts = 0;
    int fallbacks = 0;
    int max_front_rank = 0;
    std::int64_t factor_nnz() const { return dev.factor_nnz(); }
    hssmf_b200::MfFactors dev;  // the device handle
  };

  // multifrontal.hpp:473-503
  template<typename scalar_t>
  MfFactors<scalar_t> mf_factor(const SparseMatrix<scalar_t>& a, const EliminationTree& t,
                                const SolverOptions& opts, int depth = 0) {
    (void)depth;
    MfFactors<scalar_t> m;
    m.dev = hssmf_b200::mf_factor(a, t, opts, b200_device());
    m.tree = t;
    m.front_stats.reserve(m.dev.front_stats.size());
    for (const auto& s : m.dev.front_stats) {
      FrontStat f;
      f.id = s.id;
      f.level = s.level;
      f.dim = s.dim;
      f.sep = s.sep;
      f.rank = s.rank;
      f.flops = s.flops;
      f.type = s.type;
      m.front_stats.push_back(f);
    }
    m.factored = m.dev.factored;
    m.hss_fronts = m.dev.hss_fronts;
    m.fallbacks = m.dev.fallbacks;
    m.max_front_rank = m.dev.max_front_rank;
    return m;
  }

  // multifrontal.hpp:612-622
  template<typename scalar_t>
  void mf_solve(MfFactors<scalar_t>& m, DenseMatrix<scalar_t>& b, int depth = 0) {
    (void)depth;
    if (!m.factored) throw SolverError("mf solve: not factored");
    if (static_cast<int>(b.rows()) != m.tree.n) throw IoError("mf solve: rhs rows mismatch");
    hssmf_b200::mf_solve(m.dev, b);
  }

  // multifrontal.hpp:624-631
  template<typename scalar_t>
  DenseMatrix<scalar_t> mf_solve_new(MfFactors<scalar_t>& m, const DenseMatrix<scalar_t>& b,
                                     int depth = 0) {
    DenseMatrix<scalar_t> x(b);
    mf_solve(m, x, depth);
    return x;
  }

  // compressed matrix (hss_matrix.hpp:186-216), held on the device together
  // with its ULV factors
  template<typename scalar_t> class HssMatrix {
    static_assert(std::is_same_v<scalar_t, double>, "the B200 path computes in FP64");

   public:
    HssMatrix() = default;
    HssMatrix(const HssMatrix&) = delete;
    HssMatrix& operator=(const HssMatrix&) = delete;
    HssMatrix(HssMatrix&&) noexcept = default;
    HssMatrix& operator=(HssMatrix&&) noexcept = default;

    bool empty() const { return !h_; }
    int rows() const { return empty() ? 0 : tree_.root().end; }
    int cols() const { return rows(); }
    const ClusterTree& tree() const { return tree_; }
    int u_rank(int i) const { return u_[i]; }
    int v_rank(int i) const { return v_[i]; }
    // max u/v rank over the non-root nodes (hss_matrix.hpp:210-216)
    int hss_rank() const {
      int r = 0;
      for (int i = 0; i + 1 < static_cast<int>(u_.size()); i++) r = std::max({r, u_[i], v_[i]});
      return r;
    }
    hssmf_hss* handle() const { return h_.get(); }

   private:
    struct Free {
      void operator()(hssmf_hss* h) const { hssmf_hss_free(h); }
    };
    template<typename T>
    friend HssMatrix<T> hss_compress(const DenseMatrix<T>&, const ClusterTree&, const HssOptions&,
                                     HssCompressStats*,
                                     const std::function<void(const HssMatrix<T>&, int)>&);
    ClusterTree tree_;
    std::unique_ptr<hssmf_hss, Free> h_;
    std::vector<int> u_, v_;
  };

  // hss_compress.hpp:373-383 (+ the ULV factorization, hss_ulv.hpp:284-319,
  // run eagerly on the device)
  template<typename scalar_t>
  HssMatrix<scalar_t> hss_compress(
      const DenseMatrix<scalar_t>& a, const ClusterTree& tree, const HssOptions& opts,
      HssCompressStats* stats = nullptr,
      const std::function<void(const HssMatrix<scalar_t>&, int)>& round_hook = {}) {
    if (a.rows() != a.cols() || static_cast<int>(a.rows()) != tree.root().end)
      throw IoError("hss compress: matrix and cluster tree sizes disagree");
    if (round_hook) throw SolverError("hss compress: round_hook is not supported on the device");
    const int nn = tree.size();
    std::vector<int> b(nn), e(nn), c0(nn), c1(nn);
    for (int i = 0; i < nn; i++) {
      b[i] = tree.node(i).begin;
      e[i] = tree.node(i).end;
      c0[i] = tree.node(i).child0;
      c1[i] = tree.node(i).child1;
    }
    hssmf_status st{};
    hssmf_hss* h = nullptr;
    const int n = static_cast<int>(a.rows());
    const int rc = hssmf_hss_dense_tree(b200_device(), a.data(), static_cast<int>(a.ld()), n, nn,
                                        b.data(), e.data(), c0.data(), c1.data(), opts.eps,
                                        opts.d0, opts.dd, opts.p, opts.max_rank, 0, &h, &st);
    if (rc == HSSMF_ERR_RANK) throw HssRankExceeded(st.front, opts.max_rank);
    hssmf_b200::detail::check(rc, st);
    HssMatrix<scalar_t> out;
    out.tree_ = tree;
    out.h_.reset(h);
    out.u_.assign(nn, 0);
    out.v_.assign(nn, 0);
    int rounds = 0, dfin = 0;
    hssmf_hss_info(h, out.u_.data(), out.v_.data(), &rounds, &dfin, nullptr, nullptr);
    if (stats) {
      stats->rounds = rounds;
      stats->d_final = dfin;
    }
    return out;
  }

  // hss_ulv.hpp:126-285 (full factorization only; the partial one lives
  // inside mf_factor)
  template<typename scalar_t> class UlvFactors {
   public:
    explicit UlvFactors(const HssMatrix<scalar_t>& h) : hss_(&h) {}
    bool factored() const { return hss_ && !hss_->empty(); }
    void solve(DenseMatrix<scalar_t>& b, int depth = 0) const {
      (void)depth;
      if (!factored()) throw SolverError("ulv solve: factorization missing or partial");
      if (static_cast<int>(b.rows()) != hss_->rows()) throw IoError("ulv solve: rhs rows mismatch");
      hssmf_status st{};
      hssmf_b200::detail::check(hssmf_hss_solve(hss_->handle(), b.data(), static_cast<int>(b.ld()),
                                                static_cast<int>(b.cols()), 0, &st),
                                st);
    }
    DenseMatrix<scalar_t> solve_new(const DenseMatrix<scalar_t>& b, int depth = 0) const {
      DenseMatrix<scalar_t> x(b);
      solve(x, depth);
      return x;
    }

   private:
    const HssMatrix<scalar_t>* hss_;  // must not move (as in the reference)
  };

  // hss_ulv.hpp:284-285
  template<typename scalar_t>
  UlvFactors<scalar_t> ulv_factor(const HssMatrix<scalar_t>& hss, int depth = 0) {
    (void)depth;
    return UlvFactors<scalar_t>(hss);
  }

}  // namespace hssmf

#endif
