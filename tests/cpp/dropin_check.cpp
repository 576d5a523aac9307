// Source-level drop-in check: a program written against the reference's own
// names (hssmf::mf_factor / mf_solve_new / hss_compress / ulv_factor, with
// the reference's signatures) that includes include/hssmf_b200/dropin.hpp in
// place of hssmf/multifrontal.hpp, hss_compress.hpp and hss_ulv.hpp. Built in
// the build container (needs the reference's type headers), run on a GPU box by
// tests/test_cpp_wrapper.py, which compares the printed ranks with the
// oracle's.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "hssmf/cluster_tree.hpp"
#include "hssmf/dense_matrix.hpp"
#include "hssmf/elimination_tree.hpp"
#include "hssmf/errors.hpp"
#include "hssmf/grid_problems.hpp"
#include "hssmf/ordering.hpp"
#include "hssmf/solver_options.hpp"
#include "hssmf/sparse_matrix.hpp"
#include "hssmf/stats.hpp"
#include "hssmf_b200/dropin.hpp"
// a transitive include of the reference's own hot-path header is a no-op
#include "hssmf/multifrontal.hpp"

using namespace hssmf;

namespace {
  struct Problem {
    SparseMatrix<double> a;
    EliminationTree t;
  };
  Problem grid(GridKind k, int n, int leaf) {
    auto g = generate_grid_problem<double>(k, n);
    Permutation perm;
    auto st = nested_dissection_geometric(g.geom, leaf, perm);
    Problem p{g.A.permuted(perm.perm), {}};
    p.t = EliminationTree::from_separators(st, p.a.size());
    symbolic_factorization(p.a, p.t);
    p.t.compute_levels();
    return p;
  }
  double relres_sparse(const SparseMatrix<double>& a, const DenseMatrix<double>& x,
                       const DenseMatrix<double>& b) {
    std::vector<double> r(a.size());
    a.matvec(Trans::N, x.ptr(0, 0), r.data());
    double num = 0, den = 0;
    for (int i = 0; i < a.size(); i++) {
      num += (r[i] - b(i, 0)) * (r[i] - b(i, 0));
      den += b(i, 0) * b(i, 0);
    }
    return std::sqrt(num / den);
  }
  double relres_dense(const DenseMatrix<double>& a, const DenseMatrix<double>& x,
                      const DenseMatrix<double>& b) {
    const int n = a.rows();
    double num = 0, den = 0;
    for (int i = 0; i < n; i++) {
      double s = 0;
      for (int j = 0; j < n; j++) s += a(i, j) * x(j, 0);
      num += (s - b(i, 0)) * (s - b(i, 0));
      den += b(i, 0) * b(i, 0);
    }
    return std::sqrt(num / den);
  }
  DenseMatrix<double> rhs(int n) {
    DenseMatrix<double> b(n, 1);
    for (int i = 0; i < n; i++) b(i, 0) = std::sin(0.37 * i);
    return b;
  }
  // BASELINE config 2's operator, A_ij = 1/(1+|i-j|) + 4 delta_ij
  DenseMatrix<double> c2(int n) {
    DenseMatrix<double> a(n, n);
    for (int j = 0; j < n; j++)
      for (int i = 0; i < n; i++) a(i, j) = 1.0 / (1.0 + std::abs(i - j)) + (i == j ? 4.0 : 0.0);
    return a;
  }
  void print_ints(const char* key, const std::vector<int>& v) {
    std::printf("\"%s\": [", key);
    for (size_t i = 0; i < v.size(); i++) std::printf("%s%d", i ? ", " : "", v[i]);
    std::printf("]");
  }
}  // namespace

int main() {
  // 1. pure multifrontal (mode MF): exact factors
  auto p1 = grid(GridKind::P2D, 31, 16);
  SolverOptions mf;
  mf.mode = SolverMode::MF;
  auto m1 = mf_factor(p1.a, p1.t, mf);
  auto b1 = rhs(p1.a.size());
  auto x1 = mf_solve_new(m1, b1);
  const double rr1 = relres_sparse(p1.a, x1, b1);

  // 2. HSS fronts (P3D 24^3, ND leaf 16): per-front ranks for the oracle
  auto p2 = grid(GridKind::P3D, 24, 16);
  SolverOptions sh;
  sh.ls = 64;
  sh.min_hss = 250;
  sh.eps = 1e-6;
  sh.leaf = 32;
  auto m2 = mf_factor(p2.a, p2.t, sh, 3);
  auto b2 = rhs(p2.a.size());
  DenseMatrix<double> x2(b2);
  mf_solve(m2, x2);
  const double rr2 = relres_sparse(p2.a, x2, b2);
  std::vector<int> hss_ids, hss_ranks;
  for (const auto& f : m2.front_stats)
    if (f.type == "hss") {
      hss_ids.push_back(f.id);
      hss_ranks.push_back(f.rank);
    }

  // 3. standalone dense HSS on balanced and uneven cluster trees
  const int n3 = 2048;
  auto a3 = c2(n3);
  HssOptions ho;
  HssCompressStats cst;
  auto h3 = hss_compress(a3, ClusterTree::balanced(n3, 128), ho, &cst);
  auto u3 = ulv_factor(h3);
  auto b3 = rhs(n3);
  auto x3 = u3.solve_new(b3);
  const double rr3 = relres_dense(a3, x3, b3);
  std::vector<int> u3r;
  for (int i = 0; i < h3.tree().size(); i++) u3r.push_back(h3.u_rank(i));
  auto uneven = ClusterTree::join(ClusterTree::balanced(1000, 100), ClusterTree::balanced(1048, 128));
  HssCompressStats cst4;
  auto h4 = hss_compress(a3, uneven, ho, &cst4);
  auto x4 = ulv_factor(h4).solve_new(b3);
  const double rr4 = relres_dense(a3, x4, b3);
  std::vector<int> u4r;
  for (int i = 0; i < h4.tree().size(); i++) u4r.push_back(h4.u_rank(i));

  // 4. error contracts: singular front ("front 0", column 1), rank guard,
  //    size mismatch
  EliminationTree t5;
  t5.n = 3;
  t5.nodes.resize(1);
  t5.nodes[0].sep_end = 3;
  t5.compute_levels();
  std::vector<std::tuple<int, int, double>> trip = {{0, 0, 1.0}, {0, 1, 0.0}, {1, 0, 0.0}, {2, 2, 1.0}};
  auto a5 = SparseMatrix<double>::from_triplets(3, trip);
  int col = -1, front0 = 0;
  try {
    auto m5 = mf_factor(a5, t5, mf);
  } catch (const SingularMatrixError& e) {
    col = e.column();
    front0 = std::string(e.what()).find("front 0") != std::string::npos;
  }
  int rank_guard = 0, io = 0;
  try {
    HssOptions tight;
    tight.max_rank = 4;
    auto h6 = hss_compress(a3, ClusterTree::balanced(n3, 128), tight);
  } catch (const HssRankExceeded&) {
    rank_guard = 1;
  }
  try {
    auto h7 = hss_compress(a3, ClusterTree::balanced(n3 - 1, 128), ho);
  } catch (const IoError&) {
    io = 1;
  }

  std::printf("{\"mf_relres\": %.3e, \"hss_relres\": %.3e, \"hss_fronts\": %d, ", rr1, rr2,
              m2.hss_fronts);
  print_ints("hss_ids", hss_ids);
  std::printf(", ");
  print_ints("hss_ranks", hss_ranks);
  std::printf(", \"dense_relres\": %.3e, \"dense_rank\": %d, \"dense_rounds\": %d, "
              "\"dense_d_final\": %d, ", rr3, h3.hss_rank(), cst.rounds, cst.d_final);
  print_ints("dense_u", u3r);
  std::printf(", \"uneven_relres\": %.3e, \"uneven_rank\": %d, ", rr4, h4.hss_rank());
  print_ints("uneven_u", u4r);
  std::printf(", \"singular_col\": %d, \"front0\": %d, \"rank_guard\": %d, \"io\": %d, "
              "\"factor_nnz\": %lld}\n", col, front0, rank_guard, io,
              (long long)m2.factor_nnz());
  return 0;
}
