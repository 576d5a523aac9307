// Drop-in check: a program written against the reference's own types
// (proj/include/hssmf) switches mf_factor / mf_solve to hssmf_b200:: and
// compares with the reference's own mf_factor / mf_solve on the same input.
// Built in the build container (needs /root/reference headers), run on a GPU
// box by tests/test_cpp_wrapper.py.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "ref_shim.hpp"  // oracle/: the reference's nested-HSS extract fix
#include "hssmf/elimination_tree.hpp"
#include "hssmf/errors.hpp"
#include "hssmf/grid_problems.hpp"
#include "hssmf/multifrontal.hpp"
#include "hssmf/separator_reorder.hpp"
#include "hssmf/ordering.hpp"
#include "hssmf/solver_options.hpp"
#include "hssmf/sparse_matrix.hpp"
#define HSSMF_B200_REFERENCE_ERRORS
#include "hssmf_b200/hssmf.hpp"

using namespace hssmf;

int main(int argc, char** argv) {
  if (argc > 1 && !strcmp(argv[1], "--version")) {
    std::printf("%s\n", hssmf_version());
    return 0;
  }
  auto g = generate_grid_problem<double>(GridKind::P2D, 31);
  Permutation perm;
  auto st = nested_dissection_geometric(g.geom, 16, perm);
  auto a = g.A.permuted(perm.perm);
  auto t = EliminationTree::from_separators(st, a.size());
  symbolic_factorization(a, t);
  t.compute_levels();
  SolverOptions so;
  so.mode = SolverMode::MF;
  auto m = hssmf_b200::mf_factor(a, t, so);
  DenseMatrix<double> b(a.size(), 1);
  for (int i = 0; i < a.size(); i++) b(i, 0) = std::sin(0.37 * i);
  auto x = hssmf_b200::mf_solve_new(m, b);
  std::vector<double> r(a.size());
  a.matvec(Trans::N, x.ptr(0, 0), r.data());
  double num = 0, den = 0;
  for (int i = 0; i < a.size(); i++) {
    num += (r[i] - b(i, 0)) * (r[i] - b(i, 0));
    den += b(i, 0) * b(i, 0);
  }
  const double relres = std::sqrt(num / den);
  // reference error contract: singular front names the front and the column
  EliminationTree t1;
  t1.n = 3;
  t1.nodes.resize(1);
  t1.nodes[0].sep_end = 3;
  t1.compute_levels();
  std::vector<std::tuple<int, int, double>> trip = {{0, 0, 1.0}, {0, 1, 0.0}, {1, 0, 0.0}, {2, 2, 1.0}};
  auto a1 = SparseMatrix<double>::from_triplets(3, trip);
  int col = -1;
  std::string what;
  try {
    auto m1 = hssmf_b200::mf_factor(a1, t1, so);
  } catch (const SingularMatrixError& e) {
    col = e.column();
    what = e.what();
  }
  // preconditioned GMRES through the drop-in (krylov.hpp:93-184 signature
  // shape): exact factors converge at once
  std::vector<double> bv(a.size());
  for (int i = 0; i < a.size(); i++) bv[i] = b(i, 0);
  auto [xg, rep] = hssmf_b200::gmres(a, m, bv, 30, 1e-10, 0.0, 20);
  // graph ordering + the reference's own separator reordering: the drop-in
  // must compress on the reordered separator clusters (FrontNode::sep_clusters)
  // and land within +-10% of the reference's mf_factor ranks
  auto g3 = generate_grid_problem<double>(GridKind::P3D, 18);
  std::vector<int> gptr, gind;
  g3.A.symmetric_graph(gptr, gind);
  Permutation p3;
  auto st3 = nested_dissection_graph(g3.A.size(), gptr, gind, 32, p3);
  auto a3 = g3.A.permuted(p3.perm);
  auto t3 = EliminationTree::from_separators(st3, a3.size());
  symbolic_factorization(a3, t3);
  std::vector<char> sel(t3.size());
  for (int i = 0; i < t3.size(); i++) sel[i] = t3.node(i).sep_size() > 0;
  std::vector<int> pptr, pind;
  a3.symmetric_graph(pptr, pind);
  auto r3 = reorder_tree_separators(t3, sel, pptr, pind, 24);
  a3 = a3.permuted(r3.perm);
  symbolic_factorization(a3, t3);
  t3.compute_levels();
  SolverOptions sh;
  sh.ls = 64;
  sh.min_hss = 250;
  sh.eps = 1e-6;
  sh.leaf = 24;
  auto mine = hssmf_b200::mf_factor(a3, t3, sh);
  auto theirs = mf_factor(a3, t3, sh);
  int hss = 0, close = 1;
  for (size_t i = 0; i < theirs.front_stats.size(); i++) {
    const auto& f = theirs.front_stats[i];
    if (f.type != "hss") continue;
    hss++;
    const double d = std::abs((double)mine.front_stats[i].rank - f.rank);
    if (mine.front_stats[i].type != "hss" || d > std::max(0.1 * f.rank, 2.0)) close = 0;
  }
  std::printf("{\"relres\": %.3e, \"fronts\": %zu, \"singular_col\": %d, \"front0\": %d, "
              "\"gmres_iterations\": %d, \"gmres_converged\": %d, \"reorder_hss_fronts\": %d, "
              "\"reorder_ranks_close\": %d}\n",
              relres, m.front_stats.size(), col, what.find("front 0") != std::string::npos ? 1 : 0,
              rep.iterations, rep.converged ? 1 : 0, hss, close);
  return (relres < 1e-12 && col == 1 && rep.converged && rep.iterations <= 2 && hss > 0 &&
          close) ? 0 : 1;
}
