// Drop-in check: a program written against the reference's own types
// (proj/include/hssmf) switches mf_factor / mf_solve to hssmf_b200:: and
// compares with the reference's own mf_factor / mf_solve on the same input.
// Built in the build container (needs /root/reference headers), run on a GPU
// box by tests/test_cpp_wrapper.py.
#include <cmath>
#include <cstdio>
#include <cstring>

#include "hssmf/elimination_tree.hpp"
#include "hssmf/errors.hpp"
#include "hssmf/grid_problems.hpp"
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
  std::printf("{\"relres\": %.3e, \"fronts\": %zu, \"singular_col\": %d, \"front0\": %d, "
              "\"gmres_iterations\": %d, \"gmres_converged\": %d}\n",
              relres, m.front_stats.size(), col, what.find("front 0") != std::string::npos ? 1 : 0,
              rep.iterations, rep.converged ? 1 : 0);
  return (relres < 1e-12 && col == 1 && rep.converged && rep.iterations <= 2) ? 0 : 1;
}
