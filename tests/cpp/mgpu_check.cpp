// Compile-and-run check of the NCCL drop-in (include/hssmf_b200/mgpu_nccl.hpp)
// on the GPUs of one box: one process, ncclCommInitAll over the visible
// devices (1 on a gpurun box), each rank driven by its own thread; the
// assembled solution is compared with the single-GPU drop-in.
#include <cmath>
#include <cstdio>
#include <thread>
#include <vector>

#include "hssmf/elimination_tree.hpp"
#include "hssmf/grid_problems.hpp"
#include "hssmf/ordering.hpp"
#include "hssmf/solver_options.hpp"
#include "hssmf/sparse_matrix.hpp"
#include "hssmf_b200/mgpu_nccl.hpp"

using namespace hssmf;

int main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  int nranks = 1;
  while (nranks * 2 <= ndev) nranks *= 2;
  auto g = generate_grid_problem<double>(GridKind::P3D, 24);
  Permutation perm;
  auto sep = nested_dissection_geometric(g.geom, 32, perm);
  auto a = g.A.permuted(perm.perm);
  auto t = EliminationTree::from_separators(sep, a.size());
  symbolic_factorization(a, t);
  t.compute_levels();
  SolverOptions so;
  so.ls = 64;
  so.min_hss = 300;
  so.eps = 1e-6;
  so.leaf = 64;
  const int n = a.size();
  std::vector<double> b(n);
  for (int i = 0; i < n; i++) b[i] = std::sin(0.37 * i);
  // single GPU
  auto m1 = hssmf_b200::mf_factor(a, t, so, 0);
  DenseMatrix<double> bx(n, 1);
  for (int i = 0; i < n; i++) bx(i, 0) = b[i];
  auto x1 = hssmf_b200::mf_solve_new(m1, bx);
  // nranks GPUs over NCCL
  std::vector<ncclComm_t> comms(nranks);
  std::vector<int> devs(nranks);
  for (int r = 0; r < nranks; r++) devs[r] = r;
  if (ncclCommInitAll(comms.data(), nranks, devs.data()) != ncclSuccess) return 2;
  std::vector<std::vector<double>> xs(nranks, std::vector<double>(n));
  std::vector<int> owner(t.size());
  std::vector<std::thread> th;
  for (int r = 0; r < nranks; r++)
    th.emplace_back([&, r] {
      cudaSetDevice(r);
      cudaStream_t s;
      cudaStreamCreate(&s);
      hssmf_b200::NcclTransport tr(comms[r], s);
      auto m = hssmf_b200::mf_factor_mgpu(a, t, so, tr, r, nranks, r);
      double* xd = nullptr;
      cudaMalloc(&xd, n * sizeof(double));
      cudaMemcpy(xd, b.data(), n * sizeof(double), cudaMemcpyHostToDevice);
      hssmf_b200::mf_solve_mgpu(m, tr, xd, n, 1);
      cudaMemcpy(xs[r].data(), xd, n * sizeof(double), cudaMemcpyDeviceToHost);
      cudaFree(xd);
      cudaStreamDestroy(s);
    });
  for (auto& x : th) x.join();
  hssmf_tree* tt = nullptr;
  {
    hssmf_b200::detail::Inputs in;
    hssmf_b200::detail::make_inputs(a, t, in);
    hssmf_status st{};
    int ne = 0;
    hssmf_mgpu_partition(in.tr, nranks, owner.data(), &ne, &st);
  }
  (void)tt;
  double diff = 0;
  for (int i = 0; i < t.size(); i++)
    for (int k = t.node(i).sep_begin; k < t.node(i).sep_end; k++)
      diff = std::max(diff, std::abs(xs[owner[i]][k] - x1(k, 0)));
  for (auto c : comms) ncclCommDestroy(c);
  std::printf("{\"nranks\": %d, \"max_diff\": %.3e}\n", nranks, diff);
  return diff == 0.0 ? 0 : 1;
}
