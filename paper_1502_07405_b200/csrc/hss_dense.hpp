// Standalone dense HSS compression + ULV (BASELINE config 2).
#pragma once

#include <memory>
#include <vector>

namespace hssmf_b200 {

  class DenseHss {
  public:
    explicit DenseHss(int device);
    ~DenseHss();
    void run(const double* a, int lda, int n, int leaf, double eps, int d0, int dd, int p,
             int max_rank, bool on_device);
    // any postorder cluster tree over [0, n) (root last)
    void run_tree(const double* a, int lda, int n, int nnodes, const int* begin, const int* end,
                  const int* child0, const int* child1, double eps, int d0, int dd, int p,
                  int max_rank, bool on_device);
    void solve(double* b, int ldb, int nrhs, bool on_device);
    // y = op(A_hss) x on the subtree of cluster node `root` (-1: all);
    // x is node_size(root) x nc
    void matvec(char op, int root, const double* x, int ldx, int nc, double* y, int ldy,
                bool on_device);
    int node_size(int root) const;
    // out (ni x nj, ld ni) = A_hss(I, J); returns the leaves visited
    long long extract(const int* I, int ni, const int* J, int nj, double* out, bool on_device);
    void ranks(std::vector<int>& u, std::vector<int>& v) const;
    int rounds() const;
    int d_final() const;
    double compress_ms() const;
    double ulv_ms() const;
    struct Impl;

  private:
    std::unique_ptr<Impl> d_;
  };

}  // namespace hssmf_b200
