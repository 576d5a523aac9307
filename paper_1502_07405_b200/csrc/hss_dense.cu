// Standalone dense HSS (BASELINE config 2): hss_compress + ulv_factor +
// UlvFactors::solve (hss_compress.hpp:373-383, hss_ulv.hpp:150-176, 284-319).
#include "hss_dense.hpp"

#include "common.cuh"
#include "hss.hpp"

#include <stdexcept>

namespace hssmf_b200 {

  struct DenseHss::Impl {
    int device = 0, n = 0;
    cudaStream_t s = nullptr;
    double* A = nullptr;
    double* x = nullptr;
    std::unique_ptr<HssMatrixDev> h;
    double cms = 0, ums = 0;
    ~Impl() {
      h.reset();
      if (s) cudaStreamSynchronize(s);
      if (A) cudaFree(A);
      if (x) cudaFree(x);
      if (s) cudaStreamDestroy(s);
    }
  };

  DenseHss::DenseHss(int device) : d_(new Impl) {
    d_->device = device;
    HSSMF_CUDA(cudaSetDevice(device));
    HSSMF_CUDA(cudaStreamCreateWithFlags(&d_->s, cudaStreamNonBlocking));
  }
  DenseHss::~DenseHss() = default;

  void DenseHss::run(const double* a, int lda, int n, int leaf, double eps, int d0, int dd, int p,
                     int max_rank, bool on_device) {
    const ClusterTree ct = ClusterTree::balanced(n, leaf);
    std::vector<int> b, e, c0, c1;
    for (const auto& c : ct.nodes) {
      b.push_back(c.begin);
      e.push_back(c.end);
      c0.push_back(c.child0);
      c1.push_back(c.child1);
    }
    run_tree(a, lda, n, (int)ct.nodes.size(), b.data(), e.data(), c0.data(), c1.data(), eps, d0,
             dd, p, max_rank, on_device);
  }

  void DenseHss::run_tree(const double* a, int lda, int n, int nnodes, const int* begin,
                          const int* end, const int* child0, const int* child1, double eps,
                          int d0, int dd, int p, int max_rank, bool on_device) {
    // the tree must be a postorder binary partition of [0, n) (ClusterTree,
    // cluster_tree.hpp:12-97): checked here, the compression trusts it
    if (nnodes < 1 || begin[nnodes - 1] != 0 || end[nnodes - 1] != n)
      throw std::invalid_argument("hss_compress: cluster tree root must span [0, n)");
    ClusterTree ct;
    ct.nodes.resize(nnodes);
    for (int i = 0; i < nnodes; i++) {
      auto& c = ct.nodes[i];
      c.begin = begin[i];
      c.end = end[i];
      c.child0 = child0[i];
      c.child1 = child1[i];
      if ((c.child0 < 0) != (c.child1 < 0) || c.child0 >= i || c.child1 >= i || c.end < c.begin)
        throw std::invalid_argument("hss_compress: cluster tree not postorder binary");
      if (c.child0 >= 0) {
        const auto& l = ct.nodes[c.child0];
        const auto& r = ct.nodes[c.child1];
        if (l.begin != c.begin || l.end != r.begin || r.end != c.end)
          throw std::invalid_argument("hss_compress: children must split the parent range");
        ct.nodes[c.child0].parent = ct.nodes[c.child1].parent = i;
      }
    }
    auto& D = *d_;
    HSSMF_CUDA(cudaSetDevice(D.device));
    D.n = n;
    HSSMF_CUDA(cudaMalloc(&D.A, (size_t)n * n * sizeof(double) + 8));
    HSSMF_CUDA(cudaMalloc(&D.x, (size_t)n * sizeof(double) + 8));
    HSSMF_CUDA(cudaMemcpy2DAsync(D.A, n * sizeof(double), a, (size_t)lda * sizeof(double),
                                 n * sizeof(double), n,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, D.s));
    std::vector<long long> seeds(n);
    for (int i = 0; i < n; i++) seeds[i] = i;
    HssOpts o;
    o.eps = eps;
    o.d0 = d0;
    o.dd = dd;
    o.p = p;
    o.max_rank = max_rank;
    cudaEvent_t e0, e1, e2;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventCreate(&e2));
    D.h = std::make_unique<HssMatrixDev>(D.s);
    HSSMF_CUDA(cudaEventRecord(e0, D.s));
    D.h->compress(D.A, n, ct, seeds, o);
    HSSMF_CUDA(cudaEventRecord(e1, D.s));
    D.h->ulv_full();
    HSSMF_CUDA(cudaEventRecord(e2, D.s));
    HSSMF_CUDA(cudaStreamSynchronize(D.s));
    float a1 = 0, a2 = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&a1, e0, e1));
    HSSMF_CUDA(cudaEventElapsedTime(&a2, e1, e2));
    D.cms = a1;
    D.ums = a2;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
  }

  void DenseHss::solve(double* b, int ldb, int nrhs, bool on_device) {
    auto& D = *d_;
    HSSMF_CUDA(cudaSetDevice(D.device));
    for (int c = 0; c < nrhs; c++) {
      double* col = b + (size_t)c * ldb;
      if (on_device) {
        D.h->solve_full(col);
      } else {
        HSSMF_CUDA(cudaMemcpyAsync(D.x, col, D.n * sizeof(double), cudaMemcpyHostToDevice, D.s));
        D.h->solve_full(D.x);
        HSSMF_CUDA(cudaMemcpyAsync(col, D.x, D.n * sizeof(double), cudaMemcpyDeviceToHost, D.s));
      }
    }
    HSSMF_CUDA(cudaStreamSynchronize(D.s));
  }

  int DenseHss::node_size(int root) const { return d_->h->node_size(root); }

  void DenseHss::matvec(char op, int root, const double* x, int ldx, int nc, double* y, int ldy,
                        bool on_device) {
    auto& D = *d_;
    HSSMF_CUDA(cudaSetDevice(D.device));
    const int nr = D.h->node_size(root);
    if (nc <= 0 || nr <= 0) return;
    if (on_device) {
      D.h->matvec(op, root, x, ldx, nc, y, ldy);
      return;
    }
    double *dx = nullptr, *dy = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&dx, (size_t)nr * nc * sizeof(double), D.s));
    HSSMF_CUDA(cudaMallocAsync((void**)&dy, (size_t)nr * nc * sizeof(double), D.s));
    HSSMF_CUDA(cudaMemcpy2DAsync(dx, nr * sizeof(double), x, (size_t)ldx * sizeof(double),
                                 nr * sizeof(double), nc, cudaMemcpyHostToDevice, D.s));
    D.h->matvec(op, root, dx, nr, nc, dy, nr);
    HSSMF_CUDA(cudaMemcpy2DAsync(y, (size_t)ldy * sizeof(double), dy, nr * sizeof(double),
                                 nr * sizeof(double), nc, cudaMemcpyDeviceToHost, D.s));
    HSSMF_CUDA(cudaFreeAsync(dx, D.s));
    HSSMF_CUDA(cudaFreeAsync(dy, D.s));
    HSSMF_CUDA(cudaStreamSynchronize(D.s));
  }

  long long DenseHss::extract(const int* I, int ni, const int* J, int nj, double* out,
                              bool on_device) {
    auto& D = *d_;
    HSSMF_CUDA(cudaSetDevice(D.device));
    std::vector<int> vi(I, I + ni), vj(J, J + nj);
    if (on_device) return D.h->extract(vi, vj, out);
    double* dout = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&dout, (size_t)ni * nj * sizeof(double) + 8, D.s));
    const long long v = D.h->extract(vi, vj, dout);
    HSSMF_CUDA(cudaMemcpyAsync(out, dout, (size_t)ni * nj * sizeof(double), cudaMemcpyDeviceToHost,
                               D.s));
    HSSMF_CUDA(cudaFreeAsync(dout, D.s));
    HSSMF_CUDA(cudaStreamSynchronize(D.s));
    return v;
  }

  void DenseHss::ranks(std::vector<int>& u, std::vector<int>& v) const { d_->h->ranks(u, v); }
  int DenseHss::rounds() const { return d_->h->rounds(); }
  int DenseHss::d_final() const { return d_->h->d_final(); }
  double DenseHss::compress_ms() const { return d_->cms; }
  double DenseHss::ulv_ms() const { return d_->ums; }

}  // namespace hssmf_b200
