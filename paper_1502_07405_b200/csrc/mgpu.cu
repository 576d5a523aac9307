// Subtree-partitioned multi-GPU factorization and solve in C++ (SURVEY §8e),
// the native counterpart of paper_1502_07405_b200/parallel.py.
//
// With geometric nested dissection the 2^L subtrees rooted at tree level
// L = log2(P) are independent; rank r owns the r-th of them (left to right)
// and every front above level L is owned by the owner of its child0 subtree.
// The only exchanges follow tree edges whose child and parent live on
// different ranks, one message per edge and phase, in one global order
// (parent level descending, then child id), so every send meets its receive
// without a barrier:
//   factor: the child's update block (nu x nu) goes to the parent's owner;
//   forward solve: the child's bupd (nu x nrhs) goes up the same edge;
//   backward solve: x(upd(child)) (nu x nrhs) comes back down.
// The messages move through a transport: the caller's callbacks (NCCL
// send/recv over NVLink in include/hssmf_b200/mgpu_nccl.hpp, or any other
// point-to-point layer), or an in-process mailbox when all ranks share one
// process (the single-GPU check of the partitioned path).
#include "mgpu.hpp"

#include <algorithm>
#include <cmath>
#include <deque>
#include <map>
#include <stdexcept>

#include "common.cuh"

namespace hssmf_b200 {

  namespace {
    // rows of x (n x nrhs, ld ldx) at the index list idx (nu) <-> a packed
    // nu x nrhs block (ld nu)
    __global__ void gather_rows_kernel(const double* __restrict__ x, long long ldx, int nrhs,
                                       const int* __restrict__ idx, int nu, double* __restrict__ out) {
      const long long tot = (long long)nu * nrhs;
      for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
           e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % nu), c = (int)(e / nu);
        out[e] = x[idx[i] + c * ldx];
      }
    }
    __global__ void scatter_rows_kernel(double* __restrict__ x, long long ldx, int nrhs,
                                        const int* __restrict__ idx, int nu,
                                        const double* __restrict__ in) {
      const long long tot = (long long)nu * nrhs;
      for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
           e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e % nu), c = (int)(e / nu);
        x[idx[i] + c * ldx] = in[e];
      }
    }
    int grid_for(long long tot) { return (int)std::max(1LL, std::min((tot + 255) / 256, 148LL * 8)); }

    struct DevBuf {
      double* p = nullptr;
      size_t n = 0;
      void ensure(size_t cnt) {
        if (cnt <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        HSSMF_CUDA(cudaMalloc(&p, std::max<size_t>(cnt, 1) * sizeof(double)));
        n = cnt;
      }
      ~DevBuf() {
        if (p) cudaFree(p);
      }
    };
  }  // namespace

  MgpuPlan mgpu_partition(const Etree& t, int nranks) {
    if (nranks < 1 || (nranks & (nranks - 1)))
      throw std::invalid_argument("the subtree partition needs a power-of-two rank count");
    MgpuPlan P;
    P.nranks = nranks;
    P.L = 0;
    while ((1 << P.L) < nranks) P.L++;
    const int nn = (int)t.nodes.size();
    for (int i = 0; i < nn; i++)
      if (t.nodes[i].level == P.L) P.roots.push_back(i);
    if ((int)P.roots.size() != nranks)
      throw std::invalid_argument("tree has " + std::to_string(P.roots.size()) + " fronts at level " +
                                  std::to_string(P.L) + ", need " + std::to_string(nranks));
    std::vector<int> lo(nn);
    for (int i = 0; i < nn; i++) {  // postorder: children first
      lo[i] = i;
      for (int c : {t.nodes[i].child0, t.nodes[i].child1})
        if (c >= 0) lo[i] = std::min(lo[i], lo[c]);
    }
    P.owner.assign(nn, -1);
    for (int r = 0; r < nranks; r++)
      for (int i = lo[P.roots[r]]; i <= P.roots[r]; i++) P.owner[i] = r;
    for (int i = 0; i < nn; i++)
      if (P.owner[i] < 0) {
        const int c = t.nodes[i].child0 >= 0 ? t.nodes[i].child0 : t.nodes[i].child1;
        P.owner[i] = c >= 0 ? P.owner[c] : 0;
      }
    for (int i = 0; i < nn; i++)
      for (int c : {t.nodes[i].child0, t.nodes[i].child1})
        if (c >= 0 && P.owner[c] != P.owner[i])
          P.edges.push_back({c, i, P.owner[c], P.owner[i], t.nodes[c].nu(), t.nodes[i].level});
    // one global order: parent level descending, then child id
    std::sort(P.edges.begin(), P.edges.end(), [](const MgpuEdge& a, const MgpuEdge& b) {
      return a.plevel != b.plevel ? a.plevel > b.plevel : a.child < b.child;
    });
    P.nlev = 0;
    for (const auto& f : t.nodes) P.nlev = std::max(P.nlev, f.level + 1);
    return P;
  }

  void LocalTransport::send(const double* buf, long long count, int dst, int src) {
    Msg m;
    m.n = count;
    HSSMF_CUDA(cudaMalloc(&m.p, std::max<long long>(count, 1) * sizeof(double)));
    HSSMF_CUDA(cudaMemcpy(m.p, buf, count * sizeof(double), cudaMemcpyDeviceToDevice));
    q_[{src, dst}].push_back(m);
  }
  void LocalTransport::recv(double* buf, long long count, int src, int dst) {
    auto& d = q_[{src, dst}];
    if (d.empty()) throw std::runtime_error("local transport: no message from rank " +
                                            std::to_string(src) + " to " + std::to_string(dst));
    Msg m = d.front();
    d.pop_front();
    if (m.n != count) throw std::runtime_error("local transport: message size mismatch");
    HSSMF_CUDA(cudaMemcpy(buf, m.p, count * sizeof(double), cudaMemcpyDeviceToDevice));
    cudaFree(m.p);
  }
  LocalTransport::~LocalTransport() {
    for (auto& kv : q_)
      for (auto& m : kv.second) cudaFree(m.p);
  }

  // messages of the edges whose parent is at level l
  static std::vector<const MgpuEdge*> edges_into(const MgpuPlan& P, int l) {
    std::vector<const MgpuEdge*> e;
    for (const auto& x : P.edges)
      if (x.plevel == l) e.push_back(&x);
    return e;
  }

  void mgpu_factor(const MgpuPlan& P, std::map<int, Engine*>& eng, MgpuTransport& tr) {
    for (auto& kv : eng) kv.second->factor_levels(P.L, P.nlev - 1);
    DevBuf buf;
    for (int l = P.L - 1; l >= 0; l--) {
      for (const MgpuEdge* e : edges_into(P, l)) {
        const long long cnt = (long long)e->nu * e->nu;
        buf.ensure(cnt);
        if (eng.count(e->src)) {
          eng[e->src]->export_update(e->child, buf.p, true);  // synchronises its stream
          tr.send(buf.p, cnt, e->dst, e->src);
        }
        if (eng.count(e->dst)) {
          tr.recv(buf.p, cnt, e->src, e->dst);
          eng[e->dst]->import_update(e->child, buf.p, true);
        }
      }
      for (auto& kv : eng) kv.second->factor_levels(l, l);
    }
  }

  void mgpu_solve(const MgpuPlan& P, const Etree& t, std::map<int, Engine*>& eng,
                  std::map<int, double*>& x, int ldx, int nrhs, MgpuTransport& tr) {
    for (auto& kv : eng) kv.second->solve_levels(x[kv.first], ldx, nrhs, P.L, P.nlev - 1, true);
    DevBuf buf;
    for (int l = P.L - 1; l >= 0; l--) {
      for (const MgpuEdge* e : edges_into(P, l)) {
        const long long cnt = (long long)e->nu * nrhs;
        buf.ensure(cnt);
        if (eng.count(e->src)) {
          eng[e->src]->export_bupd(e->child, buf.p, nrhs);
          tr.send(buf.p, cnt, e->dst, e->src);
        }
        if (eng.count(e->dst)) {
          tr.recv(buf.p, cnt, e->src, e->dst);
          eng[e->dst]->import_bupd(e->child, buf.p, nrhs);
        }
      }
      for (auto& kv : eng) kv.second->solve_levels(x[kv.first], ldx, nrhs, l, l, true);
    }
    int* didx = nullptr;
    size_t didx_n = 0;
    for (int l = 0; l < P.L; l++) {
      for (auto& kv : eng) kv.second->solve_levels(x[kv.first], ldx, nrhs, l, l, false);
      // x at the update indices of the level-(l+1) children goes back down
      for (const MgpuEdge* e : edges_into(P, l)) {
        const auto& upd = t.nodes[e->child].upd;
        const long long cnt = (long long)e->nu * nrhs;
        buf.ensure(cnt);
        if (upd.size() > didx_n) {
          if (didx) cudaFree(didx);
          HSSMF_CUDA(cudaMalloc(&didx, upd.size() * sizeof(int)));
          didx_n = upd.size();
        }
        HSSMF_CUDA(cudaMemcpy(didx, upd.data(), upd.size() * sizeof(int), cudaMemcpyHostToDevice));
        if (eng.count(e->dst)) {
          gather_rows_kernel<<<grid_for(cnt), 256>>>(x[e->dst], ldx, nrhs, didx, e->nu, buf.p);
          HSSMF_LAUNCH_CHECK();
          HSSMF_CUDA(cudaDeviceSynchronize());
          tr.send(buf.p, cnt, e->src, e->dst);
        }
        if (eng.count(e->src)) {
          tr.recv(buf.p, cnt, e->dst, e->src);
          scatter_rows_kernel<<<grid_for(cnt), 256>>>(x[e->src], ldx, nrhs, didx, e->nu, buf.p);
          HSSMF_LAUNCH_CHECK();
          HSSMF_CUDA(cudaDeviceSynchronize());
        }
      }
    }
    if (didx) cudaFree(didx);
    for (auto& kv : eng) kv.second->solve_levels(x[kv.first], ldx, nrhs, P.L, P.nlev - 1, false);
  }

}  // namespace hssmf_b200
