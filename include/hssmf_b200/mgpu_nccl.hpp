// hssmf_b200/mgpu_nccl.hpp — the subtree-partitioned factorization and solve
// over several GPUs with NCCL point-to-point (ncclSend / ncclRecv over NVLink 5
// / NVSwitch), one process per GPU. Header-only over the C-ABI's
// hssmf_mgpu_* entry points; link the program with -lnccl.
//
//   ncclComm_t comm;  ncclCommInitRank(&comm, nranks, id, rank);   // caller's
//   hssmf_b200::NcclTransport tr(comm, stream);
//   auto m = hssmf_b200::mf_factor_mgpu(a, t, opts, tr, rank, nranks, device);
//   hssmf_b200::mf_solve_mgpu(m, tr, x_dev, n, nrhs);  // x correct on own separators
#ifndef HSSMF_B200_MGPU_NCCL_HPP
#define HSSMF_B200_MGPU_NCCL_HPP

#include <cuda_runtime.h>
#include <nccl.h>

#include "hssmf.hpp"

namespace hssmf_b200 {

  // blocking point-to-point transport on one stream of this rank's GPU
  class NcclTransport {
   public:
    NcclTransport(ncclComm_t comm, cudaStream_t s) : comm_(comm), s_(s) {}
    hssmf_transport c_api() { return hssmf_transport{this, &send_cb, &recv_cb}; }

   private:
    static int send_cb(void* ctx, const double* buf, long long n, int peer) {
      auto* t = static_cast<NcclTransport*>(ctx);
      if (ncclSend(buf, static_cast<size_t>(n), ncclDouble, peer, t->comm_, t->s_) != ncclSuccess)
        return 1;
      return cudaStreamSynchronize(t->s_) == cudaSuccess ? 0 : 1;
    }
    static int recv_cb(void* ctx, double* buf, long long n, int peer) {
      auto* t = static_cast<NcclTransport*>(ctx);
      if (ncclRecv(buf, static_cast<size_t>(n), ncclDouble, peer, t->comm_, t->s_) != ncclSuccess)
        return 1;
      return cudaStreamSynchronize(t->s_) == cudaSuccess ? 0 : 1;
    }
    ncclComm_t comm_;
    cudaStream_t s_;
  };

  // this rank's share of mf_factor (reference multifrontal.hpp:473-503); the
  // stats of the fronts it owns
  template<class Sparse, class Tree, class Opts>
  MfFactors mf_factor_mgpu(const Sparse& a, const Tree& t, const Opts& opts, NcclTransport& tr,
                           int rank, int nranks, int device) {
    detail::Inputs in;
    detail::make_inputs(a, t, in);
    hssmf_options o = detail::options(opts);
    hssmf_transport c = tr.c_api();
    hssmf_status st{};
    hssmf_factors* h = nullptr;
    detail::check(hssmf_mgpu_factor(device, in.c, in.tr, &o, rank, nranks, &c, &h, &st), st);
    MfFactors m;
    m.adopt(h, a.size());
    return m;
  }

  // this rank's share of mf_solve (reference multifrontal.hpp:612-622) on a
  // device block x (n x nrhs, ld ldx) holding b; on return x is correct on the
  // separators of the fronts this rank owns
  inline void mf_solve_mgpu(MfFactors& m, NcclTransport& tr, double* x_dev, int ldx, int nrhs) {
    hssmf_transport c = tr.c_api();
    hssmf_status st{};
    detail::check(hssmf_mgpu_solve(m.handle(), &c, x_dev, ldx, nrhs, &st), st);
  }

}  // namespace hssmf_b200

#endif
