// HSS compression (adaptive randomized, Algorithm 1 of the paper), ULV-like
// factorization, low-rank Schur update and ULV solves on the device.
//
// Reference counterparts:
//   hss_compress_adaptive / compress_pass / build_local_samples / update_done
//                                               hss_compress.hpp:101-352
//   BasisId (Pi [I; E] interpolative bases)     hss_matrix.hpp:18-172
//   ulv_eliminate / ulv_factor / partial_ulv_and_schur / LowRankSchur
//                                               hss_ulv.hpp:18-121, 284-358
//   UlvFactors::fwd/bwd/solve/partial_*         hss_ulv.hpp:150-276
//
// The compressed matrix is a dense device matrix A (a multifrontal front,
// assembled in HBM, or the standalone config-2 matrix): sampling products
// are two DMMA GEMMs per round and element extraction is an indexed gather.
// Every HSS level of a round is one batch of launches; ranks are read back
// once per level to size the next batch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "host/analysis.hpp"

namespace hssmf_b200 {

  struct HssOpts {
    double eps = 1e-8;
    int d0 = 128, dd = 128, p = 10, max_rank = 5000;
    // fronts compressed concurrently with this one (0: unknown): with few of
    // them the device idles through the pivot chains, so the next round's IDs
    // are computed speculatively beside the current ones
    int peers = 0;
  };

  struct HssRankError : std::runtime_error {
    int node, cap;
    HssRankError(int n, int c)
        : std::runtime_error("hss compression: rank cap " + std::to_string(c) +
                             " exceeded at cluster " + std::to_string(n)),
          node(n), cap(c) {}
  };

  struct HssSingular : std::runtime_error {
    int node, column;
    HssSingular(int n, int c)
        : std::runtime_error("ulv_factor cluster " + std::to_string(n) +
                             ": exactly singular, zero pivot column " + std::to_string(c)),
          node(n), column(c) {}
  };

  struct HssImpl;

  // per-phase CUDA-event timing of the HSS path (profiling / HSSMF_DEBUG only)
  void hss_set_phase_timing(bool on);

  // device-time phases of the HSS path (profiling)
  constexpr int kHssPhases = 9;
  inline const char* hss_phase_name(int i) {
    static const char* n[kHssPhases] = {"hss_sample_gemm", "hss_extract", "hss_local_samples",
                                        "hss_cpqr", "hss_id_finalize", "hss_update_done",
                                        "hss_ulv_eliminate", "hss_ulv_top", "hss_densify"};
    return n[i];
  }
  struct HssPhaseStat {
    double ms = 0, flops = 0;
    int count = 0;
    double host_ms = 0;  // host time spent issuing the phase (incl. its syncs)
  };

  class HssMatrixDev {
  public:
    HssMatrixDev(cudaStream_t s);
    ~HssMatrixDev();
    HssMatrixDev(const HssMatrixDev&) = delete;

    // compress the dense device matrix A (m x m, lda) over the cluster tree;
    // seeds[i] names the random stream of row i (host array)
    void compress(const double* A, long long lda, const ClusterTree& tree,
                  const std::vector<long long>& seeds, const HssOpts& o);
    // full ULV factorization (ulv_factor)
    void ulv_full();
    // partial ULV of the leading n_sep rows (root child0) + low-rank Schur;
    // writes the densified update  F22|hss - Theta^* Phi  (nu x nu, ld ldu)
    void ulv_partial(double* update, long long ldu);
    // release the reference to A (front storage about to be freed)
    void drop_dense();
    // stream used by later solves (factorization ran on its own stream)
    void set_stream(cudaStream_t s);
    // stream of the next solves only (no arena move; the solve scratch is
    // allocated on the owning stream first): lets the fronts of one tree level
    // run their ULV sweeps concurrently
    void set_solve_stream(cudaStream_t s);

    // solves (single right-hand side, device vectors)
    void solve_full(double* x);  // in place, length m
    // partial: forward on b1 (ns) -> subtract the coupling from bupd (nu);
    // backward from x2 = x(upd) (nu) -> x1 (ns) written in place of b1
    void partial_forward(const double* b1, double* bupd);
    void partial_backward(double* x1, const double* x2);

    // y = op(A_hss) x on the subtree of cluster node `root` (-1: the whole
    // matrix), device blocks of size(root) x nc (HssMatrix::matvec,
    // hss_matrix.hpp:234-249); needs the leaf blocks (before drop_dense)
    void matvec(char op, int root, const double* x, long long ldx, int nc, double* y,
                long long ldy);
    int node_size(int node) const;  // rows of a cluster node (-1: the root)
    // out (ni x nj, ld ni, device) = A_hss(I, J) for any index lists
    // (HssMatrix::extract, hss_matrix.hpp:261-280); returns the leaves visited
    long long extract(const std::vector<int>& I, const std::vector<int>& J, double* out);
    int rows() const;
    int rounds() const;
    int d_final() const;
    int hss_rank() const;
    void ranks(std::vector<int>& u, std::vector<int>& v) const;
    long long stored_scalars() const;
    double flops() const;
    size_t arena_bytes() const;  // device slabs held by the front's block cache
    std::vector<HssPhaseStat> phase_stats();
    void restore_phase_stats(const std::vector<HssPhaseStat>&) {}

  private:
    std::unique_ptr<HssImpl> d_;
  };

}  // namespace hssmf_b200
