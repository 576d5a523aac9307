// Device-side front descriptors and the dense-front kernels (assembly,
// partial LU, Schur update, solves). Layout per front (column-major):
//   P  m x ns, ld m : [F11; F21] -> [L11\U11; L21]       (persistent)
//   U  ns x nu, ld ns: F12 -> U12 = L11^-1 P F12          (persistent)
//   C  nu x nu, ld nu: F22 -> cb = F22 - L21 U12          (transient)
// Reference counterpart: Front<T> (multifrontal.hpp:30-63) whose dense state
// is {lu = PLU of F11, f12, f21, cb}; the Schur complement is identical in
// exact arithmetic (F21 F11^-1 F12 = L21 U12) and the solve applies the same
// operator (mf_forward / mf_backward, multifrontal.hpp:507-607).
#pragma once

#include <cstdint>
#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  struct FrontDev {
    int ns, nu, m, sep_begin;
    int child0, child1, level, hss;
    int ldu, ldc;     // leading dimensions of U and C (ns / nu for a dense front)
    double* P;
    double* U;
    double* C;        // update matrix (dense child) or densified update (HSS child)
    int* piv;         // ns, absolute row within F11 swapped at step j
    int* perm;        // ns, composed row permutation (row i of PF11 = row perm[i] of F11)
    const int* upd;   // nu global indices (sorted)
    const int* pos0;  // child0 upd -> local index in this front
    const int* pos1;
    double* bupd;     // solve scratch: nu x nrhs (ld nu)
  };

  // Partial LU of a host-described batch of fronts (dynamic shapes: HSS ULV
  // nodes, top blocks, fallback fronts): perm initialised to identity, panel
  // loop of lu_panel / l21 / swap_trsm / trailing GEMM, then the Schur GEMM.
  // Returns per front the first singular column (-1 if none).
  std::vector<int> partial_lu_dynamic(const std::vector<FrontDev>& fronts, cudaStream_t s,
                                      double* flops = nullptr);

  struct DenseKernels {
    // assembly (a4): zero is done by the caller (memset of the level's arenas)
    static void assemble_sparse(const FrontDev* f, const int* ids, int nf, const int* ptr,
                                const int* ind, const double* val, cudaStream_t s);
    // extend-add of one child slot (0 or 1) for all fronts in ids; colpre is the
    // prefix of child update sizes (warp per child column)
    static void extend_add(const FrontDev* f, const int* ids, int nf, int slot,
                           const long long* colpre, long long ncols, cudaStream_t s);
    static void lu_panel(const FrontDev* f, const int* ids, int nf, int k, int nb,
                         int* status, cudaStream_t s);
    // L21 part of panel k: rows [ns, m) <- A21 U_kk^-1 (after lu_panel)
    static void l21(const FrontDev* f, const int* ids, int nf, int k, int nb, int max_nu,
                    cudaStream_t s);
    static void swap_trsm(const FrontDev* f, const int* ids, int nf, int k, int nb,
                          int max_cols, cudaStream_t s);
    // solve
    static void fold_children(const FrontDev* f, const int* ids, int nf, int slot,
                              double* x, int ldx, int nrhs, int max_nu, cudaStream_t s);
    static void fwd_trsv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                         int nrhs, int max_ns, cudaStream_t s);
    static void fwd_gemv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                         int nrhs, int max_nu, cudaStream_t s);
    static void bwd_gemv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                         int nrhs, int max_ns, cudaStream_t s);
    static void bwd_trsv(const FrontDev* f, const int* ids, int nf, double* x, int ldx,
                         int nrhs, int max_ns, cudaStream_t s);
  };

}  // namespace hssmf_b200
