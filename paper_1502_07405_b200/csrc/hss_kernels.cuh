// Batched data-movement kernels of the HSS path: indexed copies (element
// extraction from a dense front, row/column gathers of samples, basis
// permutations, scatters of [I; E] into dense bases), max-abs reduction, and
// the per-level ULV solve kernels.
#pragma once

#include <vector>

#include "common.cuh"

namespace hssmf_b200 {

  // out(dr(i), dc(j)) (+)= alpha * src(sr(i), sc(j)), i < nr, j < nc.
  // src addressing: src[sr * srs + sc * scs]; dst is column-major (ld ldd).
  // A null index array means the identity map offset by *_off.
  struct CopyDesc {
    const double* src;
    long long srs, scs;
    const int* sr;
    const int* sc;
    int sr_off, sc_off;
    double* dst;
    long long ldd;
    const int* dr;
    const int* dc;
    int dr_off, dc_off;
    int nr, nc;
    double alpha;
    int accumulate;
    int diag;  // copy only the pairs (i, i), i < nr
  };

  inline CopyDesc copy_block(const double* src, long long lds, double* dst, long long ldd, int nr,
                             int nc) {
    return {src, 1, lds, nullptr, nullptr, 0, 0, dst, ldd, nullptr, nullptr, 0, 0, nr, nc, 1.0, 0,
            0};
  }

  // runs a host list of descriptors (uploads them stream-ordered)
  void index_copy_run(const std::vector<CopyDesc>& d, cudaStream_t s);

  // dst[off + i] = src[i], i < n, for every segment (one launch per 128)
  struct IntSeg {
    const int* src;
    int n;
    long long off;
  };
  void int_gather_run(const std::vector<IntSeg>& segs, int* dst, cudaStream_t s);

  // *out = max(*out, max |a(i, j)|) over an m x n block (ld lda); out is a
  // device double holding a non-negative value (bitwise int64 ordering)
  void maxabs_run(const double* a, long long lda, int m, int n, double* out, cudaStream_t s);
  // out[j] = L(perm[j], j), j < k: the pivot norms of a pivoted Cholesky (measurement dumps)
  void diag_gather_run(const double* L, int n, const int* perm, int k, double* out, cudaStream_t s);

  // ---- ULV solve (hss_ulv.hpp:226-276), one CTA per node of one HSS level
  struct UlvSolveNode {
    // omega / psi data
    const int* uperm;   // m (rows of U)
    const int* vperm;   // m
    const double* Eu;   // k x r, ld k
    const double* Ev;   // k x r, ld k
    // factored G (m x m, ld m): [L11\U11 | U12 ; L21 | .], pivots of the k x k block
    const double* G;
    const int* lperm;   // k: composed row permutation of the pivoting
    int m, r, k;
    // forward: input vector pieces (leaf: x + xoff contiguous m values of the
    // rhs; internal: children outputs f0 (r0) and f1 (r1))
    const double* in0;
    const double* in1;
    int n0;             // length taken from in0 (the rest from in1)
    double* ws;         // k (forward elimination result kept for backward)
    double* fout;       // r (reduced rhs passed to the parent)
    // backward: xkeep (r) input, outputs split to children or to x
    const double* xkeep;
    double* out0;       // first n0 entries of x_local
    double* out1;       // remaining entries
    double* scr;        // level scratch of the batched steps (set by the launcher)
  };
  void ulv_fwd_level(const std::vector<UlvSolveNode>& nodes, int nrhs_ld_unused, cudaStream_t s);
  void ulv_bwd_level(const std::vector<UlvSolveNode>& nodes, cudaStream_t s);

  // small dense LU solve (n x n factored in place, ld, composed row perm) of a
  // single vector: x <- U^-1 L^-1 P x ; run on one CTA
  // dout[0] = max_{i>j} |a(i,j) - a(j,i)|, dout[1] = max |a| of the m x m
  // matrix a (ld lda), stream-ordered (the caller reads them back)
  void asymmetry_async(const double* a, long long lda, int m, double* dout, cudaStream_t s);
  // a(i, j) = a(j, i) for i < j (n x n, ld): symmetrizes from the lower triangle
  void mirror_lower_run(double* a, long long ld, int n, cudaStream_t s);
  void lu_solve_vec(const double* lu, int ld, const int* perm, int n, double* x, cudaStream_t s);
  // y (+)= alpha op(A) x for one small dense matrix (one launch)
  void gemv_run(char ta, int m, int n, double alpha, const double* A, int lda, const double* x,
                double beta, double* y, cudaStream_t s);

}  // namespace hssmf_b200
