// Host orchestrator of the numeric factorization and solve on one B200.
//
// Mirrors mf_factor / mf_solve (reference multifrontal.hpp:473-631) with a
// level-synchronous schedule over the elimination tree: every kernel launch
// covers all fronts of one tree level. The dense part of the schedule is
// static (built once in Engine::analyze) and replayed through a CUDA graph.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <algorithm>
#include <string>
#include <vector>

#include "host/analysis.hpp"

namespace hssmf_b200 {

  // SolverOptions (reference solver_options.hpp:28-59), numeric subset
  struct Options {
    int ls = 0;
    double eps = 1e-8;
    int leaf = 128, d0 = 128, dd = 128, p = 10, min_hss = 512, max_rank = 0;
    int mode = 0;  // 0 auto, 1 mf (never HSS), 2 mf-hss
    int switch_level() const { return mode == 1 ? 0 : ls; }
    int resolved_max_rank(int n) const { return max_rank > 0 ? max_rank : std::min(n / 2, 5000); }
  };

  // FrontStat (reference stats.hpp:11-19); type 0 dense, 1 hss, 2 hss_dense
  struct FrontStat {
    int level = 0, dim = 0, sep = 0, rank = 0, type = 0;
    long long flops = 0;
  };



  // per-kernel-class device time + algorithmic work, for the roofline
  struct KernelStat {
    std::string name;
    int launches = 0;
    double ms = 0, flops = 0, bytes = 0;
  };

  class Engine {
  public:
    Engine(int device);
    ~Engine();

    // upload structure + values, build the static schedule. owned (optional,
    // one flag per front): only these fronts are factored and solved here;
    // the updates / bupd of their non-owned children are imported (multi-GPU
    // subtree partition)
    void analyze(const Csr& a, const Etree& t, const Options& o, const char* owned = nullptr);
    // numeric factorization from the resident values
    void factor() { factor_levels(0, nlevels() - 1); }
    // the fronts of tree levels lo..hi (deepest first); a multi-GPU run calls
    // it phase by phase with update imports in between
    void factor_levels(int lo, int hi);
    int nlevels() const;
    // update block (nu x nu, ld nu) of front f: out to dst / in from src
    void export_update(int f, double* dst, bool on_device) const;
    void import_update(int f, const double* src, bool on_device);
    // forward-sweep contribution bupd (nu x nrhs, ld nu) of front f, device memory
    void export_bupd(int f, double* dst, int nrhs) const;
    void import_bupd(int f, const double* src, int nrhs);
    // one sweep over levels lo..hi on a device x (n x nrhs, ld ldx): forward
    // deepest first, backward root first
    void solve_levels(double* x, int ldx, int nrhs, int lo, int hi, bool forward);
    // replace the matrix values (same pattern) from host or device memory
    void set_values(const double* val, bool on_device);
    // solve in place: b is n x nrhs column-major (ld = ldb), host or device
    void solve(double* b, int ldb, int nrhs, bool on_device);

    bool factored() const { return factored_; }
    int n() const { return n_; }
    const std::vector<FrontStat>& stats() const { return stats_; }
    long long factor_nnz() const;
    int hss_fronts() const, fallbacks() const, max_front_rank() const;
    // per HSS node ranks of one front (empty if dense)
    bool front_hss(int f, std::vector<int>& u, std::vector<int>& v, int& rounds,
                   int& d_final) const;
    double factor_ms() const { return factor_ms_; }
    double solve_ms() const { return solve_ms_; }
    void set_profile(bool on) { profile_ = on; }
    std::vector<KernelStat> kernel_stats() const;
    void reset_kernel_stats();
    size_t device_bytes() const;
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }

    struct Impl;

  private:
    std::unique_ptr<Impl> d_;
    int device_ = 0, n_ = 0;
    bool factored_ = false, profile_ = false;
    cudaStream_t stream_ = nullptr;
    std::vector<FrontStat> stats_;
    double factor_ms_ = 0, solve_ms_ = 0;
  };

}  // namespace hssmf_b200
