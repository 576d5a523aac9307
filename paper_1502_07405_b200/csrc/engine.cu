// Level-synchronous multifrontal factorization / solve orchestrator.
#include "engine.hpp"

#include <algorithm>
#include <cstring>
#include <numeric>

#include "common.cuh"
#include "front.cuh"
#include "gemm.cuh"

namespace hssmf_b200 {

  namespace {
    constexpr int NB = 32;  // LU panel width (reference lu_recursive base, lu.hpp:51)

    struct DevMem {
      void* p = nullptr;
      size_t bytes = 0;
      void alloc(size_t b) {
        free();
        if (b) HSSMF_CUDA(cudaMalloc(&p, b));
        bytes = b;
      }
      void free() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
      }
      template<typename T> T* as(size_t off_bytes = 0) const {
        return reinterpret_cast<T*>(static_cast<char*>(p) + off_bytes);
      }
      ~DevMem() { free(); }
    };

    template<typename T> void upload(DevMem& m, const std::vector<T>& v) {
      m.alloc(std::max<size_t>(v.size() * sizeof(T), 16));
      if (!v.empty()) HSSMF_CUDA(cudaMemcpy(m.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    }

    inline long long dense_front_flops(long long ns, long long nu) {
      return 2 * ns * ns * ns / 3 + 2 * ns * ns * nu + 2 * ns * nu * nu;
    }

    enum KClass { K_ASM, K_EXTADD, K_PANEL, K_TRSM, K_GEMM_TRAIL, K_GEMM_SCHUR, K_SOLVE_FWD,
                  K_SOLVE_BWD, K_NCLASS };
    const char* kclass_name[K_NCLASS] = {"assemble_sparse", "extend_add", "lu_panel",
                                         "swap_trsm", "gemm_trailing", "gemm_schur",
                                         "solve_forward", "solve_backward"};
  }  // namespace

  struct StepBatch {
    int k = 0, max_cols = 0;
    GemmBatchDev trail;
  };

  struct LevelPlan {
    int ids_off = 0, nf = 0;
    int max_ns = 0, max_nu = 0, max_m = 0;
    size_t p_off = 0, p_bytes = 0;    // persistent P/U region (bytes)
    size_t c_off = 0, c_bytes = 0;    // transient C region within its parity half
    size_t b_off = 0, b_count = 0;    // bupd region (doubles per rhs)
    long long ncols[2] = {0, 0};
    int max_child_nu[2] = {0, 0};
    size_t colpre_off[2] = {0, 0};
    std::vector<StepBatch> steps;
    GemmBatchDev schur;
    double flops_trail = 0, flops_schur = 0, bytes_ea = 0;
  };

  struct Engine::Impl {
    Csr a;
    Etree t;
    Options opt;
    std::vector<FrontDev> hf;
    std::vector<LevelPlan> levels;  // index = tree level
    std::vector<long long> bupd_off;
    DevMem d_ptr, d_ind, d_val, d_upd, d_pos, d_fronts, d_ids, d_colpre, d_gemm, d_gpre;
    DevMem persist, ipersist, trans[2], bupd, status, xbuf;
    int bupd_nr = 1;
    size_t bupd_total = 0;
    // profiling
    struct Ev { int cls; cudaEvent_t a, b; double flops, bytes; };
    std::vector<Ev> evs;
    std::vector<cudaEvent_t> pool;
    KernelStat kstat[K_NCLASS];
    bool profile = false;
    cudaStream_t s = nullptr;

    cudaEvent_t get_ev() {
      if (!pool.empty()) {
        auto e = pool.back();
        pool.pop_back();
        return e;
      }
      cudaEvent_t e;
      HSSMF_CUDA(cudaEventCreate(&e));
      return e;
    }
    template<typename F> void launch(int cls, double flops, double bytes, F&& f) {
      if (!profile) { f(); return; }
      Ev e{cls, get_ev(), get_ev(), flops, bytes};
      HSSMF_CUDA(cudaEventRecord(e.a, s));
      f();
      HSSMF_CUDA(cudaEventRecord(e.b, s));
      evs.push_back(e);
    }
    void collect() {
      for (auto& e : evs) {
        float ms = 0;
        HSSMF_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
        auto& k = kstat[e.cls];
        k.launches++;
        k.ms += ms;
        k.flops += e.flops;
        k.bytes += e.bytes;
        pool.push_back(e.a);
        pool.push_back(e.b);
      }
      evs.clear();
    }
    ~Impl() {
      for (auto& e : evs) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
      for (auto e : pool) cudaEventDestroy(e);
    }
    void set_bupd_capacity(int nr);
  };

  void Engine::Impl::set_bupd_capacity(int nr) {
    bupd_nr = std::max(nr, 1);
    bupd.alloc(std::max<size_t>(bupd_total * bupd_nr * sizeof(double), 16));
    for (size_t i = 0; i < hf.size(); i++) hf[i].bupd = bupd.as<double>() + bupd_off[i] * bupd_nr;
    HSSMF_CUDA(cudaMemcpy(d_fronts.p, hf.data(), hf.size() * sizeof(FrontDev),
                          cudaMemcpyHostToDevice));
  }

  Engine::Engine(int device) : d_(new Impl), device_(device) {
    HSSMF_CUDA(cudaSetDevice(device));
    HSSMF_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    d_->s = stream_;
    for (int k = 0; k < K_NCLASS; k++) d_->kstat[k].name = kclass_name[k];
  }

  Engine::~Engine() {
    cudaSetDevice(device_);
    d_.reset();
    if (stream_) cudaStreamDestroy(stream_);
  }

  void Engine::analyze(const Csr& a, const Etree& t, const Options& o) {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    if (a.n != t.n) throw SolverFailure(1, -1, -1, "mf factor: matrix and tree sizes differ");
    D.a = a;
    D.t = t;
    D.t.compute_levels();
    D.opt = o;
    n_ = a.n;
    factored_ = false;
    const int nn = (int)D.t.nodes.size();
    int nlev = 0;
    for (const auto& f : D.t.nodes) nlev = std::max(nlev, f.level + 1);

    // upload CSR
    upload(D.d_ptr, a.ptr);
    upload(D.d_ind, a.ind);
    upload(D.d_val, a.val);

    // upd sets and child position maps (front_local / child_positions,
    // multifrontal.hpp:67-94)
    std::vector<int> upd_all, pos_all;
    std::vector<long long> upd_off(nn), pos_off0(nn, -1), pos_off1(nn, -1);
    for (int i = 0; i < nn; i++) {
      upd_off[i] = upd_all.size();
      upd_all.insert(upd_all.end(), D.t.nodes[i].upd.begin(), D.t.nodes[i].upd.end());
    }
    auto local = [&](const FrontNode& f, int g) {
      if (g < f.sep_end) return g - f.sep_begin;
      auto it = std::lower_bound(f.upd.begin(), f.upd.end(), g);
      return f.ns() + (int)(it - f.upd.begin());
    };
    for (int i = 0; i < nn; i++) {
      const auto& f = D.t.nodes[i];
      for (int slot = 0; slot < 2; slot++) {
        const int c = slot ? f.child1 : f.child0;
        if (c < 0) continue;
        (slot ? pos_off1 : pos_off0)[i] = pos_all.size();
        for (int g : D.t.nodes[c].upd) pos_all.push_back(local(f, g));
      }
    }
    upload(D.d_upd, upd_all);
    upload(D.d_pos, pos_all);

    // level lists
    std::vector<std::vector<int>> lv(nlev);
    for (int i = 0; i < nn; i++) lv[D.t.nodes[i].level].push_back(i);
    D.levels.assign(nlev, LevelPlan());
    std::vector<int> ids;

    // persistent / transient layout, level-major from the deepest level
    size_t poff = 0, ipoff = 0, cmax[2] = {0, 0}, boff = 0;
    std::vector<size_t> p_at(nn), u_at(nn), c_at(nn), piv_at(nn);
    D.bupd_off.assign(nn, 0);
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      P.ids_off = (int)ids.size();
      P.nf = (int)lv[L].size();
      ids.insert(ids.end(), lv[L].begin(), lv[L].end());
      P.p_off = poff;
      size_t coff = 0;
      for (int i : lv[L]) {
        const auto& f = D.t.nodes[i];
        const size_t ns = f.ns(), nu = f.nu(), m = ns + nu;
        P.max_ns = std::max(P.max_ns, (int)ns);
        P.max_nu = std::max(P.max_nu, (int)nu);
        P.max_m = std::max(P.max_m, (int)m);
        p_at[i] = poff;
        poff += ((m * ns * 8 + 255) / 256) * 256;
        u_at[i] = poff;
        poff += ((ns * nu * 8 + 255) / 256) * 256;
        c_at[i] = coff;
        coff += ((nu * nu * 8 + 255) / 256) * 256;
        piv_at[i] = ipoff;
        ipoff += 2 * ns;
        D.bupd_off[i] = boff;
        boff += nu;
      }
      P.b_off = boff - [&] { size_t c = 0; for (int i : lv[L]) c += D.t.nodes[i].nu(); return c; }();
      P.b_count = boff - P.b_off;
      P.p_bytes = poff - P.p_off;
      P.c_off = 0;
      P.c_bytes = coff;
      cmax[L % 2] = std::max(cmax[L % 2], coff);
    }
    D.bupd_total = boff;
    D.persist.alloc(std::max<size_t>(poff, 256));
    D.ipersist.alloc(std::max<size_t>(ipoff * sizeof(int), 256));
    D.trans[0].alloc(std::max<size_t>(cmax[0], 256));
    D.trans[1].alloc(std::max<size_t>(cmax[1], 256));
    D.status.alloc(std::max<size_t>(nn * sizeof(int), 16));
    upload(D.d_ids, ids);

    D.hf.assign(nn, FrontDev());
    for (int i = 0; i < nn; i++) {
      const auto& f = D.t.nodes[i];
      auto& h = D.hf[i];
      h.ns = f.ns();
      h.nu = f.nu();
      h.m = f.m();
      h.sep_begin = f.sep_begin;
      h.child0 = f.child0;
      h.child1 = f.child1;
      h.level = f.level;
      h.hss = 0;
      h.ldu = h.ns;
      h.ldc = h.nu;
      h.P = D.persist.as<double>(p_at[i]);
      h.U = D.persist.as<double>(u_at[i]);
      h.C = D.trans[f.level % 2].as<double>(c_at[i]);
      h.piv = D.ipersist.as<int>() + piv_at[i];
      h.perm = h.piv + h.ns;
      h.upd = D.d_upd.as<int>() + upd_off[i];
      h.pos0 = pos_off0[i] >= 0 ? D.d_pos.as<int>() + pos_off0[i] : nullptr;
      h.pos1 = pos_off1[i] >= 0 ? D.d_pos.as<int>() + pos_off1[i] : nullptr;
    }
    D.d_fronts.alloc(nn * sizeof(FrontDev));
    D.set_bupd_capacity(1);

    // extend-add column prefixes and GEMM batches
    std::vector<long long> colpre;
    std::vector<GemmProblem> gp;
    std::vector<int> gpre;
    auto add_batch = [&](std::vector<GemmProblem>& probs) {
      GemmBatchDev b;
      if (probs.empty()) return b;
      auto pre = gemm_tile_prefix(probs);
      b.probs = reinterpret_cast<const GemmProblem*>(gp.size());  // offsets, fixed below
      b.prefix = reinterpret_cast<const int*>(gpre.size());
      b.nprob = (int)probs.size();
      b.tiles = pre.back();
      gp.insert(gp.end(), probs.begin(), probs.end());
      gpre.insert(gpre.end(), pre.begin(), pre.end());
      return b;
    };
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      for (int slot = 0; slot < 2; slot++) {
        P.colpre_off[slot] = colpre.size();
        long long acc = 0;
        for (int q = 0; q < P.nf; q++) {
          colpre.push_back(acc);
          const auto& f = D.t.nodes[lv[L][q]];
          const int c = slot ? f.child1 : f.child0;
          if (c >= 0) {
            const long long nuc = D.t.nodes[c].nu();
            P.max_child_nu[slot] = std::max(P.max_child_nu[slot], (int)nuc);
            acc += nuc;
            P.bytes_ea += 24.0 * nuc * nuc + 4.0 * nuc;
          }
        }
        colpre.push_back(acc);
        P.ncols[slot] = acc;
      }
      for (int k = 0; k < P.max_ns; k += NB) {
        StepBatch sb;
        sb.k = k;
        std::vector<GemmProblem> probs;
        for (int i : lv[L]) {
          const auto& h = D.hf[i];
          if (h.ns <= k) continue;
          const int nbk = std::min(NB, h.ns - k);
          sb.max_cols = std::max(sb.max_cols, h.m - nbk);
          const int k1 = k + nbk;
          if (h.ns > k1) {
            // P[k1:m, k1:ns] -= P[k1:m, k:k1] P[k:k1, k1:ns]
            probs.push_back({h.P + k1 + (size_t)k * h.m, h.P + k + (size_t)k1 * h.m,
                             h.P + k1 + (size_t)k1 * h.m, h.m - k1, h.ns - k1, nbk, h.m, h.m,
                             h.m});
            if (h.nu)  // U[k1:ns, :] -= P[k1:ns, k:k1] U[k:k1, :]
              probs.push_back({h.P + k1 + (size_t)k * h.m, h.U + k, h.U + k1, h.ns - k1, h.nu,
                               nbk, h.m, h.ldu, h.ldu});
          }
        }
        P.flops_trail += gemm_flops(probs);
        sb.trail = add_batch(probs);
        P.steps.push_back(sb);
      }
      std::vector<GemmProblem> probs;
      for (int i : lv[L]) {
        const auto& h = D.hf[i];
        if (h.ns && h.nu)  // C -= L21 U12 (Schur complement, multifrontal.hpp:340-344)
          probs.push_back({h.P + h.ns, h.U, h.C, h.nu, h.nu, h.ns, h.m, h.ldu, h.ldc});
      }
      P.flops_schur = gemm_flops(probs);
      P.schur = add_batch(probs);
    }
    upload(D.d_colpre, colpre);
    upload(D.d_gemm, gp);
    upload(D.d_gpre, gpre);
    auto fix = [&](GemmBatchDev& b) {
      if (!b.nprob) return;
      b.probs = D.d_gemm.as<GemmProblem>() + reinterpret_cast<size_t>(b.probs);
      b.prefix = D.d_gpre.as<int>() + reinterpret_cast<size_t>(b.prefix);
    };
    for (auto& P : D.levels) {
      for (auto& sb : P.steps) fix(sb.trail);
      fix(P.schur);
    }

    stats_.assign(nn, FrontStat());
    for (int i = 0; i < nn; i++) {
      const auto& f = D.t.nodes[i];
      auto& st = stats_[i];
      st.level = f.level;
      st.dim = f.m();
      st.sep = f.ns();
      st.rank = 0;
      st.type = 0;
      st.flops = dense_front_flops(f.ns(), f.nu());
    }
  }

  void Engine::set_values(const double* val, bool on_device) {
    auto& D = *d_;
    HSSMF_CUDA(cudaMemcpyAsync(D.d_val.p, val, D.a.val.size() * sizeof(double),
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               stream_));
    factored_ = false;
  }

  void Engine::factor() {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    D.profile = profile_;
    const int nn = (int)D.hf.size();
    cudaEvent_t e0, e1;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventRecord(e0, stream_));
    HSSMF_CUDA(cudaMemsetAsync(D.status.p, 0xff, nn * sizeof(int), stream_));
    const FrontDev* F = D.d_fronts.as<FrontDev>();
    const int nlev = (int)D.levels.size();
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      const int* ids = D.d_ids.as<int>() + P.ids_off;
      HSSMF_CUDA(cudaMemsetAsync(D.persist.as<char>(P.p_off), 0, P.p_bytes, stream_));
      if (P.c_bytes)
        HSSMF_CUDA(cudaMemsetAsync(D.trans[L % 2].as<char>(P.c_off), 0, P.c_bytes, stream_));
      D.launch(K_ASM, 0, 0, [&] {
        DenseKernels::assemble_sparse(F, ids, P.nf, D.d_ptr.as<int>(), D.d_ind.as<int>(),
                                      D.d_val.as<double>(), stream_);
      });
      for (int slot = 0; slot < 2; slot++)
        D.launch(K_EXTADD, 0, P.bytes_ea / 2, [&] {
          DenseKernels::extend_add(F, ids, P.nf, slot,
                                   D.d_colpre.as<long long>() + P.colpre_off[slot],
                                   P.ncols[slot], stream_);
        });
      for (auto& sb : P.steps) {
        D.launch(K_PANEL, 0, 0, [&] {
          DenseKernels::lu_panel(F, ids, P.nf, sb.k, NB, D.status.as<int>(), stream_);
        });
        D.launch(K_TRSM, 0, 0, [&] {
          DenseKernels::l21(F, ids, P.nf, sb.k, NB, P.max_nu, stream_);
          DenseKernels::swap_trsm(F, ids, P.nf, sb.k, NB, sb.max_cols, stream_);
        });
        D.launch(K_GEMM_TRAIL, 0, 0,
                 [&] { gemm_run(sb.trail, 'N', 'N', -1.0, 1.0, stream_); });
      }
      D.launch(K_GEMM_SCHUR, P.flops_schur, 0,
               [&] { gemm_run(P.schur, 'N', 'N', -1.0, 1.0, stream_); });
    }
    HSSMF_CUDA(cudaEventRecord(e1, stream_));
    std::vector<int> st(nn);
    HSSMF_CUDA(cudaMemcpyAsync(st.data(), D.status.p, nn * sizeof(int), cudaMemcpyDeviceToHost,
                               stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
    float ms = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    factor_ms_ = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (profile_) D.collect();
    // first failure in postorder = the one the sequential reference reports
    for (int i = 0; i < nn; i++)
      if (st[i] >= 0)
        throw SolverFailure(3, i, st[i],
                            "front " + std::to_string(i) +
                                ": exactly singular, zero pivot column " + std::to_string(st[i]));
    factored_ = true;
  }

  void Engine::solve(double* b, int ldb, int nrhs, bool on_device) {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    if (!factored_) throw SolverFailure(2, -1, -1, "mf solve: not factored");
    if (nrhs <= 0) return;
    D.profile = profile_;
    if (nrhs > D.bupd_nr) D.set_bupd_capacity(nrhs);
    double* x = b;
    int ldx = ldb;
    if (!on_device || ldb != n_) {
      const size_t need = (size_t)n_ * nrhs * sizeof(double);
      if (D.xbuf.bytes < need) D.xbuf.alloc(need);
      x = D.xbuf.as<double>();
      ldx = n_;
      HSSMF_CUDA(cudaMemcpy2DAsync(x, n_ * sizeof(double), b, (size_t)ldb * sizeof(double),
                                   n_ * sizeof(double), nrhs,
                                   on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                   stream_));
    }
    cudaEvent_t e0, e1;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventRecord(e0, stream_));
    const FrontDev* F = D.d_fronts.as<FrontDev>();
    const int nlev = (int)D.levels.size();
    const int nr = D.bupd_nr;
    // forward sweep, deepest level first (mf_forward, multifrontal.hpp:507-567)
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      const int* ids = D.d_ids.as<int>() + P.ids_off;
      if (P.b_count)
        HSSMF_CUDA(cudaMemsetAsync(D.bupd.as<double>() + P.b_off * nr, 0,
                                   P.b_count * nr * sizeof(double), stream_));
      D.launch(K_SOLVE_FWD, 0, 0, [&] {
        for (int slot = 0; slot < 2; slot++)
          DenseKernels::fold_children(F, ids, P.nf, slot, x, ldx, nrhs, P.max_child_nu[slot],
                                      stream_);
        DenseKernels::fwd_trsv(F, ids, P.nf, x, ldx, nrhs, P.max_ns, stream_);
        DenseKernels::fwd_gemv(F, ids, P.nf, x, ldx, nrhs, P.max_nu, stream_);
      });
    }
    // backward sweep, root first (mf_backward, multifrontal.hpp:569-607)
    for (int L = 0; L < nlev; L++) {
      auto& P = D.levels[L];
      const int* ids = D.d_ids.as<int>() + P.ids_off;
      D.launch(K_SOLVE_BWD, 0, 0, [&] {
        DenseKernels::bwd_gemv(F, ids, P.nf, x, ldx, nrhs, P.max_ns, stream_);
        DenseKernels::bwd_trsv(F, ids, P.nf, x, ldx, nrhs, P.max_ns, stream_);
      });
    }
    HSSMF_CUDA(cudaEventRecord(e1, stream_));
    if (x != b)
      HSSMF_CUDA(cudaMemcpy2DAsync(b, (size_t)ldb * sizeof(double), x, n_ * sizeof(double),
                                   n_ * sizeof(double), nrhs,
                                   on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                   stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
    float ms = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    solve_ms_ = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (profile_) D.collect();
  }

  long long Engine::factor_nnz() const {
    long long s = 0;
    for (const auto& f : d_->t.nodes) s += (long long)f.ns() * f.ns() + 2LL * f.ns() * f.nu();
    return s;
  }
  int Engine::hss_fronts() const { return 0; }
  int Engine::fallbacks() const { return 0; }
  int Engine::max_front_rank() const { return 0; }
  bool Engine::front_hss(int, std::vector<int>&, std::vector<int>&, int&, int&) const {
    return false;
  }
  std::vector<KernelStat> Engine::kernel_stats() const {
    return std::vector<KernelStat>(d_->kstat, d_->kstat + K_NCLASS);
  }
  void Engine::reset_kernel_stats() {
    for (auto& k : d_->kstat) { k.launches = 0; k.ms = k.flops = k.bytes = 0; }
  }
  size_t Engine::device_bytes() const {
    const auto& D = *d_;
    return D.persist.bytes + D.ipersist.bytes + D.trans[0].bytes + D.trans[1].bytes +
           D.bupd.bytes + D.d_val.bytes + D.d_ind.bytes + D.d_ptr.bytes + D.d_gemm.bytes;
  }

}  // namespace hssmf_b200
