// Level-synchronous multifrontal factorization / solve orchestrator.
//
// factor(): for every elimination-tree level, deepest first,
//   dense fronts  -> one static batch: zero, sparse scatter, extend-add of both
//                    children, panel LU of F11 (+ L21, U12), Schur GEMM
//   HSS fronts    -> one at a time: dense assembly in HBM, adaptive randomized
//                    HSS compression, partial ULV, densified low-rank update
//                    for the parent (factor_front_hss, multifrontal.hpp:348-377);
//                    rank-guard trip -> dense fallback on the assembled front
// solve(): forward sweep bottom-up, backward sweep top-down, same batching.
#include "engine.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <map>

#include "common.cuh"
#include "front.cuh"
#include "gemm.cuh"
#include "arena.cuh"
#include "hss.hpp"
#include "hss_kernels.cuh"

namespace hssmf_b200 {
  cudaStream_t worker_stream_take(int device);
  void worker_stream_give(int device, cudaStream_t st);

  namespace {
    constexpr int NB = 32;  // LU panel width (reference lu_recursive base, lu.hpp:51)

    struct DevMem {
      void* p = nullptr;
      size_t bytes = 0;
      DevMem() = default;
      DevMem(const DevMem&) = delete;
      DevMem(DevMem&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
      DevMem& operator=(DevMem&& o) noexcept {
        if (this != &o) {
          free();
          p = o.p;
          bytes = o.bytes;
          o.p = nullptr;
          o.bytes = 0;
        }
        return *this;
      }
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
      if (!v.empty())
        HSSMF_CUDA(cudaMemcpy(m.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    }

    // analytic per-front estimates (multifrontal.hpp:391-396)
    inline long long dense_front_flops(long long ns, long long nu) {
      return 2 * ns * ns * ns / 3 + 2 * ns * ns * nu + 2 * ns * nu * nu;
    }
    inline long long hss_front_flops(long long m, long long r, long long d) {
      return 4 * m * m * d + 8 * m * r * r;
    }

    enum KClass { K_ASM, K_EXTADD, K_PANEL, K_TRSM, K_GEMM_TRAIL, K_GEMM_SCHUR, K_HSS,
                  K_SOLVE_FWD, K_SOLVE_BWD, K_HSS_PH, K_NCLASS = K_HSS_PH + kHssPhases };
    const char* kclass_name[K_HSS_PH] = {"assemble_sparse", "extend_add", "lu_panel",
                                         "l21_swap_trsm", "gemm_trailing", "gemm_schur",
                                         "hss_front_total", "solve_forward", "solve_backward"};
  }  // namespace

  struct StepBatch {
    int k = 0, max_cols = 0;
    GemmBatchDev trail;
    double flops = 0;
  };

  struct LevelPlan {
    int ids_off = 0, nf = 0;        // all fronts of the level (fold)
    int dids_off = 0, ndf = 0;      // dense fronts (static factor plan)
    int sids_off = 0, nsf = 0;      // dense + fallback fronts (solve), rebuilt per factor
    std::vector<int> hss;           // HSS fronts (host)
    int max_ns = 0, max_nu = 0;
    size_t p_off = 0, p_bytes = 0;  // persistent P/U region (bytes)
    size_t c_bytes = 0;             // transient C region within its parity half
    size_t b_off = 0, b_count = 0;  // bupd region (doubles per rhs)
    long long ncols[2] = {0, 0};
    int max_child_nu[2] = {0, 0};
    size_t colpre_off[2] = {0, 0};
    std::vector<StepBatch> steps;
    GemmBatchDev schur;
    double flops_schur = 0, bytes_ea[2] = {0, 0}, bytes_asm = 0;
  };

  struct Engine::Impl {
    Csr a;           // sizes only (analyze)
    size_t nnz = 0;  // entries of the matrix on the device
    Etree t;
    Options opt;
    std::vector<FrontDev> hf, hf0;  // live descriptors, analysis-time descriptors
    std::vector<LevelPlan> levels;
    std::vector<std::vector<int>> lv;  // front ids per tree level
    std::vector<long long> bupd_off;
    std::vector<char> want_hss;
    DevMem d_ptr, d_ind, d_val, d_upd, d_pos, d_fronts, d_ids, d_colpre, d_gemm, d_gpre, d_sids;
    DevMem persist, ipersist, trans[2], bupd, status, xbuf, x2buf, scratch;
    std::vector<DevMem> fallback_mem;
    std::vector<std::unique_ptr<HssMatrixDev>> hss;
    std::vector<int> hss_rounds, hss_dfinal;
    int bupd_nr = 1;
    size_t bupd_total = 0;
    int n_hss = 0, n_fallback = 0, max_rank = 0;
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
      if (!profile) {
        f();
        return;
      }
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
      hss.clear();
      if (s) cudaStreamSynchronize(s);
      for (auto& e : evs) {
        cudaEventDestroy(e.a);
        cudaEventDestroy(e.b);
      }
      for (auto e : pool) cudaEventDestroy(e);
    }
    void upload_fronts() {
      HSSMF_CUDA(cudaMemcpyAsync(d_fronts.p, hf.data(), hf.size() * sizeof(FrontDev),
                                 cudaMemcpyHostToDevice, s));
      HSSMF_CUDA(cudaStreamSynchronize(s));
    }
    void upload_front(int i) {
      HSSMF_CUDA(cudaMemcpyAsync(d_fronts.as<FrontDev>() + i, &hf[i], sizeof(FrontDev),
                                 cudaMemcpyHostToDevice, s));
      HSSMF_CUDA(cudaStreamSynchronize(s));
    }
    void set_bupd_capacity(int nr) {
      bupd_nr = std::max(nr, 1);
      bupd.alloc(std::max<size_t>(bupd_total * bupd_nr * sizeof(double), 16));
      for (size_t i = 0; i < hf.size(); i++) {
        hf[i].bupd = bupd.as<double>() + bupd_off[i] * bupd_nr;
        hf0[i].bupd = hf[i].bupd;
      }
      upload_fronts();
    }
    int* scratch_ints(size_t n) {
      if (scratch.bytes < n * sizeof(int)) scratch.alloc(std::max<size_t>(n * sizeof(int), 4096));
      return scratch.as<int>();
    }
    struct HssResult {
      std::unique_ptr<HssMatrixDev> hss;
      bool fallback = false;
      FrontDev front{};
      DevMem keep, piv;
      int singular_col = -1;
      bool oom = false;  // device memory ran out while fronts ran concurrently
      std::string msg, error;
    };
    std::vector<cudaStream_t> hstreams;  // concurrent HSS fronts of one level
    // solves: the HSS fronts of one tree level sweep concurrently on the
    // worker streams (forked from / joined back into the engine stream)
    std::vector<cudaStream_t> solve_st;
    cudaEvent_t solve_fork = nullptr;
    std::vector<cudaEvent_t> solve_join;
    cudaStream_t solve_stream_of(int i) const { return solve_st[i]; }
    template <class F>
    void hss_level_concurrent(const std::vector<int>& lst, cudaStream_t main, F&& f) {
      std::vector<int> L;
      for (int i : lst)
        if (i < (int)hss.size() && hss[i]) L.push_back(i);
      if (L.empty()) return;
      if (solve_st.size() != t.nodes.size()) solve_st.assign(t.nodes.size(), main);
      const int nw = (int)std::min(L.size(), hstreams.size());
      if (nw <= 1) {
        for (int i : L) {
          solve_st[i] = main;
          hss[i]->set_solve_stream(main);
          f(i);
        }
        return;
      }
      if (!solve_fork) HSSMF_CUDA(cudaEventCreateWithFlags(&solve_fork, cudaEventDisableTiming));
      while ((int)solve_join.size() < nw) {
        cudaEvent_t e;
        HSSMF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        solve_join.push_back(e);
      }
      HSSMF_CUDA(cudaEventRecord(solve_fork, main));
      for (int w = 0; w < nw; w++) HSSMF_CUDA(cudaStreamWaitEvent(hstreams[w], solve_fork, 0));
      for (size_t q = 0; q < L.size(); q++) {
        const int i = L[q];
        cudaStream_t ws = hstreams[q % nw];
        solve_st[i] = ws;
        hss[i]->set_solve_stream(ws);
        f(i);
      }
      for (int w = 0; w < nw; w++) {
        HSSMF_CUDA(cudaEventRecord(solve_join[w], hstreams[w]));
        HSSMF_CUDA(cudaStreamWaitEvent(main, solve_join[w], 0));
      }
      for (int i : L) {
        solve_st[i] = main;
        hss[i]->set_solve_stream(main);
      }
    }
    double* assemble_hss_front(int i, cudaStream_t st);
    // every HSS front of a level at once: one zeroing per front, then one
    // sparse-scatter launch and one extend-add launch per child slot for the
    // whole list (assemble_dense semantics and order, multifrontal.hpp:141-170)
    std::vector<double*> assemble_hss_fronts(const std::vector<int>& lst, cudaStream_t st);
    void assemble_on(int i, const FrontDev& view, cudaStream_t st);
    void upload_front_on(int i, cudaStream_t st) {
      HSSMF_CUDA(cudaMemcpyAsync(d_fronts.as<FrontDev>() + i, &hf[i], sizeof(FrontDev),
                                 cudaMemcpyHostToDevice, st));
    }
    // dependency-driven factorization of the fronts from the deepest HSS
    // level up (see factor_region)
    void factor_region(const std::vector<int>& R);
    std::vector<char> owned;        // fronts factored by this engine
    std::vector<int> boundary;      // non-owned children of owned fronts
    std::vector<DevMem> imported;   // imported update blocks (per front)
    std::vector<double*> region_c;  // pool-allocated update blocks of region fronts
    std::vector<int> region_singular;  // first zero-pivot column per region front
    int region_level = -1;             // deepest level holding an HSS front
    HssResult compress_hss_front(int i, double* F, cudaStream_t st, int peers = 0);
    void factor_hss_level(const std::vector<int>& lst);
    size_t devmem_bytes() const;  // engine-owned cudaMalloc storage
  };

  Engine::Engine(int device) : d_(new Impl), device_(device) {
    HSSMF_CUDA(cudaSetDevice(device));
    stream_ = worker_stream_take(device);
    d_->s = stream_;
    for (int k = 0; k < K_NCLASS; k++)
      d_->kstat[k].name = k < K_HSS_PH ? kclass_name[k] : hss_phase_name(k - K_HSS_PH);
    // keep stream-ordered allocations (HSS path) in the pool between factorizations
    cudaMemPool_t mp;
    HSSMF_CUDA(cudaDeviceGetDefaultMemPool(&mp, device));
    unsigned long long thr = ~0ull;
    HSSMF_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
    int nw = 8;
    if (const char* e = getenv("HSSMF_HSS_STREAMS")) nw = std::max(1, atoi(e));
    // HSSMF_HSS_STREAMS_SMALL=n: width of the levels whose fronts are all < 9000 rows
    if (const char* e = getenv("HSSMF_HSS_STREAMS_SMALL")) nw = std::max(nw, atoi(e));
    for (int w = 0; w < nw; w++) d_->hstreams.push_back(worker_stream_take(device));
  }

  // worker streams outlive the engines that use them (a per-device free
  // list): an engine created after another one reuses its streams, hence
  // their side streams and pinned staging rings, instead of creating them
  // again (stream creation and cudaHostAlloc cost milliseconds and the latter
  // synchronizes)
  namespace {
    std::mutex g_ws_mu;
    std::map<int, std::vector<cudaStream_t>>& worker_free() {
      static auto* m = new std::map<int, std::vector<cudaStream_t>>();  // never destroyed
      return *m;
    }
  }  // namespace
  cudaStream_t worker_stream_take(int device) {
    {
      std::lock_guard<std::mutex> lk(g_ws_mu);
      auto& f = worker_free()[device];
      if (!f.empty()) {
        cudaStream_t st = f.back();
        f.pop_back();
        return st;
      }
    }
    // worker streams (the fronts' latency-bound chains of small launches) run
    // at the highest stream priority, their side streams (speculative sampling
    // products: full-device TMA GEMMs) at the default, lowest one: a chain's
    // next small kernel takes the SMs the moment CTAs of another front's
    // sampling product retire instead of queueing behind its whole grid
    // (HSSMF_NO_PRIO=1: all streams at the default priority)
    cudaStream_t st;
    int least = 0, greatest = 0;
    HSSMF_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    static const bool no_prio = getenv("HSSMF_NO_PRIO") != nullptr;
    HSSMF_CUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, no_prio ? least : greatest));
    return st;
  }
  void worker_stream_give(int device, cudaStream_t st) {
    cudaStreamSynchronize(st);
    std::lock_guard<std::mutex> lk(g_ws_mu);
    worker_free()[device].push_back(st);
  }

  Engine::~Engine() {
    cudaSetDevice(device_);
    auto hs = d_->hstreams;
    d_.reset();
    for (auto st : hs) worker_stream_give(device_, st);
    if (stream_) worker_stream_give(device_, stream_);
  }

  void Engine::analyze(const Csr& a, const Etree& t, const Options& o, const char* owned) {
    HSSMF_CUDA(cudaSetDevice(device_));
    const double t_an0 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    auto devmem_bytes_public = [&] { return (double)d_->devmem_bytes(); };
    auto now_s = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    double t_an[6] = {t_an0, 0, 0, 0, 0, 0};
    auto& D = *d_;
    if (a.n != t.n) throw SolverFailure(1, -1, -1, "mf factor: matrix and tree sizes differ");
    // (only the sizes of the matrix are kept on the host: its arrays go to the
    // device below, and a 128^3 copy is 180 MB per call)
    D.a = Csr();
    D.a.n = a.n;
    D.nnz = a.val.size();
    D.t = t;
    D.t.compute_levels();
    D.opt = o;
    n_ = a.n;
    factored_ = false;
    const int nn = (int)D.t.nodes.size();
    D.owned.assign(nn, 1);
    bool partial = false;
    if (owned)
      for (int i = 0; i < nn; i++) {
        D.owned[i] = owned[i] ? 1 : 0;
        partial |= !owned[i];
      }
    D.boundary.clear();
    if (partial)
      for (int i = 0; i < nn; i++) {
        if (!D.owned[i]) continue;
        for (int c : {D.t.nodes[i].child0, D.t.nodes[i].child1})
          if (c >= 0 && !D.owned[c]) D.boundary.push_back(c);
      }
    D.imported.clear();
    D.imported.resize(nn);
    int nlev = 0;
    for (const auto& f : D.t.nodes) nlev = std::max(nlev, f.level + 1);

    upload(D.d_ptr, a.ptr);
    upload(D.d_ind, a.ind);
    upload(D.d_val, a.val);

    // upd sets and child position maps (front_local / child_positions,
    // multifrontal.hpp:67-94)
    std::vector<int> upd_all, pos_all;
    std::vector<long long> upd_off(nn), pos_off0(nn, -1), pos_off1(nn, -1);
    size_t upd_total = 0;
    for (int i = 0; i < nn; i++) upd_total += D.t.nodes[i].upd.size();
    upd_all.reserve(upd_total);
    pos_all.reserve(upd_total);
    for (int i = 0; i < nn; i++) {
      upd_off[i] = upd_all.size();
      upd_all.insert(upd_all.end(), D.t.nodes[i].upd.begin(), D.t.nodes[i].upd.end());
    }
    for (int i = 0; i < nn; i++) {
      const auto& f = D.t.nodes[i];
      for (int slot = 0; slot < 2; slot++) {
        const int c = slot ? f.child1 : f.child0;
        if (c < 0) continue;
        (slot ? pos_off1 : pos_off0)[i] = pos_all.size();
        // both index lists ascend: one merge instead of a search per entry
        // (10 M entries on c5)
        size_t it = 0;
        const int ns_f = f.ns();
        for (int g : D.t.nodes[c].upd) {
          if (g < f.sep_end) {
            pos_all.push_back(g - f.sep_begin);
            continue;
          }
          while (it < f.upd.size() && f.upd[it] < g) it++;
          pos_all.push_back(ns_f + (int)it);
        }
      }
    }
    upload(D.d_upd, upd_all);
    upload(D.d_pos, pos_all);
    t_an[1] = now_s();

    // HSS selection (multifrontal.hpp:410-412)
    D.want_hss.assign(nn, 0);
    for (int i = 0; i < nn; i++) {
      const auto& f = D.t.nodes[i];
      D.want_hss[i] = D.owned[i] && f.level < o.switch_level() && f.m() >= o.min_hss && f.ns() > 0;
    }

    // HSSMF_REGION=1: the fronts from the deepest HSS level up run
    // dependency-driven (factor_region). Measured on C5 it is 10-15% slower
    // than the level-synchronous schedule (memory admission serialises the
    // top fronts more than level barriers do), so the default stays level-
    // synchronous.
    D.region_level = -1;
    static const bool use_region = [] {
      const char* e = getenv("HSSMF_REGION");
      return e && e[0] == '1';
    }();
    // HSSMF_REGION_LEVEL=k: only tree levels <= k run dependency-driven (the
    // few top fronts, where a parent can start while its cousins still run);
    // deeper levels keep their level barriers
    static const int region_top = getenv("HSSMF_REGION_LEVEL") ? atoi(getenv("HSSMF_REGION_LEVEL")) : -1;
    if ((use_region || region_top >= 0) && !partial) {
      for (int i = 0; i < nn; i++)
        if (D.want_hss[i]) D.region_level = std::max(D.region_level, D.t.nodes[i].level);
      if (region_top >= 0 && D.region_level >= 0) D.region_level = std::min(D.region_level, region_top);
    }
    D.lv.assign(nlev, {});
    auto& lv = D.lv;
    for (int i = 0; i < nn; i++)
      if (D.owned[i]) lv[D.t.nodes[i].level].push_back(i);
    D.levels.assign(nlev, LevelPlan());
    std::vector<int> ids;

    // persistent / transient layout, level-major from the deepest level
    size_t poff = 0, ipoff = 0, cmax[2] = {0, 0}, boff = 0;
    std::vector<size_t> p_at(nn, 0), u_at(nn, 0), c_at(nn), piv_at(nn, 0);
    D.bupd_off.assign(nn, 0);
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      P.ids_off = (int)ids.size();
      P.nf = (int)lv[L].size();
      ids.insert(ids.end(), lv[L].begin(), lv[L].end());
      P.p_off = poff;
      P.b_off = boff;
      size_t coff = 0;
      for (int i : lv[L]) {
        const auto& f = D.t.nodes[i];
        const size_t ns = f.ns(), nu = f.nu(), m = ns + nu;
        P.max_ns = std::max(P.max_ns, (int)ns);
        P.max_nu = std::max(P.max_nu, (int)nu);
        c_at[i] = coff;
        coff += ((nu * nu * 8 + 255) / 256) * 256;
        D.bupd_off[i] = boff;
        boff += nu;
        if (D.want_hss[i]) {
          P.hss.push_back(i);
          continue;
        }
        p_at[i] = poff;
        poff += ((m * ns * 8 + 255) / 256) * 256;
        u_at[i] = poff;
        poff += ((ns * nu * 8 + 255) / 256) * 256;
        piv_at[i] = ipoff;
        ipoff += 2 * ns;
      }
      P.b_count = boff - P.b_off;
      P.p_bytes = poff - P.p_off;
      P.c_bytes = coff;
      // region levels (above the deepest HSS level) allocate update blocks
      // per front; the static arenas only serve the levels below
      if (D.region_level < 0 || L >= D.region_level) cmax[L % 2] = std::max(cmax[L % 2], coff);
    }
    // dense-front id lists (static plan)
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      P.dids_off = (int)ids.size();
      for (int i : lv[L])
        if (!D.want_hss[i]) ids.push_back(i);
      P.ndf = (int)ids.size() - P.dids_off;
    }
    for (int c : D.boundary) {  // imported forward contributions of remote children
      D.bupd_off[c] = boff;
      boff += D.t.nodes[c].nu();
    }
    D.bupd_total = boff;
    t_an[2] = now_s();
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
      h.hss = D.want_hss[i];
      h.ldu = h.ns;
      h.ldc = h.nu;
      const bool store = D.owned[i] && !D.want_hss[i];
      h.P = store ? D.persist.as<double>(p_at[i]) : nullptr;
      h.U = store ? D.persist.as<double>(u_at[i]) : nullptr;
      const bool region = D.region_level >= 0 &&
                          (f.level < D.region_level || (f.level == D.region_level && D.want_hss[i]));
      h.C = (region || !D.owned[i]) ? nullptr : D.trans[f.level % 2].as<double>(c_at[i]);
      h.piv = store ? D.ipersist.as<int>() + piv_at[i] : nullptr;
      h.perm = h.piv ? h.piv + h.ns : nullptr;
      h.upd = D.d_upd.as<int>() + upd_off[i];
      h.pos0 = pos_off0[i] >= 0 ? D.d_pos.as<int>() + pos_off0[i] : nullptr;
      h.pos1 = pos_off1[i] >= 0 ? D.d_pos.as<int>() + pos_off1[i] : nullptr;
    }
    D.hf0 = D.hf;
    D.d_fronts.alloc(nn * sizeof(FrontDev));
    D.set_bupd_capacity(1);

    // extend-add column prefixes (dense fronts) and GEMM batches
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
      b.flops = gemm_flops(probs);
      b.ab_bytes = gemm_ab_bytes(probs);
      b.c_elems = gemm_c_elems(probs);
      gp.insert(gp.end(), probs.begin(), probs.end());
      gpre.insert(gpre.end(), pre.begin(), pre.end());
      return b;
    };
    t_an[3] = now_s();
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      std::vector<int> dl;
      for (int i : lv[L])
        if (!D.want_hss[i]) dl.push_back(i);
      int dmax_ns = 0;
      // K_ASM algorithmic bytes: the zeroing memsets of the level (bracketed
      // with the kernel) write p_bytes + c_bytes; each owned CSR entry reads
      // val + ind (12 B) and read-modify-writes its front element (16 B)
      // (ownership rule for_front_entries, multifrontal.hpp:99-119)
      P.bytes_asm = (double)P.p_bytes + (double)P.c_bytes;
      for (int i : dl) {
        dmax_ns = std::max(dmax_ns, D.hf[i].ns);
        const auto& f = D.t.nodes[i];
        long long ent = 0;
        for (int g = f.sep_begin; g < f.sep_end; g++)
          ent += a.ptr[g + 1] - (std::lower_bound(a.ind.begin() + a.ptr[g], a.ind.begin() + a.ptr[g + 1],
                                                  f.sep_begin) - a.ind.begin());
        for (int g : f.upd) {
          auto b0 = a.ind.begin() + a.ptr[g], b1 = a.ind.begin() + a.ptr[g + 1];
          ent += std::lower_bound(b0, b1, f.sep_end) - std::lower_bound(b0, b1, f.sep_begin);
        }
        P.bytes_asm += 28.0 * (double)ent;
      }
      for (int slot = 0; slot < 2; slot++) {
        P.colpre_off[slot] = colpre.size();
        long long acc = 0;
        for (int i : dl) {
          colpre.push_back(acc);
          const auto& f = D.t.nodes[i];
          const int c = slot ? f.child1 : f.child0;
          if (c >= 0) {
            const long long nuc = D.t.nodes[c].nu();
            acc += nuc;
            // read cb 8 + read-modify-write the parent 16 + map 4
            P.bytes_ea[slot] += 24.0 * nuc * nuc + 4.0 * nuc;
          }
        }
        colpre.push_back(acc);
        P.ncols[slot] = acc;
      }
      for (int i : lv[L])
        for (int slot = 0; slot < 2; slot++) {
          const int c = slot ? D.t.nodes[i].child1 : D.t.nodes[i].child0;
          if (c >= 0) P.max_child_nu[slot] = std::max(P.max_child_nu[slot], D.t.nodes[c].nu());
        }
      for (int k = 0; k < dmax_ns; k += NB) {
        StepBatch sb;
        sb.k = k;
        std::vector<GemmProblem> probs;
        for (int i : dl) {
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
        sb.flops = gemm_flops(probs);
        sb.trail = add_batch(probs);
        P.steps.push_back(sb);
      }
      std::vector<GemmProblem> probs;
      for (int i : dl) {
        const auto& h = D.hf[i];
        if (h.ns && h.nu)  // C -= L21 U12 (Schur complement, multifrontal.hpp:340-344)
          probs.push_back({h.P + h.ns, h.U, h.C, h.nu, h.nu, h.ns, h.m, h.ldu, h.ldc});
      }
      P.flops_schur = gemm_flops(probs);
      P.schur = add_batch(probs);
    }
    t_an[4] = now_s();
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
    D.hss.clear();
    D.hss.resize(nn);
    D.hss_rounds.assign(nn, 0);
    D.hss_dfinal.assign(nn, 0);

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
    if (getenv("HSSMF_DEBUG_AN")) {
      const double t1 = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
      fprintf(stderr, "[hssmf] analyze (device storage %.1f GB): %.3f s = copies + maps %.3f, layout %.3f, "
                      "allocation %.3f, level plans %.3f, uploads + stats %.3f\n",
              devmem_bytes_public() / 1e9, t1 - t_an0, t_an[1] - t_an[0], t_an[2] - t_an[1],
              t_an[3] - t_an[2], t_an[4] - t_an[3], t1 - t_an[4]);
    }
  }

  void Engine::set_values(const double* val, bool on_device) {
    auto& D = *d_;
    HSSMF_CUDA(cudaMemcpyAsync(D.d_val.p, val, D.nnz * sizeof(double),
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               stream_));
    factored_ = false;
  }

  // assembly of front i into the storage named by view (assemble_dense
  // semantics, multifrontal.hpp:141-170: sparse entries, then child0, child1
  // extend-add) on stream st; the caller has zeroed the target
  void Engine::Impl::assemble_on(int i, const FrontDev& view, cudaStream_t st) {
    const auto& fn = t.nodes[i];
    hf[i] = view;
    upload_front_on(i, st);
    long long cp[4] = {0, fn.child0 >= 0 ? t.nodes[fn.child0].nu() : 0, 0,
                       fn.child1 >= 0 ? t.nodes[fn.child1].nu() : 0};
    char* d = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&d, 64, st));
    int* did = reinterpret_cast<int*>(d + 32);
    long long* dcp = reinterpret_cast<long long*>(d);
    HSSMF_CUDA(cudaMemcpyAsync(dcp, cp, sizeof(cp), cudaMemcpyHostToDevice, st));
    HSSMF_CUDA(cudaMemcpyAsync(did, &i, sizeof(int), cudaMemcpyHostToDevice, st));
    const FrontDev* Fd = d_fronts.as<FrontDev>();
    DenseKernels::assemble_sparse(Fd, did, 1, d_ptr.as<int>(), d_ind.as<int>(), d_val.as<double>(), st);
    DenseKernels::extend_add(Fd, did, 1, 0, dcp, cp[1], st);
    DenseKernels::extend_add(Fd, did, 1, 1, dcp + 2, cp[3], st);
    HSSMF_CUDA(cudaFreeAsync(d, st));
  }

  // dense assembly of HSS front i in HBM on stream st; returns the m x m front
  double* Engine::Impl::assemble_hss_front(int i, cudaStream_t st) {
    const auto& fn = t.nodes[i];
    const int ns = fn.ns(), nu = fn.nu(), m = ns + nu;
    double* F = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&F, (size_t)m * m * sizeof(double) + 8 + (size_t)ns * 4, st));
    HSSMF_CUDA(cudaMemsetAsync(F, 0, (size_t)m * m * sizeof(double), st));
    FrontDev view = hf0[i];
    view.P = F;
    view.U = F + (size_t)ns * m;
    view.C = F + ns + (size_t)ns * m;
    view.ldu = m;
    view.ldc = m;
    view.perm = reinterpret_cast<int*>(F + (size_t)m * m + 1);  // identity written by assembly
    assemble_on(i, view, st);
    stream_sync(st);
    hf[i] = hf0[i];
    upload_front_on(i, st);
    stream_sync(st);
    return F;
  }

  std::vector<double*> Engine::Impl::assemble_hss_fronts(const std::vector<int>& lst,
                                                         cudaStream_t st) {
    std::vector<double*> F(lst.size(), nullptr);
    if (lst.empty()) return F;
    // ids, then the two slots' child-column prefixes, in one upload
    std::vector<long long> pre0{0}, pre1{0};
    for (size_t q = 0; q < lst.size(); q++) {
      const int i = lst[q];
      const auto& fn = t.nodes[i];
      const int ns = fn.ns(), nu = fn.nu(), m = ns + nu;
      HSSMF_CUDA(cudaMallocAsync((void**)&F[q], (size_t)m * m * sizeof(double) + 8 + (size_t)ns * 4, st));
      HSSMF_CUDA(cudaMemsetAsync(F[q], 0, (size_t)m * m * sizeof(double), st));
      FrontDev view = hf0[i];
      view.P = F[q];
      view.U = F[q] + (size_t)ns * m;
      view.C = F[q] + ns + (size_t)ns * m;
      view.ldu = m;
      view.ldc = m;
      view.perm = reinterpret_cast<int*>(F[q] + (size_t)m * m + 1);  // identity written by assembly
      hf[i] = view;
      upload_front_on(i, st);
      pre0.push_back(pre0.back() + (fn.child0 >= 0 ? t.nodes[fn.child0].nu() : 0));
      pre1.push_back(pre1.back() + (fn.child1 >= 0 ? t.nodes[fn.child1].nu() : 0));
    }
    const int nf = (int)lst.size();
    const size_t bytes = (2 * pre0.size()) * sizeof(long long) + nf * sizeof(int);
    std::vector<char> h(bytes);
    std::memcpy(h.data(), pre0.data(), pre0.size() * sizeof(long long));
    std::memcpy(h.data() + pre0.size() * sizeof(long long), pre1.data(),
                pre1.size() * sizeof(long long));
    std::memcpy(h.data() + 2 * pre0.size() * sizeof(long long), lst.data(), nf * sizeof(int));
    char* d = nullptr;
    HSSMF_CUDA(cudaMallocAsync((void**)&d, bytes, st));
    HSSMF_CUDA(cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, st));
    const long long* d0 = reinterpret_cast<const long long*>(d);
    const long long* d1 = d0 + pre0.size();
    const int* did = reinterpret_cast<const int*>(d + 2 * pre0.size() * sizeof(long long));
    const FrontDev* Fd = d_fronts.as<FrontDev>();
    DenseKernels::assemble_sparse(Fd, did, nf, d_ptr.as<int>(), d_ind.as<int>(), d_val.as<double>(), st);
    DenseKernels::extend_add(Fd, did, nf, 0, d0, pre0.back(), st);
    DenseKernels::extend_add(Fd, did, nf, 1, d1, pre1.back(), st);
    HSSMF_CUDA(cudaFreeAsync(d, st));
    stream_sync(st);  // h and the views are host data of this frame
    for (int i : lst) {
      hf[i] = hf0[i];
      upload_front_on(i, st);
    }
    stream_sync(st);
    return F;
  }

  // compression + ULV + densified update of an assembled HSS front on its own
  // stream (factor_front_hss, multifrontal.hpp:348-377). Runs on a worker
  // thread; the rank-guard fallback (multifrontal.hpp:414-421) factors the
  // assembled front densely in place.
  Engine::Impl::HssResult Engine::Impl::compress_hss_front(int i, double* F, cudaStream_t st,
                                                             int peers) {
    HssResult res;
    const auto& fn = t.nodes[i];
    const int ns = fn.ns(), nu = fn.nu(), m = ns + nu;
    auto tree = front_cluster_tree(fn, opt.leaf);
    std::vector<long long> seeds(m);
    for (int l = 0; l < m; l++) seeds[l] = l < ns ? fn.sep_begin + l : fn.upd[l - ns];
    HssOpts ho;
    ho.eps = opt.eps;
    ho.d0 = std::min(opt.d0, m + opt.p);
    ho.dd = opt.dd;
    ho.p = opt.p;
    ho.max_rank = std::min(opt.resolved_max_rank(t.n), m);
    ho.peers = peers;
    auto H = std::make_unique<HssMatrixDev>(st);
    bool fallback = false;
    // the compression reads the front through TMA-fed GEMMs, which need an
    // even leading dimension: an odd-sized front is compressed from a copy
    // with ld m + 1 (one extra 16 B per element of traffic; the assembled F
    // stays for the rank-guard fallback). Freed on every exit.
    struct Pad {
      double* p = nullptr;
      cudaStream_t st;
      ~Pad() {
        if (p) cudaFreeAsync(p, st);
      }
    } pad{nullptr, st};
    const double* Fc = F;
    long long ldF = m;
    static const bool no_pad = getenv("HSSMF_NO_TMA") != nullptr;
    if ((m & 1) && !no_pad) {
      ldF = m + 1;
      HSSMF_CUDA(cudaMallocAsync((void**)&pad.p, (size_t)ldF * m * sizeof(double), st));
      HSSMF_CUDA(cudaMemcpy2DAsync(pad.p, (size_t)ldF * sizeof(double), F, (size_t)m * sizeof(double),
                                   (size_t)m * sizeof(double), m, cudaMemcpyDeviceToDevice, st));
      Fc = pad.p;
    }
    try {
      H->compress(Fc, ldF, tree, seeds, ho);
      if (nu) H->ulv_partial(hf0[i].C, nu);
      else H->ulv_full();
    } catch (const HssRankError&) {
      fallback = true;
    } catch (const HssSingular& e) {
      HSSMF_CUDA(cudaFreeAsync(F, st));
      res.singular_col = e.column;
      res.msg = e.what();
      return res;
    }
    if (!fallback) {
      H->drop_dense();
      HSSMF_CUDA(cudaFreeAsync(F, st));
      stream_sync(st);
      res.hss = std::move(H);
      return res;
    }
    H.reset();
    res.keep.p = F;
    res.keep.bytes = (size_t)m * m * sizeof(double);
    res.piv.alloc(2 * (size_t)ns * sizeof(int) + 8);
    FrontDev f = hf0[i];
    f.P = F;
    f.U = F + (size_t)ns * m;
    f.C = F + ns + (size_t)ns * m;
    f.ldu = m;
    f.ldc = m;
    f.hss = 0;
    f.piv = res.piv.as<int>();
    f.perm = res.piv.as<int>() + ns;
    auto stt = partial_lu_dynamic({f}, st);
    if (stt[0] >= 0) {
      res.singular_col = stt[0];
      res.msg = "exactly singular, zero pivot column " + std::to_string(stt[0]);
      return res;
    }
    if (nu)
      HSSMF_CUDA(cudaMemcpy2DAsync(hf0[i].C, (size_t)nu * sizeof(double), f.C,
                                   (size_t)m * sizeof(double), (size_t)nu * sizeof(double), nu,
                                   cudaMemcpyDeviceToDevice, st));
    HSSMF_CUDA(cudaStreamSynchronize(st));
    f.C = hf0[i].C;
    f.ldc = nu;
    res.fallback = true;
    res.front = f;
    return res;
  }

  // the HSS fronts of one tree level: serial assembly, concurrent compression
  // on a pool of streams / host threads, serial bookkeeping
  void Engine::Impl::factor_hss_level(const std::vector<int>& lst) {
    if (lst.empty()) return;
    std::vector<double*> F(lst.size());
    F = assemble_hss_fronts(lst, s);
    // fronts of >= 9000 rows saturate the device on their own (the Gram-route
    // trailing updates are full-device, HBM-bound kernels, and concurrent
    // ones starve the 16-CTA cluster panels): at most 6 of them at a time
    // (measured on c5: 4 -> 9.01 s, 6 -> 8.81 s, 8 -> 8.84 s per step)
    int mmax = 0;
    for (int i : lst) mmax = std::max(mmax, t.nodes[i].m());
    static const int small_w = getenv("HSSMF_HSS_STREAMS_SMALL") ? atoi(getenv("HSSMF_HSS_STREAMS_SMALL")) : 8;
    static const int big_w = getenv("HSSMF_HSS_STREAMS_BIG") ? atoi(getenv("HSSMF_HSS_STREAMS_BIG")) : 6;
    size_t width = mmax >= 9000 ? std::min<size_t>(std::max(1, big_w), hstreams.size())
                                : std::min<size_t>(std::max(1, small_w), hstreams.size());
    if (const char* e = getenv("HSSMF_HSS_STREAMS")) width = std::max(1, atoi(e));
    const int nw = (int)std::min<size_t>(lst.size(), std::min(width, hstreams.size()));
    std::vector<HssResult> res(lst.size());
    std::atomic<int> next{0};
    int dev = 0;
    HSSMF_CUDA(cudaGetDevice(&dev));
    static const bool dbg = getenv("HSSMF_DEBUG") != nullptr;
    auto now = [] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t0 = now();
    std::vector<double> tq(lst.size()), tw(lst.size()), tstart(lst.size());
    std::vector<long long> nw_(lst.size());
    // admission: a front starts only while the device pool is below the
    // budget, unless nothing else runs (the rest is caught by the retry below)
    cudaMemPool_t pool;
    HSSMF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    size_t dfree = 0, dtotal = 0;
    HSSMF_CUDA(cudaMemGetInfo(&dfree, &dtotal));
    // the pool's live bytes plus the engine's own (cudaMalloc) storage
    const size_t budget = (size_t)(0.6 * (double)dtotal), fixed = devmem_bytes();
    std::atomic<int> running{0};
    // largest fronts first, so that the longest compressions start at once
    std::vector<int> order(lst.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return t.nodes[lst[a]].m() > t.nodes[lst[b]].m(); });
    auto work = [&](int w) {
      cudaSetDevice(dev);
      for (int qi = next++; qi < (int)lst.size(); qi = next++) {
        const int q = order[qi];
        for (;;) {
          size_t used = 0;
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
          if (running.load() == 0 || used + fixed < budget) break;
          std::this_thread::sleep_for(std::chrono::milliseconds(2));
        }
        running++;
        const double a = now();
        tstart[q] = a - t0;
        const SyncClock c0 = sync_clock();
        try {
          res[q] = compress_hss_front(lst[q], F[q], hstreams[w], (int)lst.size());
        } catch (const CudaError& e) {
          // the front's own buffers are released on unwinding; its assembled
          // dense front F is read-only in the HSS path, so it is retried alone
          // once the concurrent fronts are done
          res[q] = HssResult{};
          if (strstr(e.what(), "out of memory")) res[q].oom = true;
          else res[q].error = e.what();
        } catch (const std::exception& e) {
          res[q].error = e.what();
        }
        running--;
        tq[q] = now() - a;
        tw[q] = sync_clock().wait_s - c0.wait_s;
        nw_[q] = sync_clock().n - c0.n;
      }
    };
    if (nw <= 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int w = 0; w < nw; w++) th.emplace_back(work, w);
      for (auto& x : th) x.join();
    }
    for (size_t q = 0; q < lst.size(); q++) {
      if (!res[q].oom) continue;
      for (auto st : hstreams) stream_sync(st);
      if (dbg) fprintf(stderr, "[hssmf]   front %d: out of memory concurrently, retried alone\n", lst[q]);
      const double a = now();
      try {
        res[q] = compress_hss_front(lst[q], F[q], hstreams[0], 1);
      } catch (const std::exception& e) {
        res[q].error = e.what();
      }
      tq[q] = now() - a;
    }
    if (dbg) {
      cudaMemPool_t mp;
      size_t used = 0, high = 0;
      if (cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
        cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemCurrent, &used);
        cudaMemPoolGetAttribute(mp, cudaMemPoolAttrUsedMemHigh, &high);
      }
      fprintf(stderr, "[hssmf] level: %zu HSS fronts, wall %.3f s, pool used %.1f GB (high %.1f GB)\n",
              lst.size(), now() - t0, used / 1e9, high / 1e9);
      for (size_t q = 0; q < lst.size(); q++) {
        const auto& fn = t.nodes[lst[q]];
        fprintf(stderr, "[hssmf]   front %d m=%d ns=%d  start %.3f s, %.3f s (sync wait %.3f s in %lld, arena %.0f MB) rounds=%d d=%d rank=%d |",
                lst[q], fn.m(), fn.ns(), tstart[q], tq[q], tw[q], nw_[q],
                res[q].hss ? res[q].hss->arena_bytes() / 1e6 : 0.0, res[q].hss ? res[q].hss->rounds() : -1,
                res[q].hss ? res[q].hss->d_final() : -1, res[q].hss ? res[q].hss->hss_rank() : -1);
        if (res[q].hss) {
          auto ps = res[q].hss->phase_stats();
          for (int p = 0; p < kHssPhases; p++) fprintf(stderr, " %.0f", ps[p].ms);
          fprintf(stderr, " | host");
          for (int p = 0; p < kHssPhases; p++) fprintf(stderr, " %.0f", ps[p].host_ms);
          // phase_stats drains the event list: re-add so profiling still sees it
          res[q].hss->restore_phase_stats(ps);
        }
        fprintf(stderr, "\n");
      }
    }
    for (size_t q = 0; q < lst.size(); q++) {
      const int i = lst[q];
      auto& r = res[q];
      if (!r.error.empty()) throw CudaError("hss front " + std::to_string(i) + ": " + r.error);
      if (r.singular_col >= 0)
        throw SolverFailure(3, i, r.singular_col, "front " + std::to_string(i) + ": " + r.msg);
      if (r.hss) {
        r.hss->set_stream(s);
        hss[i] = std::move(r.hss);
        hf[i] = hf0[i];
        hf[i].hss = 1;
      } else {
        hf[i] = r.front;
        fallback_mem.push_back(std::move(r.keep));
        fallback_mem.push_back(std::move(r.piv));
      }
      upload_front(i);
    }
  }


  // Dependency-driven factorization of the region R: the HSS fronts of the
  // deepest HSS level and every front above it. A front starts on one of the
  // worker streams as soon as both children are done (no level barrier);
  // ready fronts are taken by their remaining critical path (sum of m^2 up to
  // the root). Update blocks of region fronts are pool allocations freed once
  // the parent has assembled them. Dense region fronts are assembled into
  // their persistent storage and factored by the dynamic partial LU.
  void Engine::Impl::factor_region(const std::vector<int>& R) {
    const int nn = (int)t.nodes.size();
    if (R.empty()) return;
    std::vector<char> inr(nn, 0);
    for (int i : R) inr[i] = 1;
    std::vector<int> pend(nn, 0);
    std::vector<double> cpath(nn, 0.0);
    for (int i = nn - 1; i >= 0; i--) {  // parents have larger ids (postorder)
      const auto& f = t.nodes[i];
      cpath[i] = (double)f.m() * f.m() + (f.parent >= 0 ? cpath[f.parent] : 0.0);
    }
    std::vector<int> ready;
    for (int i : R) {
      const auto& f = t.nodes[i];
      for (int c : {f.child0, f.child1})
        if (c >= 0 && inr[c]) pend[i]++;
      if (!pend[i]) ready.push_back(i);
    }
    region_c.assign(nn, nullptr);
    std::vector<HssResult> res(nn);
    std::vector<int> singular(nn, -1);
    std::vector<double> tq(nn, 0.0), tw(nn, 0.0), ts(nn, 0.0), peak(nn, 0.0);
    std::mutex mu;
    std::condition_variable cv;
    int remaining = (int)R.size();
    bool abort = false;
    std::string err;
    int dev = 0;
    HSSMF_CUDA(cudaGetDevice(&dev));
    size_t width = hstreams.size();
    if (const char* e = getenv("HSSMF_HSS_STREAMS")) width = std::max(1, atoi(e));
    const int nw = (int)std::min<size_t>(R.size(), std::min(width, hstreams.size()));
    cudaMemPool_t pool;
    HSSMF_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    size_t dfree = 0, dtotal = 0;
    HSSMF_CUDA(cudaMemGetInfo(&dfree, &dtotal));
    // admission by estimated peak: an HSS front holds its dense m x m front
    // plus samples, Gram matrices and per-node bases, up to about 5.5 m^2
    // doubles (C5, m = 16k: 11 GB); a dense region front its nu x nu block.
    // Running fronts are charged their full estimate on top of the pool's
    // current use (conservative: their allocations are counted twice).
    const size_t budget = (size_t)(0.92 * (double)dtotal), fixed = devmem_bytes();
    // peak per HSS front measured on C5 (serial debug runs): 4..8.6 m^2
    // doubles including the dense front and the update block
    auto est = [&](int i) {
      const auto& f = t.nodes[i];
      const double m = f.m(), nu = f.nu();
      return (long long)(want_hss[i] ? 56.0 * m * m : 8.0 * nu * nu);
    };
    // what a running front already holds: its dense front, update block and
    // everything its HSS arenas handed out (metered)
    std::unique_ptr<std::atomic<long long>[]> meter(new std::atomic<long long>[nn]);
    for (int i = 0; i < nn; i++) meter[i] = 0;
    auto fixed_part = [&](int i) {
      const auto& f = t.nodes[i];
      const double m = f.m(), nu = f.nu();
      return (long long)((want_hss[i] ? 8.0 * m * m : 0.0) + 8.0 * nu * nu);
    };
    std::vector<char> isrun(nn, 0);
    std::atomic<int> running{0};
    std::atomic<long long> charged{0};
    std::atomic<bool> exclusive{false};
    static const bool dbg = getenv("HSSMF_DEBUG") != nullptr;
    auto now = [] {
      return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
    };
    const double t0 = now();

    // one front on stream st; returns after its results are on the device
    auto process = [&](int i, cudaStream_t st) {
      const auto& fn = t.nodes[i];
      const int ns = fn.ns(), nu = fn.nu(), m = ns + nu;
      double* C = nullptr;
      if (nu) HSSMF_CUDA(cudaMallocAsync((void**)&C, (size_t)nu * nu * sizeof(double), st));
      // on an exception the front's own blocks go back to the pool (a retry
      // allocates afresh)
      struct Guard {
        double*& c;
        double* f = nullptr;
        cudaStream_t st;
        bool armed = true;
        ~Guard() {
          if (!armed) return;
          if (c) cudaFreeAsync(c, st);
          if (f) cudaFreeAsync(f, st);
          c = nullptr;
        }
      } guard{C, nullptr, st};
      if (want_hss[i]) {
        hf0[i].C = C;
        hf0[i].ldc = nu;
        double* F = assemble_hss_front(i, st);
        guard.f = F;
        HssResult r = compress_hss_front(i, F, st);
        guard.f = nullptr;  // compress_hss_front owns F from here on
        if (r.hss) {
          r.hss->set_stream(s);
          hss[i] = std::move(r.hss);
          hf[i] = hf0[i];
          hf[i].hss = 1;
        } else if (r.singular_col < 0) {
          hf[i] = r.front;  // rank-guard fallback (C = the region block)
        }
        singular[i] = r.singular_col;
        res[i] = std::move(r);
      } else {
        FrontDev f = hf0[i];
        f.C = C;
        f.ldc = nu;
        HSSMF_CUDA(cudaMemsetAsync(f.P, 0, (size_t)m * ns * sizeof(double), st));
        if (nu) {
          HSSMF_CUDA(cudaMemsetAsync(f.U, 0, (size_t)ns * nu * sizeof(double), st));
          HSSMF_CUDA(cudaMemsetAsync(C, 0, (size_t)nu * nu * sizeof(double), st));
        }
        assemble_on(i, f, st);
        auto stt = partial_lu_dynamic({f}, st);
        singular[i] = stt[0];
        hf[i] = f;
      }
      upload_front_on(i, st);
      stream_sync(st);
      // the children's update blocks have been assembled: release them
      for (int c : {fn.child0, fn.child1})
        if (c >= 0 && region_c[c]) {
          HSSMF_CUDA(cudaFreeAsync(region_c[c], st));
          region_c[c] = nullptr;
        }
      region_c[i] = C;
      guard.armed = false;
    };

    auto work = [&](int w) {
      cudaSetDevice(dev);
      const cudaStream_t st = hstreams[w];
      for (;;) {
        int i = -1;
        {
          std::unique_lock<std::mutex> lk(mu);
          cv.wait(lk, [&] { return abort || remaining == 0 || !ready.empty(); });
          if (abort || remaining == 0) return;
          auto it = std::max_element(ready.begin(), ready.end(),
                                     [&](int a, int b) { return cpath[a] < cpath[b]; });
          i = *it;
          ready.erase(it);
        }
        // admission: current use + what the running fronts may still
        // allocate + this front's estimated peak fits the budget, or nothing
        // else runs
        const long long ei = est(i);
        for (;;) {
          size_t used = 0;
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
          long long grow = 0;
          for (int r : R)
            if (isrun[r]) grow += std::max(0LL, est(r) - meter[r].load() - fixed_part(r));
          if (!exclusive && (running.load() == 0 ||
                             (long long)(used + fixed) + grow + ei < (long long)budget))
            break;
          std::this_thread::sleep_for(std::chrono::milliseconds(2));
        }
        running++;
        charged += ei;
        isrun[i] = 1;
        current_meter() = &meter[i];
        const double a = now();
        ts[i] = a;
        size_t used0 = 0;
        if (dbg && nw <= 1) {  // serial debug runs measure each front's peak footprint
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used0);
          size_t zero = 0;
          cudaMemPoolSetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &zero);
        }
        const SyncClock c0 = sync_clock();
        std::string e;
        try {
          try {
            process(i, st);
          } catch (const CudaError& x) {
            if (!strstr(x.what(), "out of memory")) throw;
            if (dbg) {
              size_t used = 0;
              cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
              fprintf(stderr, "[hssmf]   front %d m=%d: out of memory (pool %.1f GB, charged %.1f GB, "
                      "engine %.1f GB, running %d): %s\n", i, t.nodes[i].m(), used / 1e9,
                      charged.load() / 1e9, fixed / 1e9, running.load(), x.what());
            }
            // retry alone: no new front starts, the running ones drain; the
            // pool's idle reserve goes back to the driver (module loads and
            // cudaMalloc cannot use it)
            exclusive = true;
            running--;
            while (running.load() > 0) std::this_thread::sleep_for(std::chrono::milliseconds(2));
            running++;
            for (auto hs : hstreams) stream_sync(hs);
            cudaMemPoolTrimTo(pool, 0);
            if (dbg) fprintf(stderr, "[hssmf]   front %d: out of memory concurrently, retried alone\n", i);
            stream_sync(st);
            process(i, st);
            exclusive = false;
          }
        } catch (const std::exception& x) {
          e = x.what();
          exclusive = false;
        }
        running--;
        charged -= ei;
        isrun[i] = 0;
        current_meter() = nullptr;
        if (dbg && nw <= 1) {
          size_t hi = 0;
          cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &hi);
          peak[i] = (double)(hi > used0 ? hi - used0 : 0);
        }
        tq[i] = now() - a;
        tw[i] = sync_clock().wait_s - c0.wait_s;
        {
          std::lock_guard<std::mutex> lk(mu);
          if (!e.empty()) {
            if (!abort) err = "front " + std::to_string(i) + ": " + e;
            abort = true;
          } else {
            remaining--;
            const int p = t.nodes[i].parent;
            if (p >= 0 && inr[p] && --pend[p] == 0) ready.push_back(p);
          }
        }
        cv.notify_all();
      }
    };
    if (nw <= 1) {
      work(0);
    } else {
      std::vector<std::thread> th;
      for (int w = 0; w < nw; w++) th.emplace_back(work, w);
      for (auto& x : th) x.join();
    }
    for (auto st : hstreams) stream_sync(st);
    if (abort) throw CudaError(err);
    for (int i : R) {
      if (res[i].fallback) {
        fallback_mem.push_back(std::move(res[i].keep));
        fallback_mem.push_back(std::move(res[i].piv));
      }
      if (singular[i] >= 0) region_singular[i] = singular[i];
    }
    if (dbg) {
      size_t used = 0, high = 0;
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemHigh, &high);
      fprintf(stderr, "[hssmf] region: %zu fronts, wall %.3f s, pool used %.1f GB (high %.1f GB)\n",
              R.size(), now() - t0, used / 1e9, high / 1e9);
      for (int i : R) {
        if (!want_hss[i]) continue;
        const auto& fn = t.nodes[i];
        HssMatrixDev* h = hss[i].get();
        fprintf(stderr, "[hssmf]   front %d L%d m=%d ns=%d  start %.3f  %.3f s (sync wait %.3f s, peak %.2f GB = %.2f m^2 doubles) rounds=%d d=%d rank=%d |",
                i, fn.level, fn.m(), fn.ns(), ts[i] - t0, tq[i], tw[i], peak[i] / 1e9,
                peak[i] / (8.0 * fn.m() * (double)fn.m()), h ? h->rounds() : -1,
                h ? h->d_final() : -1, h ? h->hss_rank() : -1);
        if (h) {
          auto ps = h->phase_stats();
          for (int p = 0; p < kHssPhases; p++) fprintf(stderr, " %.0f", ps[p].ms);
          h->restore_phase_stats(ps);
        }
        fprintf(stderr, "\n");
      }
    }
  }

  int Engine::nlevels() const { return (int)d_->levels.size(); }

  void Engine::factor_levels(int lo, int hi) {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    D.profile = profile_;
    hss_set_phase_timing(profile_ || getenv("HSSMF_DEBUG") != nullptr);
    const int nn = (int)D.hf.size();
    const int nlev = (int)D.levels.size();
    lo = std::max(lo, 0);
    hi = std::min(hi, nlev - 1);
    const bool first = hi == nlev - 1;
    if (first) {
      // previous HSS / fallback state is rebuilt
      D.hss.clear();
      D.hss.resize(nn);
      D.fallback_mem.clear();
      D.hf = D.hf0;
      D.upload_fronts();
      D.n_hss = D.n_fallback = D.max_rank = 0;
      D.region_singular.assign(nn, -1);
      HSSMF_CUDA(cudaMemsetAsync(D.status.p, 0xff, nn * sizeof(int), stream_));
      factor_ms_ = 0;
      factored_ = false;
    }
    cudaEvent_t e0, e1;
    HSSMF_CUDA(cudaEventCreate(&e0));
    HSSMF_CUDA(cudaEventCreate(&e1));
    HSSMF_CUDA(cudaEventRecord(e0, stream_));
    const FrontDev* F = D.d_fronts.as<FrontDev>();
    const int Lh = D.region_level;
    for (int L = hi; L >= lo; L--) {
      if (Lh >= 0 && L < Lh) break;
      auto& P = D.levels[L];
      const int* ids = D.d_ids.as<int>() + P.dids_off;
      char rname[48];
      snprintf(rname, sizeof rname, "factor level %d (%d dense, %d hss)", L, P.ndf,
               (int)P.hss.size());
      NvtxRange nv(rname);
      // the level's zeroing is part of assembly: timed in the same bracket
      // as the scatter kernel, whose bytes count it (bytes_asm)
      D.launch(K_ASM, 0, P.bytes_asm, [&] {
        if (P.p_bytes)
          HSSMF_CUDA(cudaMemsetAsync(D.persist.as<char>(P.p_off), 0, P.p_bytes, stream_));
        if (P.c_bytes) HSSMF_CUDA(cudaMemsetAsync(D.trans[L % 2].p, 0, P.c_bytes, stream_));
        if (P.ndf)
          DenseKernels::assemble_sparse(F, ids, P.ndf, D.d_ptr.as<int>(), D.d_ind.as<int>(),
                                        D.d_val.as<double>(), stream_);
      });
      if (P.ndf) {
        for (int slot = 0; slot < 2; slot++)
          D.launch(K_EXTADD, 0, P.bytes_ea[slot], [&] {
            DenseKernels::extend_add(F, ids, P.ndf, slot,
                                     D.d_colpre.as<long long>() + P.colpre_off[slot],
                                     P.ncols[slot], stream_);
          });
        for (auto& sb : P.steps) {
          D.launch(K_PANEL, 0, 0, [&] {
            DenseKernels::lu_panel(F, ids, P.ndf, sb.k, NB, D.status.as<int>(), stream_);
          });
          D.launch(K_TRSM, 0, 0, [&] {
            DenseKernels::l21(F, ids, P.ndf, sb.k, NB, P.max_nu, stream_);
            DenseKernels::swap_trsm(F, ids, P.ndf, sb.k, NB, sb.max_cols, stream_);
          });
          D.launch(K_GEMM_TRAIL, sb.flops, 0,
                   [&] { gemm_run(sb.trail, 'N', 'N', -1.0, 1.0, stream_); });
        }
        D.launch(K_GEMM_SCHUR, P.flops_schur, 0,
                 [&] { gemm_run(P.schur, 'N', 'N', -1.0, 1.0, stream_); });
      }
      if (L == Lh) {
        std::vector<int> R;
        for (int i = 0; i < nn; i++) {
          const int fl = D.t.nodes[i].level;
          if (fl < Lh || (fl == Lh && D.want_hss[i])) R.push_back(i);
        }
        HSSMF_CUDA(cudaStreamSynchronize(stream_));
        D.launch(K_HSS, 0, 0, [&] { D.factor_region(R); });
        double hfl = 0;
        for (int i : R)
          if (D.hss[i]) hfl += D.hss[i]->flops();
        if (profile_ && !D.evs.empty()) D.evs.back().flops = hfl;
      } else if (!P.hss.empty()) {
        HSSMF_CUDA(cudaStreamSynchronize(stream_));
        D.launch(K_HSS, 0, 0, [&] { D.factor_hss_level(P.hss); });
        double hfl = 0;
        for (int i : P.hss)
          if (D.hss[i]) hfl += D.hss[i]->flops();
        if (profile_ && !D.evs.empty()) D.evs.back().flops = hfl;
      }
    }
    HSSMF_CUDA(cudaEventRecord(e1, stream_));
    std::vector<int> st(nn);
    HSSMF_CUDA(cudaMemcpyAsync(st.data(), D.status.p, nn * sizeof(int), cudaMemcpyDeviceToHost,
                               stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
    float ms = 0;
    HSSMF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    factor_ms_ += ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (profile_) {
      D.collect();
      for (auto& h : D.hss) {
        if (!h) continue;
        auto ps = h->phase_stats();
        for (int p = 0; p < kHssPhases; p++) {
          auto& k = D.kstat[K_HSS_PH + p];
          k.launches += ps[p].count;
          k.ms += ps[p].ms;
          k.flops += ps[p].flops;
        }
      }
    }
    // first failure in postorder = the one the sequential reference reports
    for (int i = 0; i < nn; i++) {
      const int col = st[i] >= 0 ? st[i] : D.region_singular[i];
      if (col >= 0)
        throw SolverFailure(3, i, col,
                            "front " + std::to_string(i) +
                                ": exactly singular, zero pivot column " + std::to_string(col));
    }
    // stats (multifrontal.hpp:432-445, 496-500) and the solve lists
    std::vector<int> sids;
    for (int L = nlev - 1; L >= 0; L--) {
      auto& P = D.levels[L];
      P.sids_off = (int)sids.size();
      for (int i : D.lv[L])
        if (!D.hss[i]) sids.push_back(i);
      P.nsf = (int)sids.size() - P.sids_off;
    }
    upload(D.d_sids, sids);
    for (int i = 0; i < nn; i++) {
      auto& s = stats_[i];
      const auto& f = D.t.nodes[i];
      if (D.hss[i]) {
        s.type = 1;
        s.rank = D.hss[i]->hss_rank();
        s.flops = hss_front_flops(f.m(), s.rank, D.hss[i]->d_final());
        D.n_hss++;
      } else {
        s.rank = 0;
        s.type = D.want_hss[i] ? 2 : 0;
        s.flops = dense_front_flops(f.ns(), f.nu());
        if (D.want_hss[i]) D.n_fallback++;
      }
      D.max_rank = std::max(D.max_rank, s.rank);
    }
    factored_ = lo == 0;
  }

  void Engine::export_update(int f, double* dst, bool on_device) const {
    const auto& D = *d_;
    const int nu = D.t.nodes[f].nu();
    const FrontDev& h = D.hf[f];
    if (!nu) return;
    if (!h.C) throw SolverFailure(2, f, -1, "export_update: front has no update block here");
    HSSMF_CUDA(cudaMemcpy2DAsync(dst, (size_t)nu * sizeof(double), h.C, (size_t)h.ldc * sizeof(double),
                                 (size_t)nu * sizeof(double), nu,
                                 on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
  }

  void Engine::import_update(int f, const double* src, bool on_device) {
    auto& D = *d_;
    const int nu = D.t.nodes[f].nu();
    if (!nu) return;
    auto& m = D.imported[f];
    if (m.bytes < (size_t)nu * nu * sizeof(double)) m.alloc((size_t)nu * nu * sizeof(double));
    HSSMF_CUDA(cudaMemcpyAsync(m.p, src, (size_t)nu * nu * sizeof(double),
                               on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream_));
    D.hf[f].C = m.as<double>();
    D.hf[f].ldc = nu;
    D.upload_front(f);  // synchronises the stream
  }

  void Engine::export_bupd(int f, double* dst, int nrhs) const {
    const auto& D = *d_;
    const int nu = D.t.nodes[f].nu();
    if (!nu || nrhs <= 0) return;
    HSSMF_CUDA(cudaMemcpyAsync(dst, D.hf[f].bupd, (size_t)nu * nrhs * sizeof(double),
                               cudaMemcpyDeviceToDevice, stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
  }

  void Engine::import_bupd(int f, const double* src, int nrhs) {
    auto& D = *d_;
    const int nu = D.t.nodes[f].nu();
    if (!nu || nrhs <= 0) return;
    if (nrhs > D.bupd_nr) D.set_bupd_capacity(nrhs);
    HSSMF_CUDA(cudaMemcpyAsync(D.hf[f].bupd, src, (size_t)nu * nrhs * sizeof(double),
                               cudaMemcpyDeviceToDevice, stream_));
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
  }

  void Engine::solve(double* b, int ldb, int nrhs, bool on_device) {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    if (!factored_) throw SolverFailure(2, -1, -1, "mf solve: not factored");
    if (nrhs <= 0) return;
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
    const int nlev = (int)D.levels.size();
    solve_levels(x, ldx, nrhs, 0, nlev - 1, true);
    solve_levels(x, ldx, nrhs, 0, nlev - 1, false);
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

  void Engine::solve_levels(double* x, int ldx, int nrhs, int lo, int hi, bool forward) {
    HSSMF_CUDA(cudaSetDevice(device_));
    auto& D = *d_;
    if (nrhs <= 0) return;
    D.profile = profile_;
    if (nrhs > D.bupd_nr) D.set_bupd_capacity(nrhs);
    size_t max_nu = 0;
    for (const auto& P : D.levels) {
      size_t sum = 0;
      for (int i : P.hss) sum += D.t.nodes[i].nu();
      max_nu = std::max(max_nu, sum);
    }
    for (const auto& f : D.t.nodes) max_nu = std::max(max_nu, (size_t)f.nu());
    if (D.x2buf.bytes < max_nu * sizeof(double) + 8)
      D.x2buf.alloc(max_nu * sizeof(double) + 8);
    const FrontDev* F = D.d_fronts.as<FrontDev>();
    const int nlev = (int)D.levels.size();
    lo = std::max(lo, 0);
    hi = std::min(hi, nlev - 1);
    const int nr = D.bupd_nr;
    NvtxRange nv(forward ? "solve forward" : "solve backward");
    if (forward) {
      // forward sweep, deepest level first (mf_forward, multifrontal.hpp:507-567)
      for (int L = hi; L >= lo; L--) {
        auto& P = D.levels[L];
        const int* ids = D.d_ids.as<int>() + P.ids_off;
        const int* sids = D.d_sids.as<int>() + P.sids_off;
        if (P.b_count)
          HSSMF_CUDA(cudaMemsetAsync(D.bupd.as<double>() + P.b_off * nr, 0,
                                     P.b_count * nr * sizeof(double), stream_));
        D.launch(K_SOLVE_FWD, 0, 0, [&] {
          for (int slot = 0; slot < 2; slot++)
            DenseKernels::fold_children(F, ids, P.nf, slot, x, ldx, nrhs, P.max_child_nu[slot],
                                        stream_);
          if (P.nsf) {
            DenseKernels::fwd_trsv(F, sids, P.nsf, x, ldx, nrhs, P.max_ns, stream_);
            DenseKernels::fwd_gemv(F, sids, P.nsf, x, ldx, nrhs, P.max_nu, stream_);
          }
          D.hss_level_concurrent(P.hss, stream_, [&](int i) {
            const auto& h = D.hf[i];
            for (int r = 0; r < nrhs; r++) {
              double* xr = x + (size_t)r * ldx + h.sep_begin;
              if (h.nu) D.hss[i]->partial_forward(xr, h.bupd + (size_t)r * h.nu);
              else D.hss[i]->solve_full(xr);
            }
          });
        });
      }
    } else {
      // backward sweep, root first (mf_backward, multifrontal.hpp:569-607)
      for (int L = lo; L <= hi; L++) {
        auto& P = D.levels[L];
        const int* sids = D.d_sids.as<int>() + P.sids_off;
        D.launch(K_SOLVE_BWD, 0, 0, [&] {
          if (P.nsf) {
            DenseKernels::bwd_gemv(F, sids, P.nsf, x, ldx, nrhs, P.max_ns, stream_);
            DenseKernels::bwd_trsv(F, sids, P.nsf, x, ldx, nrhs, P.max_ns, stream_);
          }
          // x(upd) of every front of the level into its own slice of x2buf
          std::vector<size_t> x2off(D.t.nodes.size(), 0);
          size_t o2 = 0;
          for (int i : P.hss) {
            x2off[i] = o2;
            o2 += D.t.nodes[i].nu();
          }
          D.hss_level_concurrent(P.hss, stream_, [&](int i) {
            const auto& h = D.hf[i];
            if (!h.nu) return;
            double* x2 = D.x2buf.as<double>() + x2off[i];
            for (int r = 0; r < nrhs; r++) {
              double* xr = x + (size_t)r * ldx;
              CopyDesc g{xr, 1, 0, h.upd, nullptr, 0, 0, x2, h.nu, nullptr,
                         nullptr, 0, 0, h.nu, 1, 1.0, 0, 0};
              index_copy_run({g}, D.solve_stream_of(i));
              D.hss[i]->partial_backward(xr + h.sep_begin, x2);
            }
          });
        });
      }
    }
    HSSMF_CUDA(cudaStreamSynchronize(stream_));
  }

  long long Engine::factor_nnz() const {
    long long s = 0;
    const auto& D = *d_;
    for (size_t i = 0; i < D.t.nodes.size(); i++) {
      const auto& f = D.t.nodes[i];
      if (i < D.hss.size() && D.hss[i]) {
        s += D.hss[i]->stored_scalars();
        s += 2LL * f.nu() * D.hss[i]->hss_rank();  // Theta, Phi
      } else {
        s += (long long)f.ns() * f.ns() + 2LL * f.ns() * f.nu();
      }
    }
    return s;
  }
  int Engine::hss_fronts() const { return d_->n_hss; }
  int Engine::fallbacks() const { return d_->n_fallback; }
  int Engine::max_front_rank() const { return d_->max_rank; }
  bool Engine::front_hss(int f, std::vector<int>& u, std::vector<int>& v, int& rounds,
                         int& d_final) const {
    if (f < 0 || f >= (int)d_->hss.size() || !d_->hss[f]) return false;
    d_->hss[f]->ranks(u, v);
    rounds = d_->hss[f]->rounds();
    d_final = d_->hss[f]->d_final();
    return true;
  }
  std::vector<KernelStat> Engine::kernel_stats() const {
    return std::vector<KernelStat>(d_->kstat, d_->kstat + K_NCLASS);
  }
  void Engine::reset_kernel_stats() {
    for (auto& k : d_->kstat) {
      k.launches = 0;
      k.ms = k.flops = k.bytes = 0;
    }
  }
  size_t Engine::Impl::devmem_bytes() const {
    size_t b = persist.bytes + ipersist.bytes + trans[0].bytes + trans[1].bytes + bupd.bytes +
               d_val.bytes + d_ind.bytes + d_ptr.bytes + d_gemm.bytes;
    for (auto& m : fallback_mem) b += m.bytes;
    return b;
  }
  size_t Engine::device_bytes() const { return d_->devmem_bytes(); }

}  // namespace hssmf_b200
