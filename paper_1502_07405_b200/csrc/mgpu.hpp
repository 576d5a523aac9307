// Subtree-partitioned multi-GPU factorization / solve (mgpu.cu).
#pragma once

#include <deque>
#include <map>
#include <utility>
#include <vector>

#include "engine.hpp"

namespace hssmf_b200 {

  struct MgpuEdge {
    int child, parent, src, dst, nu, plevel;  // src = owner of child, dst = owner of parent
  };
  struct MgpuPlan {
    int nranks = 1, L = 0, nlev = 0;
    std::vector<int> owner;  // per front
    std::vector<int> roots;  // subtree root per rank
    std::vector<MgpuEdge> edges;  // exchange order
  };
  MgpuPlan mgpu_partition(const Etree& t, int nranks);

  // point-to-point transport of device buffers (blocking: a sent buffer may
  // be reused on return, a received one holds the data on return)
  struct MgpuTransport {
    virtual ~MgpuTransport() = default;
    virtual void send(const double* buf, long long count, int dst, int src) = 0;
    virtual void recv(double* buf, long long count, int src, int dst) = 0;
  };
  // all ranks in one process: FIFO per (src, dst) of device copies
  class LocalTransport : public MgpuTransport {
   public:
    ~LocalTransport() override;
    void send(const double* buf, long long count, int dst, int src) override;
    void recv(double* buf, long long count, int src, int dst) override;

   private:
    struct Msg {
      double* p = nullptr;
      long long n = 0;
    };
    std::map<std::pair<int, int>, std::deque<Msg>> q_;
  };

  // engines: the ranks living in this process (each analysed with its
  // ownership mask); x: per rank, a device n x nrhs block solved in place
  void mgpu_factor(const MgpuPlan& P, std::map<int, Engine*>& eng, MgpuTransport& tr);
  void mgpu_solve(const MgpuPlan& P, const Etree& t, std::map<int, Engine*>& eng,
                  std::map<int, double*>& x, int ldx, int nrhs, MgpuTransport& tr);

}  // namespace hssmf_b200
