#include <stdexcept>

#include "hss_dense.hpp"

namespace hssmf_b200 {
  struct DenseHss::Impl {};
  DenseHss::DenseHss(int) : d_(new Impl) {}
  DenseHss::~DenseHss() = default;
  void DenseHss::run(const double*, int, int, int, double, int, int, int, int, bool) {
    throw std::runtime_error("dense HSS: not built yet");
  }
  void DenseHss::solve(double*, int, int, bool) { throw std::runtime_error("dense HSS: not built yet"); }
  void DenseHss::ranks(std::vector<int>&, std::vector<int>&) const {}
  int DenseHss::rounds() const { return 0; }
  int DenseHss::d_final() const { return 0; }
  double DenseHss::compress_ms() const { return 0; }
  double DenseHss::ulv_ms() const { return 0; }
}  // namespace hssmf_b200
