// ORACLE — test infrastructure only. Not part of the product.
//
// The one semantics-preserving shim applied to the reference (see
// ref_driver.cpp's header): an explicit specialization of
// LowRankSchur<double>::extract (reference hss_ulv.hpp:46-60) that sorts the
// requested index lists before the reference's own HssMatrix::extract and
// scatters the block back. Included before multifrontal.hpp by every program
// that instantiates the reference's mf_factor (oracle/ref_driver.cpp,
// tests/cpp/wrapper_check.cpp).
#pragma once

#include <algorithm>
#include <numeric>
#include <vector>

#include "hssmf/hss_ulv.hpp"

namespace hssmf {
  template<>
  DenseMatrix<double> LowRankSchur<double>::extract(const HssMatrix<double>& hss,
                                                    const std::vector<int>& i,
                                                    const std::vector<int>& j) const {
    std::vector<int> pi(i.size()), pj(j.size());
    std::iota(pi.begin(), pi.end(), 0);
    std::iota(pj.begin(), pj.end(), 0);
    std::stable_sort(pi.begin(), pi.end(), [&](int a, int b) { return i[a] < i[b]; });
    std::stable_sort(pj.begin(), pj.end(), [&](int a, int b) { return j[a] < j[b]; });
    std::vector<int> si(i.size()), sj(j.size());
    for (std::size_t x = 0; x < i.size(); x++) si[x] = i[pi[x]];
    for (std::size_t y = 0; y < j.size(); y++) sj[y] = j[pj[y]];
    const int c1 = hss.tree().root().child1;
    auto sorted = hss.extract(si, sj, c1);
    const int r = rank();
    DenseMatrix<double> out(i.size(), j.size());
    for (std::size_t y = 0; y < j.size(); y++)
      for (std::size_t x = 0; x < i.size(); x++) {
        double s = 0;
        for (int l = 0; l < r; l++) s += theta(l, si[x]) * phi(l, sj[y]);
        out(pi[x], pj[y]) = sorted(x, y) - s;
      }
    return out;
  }
}
