// Equilibration + static pivoting and Matrix Market I/O on the host (SURVEY
// §8f row 3). Bit-exact with the reference's
//   equilibrate_and_permute   scaling.hpp:40-139
//   read/write_matrix_market  matrix_market.cpp:10-77
//   from_triplets / col_permuted  sparse_matrix.hpp:25-47, 104-124
// (pinned by tests/test_scaling_io.py against oracle/_ref): the same
// floating-point operations in the same order, so the scaled matrix, the
// scaling vectors and the matching are identical bit for bit.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <tuple>

#include "analysis.hpp"

namespace hssmf_b200 {

  Csr csr_from_triplets(int n, std::vector<std::tuple<int, int, double>>& t) {
    std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
      return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                              : std::get<1>(a) < std::get<1>(b);
    });
    Csr m;
    m.n = n;
    m.ptr.assign(n + 1, 0);
    m.ind.reserve(t.size());
    m.val.reserve(t.size());
    size_t k = 0;
    while (k < t.size()) {
      const int i = std::get<0>(t[k]), j = std::get<1>(t[k]);
      double v = 0.0;  // duplicates summed in sorted order
      for (; k < t.size() && std::get<0>(t[k]) == i && std::get<1>(t[k]) == j; k++)
        v += std::get<2>(t[k]);
      m.ind.push_back(j);
      m.val.push_back(v);
      m.ptr[i + 1]++;
    }
    for (int i = 0; i < n; i++) m.ptr[i + 1] += m.ptr[i];
    return m;
  }

  Csr Csr::col_permuted(const std::vector<int>& q) const {
    std::vector<int> inv(n);
    for (int j = 0; j < n; j++) inv[q[j]] = j;
    Csr m;
    m.n = n;
    m.ptr = ptr;
    m.ind.resize(ind.size());
    m.val.resize(val.size());
    std::vector<std::pair<int, double>> row;
    for (int i = 0; i < n; i++) {
      row.clear();
      for (int k = ptr[i]; k < ptr[i + 1]; k++) row.push_back({inv[ind[k]], val[k]});
      std::sort(row.begin(), row.end());
      for (int k = ptr[i]; k < ptr[i + 1]; k++) {
        m.ind[k] = row[k - ptr[i]].first;
        m.val[k] = row[k - ptr[i]].second;
      }
    }
    return m;
  }

  namespace {
    struct Matching {
      const Csr& s;
      std::vector<int> row_to_col, col_to_row, seen;
      // augmenting path from row i0 over nonzero entries (depth first, the
      // entries of a row in CSR order), iterative so deep paths cannot
      // exhaust the stack; same visiting order as the recursive search
      bool augment(int i0, int stamp) {
        struct Frame { int i, k; };
        std::vector<Frame> st{{i0, s.ptr[i0]}};
        while (!st.empty()) {
          Frame& f = st.back();
          bool descended = false;
          for (; f.k < s.ptr[f.i + 1]; f.k++) {
            const int j = s.ind[f.k];
            if (s.val[f.k] == 0.0 || seen[j] == stamp) continue;
            seen[j] = stamp;
            if (col_to_row[j] < 0) {
              // free column: flip the path
              for (auto it = st.rbegin(); it != st.rend(); ++it) {
                const int c = s.ind[it->k];
                row_to_col[it->i] = c;
                col_to_row[c] = it->i;
              }
              return true;
            }
            st.push_back({col_to_row[j], s.ptr[col_to_row[j]]});
            descended = true;
            break;
          }
          if (descended) continue;
          st.pop_back();
          if (!st.empty()) st.back().k++;
        }
        return false;
      }
    };
  }  // namespace

  Csr equilibrate_and_permute(const Csr& a, Scaling& sc) {
    const int n = a.n;
    sc.dr.assign(n, 1.0);
    sc.dc.assign(n, 1.0);
    sc.qc.assign(n, 0);
    sc.sweeps = 0;
    Csr s = a;
    std::vector<double> rmax(n), cmax(n);
    auto in_range = [](double v) { return v >= 0.5 && v <= 2.0; };
    for (int sweep = 0; sweep < 10; sweep++) {
      std::fill(rmax.begin(), rmax.end(), 0.0);
      std::fill(cmax.begin(), cmax.end(), 0.0);
      for (int i = 0; i < n; i++)
        for (int k = s.ptr[i]; k < s.ptr[i + 1]; k++) {
          const double v = std::fabs(s.val[k]);
          rmax[i] = std::max(rmax[i], v);
          cmax[s.ind[k]] = std::max(cmax[s.ind[k]], v);
        }
      bool done = true;
      for (int i = 0; i < n && done; i++) done = in_range(rmax[i]) && in_range(cmax[i]);
      if (done) break;
      sc.sweeps++;
      // rows by their maxima, then columns by the maxima of the row-scaled matrix
      for (int i = 0; i < n; i++) {
        if (rmax[i] == 0.0)
          throw SolverFailure(9, -1, i, "equilibration: row " + std::to_string(i) + " is empty");
        const double f = 1.0 / rmax[i];
        sc.dr[i] *= f;
        for (int k = s.ptr[i]; k < s.ptr[i + 1]; k++) s.val[k] *= f;
      }
      std::fill(cmax.begin(), cmax.end(), 0.0);
      for (int i = 0; i < n; i++)
        for (int k = s.ptr[i]; k < s.ptr[i + 1]; k++)
          cmax[s.ind[k]] = std::max(cmax[s.ind[k]], std::fabs(s.val[k]));
      for (int j = 0; j < n; j++)
        if (cmax[j] == 0.0)
          throw SolverFailure(9, -1, j,
                              "equilibration: column " + std::to_string(j) + " is empty");
      std::vector<double> cf(n);
      for (int j = 0; j < n; j++) cf[j] = 1.0 / cmax[j];
      for (int j = 0; j < n; j++) sc.dc[j] *= cf[j];
      for (int i = 0; i < n; i++)
        for (int k = s.ptr[i]; k < s.ptr[i + 1]; k++) s.val[k] *= cf[s.ind[k]];
    }
    // greedy: every row takes its largest still-free column (first on ties)
    Matching mt{s, std::vector<int>(n, -1), std::vector<int>(n, -1), std::vector<int>(n, -1)};
    for (int i = 0; i < n; i++) {
      int best = -1;
      double bv = -1.0;
      for (int k = s.ptr[i]; k < s.ptr[i + 1]; k++) {
        const int j = s.ind[k];
        if (mt.col_to_row[j] >= 0) continue;
        const double v = std::fabs(s.val[k]);
        if (v > bv) {
          bv = v;
          best = j;
        }
      }
      if (best >= 0 && bv > 0.0) {
        mt.row_to_col[i] = best;
        mt.col_to_row[best] = i;
      }
    }
    for (int i = 0; i < n; i++) {
      if (mt.row_to_col[i] >= 0) continue;
      if (!mt.augment(i, i))
        throw SolverFailure(9, -1, -1,
                            "matching: no zero-free diagonal exists (structurally singular)");
    }
    for (int j = 0; j < n; j++) sc.qc[j] = mt.row_to_col[j];
    return s.col_permuted(sc.qc);
  }

  Csr read_matrix_market(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw SolverFailure(1, -1, -1, "cannot open '" + path + "'");
    auto bad = [&](const std::string& why) { return SolverFailure(1, -1, -1, path + ": " + why); };
    std::string line;
    if (!std::getline(f, line)) throw bad("empty file");
    std::istringstream hdr(line);
    std::string banner, object, format, field, symmetry;
    hdr >> banner >> object >> format >> field >> symmetry;
    for (auto* w : {&object, &format, &field, &symmetry})
      for (auto& c : *w) c = (char)std::tolower((unsigned char)c);
    if (banner != "%%MatrixMarket" || object != "matrix") throw bad("not a MatrixMarket matrix file");
    if (format != "coordinate") throw bad("only coordinate format is supported");
    if (field != "real" && field != "integer") throw bad("unsupported field '" + field + "'");
    const bool sym = symmetry == "symmetric";
    if (!sym && symmetry != "general") throw bad("unsupported symmetry '" + symmetry + "'");
    while (std::getline(f, line))
      if (!line.empty() && line[0] != '%') break;
    std::istringstream sz(line);
    long long rows = -1, cols = -1, nnz = -1;
    sz >> rows >> cols >> nnz;
    if (rows < 0 || cols < 0 || nnz < 0) throw bad("malformed size line");
    if (rows != cols)
      throw bad("matrix must be square (" + std::to_string(rows) + "x" + std::to_string(cols) + ")");
    std::vector<std::tuple<int, int, double>> t;
    t.reserve((size_t)(sym ? 2 * nnz : nnz));
    long long got = 0;
    while (got < nnz && std::getline(f, line)) {
      if (line.empty() || line[0] == '%') continue;
      long long i, j;
      double v;
      if (std::sscanf(line.c_str(), "%lld %lld %lf", &i, &j, &v) != 3)
        throw bad("malformed entry on line '" + line + "'");
      if (i < 1 || i > rows || j < 1 || j > cols)
        throw bad("entry (" + std::to_string(i) + "," + std::to_string(j) + ") out of range");
      t.emplace_back((int)(i - 1), (int)(j - 1), v);
      if (sym && i != j) t.emplace_back((int)(j - 1), (int)(i - 1), v);
      got++;
    }
    if (got != nnz)
      throw bad("expected " + std::to_string(nnz) + " entries, got " + std::to_string(got));
    return csr_from_triplets((int)rows, t);
  }

  void write_matrix_market(const Csr& a, const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    if (!f) throw SolverFailure(1, -1, -1, "cannot open '" + path + "' for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n");
    std::fprintf(f, "%d %d %lld\n", a.n, a.n, (long long)a.nnz());
    for (int i = 0; i < a.n; i++)
      for (int k = a.ptr[i]; k < a.ptr[i + 1]; k++)
        std::fprintf(f, "%d %d %.17g\n", i + 1, a.ind[k] + 1, a.val[k]);
    if (std::fclose(f) != 0) throw SolverFailure(1, -1, -1, "error closing '" + path + "'");
  }

}  // namespace hssmf_b200
