#include "analysis.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>

namespace hssmf_b200 {

  double Csr::get(int i, int j) const {
    auto b = ind.begin() + ptr[i], e = ind.begin() + ptr[i + 1];
    auto it = std::lower_bound(b, e, j);
    return (it != e && *it == j) ? val[it - ind.begin()] : 0.0;
  }

  Csr Csr::permuted(const std::vector<int>& p) const {
    // rows of B are rows p[i] of A re-sorted by permuted column; entries are
    // unique so the (row, col) sort of from_triplets is reproduced exactly
    Csr b;
    b.n = n;
    std::vector<int> inv(n);
    for (int i = 0; i < n; i++) inv[p[i]] = i;
    b.ptr.assign(n + 1, 0);
    b.ind.resize(ind.size());
    b.val.resize(val.size());
    std::vector<std::pair<int, double>> row;
    for (int r = 0; r < n; r++) {
      const int o = inv[r];
      row.clear();
      for (int k = ptr[o]; k < ptr[o + 1]; k++) row.emplace_back(p[ind[k]], val[k]);
      std::sort(row.begin(), row.end(),
                [](const auto& x, const auto& y) { return x.first < y.first; });
      // duplicates (impossible for a valid CSR) would be summed by from_triplets
      int w = b.ptr[r];
      for (std::size_t q = 0; q < row.size(); q++) {
        if (q && row[q].first == row[q - 1].first) {
          b.val[w - 1] += row[q].second;
          continue;
        }
        b.ind[w] = row[q].first;
        b.val[w] = row[q].second;
        w++;
      }
      b.ptr[r + 1] = w;
    }
    b.ind.resize(b.ptr[n]);
    b.val.resize(b.ptr[n]);
    return b;
  }

  void Csr::symmetric_graph(std::vector<int>& gptr, std::vector<int>& gind) const {
    std::vector<int> cnt(n + 1, 0);
    for (int i = 0; i < n; i++)
      for (int k = ptr[i]; k < ptr[i + 1]; k++) {
        const int j = ind[k];
        if (j == i) continue;
        cnt[i + 1]++;
        cnt[j + 1]++;
      }
    for (int i = 0; i < n; i++) cnt[i + 1] += cnt[i];
    std::vector<int> adj(cnt[n]), fill(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < n; i++)
      for (int k = ptr[i]; k < ptr[i + 1]; k++) {
        const int j = ind[k];
        if (j == i) continue;
        adj[fill[i]++] = j;
        adj[fill[j]++] = i;
      }
    gptr.assign(n + 1, 0);
    gind.clear();
    gind.reserve(adj.size());
    for (int i = 0; i < n; i++) {
      auto b = adj.begin() + cnt[i], e = adj.begin() + cnt[i + 1];
      std::sort(b, e);
      e = std::unique(b, e);
      gind.insert(gind.end(), b, e);
      gptr[i + 1] = (int)gind.size();
    }
  }

  namespace {
    inline void upwind(double v, double h, double& diag, double& lo, double& hi) {
      diag += h * std::abs(v);
      lo -= h * std::max(v, 0.0);
      hi += h * std::min(v, 0.0);
    }

    // rows are emitted directly in sorted column order: l-1, j-1, i-1, diag,
    // i+1, j+1, l+1 (ascending for a lexicographic x-fastest grid)
    template<typename Coef>
    Csr stencil(const Geometry& g, bool threed, Coef&& coef) {
      const int kx = g.dims[0], ky = g.dims[1], kz = g.dims[2];
      Csr a;
      a.n = kx * ky * kz;
      a.ptr.assign(a.n + 1, 0);
      a.ind.reserve((std::size_t)a.n * (threed ? 7 : 5));
      a.val.reserve(a.ind.capacity());
      double c[7];  // diag, w, e, s, n, dn, up
      for (int l = 0; l < kz; l++)
        for (int j = 0; j < ky; j++)
          for (int i = 0; i < kx; i++) {
            const int row = g.vertex(i, j, l);
            coef(i, j, l, c);
            auto put = [&](int col, double v) {
              a.ind.push_back(col);
              a.val.push_back(v);
            };
            if (threed && l > 0) put(g.vertex(i, j, l - 1), c[5]);
            if (j > 0) put(g.vertex(i, j - 1, l), c[3]);
            if (i > 0) put(g.vertex(i - 1, j, l), c[1]);
            put(row, c[0]);
            if (i < kx - 1) put(g.vertex(i + 1, j, l), c[2]);
            if (j < ky - 1) put(g.vertex(i, j + 1, l), c[4]);
            if (threed && l < kz - 1) put(g.vertex(i, j, l + 1), c[6]);
            a.ptr[row + 1] = (int)a.ind.size();
          }
      return a;
    }
  }  // namespace

  Csr grid_problem(int kind, int k, double nu, Geometry& g) {
    if (k < 1) throw std::invalid_argument("grid size k must be >= 1");
    const bool threed = kind == P3D || kind == C3D;
    const bool convect = kind == C2D || kind == C3D;
    const int kz = threed ? k : 1;
    g.dims = {k, k, kz};
    g.ndims = threed ? 3 : 2;
    const double h = 1.0 / (k + 1);
    const double dcoef = convect ? nu : 1.0;
    return stencil(g, threed, [&](int i, int j, int l, double* c) {
      const double x = (i + 1) * h, y = (j + 1) * h, z = (l + 1) * h;
      double diag = (threed ? 6.0 : 4.0) * dcoef;
      double w = -dcoef, e = -dcoef, s = -dcoef, n = -dcoef, dn = -dcoef, up = -dcoef;
      if (convect) {
        double vx, vy, vz = 0;
        if (threed) {
          vx = 2 * x * (1 - x) * (2 * y - 1) * z;
          vy = -y * (1 - y) * (2 * x - 1);
          vz = -(2 * x - 1) * (2 * y - 1) * z * (1 - z);
        } else {
          vx = x * (1 - x) * (2 * y - 1);
          vy = y * (1 - y) * (2 * x - 1);
        }
        upwind(vx, h, diag, w, e);
        upwind(vy, h, diag, s, n);
        if (threed) upwind(vz, h, diag, dn, up);
      }
      c[0] = diag; c[1] = w; c[2] = e; c[3] = s; c[4] = n; c[5] = dn; c[6] = up;
    });
  }

  Csr convdiff3d_const(int k, double scale, Geometry& g) {
    g.dims = {k, k, k};
    g.ndims = 3;
    const double h = 1.0 / (k + 1);
    const double bx = scale * 1.0 / h, by = scale * 0.5 / h, bz = scale * 0.25 / h;
    return stencil(g, true, [&](int, int, int, double* c) {
      double diag = 6.0, w = -1, e = -1, s = -1, n = -1, dn = -1, up = -1;
      upwind(bx, h, diag, w, e);
      upwind(by, h, diag, s, n);
      upwind(bz, h, diag, dn, up);
      c[0] = diag; c[1] = w; c[2] = e; c[3] = s; c[4] = n; c[5] = dn; c[6] = up;
    });
  }

  void Etree::compute_levels() {
    if (nodes.empty()) return;
    nodes.back().level = 0;
    for (int i = root(); i >= 0; i--) {
      if (nodes[i].child0 >= 0) nodes[nodes[i].child0].level = nodes[i].level + 1;
      if (nodes[i].child1 >= 0) nodes[nodes[i].child1].level = nodes[i].level + 1;
    }
  }

  namespace {
    struct Nd {
      const Geometry& g;
      int leaf;
      std::vector<int> iperm;
      std::vector<FrontNode> tree;
      int next = 0;

      void emit(const int lo[3], const int sz[3]) {
        for (int l = lo[2]; l < lo[2] + sz[2]; l++)
          for (int j = lo[1]; j < lo[1] + sz[1]; j++)
            for (int i = lo[0]; i < lo[0] + sz[0]; i++) iperm[next++] = g.vertex(i, j, l);
      }
      int push(int b, int c0, int c1) {
        FrontNode f;
        f.sep_begin = b;
        f.sep_end = next;
        f.child0 = c0;
        f.child1 = c1;
        tree.push_back(std::move(f));
        const int id = (int)tree.size() - 1;
        if (c0 >= 0) tree[c0].parent = id;
        if (c1 >= 0) tree[c1].parent = id;
        return id;
      }
      // middle-plane bisection along the longest axis (lowest on ties)
      int rec(const int lo[3], const int sz[3]) {
        const long nv = (long)sz[0] * sz[1] * sz[2];
        int d = 0;
        for (int a = 1; a < g.ndims; a++)
          if (sz[a] > sz[d]) d = a;
        if (nv <= leaf || sz[d] < 3) {
          const int b = next;
          emit(lo, sz);
          return push(b, -1, -1);
        }
        const int m = lo[d] + sz[d] / 2;
        int l1[3] = {lo[0], lo[1], lo[2]}, s1[3] = {sz[0], sz[1], sz[2]};
        s1[d] = sz[d] / 2;
        const int c0 = rec(l1, s1);
        l1[d] = m + 1;
        s1[d] = sz[d] - sz[d] / 2 - 1;
        const int c1 = rec(l1, s1);
        const int b = next;
        l1[d] = m;
        s1[d] = 1;
        emit(l1, s1);
        return push(b, c0, c1);
      }
    };
  }  // namespace

  Etree nested_dissection_geometric(const Geometry& g, int leaf, std::vector<int>& perm) {
    Nd nd{g, std::max(leaf, 1), {}, {}, 0};
    const int n = g.dims[0] * g.dims[1] * g.dims[2];
    nd.iperm.resize(n);
    const int lo[3] = {0, 0, 0};
    nd.rec(lo, g.dims.data());
    perm.assign(n, -1);
    for (int k = 0; k < n; k++) perm[nd.iperm[k]] = k;
    Etree t;
    t.n = n;
    t.nodes = std::move(nd.tree);
    t.compute_levels();
    return t;
  }

  void symbolic_factorization(const Csr& a, Etree& t) {
    std::vector<int> gptr, gind;
    a.symmetric_graph(gptr, gind);
    // postorder ids: children always precede parents, so a forward sweep
    // sees finished children
    std::vector<int> s;
    for (auto& nd : t.nodes) {
      s.clear();
      for (int c = nd.sep_begin; c < nd.sep_end; c++)
        for (int k = gptr[c]; k < gptr[c + 1]; k++)
          if (gind[k] >= nd.sep_end) s.push_back(gind[k]);
      for (int c : {nd.child0, nd.child1}) {
        if (c < 0) continue;
        const auto& u = t.nodes[c].upd;
        s.insert(s.end(), std::lower_bound(u.begin(), u.end(), nd.sep_end), u.end());
      }
      std::sort(s.begin(), s.end());
      s.erase(std::unique(s.begin(), s.end()), s.end());
      nd.upd = s;
    }
  }

  namespace {
    int build_balanced(ClusterTree& t, int b, int e, int leaf) {
      if (e - b <= leaf) {
        t.nodes.push_back({b, e, -1, -1, -1});
        return (int)t.nodes.size() - 1;
      }
      const int mid = b + (e - b) / 2;
      const int c0 = build_balanced(t, b, mid, leaf);
      const int c1 = build_balanced(t, mid, e, leaf);
      t.nodes.push_back({b, e, c0, c1, -1});
      const int id = (int)t.nodes.size() - 1;
      t.nodes[c0].parent = t.nodes[c1].parent = id;
      return id;
    }
  }  // namespace

  ClusterTree ClusterTree::balanced(int n, int leaf) {
    ClusterTree t;
    if (n == 0) {
      t.nodes.push_back({0, 0, -1, -1, -1});
      return t;
    }
    build_balanced(t, 0, n, leaf);
    return t;
  }

  ClusterTree ClusterTree::join(const ClusterTree& a, const ClusterTree& b) {
    ClusterTree t;
    t.nodes = a.nodes;
    const int off = (int)t.nodes.size();
    const int shift = a.nodes.back().end;
    for (auto n : b.nodes) {
      n.begin += shift;
      n.end += shift;
      if (n.child0 >= 0) {
        n.child0 += off;
        n.child1 += off;
      }
      if (n.parent >= 0) n.parent += off;
      t.nodes.push_back(n);
    }
    const int c0 = off - 1, c1 = (int)t.nodes.size() - 1;
    t.nodes.push_back({t.nodes[c0].begin, t.nodes[c1].end, c0, c1, -1});
    t.nodes[c0].parent = t.nodes[c1].parent = (int)t.nodes.size() - 1;
    return t;
  }

  ClusterTree front_cluster_tree(int ns, int nu, int leaf) {
    ClusterTree sep = ClusterTree::balanced(ns, leaf);
    if (!nu) return sep;
    return ClusterTree::join(sep, ClusterTree::balanced(nu, leaf));
  }

}  // namespace hssmf_b200
