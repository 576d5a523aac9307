// Graph nested dissection and separator reordering on the host.
//
// Integer structure only; outputs are bit-exact with the reference's
//   level-set bisection        ordering.cpp:15-119
//   graph nested dissection    ordering.cpp:171-236
//   enriched separator graph   separator_reorder.cpp:10-41
//   separator cluster bisection separator_reorder.cpp:43-94
//   tree-wide reordering       separator_reorder.cpp:96-135
// (pinned by tests/test_analysis.py against oracle/_ref). Written from the
// documented semantics: BFS level structures from a pseudo-peripheral vertex,
// a level cut at the half-weight point, and the smaller boundary side of the
// edge cut as vertex separator.
#include <algorithm>
#include <cstdlib>

#include "analysis.hpp"

namespace hssmf_b200 {

  namespace {
    // Breadth-first levels over the subset verts (members hold -1 in lev);
    // when the BFS runs dry before covering the subset it restarts from the
    // first unvisited member, one level above the deepest so far. Returns the
    // last vertex taken from the queue.
    int bfs_sweep(const std::vector<int>& verts, const int* gptr, const int* gind,
                  std::vector<int>& lev, int start, std::vector<int>& q) {
      q.clear();
      q.push_back(start);
      lev[start] = 0;
      int last = start, deepest = 0;
      size_t head = 0, scan = 0;
      for (;;) {
        while (head < q.size()) {
          const int v = q[head++];
          last = v;
          if (lev[v] > deepest) deepest = lev[v];
          for (int k = gptr[v]; k < gptr[v + 1]; k++) {
            const int w = gind[k];
            if (lev[w] == -1) {
              lev[w] = lev[v] + 1;
              q.push_back(w);
            }
          }
        }
        if (q.size() == verts.size()) return last;
        while (lev[verts[scan]] != -1) scan++;
        lev[verts[scan]] = deepest + 1;
        q.push_back(verts[scan]);
      }
    }
  }  // namespace

  Bisection level_set_bisection(const std::vector<int>& verts, const int* gptr,
                                const int* gind, std::vector<int>& level, bool extract_sep) {
    Bisection out;
    const int tot = (int)verts.size();
    if (tot < 2) {
      out.part0 = verts;
      for (int v : verts) level[v] = -2;
      return out;
    }
    std::vector<int> q;
    q.reserve(tot);
    for (int v : verts) level[v] = -1;
    const int far = bfs_sweep(verts, gptr, gind, level, verts[0], q);
    for (int v : verts) level[v] = -1;
    bfs_sweep(verts, gptr, gind, level, far, q);
    int top = 0;
    for (int v : verts) top = std::max(top, level[v]);
    std::vector<int> width(top + 1, 0);
    for (int v : verts) width[level[v]]++;
    int cut = 1;
    if (extract_sep) {
      // smallest cut whose prefix holds half the vertices, below the top level
      int below = width[0];
      while (cut < top && 2 * below < tot) below += width[cut++];
    } else {
      // level boundary closest to the half (the lower cut wins ties)
      int below = width[0], best = std::abs(2 * below - tot);
      for (int c = 2; c <= top; c++) {
        below += width[c - 1];
        const int dev = std::abs(2 * below - tot);
        if (dev < best) {
          best = dev;
          cut = c;
        }
      }
    }
    for (int v : verts) (level[v] < cut ? out.part0 : out.part1).push_back(v);
    if (extract_sep) {
      // boundary vertices of each side of the edge cut; the smaller set (side
      // 0 on ties) becomes the separator and leaves its side
      std::vector<int> bd0, bd1;
      for (int v : out.part0)
        for (int k = gptr[v]; k < gptr[v + 1]; k++)
          if (level[gind[k]] >= cut) {
            bd0.push_back(v);
            break;
          }
      for (int v : out.part1)
        for (int k = gptr[v]; k < gptr[v + 1]; k++) {
          const int lw = level[gind[k]];
          if (lw >= 0 && lw < cut) {
            bd1.push_back(v);
            break;
          }
        }
      const bool side0 = bd0.size() <= bd1.size();
      out.sep = side0 ? std::move(bd0) : std::move(bd1);
      std::vector<int>& side = side0 ? out.part0 : out.part1;
      for (int v : out.sep) level[v] = -3;
      side.erase(std::remove_if(side.begin(), side.end(), [&](int v) { return level[v] == -3; }),
                 side.end());
    }
    for (int v : verts) level[v] = -2;
    return out;
  }

  namespace {
    struct GraphDissection {
      const int* gptr;
      const int* gind;
      int leaf;
      std::vector<int> iperm, level;
      std::vector<FrontNode> nodes;
      int next = 0;

      int add(int begin, int c0, int c1) {
        FrontNode f;
        f.sep_begin = begin;
        f.sep_end = next;
        f.child0 = c0;
        f.child1 = c1;
        nodes.push_back(std::move(f));
        const int id = (int)nodes.size() - 1;
        if (c0 >= 0) nodes[c0].parent = id;
        if (c1 >= 0) nodes[c1].parent = id;
        return id;
      }
      // children first (postorder), then the separator; a missing child is
      // always child1
      int split(std::vector<int>& verts) {
        if ((int)verts.size() <= leaf) {
          const int b = next;
          for (int v : verts) iperm[next++] = v;
          return add(b, -1, -1);
        }
        Bisection bs = level_set_bisection(verts, gptr, gind, level, true);
        std::vector<int>().swap(verts);
        int c0 = bs.part0.empty() ? -1 : split(bs.part0);
        int c1 = bs.part1.empty() ? -1 : split(bs.part1);
        if (c0 < 0) std::swap(c0, c1);
        const int b = next;
        for (int v : bs.sep) iperm[next++] = v;
        return add(b, c0, c1);
      }
    };
  }  // namespace

  Etree nested_dissection_graph(int n, const std::vector<int>& gptr,
                                const std::vector<int>& gind, int leaf, std::vector<int>& perm) {
    GraphDissection gd{gptr.data(), gind.data(), std::max(leaf, 1), std::vector<int>(n),
                       std::vector<int>(n, -2), {}, 0};
    std::vector<int> all(n);
    for (int i = 0; i < n; i++) all[i] = i;
    gd.split(all);
    perm.assign(n, -1);
    for (int k = 0; k < n; k++) perm[gd.iperm[k]] = k;
    Etree t;
    t.n = n;
    t.nodes = std::move(gd.nodes);
    t.compute_levels();
    return t;
  }

  void separator_enriched_graph(const std::vector<int>& sep_verts, int n,
                                const std::vector<int>& gptr, const std::vector<int>& gind,
                                std::vector<int>& sptr, std::vector<int>& sind) {
    const int s = (int)sep_verts.size();
    std::vector<int> local(n, -1);
    for (int t = 0; t < s; t++) local[sep_verts[t]] = t;
    sptr.assign(s + 1, 0);
    sind.clear();
    std::vector<int> nb;
    for (int t = 0; t < s; t++) {
      nb.clear();
      const int v = sep_verts[t];
      for (int k = gptr[v]; k < gptr[v + 1]; k++) {
        const int w = gind[k];
        if (local[w] >= 0) {
          if (local[w] != t) nb.push_back(local[w]);
          continue;
        }
        // separator vertices two steps away through an outside vertex
        for (int k2 = gptr[w]; k2 < gptr[w + 1]; k2++) {
          const int u = local[gind[k2]];
          if (u >= 0 && u != t) nb.push_back(u);
        }
      }
      std::sort(nb.begin(), nb.end());
      nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
      sind.insert(sind.end(), nb.begin(), nb.end());
      sptr[t + 1] = (int)sind.size();
    }
  }

  namespace {
    struct SepClusters {
      const int* sptr;
      const int* sind;
      int b;
      std::vector<int> level, order;
      ClusterTree tree;
      int next = 0;

      int split(std::vector<int>& vs) {
        if ((int)vs.size() <= b) {
          const int begin = next;
          for (int v : vs) order[next++] = v;
          tree.nodes.push_back({begin, next, -1, -1, -1});
          return (int)tree.nodes.size() - 1;
        }
        Bisection bs = level_set_bisection(vs, sptr, sind, level, false);
        std::vector<int>().swap(vs);
        const int c0 = split(bs.part0);
        const int c1 = split(bs.part1);
        tree.nodes.push_back({tree.nodes[c0].begin, tree.nodes[c1].end, c0, c1, -1});
        const int id = (int)tree.nodes.size() - 1;
        tree.nodes[c0].parent = tree.nodes[c1].parent = id;
        return id;
      }
    };
  }  // namespace

  ClusterTree reorder_separator(const std::vector<int>& sep_verts, int n,
                                const std::vector<int>& gptr, const std::vector<int>& gind,
                                int b, std::vector<int>& new_to_old) {
    const int s = (int)sep_verts.size();
    b = std::max(b, 1);
    if (s <= b) {
      new_to_old.resize(s);
      for (int t = 0; t < s; t++) new_to_old[t] = t;
      ClusterTree one;
      one.nodes.push_back({0, s, -1, -1, -1});
      return one;
    }
    std::vector<int> sptr, sind;
    separator_enriched_graph(sep_verts, n, gptr, gind, sptr, sind);
    SepClusters sc{sptr.data(), sind.data(), b, std::vector<int>(s, -2), std::vector<int>(s), {},
                   0};
    std::vector<int> all(s);
    for (int t = 0; t < s; t++) all[t] = t;
    sc.split(all);
    new_to_old = std::move(sc.order);
    return std::move(sc.tree);
  }

  std::vector<int> reorder_tree_separators(Etree& t, const std::vector<char>& selected,
                                           const std::vector<int>& gptr,
                                           const std::vector<int>& gind, int b) {
    // the separators are disjoint index ranges: every front relabels its own
    // range independently (the reference's task order does not matter)
    std::vector<int> iperm(t.n);
    for (int k = 0; k < t.n; k++) iperm[k] = k;
    for (int i = 0; i < (int)t.nodes.size(); i++) {
      FrontNode& f = t.nodes[i];
      if (!selected[i] || f.ns() <= 0) continue;
      std::vector<int> verts(f.ns()), n2o;
      for (int c = f.sep_begin; c < f.sep_end; c++) verts[c - f.sep_begin] = c;
      f.sep_clusters = reorder_separator(verts, t.n, gptr, gind, b, n2o);
      for (int k = 0; k < f.ns(); k++) iperm[f.sep_begin + k] = f.sep_begin + n2o[k];
    }
    std::vector<int> perm(t.n);
    for (int k = 0; k < t.n; k++) perm[iperm[k]] = k;
    return perm;
  }

  ClusterTree front_cluster_tree(const FrontNode& f, int leaf) {
    const bool own = !f.sep_clusters.nodes.empty() && f.sep_clusters.nodes.back().end == f.ns();
    ClusterTree sep = own ? f.sep_clusters : ClusterTree::balanced(f.ns(), leaf);
    if (!f.nu()) return sep;
    return ClusterTree::join(sep, ClusterTree::balanced(f.nu(), leaf));
  }

}  // namespace hssmf_b200
