// Host-side symbolic analysis for the HSS-multifrontal path.
//
// Everything here is integer structure (plus the grid generators' values)
// whose outputs must be bit-exact with the reference; it stays on the host
// as the north star allows. Written fresh against the reference semantics:
//   grid generators       grid_problems.hpp:65-117
//   CSR permutation       sparse_matrix.hpp:24-46, 95-102
//   geometric ND          ordering.cpp:123-169, 213-222
//   etree from separators elimination_tree.cpp:10-35
//   symbolic upd sets     elimination_tree.cpp:148-189
//   cluster trees         cluster_tree.hpp:38-61, 90-96
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

namespace hssmf_b200 {

  // error with a C-ABI status code (include/hssmf_b200.h), the failing front
  // and column where they apply
  struct SolverFailure : std::runtime_error {
    int code, front, column;
    SolverFailure(int c, int f, int col, const std::string& m)
        : std::runtime_error(m), code(c), front(f), column(col) {}
  };
  // square CSR, sorted duplicate-free rows (sparse_matrix.hpp:14-47)
  struct Csr {
    int n = 0;
    std::vector<int> ptr{0}, ind;
    std::vector<double> val;
    std::int64_t nnz() const { return (std::int64_t)ind.size(); }
    double get(int i, int j) const;
    // symmetric permutation B[p[i]][p[j]] = A[i][j]
    Csr permuted(const std::vector<int>& p) const;
    // column permutation B[i][j] = A[i][q[j]] (sparse_matrix.hpp:104-124)
    Csr col_permuted(const std::vector<int>& q) const;
    // structurally symmetrized adjacency without the diagonal
    void symmetric_graph(std::vector<int>& gptr, std::vector<int>& gind) const;
  };

  // SparseMatrix::from_triplets (sparse_matrix.hpp:25-47): rows sorted,
  // duplicates summed; t is sorted in place
  Csr csr_from_triplets(int n, std::vector<std::tuple<int, int, double>>& t);

  // ScalingState (scaling.hpp:15-32): As = Dr A Dc Qc; xs[j] = x[qc[j]] / dc[qc[j]]
  struct Scaling {
    std::vector<double> dr, dc;
    std::vector<int> qc;
    int sweeps = 0;
  };
  // equilibrate_and_permute (scaling.hpp:40-139); throws code 9 (structurally
  // singular) on an empty row / column or when no zero-free diagonal exists
  Csr equilibrate_and_permute(const Csr& a, Scaling& sc);
  // read_matrix_market / write_matrix_market (matrix_market.cpp:10-77):
  // coordinate real|integer, general|symmetric; errors are code 1 (IoError)
  Csr read_matrix_market(const std::string& path);
  void write_matrix_market(const Csr& a, const std::string& path);

  struct Geometry {
    std::array<int, 3> dims{1, 1, 1};
    int ndims = 0;
    int vertex(int i, int j, int l) const { return i + dims[0] * (j + dims[1] * l); }
  };

  enum GridKind { P2D = 0, P3D = 1, C2D = 2, C3D = 3 };

  Csr grid_problem(int kind, int k, double nu, Geometry& g);
  // config 4: h^2-scaled -lap(u) + beta.grad(u) on k^3, beta = scale*(1,.5,.25)/h,
  // first-order upwind with the reference's upwind rule (grid_problems.hpp:57-61)
  Csr convdiff3d_const(int k, double scale, Geometry& g);

  struct Cluster {
    int begin = 0, end = 0, child0 = -1, child1 = -1, parent = -1;
    bool leaf() const { return child0 < 0; }
    int size() const { return end - begin; }
  };
  struct ClusterTree {
    std::vector<Cluster> nodes;  // postorder, root last
    int root() const { return (int)nodes.size() - 1; }
    static ClusterTree balanced(int n, int leaf);
    static ClusterTree join(const ClusterTree& a, const ClusterTree& b);
  };
  struct FrontNode {
    int sep_begin = 0, sep_end = 0;
    int child0 = -1, child1 = -1, parent = -1, level = 0;
    std::vector<int> upd;
    // HSS clusters of the separator from separator reordering
    // (FrontNode::sep_clusters, elimination_tree.hpp:20); empty = balanced
    ClusterTree sep_clusters;
    int ns() const { return sep_end - sep_begin; }
    int nu() const { return (int)upd.size(); }
    int m() const { return ns() + nu(); }
    bool leaf() const { return child0 < 0 && child1 < 0; }
  };

  struct Etree {
    int n = 0;
    std::vector<FrontNode> nodes;  // postorder, root last
    int root() const { return (int)nodes.size() - 1; }
    void compute_levels();
  };

  // geometric nested dissection; perm[old] = new. nodes carry separators only
  Etree nested_dissection_geometric(const Geometry& g, int leaf, std::vector<int>& perm);
  void symbolic_factorization(const Csr& a, Etree& t);

  // front_cluster_tree (multifrontal.hpp:318-326): balanced separator
  // clusters, or the front's own when they cover the separator exactly
  ClusterTree front_cluster_tree(int ns, int nu, int leaf);
  ClusterTree front_cluster_tree(const FrontNode& f, int leaf);

  // ---- graph ordering and separator reordering (ordering.cpp:47-119,
  // 171-236; separator_reorder.cpp:10-135), integer outputs bit-exact ----
  struct Bisection {
    std::vector<int> part0, part1, sep;
  };
  // level-set bisection of the vertex subset verts; level is scratch of size
  // >= n holding -2 everywhere (restored on return)
  Bisection level_set_bisection(const std::vector<int>& verts, const int* gptr,
                                const int* gind, std::vector<int>& level, bool extract_sep);
  // nested dissection of a symmetric adjacency (no diagonal); perm[old] = new;
  // nodes carry separators only (upd empty)
  Etree nested_dissection_graph(int n, const std::vector<int>& gptr,
                                const std::vector<int>& gind, int leaf, std::vector<int>& perm);
  void separator_enriched_graph(const std::vector<int>& sep_verts, int n,
                                const std::vector<int>& gptr, const std::vector<int>& gind,
                                std::vector<int>& sptr, std::vector<int>& sind);
  ClusterTree reorder_separator(const std::vector<int>& sep_verts, int n,
                                const std::vector<int>& gptr, const std::vector<int>& gind,
                                int b, std::vector<int>& new_to_old);
  // relabels the separators of the selected fronts (sep_clusters set);
  // returns perm[old] = new on the current numbering
  std::vector<int> reorder_tree_separators(Etree& t, const std::vector<char>& selected,
                                           const std::vector<int>& gptr,
                                           const std::vector<int>& gind, int b);

}  // namespace hssmf_b200
