// plan.hpp — host-side plan builder of the fast GFT (Lu & Ortega, arXiv 1907.07875).
//
// Everything graph-dependent happens here once, in double precision:
//   P1 Laplacian                          eq:l_from_sw
//   P2 phi validation / partition         Def. 1-2, eq:B_phi
//   P3 involution search                  Sec. V-F
//   P4 decomposition G -> (G+, G-)        Theorem 4
//      recursion "until a symmetry property cannot be found"
//   P5 leaf eigensolves (cyclic Jacobi)
//   P6 realise columns, canonical signs, ascending-eigenvalue order
//   P7 fold the Haar 1/sqrt2 factors into the leaves
//   P8 op counts (tab:runtime conventions)
// The device kernels (codegen.cpp) consume `Plan` only.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gft {

// Error with a gft_status code (thrown inside the library, caught at the C ABI).
struct Error {
  int status;
  std::string msg;
};
[[noreturn]] void fail(int status, const std::string& msg);

// A weighted undirected graph in (W, s) form: W dense k x k symmetric with zero
// diagonal (w_ij, i != j) and s the self-loop weights.
struct SubGraph {
  int k = 0;
  std::vector<double> W;   // row-major k*k
  std::vector<double> s;   // k
  double w(int i, int j) const { return W[(size_t)i * k + j]; }
  std::vector<double> laplacian() const;   // l_ii = s_i + sum_{j!=i} w_ij, l_ij = -w_ij
  double scale() const;                    // max(|W|, |s|, 1e-300)
};

// Build a SubGraph from a Laplacian (eq:sw_from_l): s_i = sum_j l_ij.
SubGraph subgraph_from_laplacian(int n, const double* L);

// One operation of the unnormalised butterfly network, in forward order.
//   UNIT: (x_a, x_b) <- (x_a + x_b, x_a - x_b)       a in V_X, b = phi(a) in V_Y (A-6)
//   FIX:  x_a <- x_a * 2^(m/2)                         equalises deferred Haar scales
struct Op {
  enum Kind { UNIT = 0, FIX = 1 } kind;
  int a, b;     // positions (b unused for FIX)
  int m;        // FIX exponent
  int level;    // butterfly level (depth of the decomposition node)
};

// One Givens rotation of an approximate leaf (local indices p < q): G = I except
// G[p][p] = G[q][q] = c, G[p][q] = s, G[q][p] = -s; the leaf's A <- G^T A G.
struct Givens {
  int p, q;
  double c, s;
};

// A dense sub-GFT block.  Forward: y[slot[r]] = sum_c M[r*k + c] * x[pos[c]],
// inverse: x[pos[c]] = sum_r M[r*k + c] * y[slot[r]]  (M = V^T diag(2^(-d/2))).
struct Leaf {
  int k = 0;
  std::vector<int> pos;        // positions (signal indices) feeding the leaf
  std::vector<int> slot;       // output coefficient index of local eigenvector r
  std::vector<double> lam;     // eigenvalues (ascending within the leaf)
  std::vector<double> V;       // eigenvectors, row-major V[c*k + r] = v_r(c), canonical sign
  std::vector<double> M;       // folded matrix, row-major M[r*k + c]
  int level = 0;               // depth at which the leaf was emitted
  // right Haar stage membership: index into Plan::rights, side 0 = E (part S1), 1 = F (S2),
  // pair[r] = pair index of output r or -1 (unpaired, passes through)
  int right = -1, side = 0;
  std::vector<int> pair;
  // approximate leaf (NEXT-4): J layers of parallel Givens rotations from
  // the truncated Jacobi algorithm, then output r = rotated local index perm[r]; V holds the
  // realised U_hat_l = G_1...G_J Pi, lam the final (sorted) diagonal; scale[c] = 2^(-d/2)
  bool approx = false;
  std::vector<std::vector<Givens>> layers;
  std::vector<int> perm;
  std::vector<double> scale;
};

struct PlanOptions {
  int max_depth = -1;
  int min_leaf = 1;
  int64_t search_budget = 1000000;
  double sym_rtol = 1e-12;
  bool normalized = false;   // GFT of D^{-1/2} L D^{-1/2}
  bool right_haar = true;    // right Haar stages on constant-diagonal bipartite components
  int approx_layers = -1;    // >= 0: leaves with k >= approx_min_leaf become J Givens layers
  int approx_min_leaf = 2;
};

// A right Haar stage (eq:right_gft / eq:right_pm, Theorems 1-2): on a
// bipartite component whose Laplacian has a constant diagonal c (a k-regular bipartite
// graph, or the normalised Laplacian of any bipartite graph), eigenvectors pair as
// (mu1; mu2) <-> (mu1; -mu2) with eigenvalues lambda <-> 2c - lambda (Lemma 1), so
//   U^T x = B diag(E^T, F^T) x:  a = E^T x_S1, b = F^T x_S2 (two dense leaves), then a
// butterfly on coefficient pairs.  Unpaired eigenvectors (lambda = c) are supported on one
// part only and pass through.
struct PostUnit {
  int p, q;   // coefficient slots: y_p <- a + b (eigenvalue lambda), y_q <- s (a - b) (2c - lambda)
  int s;      // +1 / -1, chosen so that both realised columns have the canonical sign
};

struct RightStage {
  int leafE = -1, leafF = -1;        // indices in Plan::leaves (E on part S1, F on part S2)
  std::vector<int> rE, rF;           // paired local outputs
  std::vector<int> sign;             // s per pair
};

struct Plan {
  int n = 0;
  std::vector<Op> ops;               // forward order
  std::vector<Leaf> leaves;          // emission order
  std::vector<RightStage> rights;    // right Haar stages (pairs of leaves)
  std::vector<PostUnit> post;        // forward: applied to the coefficients after the leaves
  std::vector<int> dexp;             // final Haar scale exponent per position
  std::vector<double> lambda;        // ascending, size n
  std::vector<double> U;             // realised basis row-major U[i*n+k]
  std::vector<double> L;             // Laplacian of the input graph
  // statistics
  int depth = 0;
  std::vector<int> units_per_level;
  int n_units = 0, n_fix = 0, n_vz_total = 0, max_leaf = 0, n_clusters = 0, n_post = 0;
  int n_givens = 0, n_approx_scale = 0, n_approx_leaves = 0;
  int64_t sum_k2 = 0, sum_kk1 = 0;
  double residual = 0, orth_error = 0;
};

// Validates the input graph (rules of gft.h) and returns (W, s) of the graph.
SubGraph graph_from_edges(int n, int64_t n_edges, const int32_t* src, const int32_t* dst,
                          const double* w, const double* self_loops);

// Definition 1-2 checks.  Throws GFT_ERR_NOT_INVOLUTION / GFT_ERR_NOT_SYMMETRIC.
void check_involution(int n, const int32_t* phi);
bool is_phi_symmetric(const SubGraph& g, const std::vector<int>& phi, double rtol);

// Node partition: V_X such that "nodes in those sets belong to
// different sides of the symmetry axis": pairs are oriented by propagating a side label
// along edges that do not cross the axis (seeded with the smaller index).  Returns V_X
// ascending.  `smaller_index` = true gives the plain rule V_X = min(i, phi(i)).
std::vector<int> orient_pairs(const SubGraph& g, const std::vector<int>& phi, bool smaller_index);

// Theorem 4 for the partition V_X = X (one node of every pair).
// plus: X in the given order, then V_Z ascending; minus: phi(X) in the same order.
// Entries with magnitude <= flush (absolute) are set to exactly 0.
void theorem4(const SubGraph& g, const std::vector<int>& phi, const std::vector<int>& X,
              double flush, SubGraph& plus, SubGraph& minus, std::vector<int>& plus_nodes,
              std::vector<int>& minus_nodes);

// Involution search (Sec. V-F): max p_phi, ties -> lexicographically smallest phi.
struct SearchResult {
  std::vector<int> phi;
  int p = 0;
  bool complete = true;
  int64_t steps = 0;
};
SearchResult find_involution(const SubGraph& g, double rtol, int64_t budget);

// Connected components (edges with |w| > 0).
std::vector<std::vector<int>> components(const SubGraph& g);

// Cyclic Jacobi eigensolver for a dense symmetric k x k matrix (row-major).
// Returns eigenvalues ascending and eigenvectors V[c*k + r] (column r).
void jacobi_eigh(int k, const std::vector<double>& A, std::vector<double>& lam,
                 std::vector<double>& V);

// Parallel truncated Jacobi (reading R-4 of DESIGN.md): up to J layers, each
// greedily rotating disjoint pairs by decreasing |a_pq| (relative ties 1e-12 -> lexicographic
// (p, q)) while |a_pq| > 1e-14 max(1, max|A|); an empty layer stops.  Returns the layers,
// perm (ascending final diagonal, stable), lam = sorted diagonal and V[c*k + r] = column r of
// U_hat = G_1...G_J Pi.
void truncated_jacobi(int k, const std::vector<double>& A, int J, std::vector<std::vector<Givens>>& layers,
                      std::vector<int>& perm, std::vector<double>& lam, std::vector<double>& V);

Plan build_plan(const SubGraph& g, const int32_t* user_phi, const PlanOptions& opt);

// Plan persistence (serialize.cpp): a versioned byte string of the whole factorisation;
// deserialize validates every index and size and throws GFT_ERR_INVALID_ARG on malformed input.
std::vector<uint8_t> serialize_plan(const Plan& P);
// consumed (optional): bytes of `buf` the plan occupies; without it, trailing bytes are an error
Plan deserialize_plan(const uint8_t* buf, size_t size, size_t* consumed = nullptr);

}  // namespace gft
