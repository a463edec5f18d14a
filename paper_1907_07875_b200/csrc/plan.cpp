// plan.cpp — graph validation, Theorem 4 decomposition, recursion, leaf solves,
// realisation / canonicalisation / ordering, sqrt2 folding (see plan.hpp for the map).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <utility>

#include "../../include/gft.h"

namespace gft {

[[noreturn]] void fail(int status, const std::string& msg) { throw Error{status, msg}; }

static const double kSqrt2 = 1.41421356237309504880;

std::vector<double> SubGraph::laplacian() const {
  // eq:l_from_sw
  std::vector<double> L((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) {
    double d = s[i];
    for (int j = 0; j < k; ++j) {
      if (j == i) continue;
      L[(size_t)i * k + j] = -w(i, j);
      d += w(i, j);
    }
    L[(size_t)i * k + i] = d;
  }
  return L;
}

double SubGraph::scale() const {
  double m = 0;
  for (double v : W) m = std::max(m, std::fabs(v));
  for (double v : s) m = std::max(m, std::fabs(v));
  return m > 0 ? m : 1e-300;
}

SubGraph subgraph_from_laplacian(int n, const double* L) {
  // eq:sw_from_l: s_i = sum_j l_ij, w_ij = -l_ij
  SubGraph g;
  g.k = n;
  g.W.assign((size_t)n * n, 0.0);
  g.s.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double rs = 0;
    for (int j = 0; j < n; ++j) {
      double v = L[(size_t)i * n + j];
      if (!std::isfinite(v)) fail(GFT_ERR_INVALID_ARG, "non-finite Laplacian entry");
      rs += v;
      if (j != i) g.W[(size_t)i * n + j] = -v;
    }
    g.s[i] = rs;
  }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double a = g.W[(size_t)i * n + j], b = g.W[(size_t)j * n + i];
      if (std::fabs(a - b) > 1e-12 * std::max(1.0, std::max(std::fabs(a), std::fabs(b))))
        fail(GFT_ERR_INVALID_ARG, "Laplacian is not symmetric");
      double m = 0.5 * (a + b);
      g.W[(size_t)i * n + j] = g.W[(size_t)j * n + i] = m;
    }
  return g;
}

SubGraph graph_from_edges(int n, int64_t n_edges, const int32_t* src, const int32_t* dst,
                          const double* w, const double* self_loops) {
  if (n < 1) fail(GFT_ERR_INVALID_ARG, "n must be >= 1");
  if (n > 8192) fail(GFT_ERR_UNSUPPORTED, "n > 8192 not supported by the dense planner");
  if (n_edges < 0) fail(GFT_ERR_INVALID_ARG, "n_edges < 0");
  if (n_edges > 0 && (!src || !dst || !w)) fail(GFT_ERR_INVALID_ARG, "NULL edge arrays");
  SubGraph g;
  g.k = n;
  g.W.assign((size_t)n * n, 0.0);
  g.s.assign(n, 0.0);
  std::vector<char> seen((size_t)n * n, 0);
  for (int64_t e = 0; e < n_edges; ++e) {
    int i = src[e], j = dst[e];
    double wt = w[e];
    if (i < 0 || i >= n || j < 0 || j >= n)
      fail(GFT_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": node index out of range");
    if (i == j)
      fail(GFT_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": self-edge (use self_loops)");
    if (!std::isfinite(wt)) fail(GFT_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": non-finite weight");
    size_t a = (size_t)std::min(i, j) * n + std::max(i, j);
    if (seen[a]) fail(GFT_ERR_INVALID_ARG, "edge " + std::to_string(e) + ": duplicate node pair");
    seen[a] = 1;
    if (wt == 0.0) continue;   // zero weight = no edge
    g.W[(size_t)i * n + j] = wt;
    g.W[(size_t)j * n + i] = wt;
  }
  if (self_loops) {
    for (int i = 0; i < n; ++i) {
      if (!std::isfinite(self_loops[i])) fail(GFT_ERR_INVALID_ARG, "non-finite self-loop");
      g.s[i] = self_loops[i];
    }
  }
  return g;
}

void check_involution(int n, const int32_t* phi) {
  // Definition 1: a permutation with phi(phi(i)) = i.
  for (int i = 0; i < n; ++i) {
    int j = phi[i];
    if (j < 0 || j >= n) fail(GFT_ERR_NOT_INVOLUTION, "phi[" + std::to_string(i) + "] out of range");
    if (phi[j] != i)
      fail(GFT_ERR_NOT_INVOLUTION, "phi(phi(" + std::to_string(i) + ")) != " + std::to_string(i));
  }
}

bool is_phi_symmetric(const SubGraph& g, const std::vector<int>& phi, double rtol) {
  // Definition 2, including self-loops s_i = s_phi(i).
  const double tol = rtol * g.scale();
  for (int i = 0; i < g.k; ++i) {
    if (std::fabs(g.s[i] - g.s[phi[i]]) > tol) return false;
    for (int j = i + 1; j < g.k; ++j)
      if (std::fabs(g.w(i, j) - g.w(phi[i], phi[j])) > tol) return false;
  }
  return true;
}

std::vector<int> orient_pairs(const SubGraph& g, const std::vector<int>& phi, bool smaller_index) {
  const int k = g.k;
  std::vector<int> side(k, -1);   // 0 = V_X, 1 = V_Y
  for (int a = 0; a < k; ++a) {
    if (phi[a] == a || side[a] >= 0) continue;
    side[a] = 0;
    side[phi[a]] = 1;
    if (smaller_index) continue;
    std::vector<int> q{a, phi[a]};
    for (size_t h = 0; h < q.size(); ++h) {
      const int u = q[h];
      for (int v = 0; v < k; ++v) {
        if (v == u || phi[v] == v || v == phi[u] || side[v] >= 0 || g.w(u, v) == 0.0) continue;
        side[v] = side[u];            // same side as its neighbour (edge does not cross the axis)
        side[phi[v]] = 1 - side[u];
        q.push_back(v);
        q.push_back(phi[v]);
      }
    }
  }
  std::vector<int> X;
  for (int i = 0; i < k; ++i)
    if (side[i] == 0) X.push_back(i);
  return X;
}

void theorem4(const SubGraph& g, const std::vector<int>& phi, const std::vector<int>& Xin,
              double flush, SubGraph& plus, SubGraph& minus, std::vector<int>& plus_nodes,
              std::vector<int>& minus_nodes) {
  // Node partition: V_Z fixed points, V_X = Xin (one node of every
  // pair), V_Y = phi(V_X).  G+ lives on V_X u V_Z, G- on V_Y.
  const int k = g.k;
  std::vector<int> X(Xin), Y, Z;
  std::vector<char> inX(k, 0), inZ(k, 0);
  for (int i = 0; i < k; ++i)
    if (phi[i] == i) { Z.push_back(i); inZ[i] = 1; }
  for (int x : X) {
    if (phi[x] == x || inX[x] || inX[phi[x]]) fail(GFT_ERR_INVALID_ARG, "bad V_X for theorem4");
    inX[x] = 1;
  }
  if ((int)(2 * X.size() + Z.size()) != k) fail(GFT_ERR_INVALID_ARG, "V_X does not cover every pair");
  for (int x : X) Y.push_back(phi[x]);
  plus_nodes = X;
  plus_nodes.insert(plus_nodes.end(), Z.begin(), Z.end());
  minus_nodes = Y;
  const int kp = (int)plus_nodes.size(), km = (int)minus_nodes.size();
  auto fl = [flush](double v) { return std::fabs(v) <= flush ? 0.0 : v; };

  // ---- G+ (Theorem 4) ----
  plus.k = kp;
  plus.W.assign((size_t)kp * kp, 0.0);
  plus.s.assign(kp, 0.0);
  for (int a = 0; a < kp; ++a) {
    const int i = plus_nodes[a];
    for (int b = a + 1; b < kp; ++b) {
      const int j = plus_nodes[b];
      double v;
      if (inX[i] && inX[j]) v = g.w(i, j) + g.w(i, phi[j]);          // X-X
      else if (inZ[i] && inZ[j]) v = g.w(i, j);                        // Z-Z
      else v = kSqrt2 * g.w(i, j);                                     // X-Z / Z-X
      v = fl(v);
      plus.W[(size_t)a * kp + b] = plus.W[(size_t)b * kp + a] = v;
    }
    double sv;
    if (inX[i]) {
      double sz = 0;
      for (int z : Z) sz += g.w(i, z);
      sv = g.s[i] - (kSqrt2 - 1.0) * sz;                               // s+_i, i in V_X
    } else {
      double sx = 0;
      for (int x : X) sx += g.w(i, x);
      sv = g.s[i] + (2.0 - kSqrt2) * sx;                               // s+_i, i in V_Z
    }
    plus.s[a] = fl(sv);
  }
  // ---- G- (Theorem 4) ----
  minus.k = km;
  minus.W.assign((size_t)km * km, 0.0);
  minus.s.assign(km, 0.0);
  for (int a = 0; a < km; ++a) {
    const int i = minus_nodes[a];
    for (int b = a + 1; b < km; ++b) {
      const int j = minus_nodes[b];
      double v = fl(g.w(i, j) - g.w(i, phi[j]));
      minus.W[(size_t)a * km + b] = minus.W[(size_t)b * km + a] = v;
    }
    double sx = 0, sz = 0;
    for (int x : X) sx += g.w(i, x);
    for (int z : Z) sz += g.w(i, z);
    minus.s[a] = fl(g.s[i] + 2.0 * sx + sz);
  }
}

std::vector<std::vector<int>> components(const SubGraph& g) {
  std::vector<int> comp(g.k, -1);
  std::vector<std::vector<int>> out;
  for (int r = 0; r < g.k; ++r) {
    if (comp[r] >= 0) continue;
    std::vector<int> members{r};
    comp[r] = (int)out.size();
    for (size_t q = 0; q < members.size(); ++q) {
      int u = members[q];
      for (int v = 0; v < g.k; ++v)
        if (v != u && comp[v] < 0 && g.w(u, v) != 0.0) {
          comp[v] = comp[r];
          members.push_back(v);
        }
    }
    std::sort(members.begin(), members.end());
    out.push_back(members);
  }
  return out;
}

static SubGraph induced(const SubGraph& g, const std::vector<int>& nodes) {
  SubGraph h;
  h.k = (int)nodes.size();
  h.W.assign((size_t)h.k * h.k, 0.0);
  h.s.assign(h.k, 0.0);
  for (int a = 0; a < h.k; ++a) {
    h.s[a] = g.s[nodes[a]];
    for (int b = 0; b < h.k; ++b)
      if (a != b) h.W[(size_t)a * h.k + b] = g.w(nodes[a], nodes[b]);
  }
  return h;
}

// ---------------------------------------------------------------------------------
// Recursive builder
// ---------------------------------------------------------------------------------
namespace {
struct Builder {
  const PlanOptions& opt;
  Plan& P;
  std::vector<int> d;   // running Haar scale exponent per position

  Builder(const PlanOptions& o, Plan& p) : opt(o), P(p), d(p.n, 0) {}

  double internal_rtol() const { return std::max(opt.sym_rtol, 1e-10); }

  void emit_leaf(const SubGraph& g, const std::vector<int>& pos, int depth) {
    Leaf lf;
    lf.k = g.k;
    lf.pos = pos;
    lf.level = depth;
    if (opt.approx_layers >= 0 && g.k >= std::max(2, opt.approx_min_leaf)) {
      // Haar + approximate GFT: the sub-GFT becomes J Givens layers
      lf.approx = true;
      truncated_jacobi(g.k, g.laplacian(), opt.approx_layers, lf.layers, lf.perm, lf.lam, lf.V);
    } else {
      jacobi_eigh(g.k, g.laplacian(), lf.lam, lf.V);
    }
    P.leaves.push_back(std::move(lf));
  }

  // Right Haar stage: needs a bipartite component whose Laplacian has a
  // constant diagonal c; builds E (part S1) and F (part S2) from the component's
  // eigenvectors paired by sigma = diag(+1 on S1, -1 on S2) (Lemma 1 / Theorem 1
  // construction).  Returns false (caller emits a dense leaf) if any check fails.
  // The preconditions of a right Haar stage on a connected (sub)graph: constant Laplacian
  // diagonal and a 2-colouring; returns the parts S1 (colour of node 0) and S2.
  static bool right_parts(const SubGraph& g, std::vector<int>& S1, std::vector<int>& S2) {
    const int k = g.k;
    if (k < 2) return false;
    const std::vector<double> L = g.laplacian();
    double lmax = 0;
    for (double v : L) lmax = std::max(lmax, std::fabs(v));
    const double tol = 1e-9 * std::max(1.0, lmax);
    for (int i = 0; i < k; ++i)
      if (std::fabs(L[(size_t)i * k + i] - L[0]) > tol) return false;
    std::vector<int> col(k, -1);
    col[0] = 0;
    std::vector<int> q{0};
    for (size_t h = 0; h < q.size(); ++h) {
      const int u = q[h];
      for (int v = 0; v < k; ++v) {
        if (v == u || g.w(u, v) == 0.0) continue;
        if (col[v] < 0) { col[v] = 1 - col[u]; q.push_back(v); }
        else if (col[v] == col[u]) return false;   // odd cycle: not bipartite
      }
    }
    S1.clear();
    S2.clear();
    for (int i = 0; i < k; ++i) (col[i] == 0 ? S1 : S2).push_back(i);
    return !S2.empty() && (int)q.size() == k;
  }

  bool try_right(const SubGraph& g, const std::vector<int>& pos, int depth) {
    const int k = g.k;
    std::vector<int> S1, S2;
    if (!right_parts(g, S1, S2)) return false;
    const std::vector<double> L = g.laplacian();
    double lmax = 0;
    for (double v : L) lmax = std::max(lmax, std::fabs(v));
    const double tol = 1e-9 * std::max(1.0, lmax);
    const double c = L[0];
    std::vector<double> lam, V;
    jacobi_eigh(k, L, lam, V);
    auto comp = [&](int j, const std::vector<int>& S, double scale) {
      std::vector<double> e(S.size());
      for (size_t a = 0; a < S.size(); ++a) e[a] = scale * V[(size_t)S[a] * k + j];
      return e;
    };
    std::vector<std::vector<double>> Ecol, Fcol;
    std::vector<double> lamE, lamF;
    std::vector<int> pairE, pairF;
    // clusters of (nearly) equal eigenvalues
    std::vector<std::pair<int, int>> cl;   // [begin, end)
    for (int j = 0; j < k;) {
      int e = j + 1;
      while (e < k && lam[e] - lam[e - 1] <= tol) ++e;
      cl.push_back({j, e});
      j = e;
    }
    const double s2 = std::sqrt(2.0);
    std::vector<char> used(cl.size(), 0);
    for (size_t a = 0; a < cl.size(); ++a) {
      const int b0 = cl[a].first, b1 = cl[a].second;
      const double la = lam[b0];
      if (la < c - tol) {
        // partner cluster at 2c - lambda with the same multiplicity
        size_t bpart = cl.size();
        for (size_t b = 0; b < cl.size(); ++b)
          if (!used[b] && std::fabs(lam[cl[b].first] - (2 * c - la)) <= 10 * tol &&
              cl[b].second - cl[b].first == b1 - b0)
            bpart = b;
        if (bpart == cl.size()) return false;
        used[a] = used[bpart] = 1;
        for (int j = b0; j < b1; ++j) {
          pairE.push_back((int)Ecol.size());
          pairF.push_back((int)Fcol.size());
          Ecol.push_back(comp(j, S1, s2));
          Fcol.push_back(comp(j, S2, s2));
          lamE.push_back(lam[j]);
          lamF.push_back(lam[cl[bpart].first + (j - b0)]);
        }
      } else if (std::fabs(la - c) <= tol) {
        // sigma-invariant eigenspace: split into S1-supported and S2-supported halves
        used[a] = 1;
        for (int part = 0; part < 2; ++part) {
          const std::vector<int>& S = part == 0 ? S1 : S2;
          std::vector<std::vector<double>> basis;
          for (int j = b0; j < b1; ++j) {
            std::vector<double> v = comp(j, S, 1.0);
            for (const auto& u : basis) {   // Gram-Schmidt (twice for stability)
              for (int rep = 0; rep < 2; ++rep) {
                double dot = 0;
                for (size_t t = 0; t < v.size(); ++t) dot += v[t] * u[t];
                for (size_t t = 0; t < v.size(); ++t) v[t] -= dot * u[t];
              }
            }
            double nv = 0;
            for (double x : v) nv += x * x;
            nv = std::sqrt(nv);
            if (nv > 1e-6) {
              for (double& x : v) x /= nv;
              basis.push_back(v);
            }
          }
          for (auto& v : basis) {
            if (part == 0) { Ecol.push_back(v); lamE.push_back(la); }
            else { Fcol.push_back(v); lamF.push_back(la); }
          }
        }
      }
    }
    for (size_t a = 0; a < cl.size(); ++a)
      if (!used[a]) return false;
    if (Ecol.size() != S1.size() || Fcol.size() != S2.size()) return false;
    auto orth_ok = [](const std::vector<std::vector<double>>& C) {
      for (size_t a = 0; a < C.size(); ++a)
        for (size_t b = a; b < C.size(); ++b) {
          double dot = 0;
          for (size_t t = 0; t < C[a].size(); ++t) dot += C[a][t] * C[b][t];
          if (std::fabs(dot - (a == b ? 1.0 : 0.0)) > 1e-9) return false;
        }
      return true;
    };
    if (!orth_ok(Ecol) || !orth_ok(Fcol)) return false;
    // emit the two leaves and the stage
    const int ri = (int)P.rights.size();
    RightStage rs;
    for (int side = 0; side < 2; ++side) {
      const std::vector<int>& S = side == 0 ? S1 : S2;
      const auto& C = side == 0 ? Ecol : Fcol;
      Leaf lf;
      lf.k = (int)S.size();
      for (int i : S) lf.pos.push_back(pos[i]);
      lf.level = depth;
      lf.lam = side == 0 ? lamE : lamF;
      lf.V.assign((size_t)lf.k * lf.k, 0.0);
      for (int r = 0; r < lf.k; ++r)
        for (int cc = 0; cc < lf.k; ++cc) lf.V[(size_t)cc * lf.k + r] = C[r][cc];
      lf.right = ri;
      lf.side = side;
      lf.pair.assign(lf.k, -1);
      const auto& pl = side == 0 ? pairE : pairF;
      for (size_t j = 0; j < pl.size(); ++j) lf.pair[pl[j]] = (int)j;
      (side == 0 ? rs.leafE : rs.leafF) = (int)P.leaves.size();
      P.leaves.push_back(std::move(lf));
    }
    rs.rE = pairE;
    rs.rF = pairF;
    rs.sign.assign(pairE.size(), 1);
    P.rights.push_back(rs);
    P.n_post += (int)pairE.size();
    return true;
  }

  void emit_stage(const SubGraph& g, const std::vector<int>& pos, int depth,
                  const std::vector<int>& phi) {
    int p = 0, nz = 0;
    for (int i = 0; i < g.k; ++i) nz += phi[i] == i;
    const std::vector<int> X = orient_pairs(g, phi, false);
    for (int i : X) {
      ++p;
      const int a = pos[i], b = pos[phi[i]];
      if (d[a] != d[b]) {
        // partners carry different deferred 2^(d/2) scales: equalise explicitly
        const int lo = d[a] < d[b] ? a : b, hi = d[a] < d[b] ? b : a;
        P.ops.push_back(Op{Op::FIX, lo, -1, d[hi] - d[lo], depth});
        d[lo] = d[hi];
        ++P.n_fix;
      }
      P.ops.push_back(Op{Op::UNIT, a, b, 0, depth});   // sum -> a (V_X), difference -> b (V_Y)
      ++d[a];
      ++d[b];
    }
    if ((int)P.units_per_level.size() <= depth) P.units_per_level.resize(depth + 1, 0);
    P.units_per_level[depth] += p;
    P.n_units += p;
    P.n_vz_total += nz;
    SubGraph plus, minus;
    std::vector<int> pn, mn;
    theorem4(g, phi, X, internal_rtol() * g.scale(), plus, minus, pn, mn);
    std::vector<int> pos_plus(pn.size()), pos_minus(mn.size());
    for (size_t a = 0; a < pn.size(); ++a) pos_plus[a] = pos[pn[a]];
    for (size_t a = 0; a < mn.size(); ++a) pos_minus[a] = pos[mn[a]];
    node(plus, pos_plus, depth + 1, nullptr);
    node(minus, pos_minus, depth + 1, nullptr);
  }

  void node(const SubGraph& g, const std::vector<int>& pos, int depth, const int32_t* top_phi) {
    if (g.k == 0) return;
    const bool depth_ok = opt.max_depth < 0 || depth < opt.max_depth;
    if (top_phi) {
      std::vector<int> phi(top_phi, top_phi + g.k);
      int p = 0;
      for (int i = 0; i < g.k; ++i) p += phi[i] > i;
      if (p > 0 && depth_ok) {
        emit_stage(g, pos, depth, phi);
        return;
      }
    }
    // Split into connected components before searching (reading A-9)
    auto comps = components(g);
    if (comps.size() > 1) {
      for (auto& c : comps) {
        std::vector<int> cp(c.size());
        for (size_t a = 0; a < c.size(); ++a) cp[a] = pos[c[a]];
        node(induced(g, c), cp, depth, nullptr);
      }
      return;
    }
    if (g.k <= opt.min_leaf || !depth_ok) {
      emit_leaf(g, pos, depth);
      return;
    }
    SearchResult r = find_involution(g, internal_rtol(), opt.search_budget);
    if (r.p == 0) {
      if (!(opt.right_haar && try_right(g, pos, depth))) emit_leaf(g, pos, depth);
      return;
    }
    // both stage types available (a symmetric k-RBG / normalised bipartite graph): take the
    // one with fewer leaf multiplications at this level -- p^2 + (n-p)^2 for the left stage
    // (PAPER.md:721), |S1|^2 + |S2|^2 for the right stage (reading R-7)
    std::vector<int> S1, S2;
    if (opt.right_haar && right_parts(g, S1, S2)) {
      const int64_t kr = (int64_t)S1.size() * S1.size() + (int64_t)S2.size() * S2.size();
      const int64_t kl = (int64_t)r.p * r.p + (int64_t)(g.k - r.p) * (g.k - r.p);
      if (kr < kl && try_right(g, pos, depth)) return;
    }
    emit_stage(g, pos, depth, r.phi);
  }
};
}  // namespace

SubGraph normalized_graph(const SubGraph& g) {
  // symmetric normalised Laplacian D^{-1/2} L D^{-1/2}, d_i = sum_j w_ij with
  // w_ii = s_i, i.e. d_i = l_ii; returned in (W, s) form via eq:sw_from_l
  const int k = g.k;
  std::vector<double> L = g.laplacian(), isd(k);
  for (int i = 0; i < k; ++i) {
    const double d = L[(size_t)i * k + i];
    if (!(d > 0) || !std::isfinite(d))
      fail(GFT_ERR_INVALID_ARG, "normalized Laplacian needs positive degrees (node " + std::to_string(i) + ")");
    isd[i] = 1.0 / std::sqrt(d);
  }
  SubGraph h;
  h.k = k;
  h.W.assign((size_t)k * k, 0.0);
  h.s.assign(k, 0.0);
  for (int i = 0; i < k; ++i) {
    double rs = 0;
    for (int j = 0; j < k; ++j) {
      const double v = L[(size_t)i * k + j] * isd[i] * isd[j];
      rs += v;
      if (j != i) h.W[(size_t)i * k + j] = -v;
    }
    h.s[i] = rs;
  }
  return h;
}

Plan build_plan(const SubGraph& g0, const int32_t* user_phi, const PlanOptions& opt) {
  Plan P;
  P.n = g0.k;
  if (user_phi) {
    check_involution(g0.k, user_phi);
    std::vector<int> phi(user_phi, user_phi + g0.k);
    if (!is_phi_symmetric(g0, phi, opt.sym_rtol))
      fail(GFT_ERR_NOT_SYMMETRIC, "graph is not phi-symmetric within sym_rtol (Definition 2)");
  }
  // Theorem 3 "holds for normalized Laplacian as well": the same
  // decomposition runs on the (W, s) form of D^{-1/2} L D^{-1/2}, which is phi-symmetric
  // whenever the graph is (degrees are phi-invariant)
  const SubGraph g = opt.normalized ? normalized_graph(g0) : g0;
  P.L = g.laplacian();
  Builder B(opt, P);
  std::vector<int> pos(g.k);
  std::iota(pos.begin(), pos.end(), 0);
  B.node(g, pos, 0, user_phi);
  P.dexp = B.d;
  P.depth = (int)P.units_per_level.size();
  while (P.depth > 0 && P.units_per_level[P.depth - 1] == 0) --P.depth;
  P.units_per_level.resize(P.depth);

  const int n = P.n;
  // ---- P6: realise columns u = B_1 ... B_D (embedded v), canonicalise signs ----
  // Q = B_D...B_1 (normalised butterflies) so U = Q^T blockdiag(V) and Q^T applies the
  // units in reverse order; each B_phi is symmetric.
  struct Col { double lam; int leaf, r; };
  std::vector<Col> cols;
  std::vector<std::vector<double>> realised;   // per (leaf, r) in cols order
  const double r2 = 1.0 / kSqrt2;
  auto apply_units_T = [&](std::vector<double>& u) {
    for (auto it = P.ops.rbegin(); it != P.ops.rend(); ++it) {
      if (it->kind != Op::UNIT) continue;
      const double a = u[it->a], b = u[it->b];
      u[it->a] = (a + b) * r2;
      u[it->b] = (a - b) * r2;
    }
  };
  // sign rule: first entry with |u_i| > 1e-8 positive (reading A-3)
  auto first_sign = [&](const std::vector<double>& u) {
    for (int i = 0; i < n; ++i)
      if (std::fabs(u[i]) > 1e-8) return u[i] < 0 ? -1 : 1;
    return 1;
  };
  auto negate_col = [](Leaf& lf, int r) {
    for (int c = 0; c < lf.k; ++c) lf.V[(size_t)c * lf.k + r] = -lf.V[(size_t)c * lf.k + r];
  };
  for (int l = 0; l < (int)P.leaves.size(); ++l) {
    Leaf& lf = P.leaves[l];
    P.max_leaf = std::max(P.max_leaf, lf.k);
    if (lf.approx) {
      ++P.n_approx_leaves;
      for (const auto& layer : lf.layers) P.n_givens += (int)layer.size();
      P.n_approx_scale += lf.k;   // one output multiply per position (scaled rotations)
    } else {
      P.sum_k2 += (int64_t)lf.k * lf.k;
      P.sum_kk1 += (int64_t)lf.k * (lf.k - 1);
    }
    for (int r = 0; r < lf.k; ++r) {
      if (lf.right >= 0 && lf.pair[r] >= 0) {
        // right Haar pair: u_A = (e; f)/sqrt2 (lambda), u_B = s (e; -f)/sqrt2
        // (2c - lambda); realised together when the E leaf is visited
        if (lf.side == 1) continue;
        RightStage& rs = P.rights[lf.right];
        const int j = lf.pair[r];
        Leaf& lF = P.leaves[rs.leafF];
        const int rf = rs.rF[j];
        std::vector<double> uA(n, 0.0), uB(n, 0.0);
        for (int c = 0; c < lf.k; ++c) uA[lf.pos[c]] = uB[lf.pos[c]] = lf.V[(size_t)c * lf.k + r] * r2;
        for (int c = 0; c < lF.k; ++c) {
          const double v = lF.V[(size_t)c * lF.k + rf] * r2;
          uA[lF.pos[c]] = v;
          uB[lF.pos[c]] = -v;
        }
        apply_units_T(uA);
        apply_units_T(uB);
        if (first_sign(uA) < 0) {   // flip (e, f) jointly: u_A -> -u_A, u_B -> -u_B
          for (double& v : uA) v = -v;
          for (double& v : uB) v = -v;
          negate_col(lf, r);
          negate_col(lF, rf);
        }
        rs.sign[j] = 1;
        if (first_sign(uB) < 0) {
          for (double& v : uB) v = -v;
          rs.sign[j] = -1;
        }
        cols.push_back(Col{lf.lam[r], l, r});
        realised.push_back(std::move(uA));
        cols.push_back(Col{lF.lam[rf], rs.leafF, rf});
        realised.push_back(std::move(uB));
        continue;
      }
      std::vector<double> u(n, 0.0);
      for (int c = 0; c < lf.k; ++c) u[lf.pos[c]] = lf.V[(size_t)c * lf.k + r];
      apply_units_T(u);
      // approximate columns keep the signs the rotations give (the paper's delta / epsilon
      // take absolute values); the rotations themselves are the code
      if (!lf.approx && first_sign(u) < 0) {
        for (double& v : u) v = -v;
        negate_col(lf, r);
      }
      cols.push_back(Col{lf.lam[r], l, r});
      realised.push_back(std::move(u));
    }
  }
  std::vector<int> order(cols.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return cols[a].lam < cols[b].lam; });
  P.lambda.assign(n, 0.0);
  P.U.assign((size_t)n * n, 0.0);
  for (auto& lf : P.leaves) lf.slot.assign(lf.k, -1);
  for (int rank = 0; rank < (int)order.size(); ++rank) {
    const Col& c = cols[order[rank]];
    P.lambda[rank] = c.lam;
    P.leaves[c.leaf].slot[c.r] = rank;
    const auto& u = realised[order[rank]];
    for (int i = 0; i < n; ++i) P.U[(size_t)i * n + rank] = u[i];
  }
  // right Haar post-units on the coefficient slots (forward order = stage order)
  for (const RightStage& rs : P.rights)
    for (size_t j = 0; j < rs.rE.size(); ++j)
      P.post.push_back(PostUnit{P.leaves[rs.leafE].slot[rs.rE[j]], P.leaves[rs.leafF].slot[rs.rF[j]],
                                rs.sign[j]});
  // ---- P7: fold 2^(-d/2) into the leaves: M[r][c] = v_r(c) * 2^(-d_pos(c)/2), and the
  // 1/sqrt2 of a right Haar pair into its rows (post-units are unnormalised (a+b, a-b)) ----
  for (auto& lf : P.leaves) {
    if (lf.approx) {
      lf.scale.resize(lf.k);
      for (int c = 0; c < lf.k; ++c) lf.scale[c] = std::pow(2.0, -0.5 * P.dexp[lf.pos[c]]);
    }
    lf.M.assign((size_t)lf.k * lf.k, 0.0);
    for (int r = 0; r < lf.k; ++r) {
      const double pr = (lf.right >= 0 && lf.pair[r] >= 0) ? r2 : 1.0;
      for (int c = 0; c < lf.k; ++c)
        lf.M[(size_t)r * lf.k + c] =
            lf.V[(size_t)c * lf.k + r] * std::pow(2.0, -0.5 * P.dexp[lf.pos[c]]) * pr;
    }
  }
  // ---- self-check of the realised basis ----
  double lmax = 0;
  for (double v : P.L) lmax = std::max(lmax, std::fabs(v));
  double res = 0, orth = 0;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < n; ++k) {
      double acc = 0;
      for (int j = 0; j < n; ++j) acc += P.L[(size_t)i * n + j] * P.U[(size_t)j * n + k];
      res = std::max(res, std::fabs(acc - P.U[(size_t)i * n + k] * P.lambda[k]));
    }
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) {
      double acc = 0;
      for (int i = 0; i < n; ++i) acc += P.U[(size_t)i * n + a] * P.U[(size_t)i * n + b];
      orth = std::max(orth, std::fabs(acc - (a == b ? 1.0 : 0.0)));
    }
  P.residual = res;
  P.orth_error = orth;
  // an approximate plan is orthogonal but not an eigenbasis: only orthogonality is checked
  if ((P.n_approx_leaves == 0 && !(res <= 1e-8 * std::max(1.0, lmax))) || !(orth <= 1e-10))
    fail(GFT_ERR_EIG_NOCONVERGE, "realised basis failed self-check (residual " +
                                     std::to_string(res) + ", orthogonality " +
                                     std::to_string(orth) + ")");
  // ---- clusters (reading A-5) ----
  double lm = 0;
  for (double v : P.lambda) lm = std::max(lm, std::fabs(v));
  const double ctol = 1e-9 * std::max(1.0, lm);
  P.n_clusters = n > 0 ? 1 : 0;
  for (int k = 1; k < n; ++k)
    if (P.lambda[k] - P.lambda[k - 1] > ctol) ++P.n_clusters;
  return P;
}

// ---------------------------------------------------------------------------------
// Cyclic-by-row Jacobi (classical two-sided rotations; stable tan formula)
// ---------------------------------------------------------------------------------
void jacobi_eigh(int k, const std::vector<double>& A0, std::vector<double>& lam,
                 std::vector<double>& V) {
  std::vector<double> a(A0);
  V.assign((size_t)k * k, 0.0);
  for (int i = 0; i < k; ++i) V[(size_t)i * k + i] = 1.0;
  auto A = [&](int i, int j) -> double& { return a[(size_t)i * k + j]; };
  bool converged = (k <= 1);
  for (int sweep = 0; sweep < 100 && !converged; ++sweep) {
    double off = 0, diag = 0;
    for (int i = 0; i < k; ++i) {
      diag += A(i, i) * A(i, i);
      for (int j = i + 1; j < k; ++j) off += A(i, j) * A(i, j);
    }
    if (off == 0.0 || std::sqrt(off) <= 1e-17 * std::sqrt(diag + 2 * off)) {
      converged = true;
      break;
    }
    for (int p = 0; p < k - 1; ++p)
      for (int q = p + 1; q < k; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double app = A(p, p), aqq = A(q, q);
        // underflow rule: drop a_pq once it no longer changes the diagonal
        if (sweep > 3 && std::fabs(app) + 100 * std::fabs(apq) == std::fabs(app) &&
            std::fabs(aqq) + 100 * std::fabs(apq) == std::fabs(aqq)) {
          A(p, q) = A(q, p) = 0.0;
          continue;
        }
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < k; ++r) {              // columns p, q
          const double xp = A(r, p), xq = A(r, q);
          A(r, p) = c * xp - s * xq;
          A(r, q) = s * xp + c * xq;
        }
        for (int r = 0; r < k; ++r) {              // rows p, q
          const double xp = A(p, r), xq = A(q, r);
          A(p, r) = c * xp - s * xq;
          A(q, r) = s * xp + c * xq;
        }
        A(p, q) = A(q, p) = 0.0;
        for (int r = 0; r < k; ++r) {
          const double vp = V[(size_t)r * k + p], vq = V[(size_t)r * k + q];
          V[(size_t)r * k + p] = c * vp - s * vq;
          V[(size_t)r * k + q] = s * vp + c * vq;
        }
      }
  }
  if (!converged) {
    double off = 0, fro = 0;
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < k; ++j) {
        fro += A(i, j) * A(i, j);
        if (i != j) off += A(i, j) * A(i, j);
      }
    if (std::sqrt(off) > 1e-13 * std::sqrt(fro))
      fail(GFT_ERR_EIG_NOCONVERGE, "Jacobi did not converge in 100 sweeps");
  }
  // ascending order (stable)
  std::vector<int> idx(k);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
  lam.resize(k);
  std::vector<double> Vs((size_t)k * k);
  for (int r = 0; r < k; ++r) {
    lam[r] = A(idx[r], idx[r]);
    for (int c = 0; c < k; ++c) Vs[(size_t)c * k + r] = V[(size_t)c * k + idx[r]];
  }
  V.swap(Vs);
}

// ---------------------------------------------------------------------------------
// Parallel truncated Jacobi (approximate sub-GFTs; reading R-4)
// ---------------------------------------------------------------------------------
void truncated_jacobi(int k, const std::vector<double>& A0, int J, std::vector<std::vector<Givens>>& layers,
                      std::vector<int>& perm, std::vector<double>& lam, std::vector<double>& V) {
  std::vector<double> a(A0);
  auto A = [&](int i, int j) -> double& { return a[(size_t)i * k + j]; };
  std::vector<double> W((size_t)k * k, 0.0);   // accumulated G_1 G_2 ... (row-major)
  for (int i = 0; i < k; ++i) W[(size_t)i * k + i] = 1.0;
  double amax = 0;
  for (double v : a) amax = std::max(amax, std::fabs(v));
  const double zt = 1e-14 * std::max(1.0, amax);
  layers.clear();
  for (int layer = 0; layer < J; ++layer) {
    std::vector<char> used(k, 0);
    std::vector<Givens> rots;
    for (;;) {
      double m = -1;
      for (int p = 0; p < k; ++p) {
        if (used[p]) continue;
        for (int q = p + 1; q < k; ++q)
          if (!used[q]) m = std::max(m, std::fabs(A(p, q)));
      }
      if (!(m > zt)) break;
      // lexicographically first pair within the relative tie band of the maximum
      const double thr = m * (1.0 - 1e-12);
      int bp = -1, bq = -1;
      for (int p = 0; p < k && bp < 0; ++p) {
        if (used[p]) continue;
        for (int q = p + 1; q < k; ++q)
          if (!used[q] && std::fabs(A(p, q)) >= thr) { bp = p; bq = q; break; }
      }
      const int p = bp, q = bq;
      const double apq = A(p, q), app = A(p, p), aqq = A(q, q), tau = (aqq - app) / (2.0 * apq);
      double t;
      // numerically equal diagonals -> the 45 degree rotation (a rounding-level tau must
      // not decide the rotation direction)
      if (std::fabs(aqq - app) <= 1e-12 * std::max(std::fabs(app), std::max(std::fabs(aqq), std::fabs(apq)))) t = 1.0;
      else if (std::fabs(tau) > 1e150) t = 1.0 / (2.0 * tau);
      else t = (tau >= 0 ? 1.0 : -1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
      const double c = 1.0 / std::sqrt(1.0 + t * t), s = t * c;
      for (int r = 0; r < k; ++r) {              // columns p, q
        const double xp = A(r, p), xq = A(r, q);
        A(r, p) = c * xp - s * xq;
        A(r, q) = s * xp + c * xq;
      }
      for (int r = 0; r < k; ++r) {              // rows p, q
        const double xp = A(p, r), xq = A(q, r);
        A(p, r) = c * xp - s * xq;
        A(q, r) = s * xp + c * xq;
      }
      A(p, q) = A(q, p) = 0.0;
      for (int r = 0; r < k; ++r) {
        const double wp = W[(size_t)r * k + p], wq = W[(size_t)r * k + q];
        W[(size_t)r * k + p] = c * wp - s * wq;
        W[(size_t)r * k + q] = s * wp + c * wq;
      }
      used[p] = used[q] = 1;
      rots.push_back(Givens{p, q, c, s});
    }
    if (rots.empty()) break;
    layers.push_back(std::move(rots));
  }
  perm.resize(k);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return A(x, x) < A(y, y); });
  lam.resize(k);
  V.assign((size_t)k * k, 0.0);
  for (int r = 0; r < k; ++r) {
    lam[r] = A(perm[r], perm[r]);
    for (int c = 0; c < k; ++c) V[(size_t)c * k + r] = W[(size_t)c * k + perm[r]];
  }
}

}  // namespace gft
