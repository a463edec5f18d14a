// search.cpp — involution search (Sec. V-F).
//
// The paper prunes the T(n) candidate involutions with the degree list (equal degrees
// of i and phi(i)).  We use a slightly stronger sound signature per node: (self-loop,
// sorted incident-weight multiset), compared with a tolerance because sub-graph
// weights from Theorem 4 are irrational (sqrt2, 2-sqrt2, w +- w').  Within a connected
// component the search assigns phi in BFS order: for every non-root node u with BFS
// parent v, phi(u) must be a neighbour of phi(v) joined by an edge of the same weight,
// so a partial assignment propagates like an automorphism search.  Each extension is
// checked against all assigned nodes (Definition 2 restricted to assigned nodes, both
// for u and for phi(u)); a complete assignment is therefore phi-symmetric.  Among all
// complete assignments the one with max p_phi wins (motivated by the p^2 + (n-p)^2
// complexity), ties broken by the lexicographically smallest phi
// (reading A-8).  A budget bounds the enumeration.
//
// Trees ("searching of identical tree branches"): when the budget runs
// out on a component that is a tree, an O(n log n) canonical-label search takes over (the
// report [lu2019search] with the paper's algorithm is not available; this is the standard
// AHU rooted-tree labelling, weights and self-loops included).  Every involutive
// automorphism fixes the tree's centre (or swaps a bicentre), so rooted at the centre a
// max-p_phi involution swaps floor(m/2) pairs among each class of m identical child
// branches and recurses only into the unpaired one -- swapping two identical branches of
// size s pairs s nodes, more than any involution inside them.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <map>
#include <numeric>

#include "plan.hpp"

namespace gft {
namespace {

struct Ctx {
  const SubGraph& g;
  double tol;
  int64_t budget;
  std::vector<int> nodes;            // component nodes (ascending)
  std::vector<int> order, parent;    // BFS order / parent (local node ids)
  std::vector<std::vector<int>> nbr;
  std::vector<std::vector<char>> compat;
  std::vector<int> phi;              // -1 unassigned
  std::vector<int> assigned;
  std::vector<int> best;
  int best_p = 0;
  int64_t steps = 0;
  bool complete = true;

  Ctx(const SubGraph& gg, double t, int64_t b) : g(gg), tol(t), budget(b) {}

  bool consistent(int u, int j) const {
    for (int a : assigned) {
      if (std::fabs(g.w(u, a) - g.w(j, phi[a])) > tol) return false;
      if (j != u && std::fabs(g.w(j, a) - g.w(u, phi[a])) > tol) return false;
    }
    return true;
  }

  void record(int pairs) {
    bool better = pairs > best_p;
    if (!better && pairs == best_p) {
      for (int v : nodes) {
        if (phi[v] != best[v]) { better = phi[v] < best[v]; break; }
      }
    }
    if (better) {
      best_p = pairs;
      for (int v : nodes) best[v] = phi[v];
    }
  }

  void dfs(size_t idx, int pairs, int unassigned) {
    while (idx < order.size() && phi[order[idx]] >= 0) ++idx;
    if (idx == order.size()) { record(pairs); return; }
    if (steps >= budget) { complete = false; return; }
    const int u = order[idx];
    std::vector<int> cand;
    if (parent[u] < 0) {
      for (int j : nodes) if (compat[u][j]) cand.push_back(j);
    } else {
      const int v = phi[parent[u]];
      const double wt = g.w(u, parent[u]);
      for (int j : nbr[v])
        if (compat[u][j] && std::fabs(g.w(j, v) - wt) <= tol) cand.push_back(j);
    }
    // pairs first (ascending), the fixed point last: reaches large p_phi early
    std::sort(cand.begin(), cand.end(), [u](int a, int b) {
      if ((a == u) != (b == u)) return b == u;
      return a < b;
    });
    for (int j : cand) {
      if (j != u && phi[j] >= 0) continue;
      if (!consistent(u, j)) continue;
      if (++steps > budget) { complete = false; return; }
      phi[u] = j;
      phi[j] = u;
      assigned.push_back(u);
      if (j != u) assigned.push_back(j);
      const int np = pairs + (j != u);
      const int rem = unassigned - (j != u ? 2 : 1);
      if (np + rem / 2 >= best_p) dfs(idx + 1, np, rem);
      assigned.pop_back();
      if (j != u) assigned.pop_back();
      phi[u] = phi[j] = -1;
    }
  }
};

// Max-p involution of a tree component (see the header).  nodes = the component,
// nbr = neighbour lists over |w| > tol.  Returns p and writes phi on the component.
int tree_involution(const SubGraph& g, const std::vector<int>& nodes, const std::vector<std::vector<int>>& nbr,
                    double tol, std::vector<int>& phi) {
  const int k = g.k;
  const double quantum = tol > 0 ? tol : 1e-300;
  auto q = [quantum](double v) { return (int64_t)std::llround(v / quantum); };
  // centre(s) by peeling leaves
  std::vector<int> deg(k, 0), layer;
  for (int v : nodes) {
    deg[v] = (int)nbr[v].size();
    if (deg[v] <= 1) layer.push_back(v);
  }
  int remaining = (int)nodes.size();
  std::vector<char> gone(k, 0);
  while (remaining > 2) {
    std::vector<int> next;
    for (int v : layer) {
      gone[v] = 1;
      --remaining;
      for (int u : nbr[v])
        if (!gone[u] && --deg[u] == 1) next.push_back(u);
    }
    layer.swap(next);
  }
  std::vector<int> centres;
  for (int v : nodes) if (!gone[v]) centres.push_back(v);
  // canonical labels of rooted subtrees (parent excluded)
  std::map<std::vector<int64_t>, int> ids;
  std::vector<int> label(k, -1);
  std::function<int(int, int)> lab = [&](int v, int parent) -> int {
    std::vector<std::pair<int64_t, int>> ch;
    for (int c : nbr[v])
      if (c != parent) ch.push_back({q(g.w(v, c)), lab(c, v)});
    std::sort(ch.begin(), ch.end());
    std::vector<int64_t> key{q(g.s[v])};
    for (auto& e : ch) { key.push_back(e.first); key.push_back(e.second); }
    auto it = ids.emplace(key, (int)ids.size()).first;
    return label[v] = it->second;
  };
  auto children = [&](int v, int parent) {
    std::vector<int> ch;
    for (int c : nbr[v]) if (c != parent) ch.push_back(c);
    std::sort(ch.begin(), ch.end(), [&](int a, int b) {
      const auto ka = std::make_pair(q(g.w(v, a)), label[a]), kb = std::make_pair(q(g.w(v, b)), label[b]);
      return ka != kb ? ka < kb : a < b;
    });
    return ch;
  };
  int p = 0;
  // map the isomorphic subtrees rooted at a (parent pa) and b (parent pb) onto each other
  std::function<void(int, int, int, int)> iso = [&](int a, int pa, int b, int pb) {
    phi[a] = b;
    phi[b] = a;
    ++p;
    const auto ca = children(a, pa), cb = children(b, pb);
    for (size_t t = 0; t < ca.size(); ++t) iso(ca[t], a, cb[t], b);
  };
  std::function<void(int, int)> build = [&](int v, int parent) {
    phi[v] = v;
    const auto ch = children(v, parent);
    for (size_t a = 0; a < ch.size();) {
      size_t b = a;
      const auto key = std::make_pair(q(g.w(v, ch[a])), label[ch[a]]);
      while (b < ch.size() && std::make_pair(q(g.w(v, ch[b])), label[ch[b]]) == key) ++b;
      // class ch[a..b): the smallest-index branch stays (when m is odd), the rest pair up
      size_t t = a;
      if ((b - a) % 2 == 1) build(ch[t++], v);
      for (; t + 1 < b; t += 2) iso(ch[t], v, ch[t + 1], v);
      a = b;
    }
  };
  if (centres.size() == 2) {
    const int c1 = centres[0], c2 = centres[1];
    if (lab(c1, c2) == lab(c2, c1)) {
      iso(c1, c2, c2, c1);
      return p;
    }
  }
  lab(centres[0], -1);
  build(centres[0], -1);
  return p;
}

}  // namespace

SearchResult find_involution(const SubGraph& g, double rtol, int64_t budget) {
  SearchResult res;
  const int k = g.k;
  res.phi.resize(k);
  std::iota(res.phi.begin(), res.phi.end(), 0);
  if (k <= 1) return res;
  const double tol = rtol * g.scale();

  // neighbour lists and the node signature (PAPER.md:714-715 degree pruning, refined)
  std::vector<std::vector<int>> nbr(k);
  std::vector<std::vector<double>> sig(k);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j)
      if (j != i && std::fabs(g.w(i, j)) > tol) {
        nbr[i].push_back(j);
        sig[i].push_back(g.w(i, j));
      }
  for (auto& s : sig) std::sort(s.begin(), s.end());
  std::vector<std::vector<char>> compat(k, std::vector<char>(k, 0));
  std::vector<int> class_size(k, 0);
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) {
      bool ok = std::fabs(g.s[i] - g.s[j]) <= tol && sig[i].size() == sig[j].size();
      for (size_t t = 0; ok && t < sig[i].size(); ++t) ok = std::fabs(sig[i][t] - sig[j][t]) <= tol;
      compat[i][j] = ok;
      class_size[i] += ok;
    }

  // connected components over |w| > tol; each is searched independently
  std::vector<int> comp(k, -1);
  int ncomp = 0;
  for (int r = 0; r < k; ++r) {
    if (comp[r] >= 0) continue;
    std::vector<int> q{r};
    comp[r] = ncomp;
    for (size_t a = 0; a < q.size(); ++a)
      for (int v : nbr[q[a]])
        if (comp[v] < 0) { comp[v] = ncomp; q.push_back(v); }
    ++ncomp;
  }
  for (int c = 0; c < ncomp; ++c) {
    Ctx ctx(g, tol, budget);
    ctx.nbr = nbr;
    ctx.compat = compat;
    for (int i = 0; i < k; ++i) if (comp[i] == c) ctx.nodes.push_back(i);
    for (int i = 0; i < k; ++i)            // restrict compat to the component
      for (int j = 0; j < k; ++j)
        if (comp[i] != c || comp[j] != c) ctx.compat[i][j] = 0;
    // root: node of the rarest signature class (ties: smallest index)
    int root = ctx.nodes[0];
    for (int v : ctx.nodes) if (class_size[v] < class_size[root]) root = v;
    ctx.parent.assign(k, -1);
    std::vector<char> seen(k, 0);
    ctx.order.push_back(root);
    seen[root] = 1;
    for (size_t a = 0; a < ctx.order.size(); ++a) {
      const int u = ctx.order[a];
      for (int v : nbr[u])
        if (!seen[v]) { seen[v] = 1; ctx.parent[v] = u; ctx.order.push_back(v); }
    }
    ctx.phi.assign(k, -1);
    ctx.best.resize(k);
    for (int v : ctx.nodes) ctx.best[v] = v;   // identity is always valid (p = 0)
    ctx.dfs(0, 0, (int)ctx.nodes.size());
    if (!ctx.complete) {
      // budget exhausted: on a tree, the identical-branch search gives a
      // max-p involution in O(n log n); used if it beats the partial enumeration and passes
      // Definition 2 on the component
      size_t twice_edges = 0;
      for (int v : ctx.nodes) twice_edges += nbr[v].size();
      if (twice_edges == 2 * (ctx.nodes.size() - 1)) {
        std::vector<int> tphi(k);
        std::iota(tphi.begin(), tphi.end(), 0);
        const int tp = tree_involution(g, ctx.nodes, nbr, tol, tphi);
        bool ok = tp > ctx.best_p;
        for (size_t a = 0; ok && a < ctx.nodes.size(); ++a) {
          const int i = ctx.nodes[a];
          ok = std::fabs(g.s[i] - g.s[tphi[i]]) <= tol && tphi[tphi[i]] == i;
          for (size_t b = a + 1; ok && b < ctx.nodes.size(); ++b) {
            const int j = ctx.nodes[b];
            ok = std::fabs(g.w(i, j) - g.w(tphi[i], tphi[j])) <= tol;
          }
        }
        if (ok) {
          ctx.best_p = tp;
          for (int v : ctx.nodes) ctx.best[v] = tphi[v];
        }
      }
    }
    for (int v : ctx.nodes) res.phi[v] = ctx.best[v];
    res.p += ctx.best_p;
    res.steps += ctx.steps;
    res.complete = res.complete && ctx.complete;
  }
  return res;
}

}  // namespace gft
