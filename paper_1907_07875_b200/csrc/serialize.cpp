// serialize.cpp — plan persistence: the complete factorisation (butterfly ops, leaves with
// their matrices / Givens layers, right Haar stages, realised basis, statistics) as a
// versioned little-endian byte string, so that a plan can be rebuilt without the
// involution search and the eigensolves.  Kernels are regenerated from the loaded plan; the
// generator is deterministic, so they get the same names (source hashes) and hit the same
// AOT / NVRTC cubin caches.
#include <cstring>

#include "../../include/gft.h"
#include "plan.hpp"

namespace gft {
namespace {

constexpr char kMagic[8] = {'G', 'F', 'T', 'P', 'L', 'A', 'N', '1'};
constexpr uint32_t kVersion = 1;

struct Writer {
  std::vector<uint8_t> b;
  template <class T>
  void pod(const T& v) {
    const uint8_t* p = reinterpret_cast<const uint8_t*>(&v);
    b.insert(b.end(), p, p + sizeof(T));
  }
  template <class T>
  void vec(const std::vector<T>& v) {
    pod<uint64_t>(v.size());
    for (const T& x : v) pod(x);
  }
};

struct Reader {
  const uint8_t* p;
  size_t n, off = 0;
  template <class T>
  T pod() {
    if (off + sizeof(T) > n) fail(GFT_ERR_INVALID_ARG, "serialized plan: truncated");
    T v;
    std::memcpy(&v, p + off, sizeof(T));
    off += sizeof(T);
    return v;
  }
  template <class T>
  std::vector<T> vec(size_t max_count) {
    const uint64_t c = pod<uint64_t>();
    if (c > max_count || off + c * sizeof(T) > n) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad array length");
    std::vector<T> v(c);
    for (auto& x : v) x = pod<T>();
    return v;
  }
};

void check_index(int v, int hi, const char* what) {
  if (v < 0 || v >= hi) fail(GFT_ERR_INVALID_ARG, std::string("serialized plan: ") + what + " out of range");
}

}  // namespace

std::vector<uint8_t> serialize_plan(const Plan& P) {
  Writer w;
  w.b.insert(w.b.end(), kMagic, kMagic + 8);
  w.pod(kVersion);
  w.pod<int32_t>(P.n);
  w.pod<uint64_t>(P.ops.size());
  for (const Op& op : P.ops) {
    w.pod<int32_t>(op.kind);
    w.pod<int32_t>(op.a);
    w.pod<int32_t>(op.b);
    w.pod<int32_t>(op.m);
    w.pod<int32_t>(op.level);
  }
  w.pod<uint64_t>(P.leaves.size());
  for (const Leaf& lf : P.leaves) {
    w.pod<int32_t>(lf.k);
    w.vec(lf.pos);
    w.vec(lf.slot);
    w.vec(lf.lam);
    w.vec(lf.V);
    w.vec(lf.M);
    w.pod<int32_t>(lf.level);
    w.pod<int32_t>(lf.right);
    w.pod<int32_t>(lf.side);
    w.vec(lf.pair);
    w.pod<int32_t>(lf.approx ? 1 : 0);
    w.pod<uint64_t>(lf.layers.size());
    for (const auto& layer : lf.layers) {
      w.pod<uint64_t>(layer.size());
      for (const Givens& g : layer) {
        w.pod<int32_t>(g.p);
        w.pod<int32_t>(g.q);
        w.pod<double>(g.c);
        w.pod<double>(g.s);
      }
    }
    w.vec(lf.perm);
    w.vec(lf.scale);
  }
  w.pod<uint64_t>(P.rights.size());
  for (const RightStage& r : P.rights) {
    w.pod<int32_t>(r.leafE);
    w.pod<int32_t>(r.leafF);
    w.vec(r.rE);
    w.vec(r.rF);
    w.vec(r.sign);
  }
  w.pod<uint64_t>(P.post.size());
  for (const PostUnit& u : P.post) {
    w.pod<int32_t>(u.p);
    w.pod<int32_t>(u.q);
    w.pod<int32_t>(u.s);
  }
  w.vec(P.dexp);
  w.vec(P.lambda);
  w.vec(P.U);
  w.vec(P.L);
  w.pod<int32_t>(P.depth);
  w.vec(P.units_per_level);
  for (int v : {P.n_units, P.n_fix, P.n_vz_total, P.max_leaf, P.n_clusters, P.n_post, P.n_givens,
                P.n_approx_scale, P.n_approx_leaves})
    w.pod<int32_t>(v);
  w.pod<int64_t>(P.sum_k2);
  w.pod<int64_t>(P.sum_kk1);
  w.pod<double>(P.residual);
  w.pod<double>(P.orth_error);
  return w.b;
}

Plan deserialize_plan(const uint8_t* buf, size_t size, size_t* consumed) {
  Reader r{buf, size};
  if (size < 12 || std::memcmp(buf, kMagic, 8) != 0) fail(GFT_ERR_INVALID_ARG, "not a serialized gft plan");
  r.off = 8;
  if (r.pod<uint32_t>() != kVersion) fail(GFT_ERR_UNSUPPORTED, "serialized plan: unknown format version");
  Plan P;
  P.n = r.pod<int32_t>();
  if (P.n < 1 || P.n > 8192) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad n");
  const size_t n = (size_t)P.n, nn = n * n, big = 1u << 26;
  const uint64_t nops = r.pod<uint64_t>();
  if (nops > 4 * n) fail(GFT_ERR_INVALID_ARG, "serialized plan: too many ops");
  for (uint64_t i = 0; i < nops; ++i) {
    Op op;
    op.kind = (Op::Kind)r.pod<int32_t>();
    op.a = r.pod<int32_t>();
    op.b = r.pod<int32_t>();
    op.m = r.pod<int32_t>();
    op.level = r.pod<int32_t>();
    if (op.kind != Op::UNIT && op.kind != Op::FIX) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad op kind");
    check_index(op.a, P.n, "op position");
    if (op.kind == Op::UNIT) check_index(op.b, P.n, "op position");
    P.ops.push_back(op);
  }
  const uint64_t nleaves = r.pod<uint64_t>();
  if (nleaves > n) fail(GFT_ERR_INVALID_ARG, "serialized plan: too many leaves");
  size_t covered = 0;
  for (uint64_t l = 0; l < nleaves; ++l) {
    Leaf lf;
    lf.k = r.pod<int32_t>();
    if (lf.k < 1 || lf.k > P.n) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad leaf size");
    const size_t k = (size_t)lf.k;
    lf.pos = r.vec<int>(k);
    lf.slot = r.vec<int>(k);
    lf.lam = r.vec<double>(k);
    lf.V = r.vec<double>(k * k);
    lf.M = r.vec<double>(k * k);
    if (lf.pos.size() != k || lf.slot.size() != k || lf.lam.size() != k || lf.V.size() != k * k ||
        lf.M.size() != k * k)
      fail(GFT_ERR_INVALID_ARG, "serialized plan: leaf arrays inconsistent");
    for (int v : lf.pos) check_index(v, P.n, "leaf position");
    for (int v : lf.slot) check_index(v, P.n, "leaf slot");
    lf.level = r.pod<int32_t>();
    lf.right = r.pod<int32_t>();
    lf.side = r.pod<int32_t>();
    lf.pair = r.vec<int>(k);
    lf.approx = r.pod<int32_t>() != 0;
    const uint64_t nlayers = r.pod<uint64_t>();
    if (nlayers > big) fail(GFT_ERR_INVALID_ARG, "serialized plan: too many Givens layers");
    for (uint64_t j = 0; j < nlayers; ++j) {
      const uint64_t nr = r.pod<uint64_t>();
      if (nr > k) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad Givens layer");
      std::vector<Givens> layer;
      for (uint64_t q = 0; q < nr; ++q) {
        Givens g;
        g.p = r.pod<int32_t>();
        g.q = r.pod<int32_t>();
        g.c = r.pod<double>();
        g.s = r.pod<double>();
        check_index(g.p, lf.k, "Givens index");
        check_index(g.q, lf.k, "Givens index");
        layer.push_back(g);
      }
      lf.layers.push_back(std::move(layer));
    }
    lf.perm = r.vec<int>(k);
    lf.scale = r.vec<double>(k);
    if (lf.approx && (lf.perm.size() != k || lf.scale.size() != k))
      fail(GFT_ERR_INVALID_ARG, "serialized plan: approximate leaf arrays inconsistent");
    for (int v : lf.perm) check_index(v, lf.k, "leaf permutation");
    covered += k;
    P.leaves.push_back(std::move(lf));
  }
  if (covered != n) fail(GFT_ERR_INVALID_ARG, "serialized plan: leaves do not cover the positions");
  // every position is read by exactly one leaf and every coefficient slot written by exactly
  // one: the sizes summing to n is not enough (a duplicate would compile into a kernel that
  // reads one position twice and leaves another coefficient unwritten)
  {
    std::vector<char> seen_pos(n, 0), seen_slot(n, 0);
    for (const Leaf& lf : P.leaves)
      for (int i = 0; i < lf.k; ++i) {
        if (seen_pos[lf.pos[i]]++) fail(GFT_ERR_INVALID_ARG, "serialized plan: position read by two leaves");
        if (seen_slot[lf.slot[i]]++) fail(GFT_ERR_INVALID_ARG, "serialized plan: coefficient slot written twice");
      }
  }
  for (const Leaf& lf : P.leaves)
    for (int v : lf.pair)
      if (v < -1 || v >= lf.k) fail(GFT_ERR_INVALID_ARG, "serialized plan: bad right-stage pair index");
  const uint64_t nr = r.pod<uint64_t>();
  if (nr > n) fail(GFT_ERR_INVALID_ARG, "serialized plan: too many right stages");
  for (uint64_t i = 0; i < nr; ++i) {
    RightStage rs;
    rs.leafE = r.pod<int32_t>();
    rs.leafF = r.pod<int32_t>();
    check_index(rs.leafE, (int)P.leaves.size(), "right-stage leaf");
    check_index(rs.leafF, (int)P.leaves.size(), "right-stage leaf");
    rs.rE = r.vec<int>(n);
    rs.rF = r.vec<int>(n);
    rs.sign = r.vec<int>(n);
    if (rs.rE.size() != rs.rF.size() || rs.sign.size() != rs.rE.size())
      fail(GFT_ERR_INVALID_ARG, "serialized plan: right-stage arrays inconsistent");
    for (size_t j = 0; j < rs.rE.size(); ++j) {
      check_index(rs.rE[j], P.leaves[rs.leafE].k, "right-stage output");
      check_index(rs.rF[j], P.leaves[rs.leafF].k, "right-stage output");
    }
    P.rights.push_back(std::move(rs));
  }
  const uint64_t np = r.pod<uint64_t>();
  if (np > n) fail(GFT_ERR_INVALID_ARG, "serialized plan: too many coefficient butterflies");
  for (uint64_t i = 0; i < np; ++i) {
    PostUnit u;
    u.p = r.pod<int32_t>();
    u.q = r.pod<int32_t>();
    u.s = r.pod<int32_t>();
    check_index(u.p, P.n, "coefficient slot");
    check_index(u.q, P.n, "coefficient slot");
    P.post.push_back(u);
  }
  P.dexp = r.vec<int>(n);
  P.lambda = r.vec<double>(n);
  P.U = r.vec<double>(nn);
  P.L = r.vec<double>(nn);
  if (P.dexp.size() != n || P.lambda.size() != n || P.U.size() != nn || P.L.size() != nn)
    fail(GFT_ERR_INVALID_ARG, "serialized plan: basis arrays inconsistent");
  P.depth = r.pod<int32_t>();
  P.units_per_level = r.vec<int>(64);
  if (P.depth < 0 || P.depth > (int)P.units_per_level.size())
    fail(GFT_ERR_INVALID_ARG, "serialized plan: bad depth");
  for (const Leaf& lf : P.leaves) {
    if (lf.right < -1 || lf.right >= (int)P.rights.size() || (lf.side != 0 && lf.side != 1))
      fail(GFT_ERR_INVALID_ARG, "serialized plan: bad right-stage membership");
    if (lf.right >= 0 && (int)lf.pair.size() != lf.k)
      fail(GFT_ERR_INVALID_ARG, "serialized plan: right-stage leaf without pair map");
  }
  int* stats[] = {&P.n_units, &P.n_fix, &P.n_vz_total, &P.max_leaf, &P.n_clusters, &P.n_post, &P.n_givens,
                  &P.n_approx_scale, &P.n_approx_leaves};
  for (int* s : stats) *s = r.pod<int32_t>();
  P.sum_k2 = r.pod<int64_t>();
  P.sum_kk1 = r.pod<int64_t>();
  P.residual = r.pod<double>();
  P.orth_error = r.pod<double>();
  if (consumed) *consumed = r.off;
  else if (r.off != size) fail(GFT_ERR_INVALID_ARG, "serialized plan: trailing bytes");
  return P;
}

}  // namespace gft
