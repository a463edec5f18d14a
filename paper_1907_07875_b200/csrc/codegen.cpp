// codegen.cpp — per-plan CUDA source generation.
//
// Every graph-dependent quantity of the fast GFT becomes code: the Haar units
// (eq:B_phi) become register add/sub pairs, the folded sub-GFT
// coefficients (Theorem 4 leaves, 1/sqrt2 absorbed as PAPER.md:158
// suggests) become FFMA/DFMA immediates, and the ascending-eigenvalue permutation
// becomes the register index the result is written to.  There are no
// tables to fetch on the device: per signal the kernel executes exactly
// 2*units + sum_k k^2 arithmetic instructions (+ explicit scale fixes, if any).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "../../include/gft.h"
#include "kernels.hpp"

namespace gft {

// The device skeletons, embedded at build time (build.py writes *_inc.h).
static const char* kSkeleton =
#include "skeleton_inc.h"
    ;
static const char* kSkeletonTC =
#include "skeleton_tc_inc.h"
    ;
static const char* kSkeletonTC2 =
#include "skeleton_tc2_inc.h"
    ;
static const char* kSkeletonTC3 =
#include "skeleton_tc3_inc.h"
    ;
static const char* kSkeletonDense =
#include "skeleton_dense_inc.h"
    ;

KernelCfg choose_cfg(int n, int dtype, int64_t work, const CfgOverride* ov, int kind) {
  KernelCfg c;
  c.n = n;
  c.elem = dtype == GFT_F64 ? 8 : 4;
  const int row = n * c.elem;
  if (row % 16 == 0) {
    c.mode = 0;
    c.vec = 16 / c.elem;
    if (row % 128 == 0) { c.boxc = 128 / c.elem; c.swz_mask = 7; }
    else if (row % 64 == 0) { c.boxc = 64 / c.elem; c.swz_mask = 3; }
    else if (row % 32 == 0) { c.boxc = 32 / c.elem; c.swz_mask = 1; }
    else { c.boxc = n; c.swz_mask = 0; }   // 16*odd bytes: odd chunk pitch, conflict-free
    // rows of 16/32/64 bytes: TMA boxes that narrow move few bytes per request (n = 8 f32:
    // ~5.4 TB/s whatever the geometry, tools/gpu_r01_persist_cfg1.sh).  Packed view instead:
    // [batch / g, g*n] with g = 128 / row, one 128-byte box row = g signals, 128B swizzle --
    // thread-per-row 16-byte LDS stay conflict-free (8 threads of a phase cover two box rows
    // whose chunk parities the swizzle separates).  GFT_PACK=0 disables.
    const char* pk = getenv("GFT_PACK");
    const bool pack_on = pk ? pk[0] != '0' : (row <= 32);
    if (row < 128 && 128 % row == 0 && pack_on) {
      c.mode = 2;
      c.pack = 128 / row;
      c.boxc = n;
      c.swz_mask = 7;
    }
  } else {
    // unaligned row pitch: 1-D bulk copies of whole tiles (TMA copies of a 4-signal super-row
    // view were measured 3% slower on cfg3 in round 1 and removed)
    c.mode = 1;
    c.pack = 1;
    c.boxc = n;
    c.swz_mask = 0;
    // odd row pitch in vector units makes thread-per-row accesses conflict-free
    c.vec = (c.elem == 4 && n % 2 == 0) ? 2 : 1;
  }
  // Default geometry for an (n, dtype) without a tuning entry: the largest warp tile of at
  // most 8 KiB, double-buffered, as many warps (<= 12) as ~150 KiB of SMEM holds -- one
  // persistent CTA per SM.  The measured geometry search of gft_plan_tune on graphs outside
  // the table picked 4-8 KiB tiles with 12 warps (n = 40, 48: +15%, +36% over the previous
  // default of >= 8 KiB tiles and <= 8 warps; tools/tune_probe.py).
  c.R = 1;
  while (c.R < 8 && 2 * c.tile_bytes() <= 8192) c.R *= 2;
  c.stages = 2;
  c.warps = std::max(2, std::min(12, (150 * 1024) / (c.stages * c.tile_bytes())));
  // measured geometry for this (n, dtype) if the tuning table has one (tools/gpu_autotune.py)
  int tR, tS, tW, tP, tO;
  if (tuned_geometry(n, dtype, work, kind, tR, tS, tW, tP, tO)) {
    c.R = tR;
    c.stages = tS;
    c.warps = tW;
    c.pace_ns = tP;
    c.obuf = tO;
  }
  // tuning knobs for experiments (GFT_TUNE_R / _STAGES / _WARPS); defaults above
  auto env_int = [](const char* k, int v) { const char* e = getenv(k); return (e && *e) ? atoi(e) : v; };
  c.R = std::max(1, std::min(8, env_int("GFT_TUNE_R", c.R)));
  c.stages = std::max(2, std::min(8, env_int("GFT_TUNE_STAGES", c.stages)));
  c.warps = std::max(1, std::min(16, env_int("GFT_TUNE_WARPS", c.warps)));
  c.pace_ns = std::max(0, std::min(100000, env_int("GFT_PACE_NS", c.pace_ns)));
  c.obuf = std::max(0, std::min(2, env_int("GFT_FMA_OBUF", c.obuf)));   // experiments
  if (ov) {
    if (ov->R > 0) c.R = std::min(8, ov->R);
    if (ov->stages > 0) c.stages = std::max(2, std::min(8, ov->stages));
    if (ov->warps > 0) c.warps = std::min(16, ov->warps);
    if (ov->pace_ns >= 0) c.pace_ns = std::min(100000, ov->pace_ns);
  }
  // the 128B swizzle atom needs 1024-byte aligned tile buffers; TMA boxes hold <= 256 rows
  while (c.mode == 2 && c.swz_mask && c.tile_bytes() % 1024 != 0 && c.R < 8) c.R *= 2;
  if (c.smem_bytes() > 227 * 1024) c.obuf = 0;
  if (c.smem_bytes() > 227 * 1024) c.stages = 2;
  if (c.smem_bytes() > 227 * 1024) c.warps = 2;
  return c;
}

namespace {

std::string lit(double v, int dtype) {
  char buf[64];
  if (dtype == GFT_F64) {
    std::snprintf(buf, sizeof buf, "%a", v);
    return std::string("(") + buf + ")";
  }
  std::snprintf(buf, sizeof buf, "%af", (double)(float)v);
  return std::string("(") + buf + ")";
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : s) { h ^= ch; h *= 1099511628211ull; }
  return h;
}

// out = sum_t coef[t] * in[idx[t]]  as an FMA chain (exact zeros skipped)
void emit_dot(std::ostringstream& o, const std::string& out, const std::vector<double>& coef,
              const std::vector<std::string>& in, int dtype) {
  bool first = true;
  std::string fma = dtype == GFT_F64 ? "__fma_rn" : "__fmaf_rn";
  std::string mul = dtype == GFT_F64 ? "__dmul_rn" : "__fmul_rn";
  o << "  { elem_t acc = (elem_t)0;";
  for (size_t t = 0; t < coef.size(); ++t) {
    if (coef[t] == 0.0) continue;
    if (first) { o << " acc = " << mul << "(" << in[t] << ", " << lit(coef[t], dtype) << ");"; first = false; }
    else o << " acc = " << fma << "(" << in[t] << ", " << lit(coef[t], dtype) << ", acc);";
  }
  o << " " << out << " = acc; }\n";
}

std::string xs(const char* arr, int i) { return std::string(arr) + "[" + std::to_string(i) + "]"; }

// Transform direction of a fast kernel: which index a leaf reads / writes and whether the
// butterfly network runs before (forward) and / or reversed after (inverse) the leaves.
//   FWD:    x -> units -> y[slot[r]] = sum_c M[r][c] x[pos[c]]
//   INV:    y[pos[c]] = sum_r M[r][c] x[slot[r]] -> reverse units
//   FILTER: x -> units -> y[pos[c]] = sum_c' F[c][c'] x[pos[c']] -> reverse units, with the
//           leaf matrix field holding F = M^T diag(h) M (fused U diag(h) U^T)
enum Dir { DIR_FWD = 0, DIR_INV = 1, DIR_FILTER = 2 };
int in_idx(const Leaf& lf, Dir d, int i) { return d == DIR_INV ? lf.slot[i] : lf.pos[i]; }
int out_idx(const Leaf& lf, Dir d, int o) { return d == DIR_FWD ? lf.slot[o] : lf.pos[o]; }
double leaf_coef(const Leaf& lf, Dir d, int o, int i) {
  return d == DIR_INV ? lf.M[(size_t)i * lf.k + o] : lf.M[(size_t)o * lf.k + i];
}

// fp32 Haar unit as ONE packed FFMA2 (sm_100 fma.rn.f32x2 with both scalar operands broadcast):
// {P, P} * {pm.lo, pm.hi} + {Q, Q}, pm = {1, -1} or {-1, 1}; fma(P, +-1, Q) is the exactly rounded
// Q +- P, so the result is bit-identical to two FADDs and the butterfly costs half the issue
// slots (the outputs form the destination register pair; the inputs need no packing).
// Opt-in (GFT_FFMA2_UNITS=1), tcgen05 kernels' stager / drainer only: timed alone it lifts the
// IO-split kernels 0.4-1.3% (cfg5b, right-Haar 64|64), but inside the headline step, interleaved
// in one process, it is 0.2-0.5% SLOWER (the pair destinations cost ~140 extra MOVs per row
// elsewhere); in the CUDA-core FMA skeleton it cost up to 18% (cfg2 fwd 1.036 -> 0.851, cfg4 inv
// 1.047 -> 0.872, cfg5a filter 0.975 -> 0.927) and is never used there
// (profiles/r02/r02_ffma2_units.log).
bool ffma2_units() {
  const char* e = getenv("GFT_FFMA2_UNITS");
  return e && e[0] == '1';
}
// (dst0, dst1) <- (Q + pm.lo * P, Q + pm.hi * P); minus_first: pm = {-1, 1} instead of {1, -1}
std::string unit2(const std::string& d0, const std::string& d1, const std::string& P_, const std::string& Q_,
                  bool minus_first) {
  return "{ unsigned long long d_; asm(\"{ .reg .b64 t0, t1; mov.b64 t0, {%1, %1}; mov.b64 t1, {%2, %2}; "
         "fma.rn.f32x2 %0, t1, %3, t0; }\" : \"=l\"(d_) : \"f\"(" + Q_ + "), \"f\"(" + P_ + "), \"l\"(" +
         (minus_first ? "0x3F800000BF800000ull" : "0xBF8000003F800000ull") +
         ")); asm(\"mov.b64 {%0, %1}, %2;\" : \"=f\"(" + d0 + "), \"=f\"(" + d1 + ") : \"l\"(d_)); }";
}
std::string unit_ab(const char* arr, int a, int b) {   // (x_a, x_b) <- (x_a + x_b, x_a - x_b)
  const std::string A = xs(arr, a), B = xs(arr, b);
  return unit2(A, B, B, A, false);
}

void emit_units_elem(std::ostringstream& o, const Plan& P, const char* arr, bool reverse, int dtype) {
  o << "  { elem_t a_, b_;\n";
  int lvl = -1;
  auto one = [&](const Op& op) {
    if (op.level != lvl) {
      lvl = op.level;
      o << "  // ---- butterfly level " << lvl << (reverse ? " (reverse)" : "") << "\n";
    }
    if (op.kind == Op::UNIT)
      o << "  a_ = " << arr << "[" << op.a << "]; b_ = " << arr << "[" << op.b << "]; " << arr << "["
        << op.a << "] = a_ + b_; " << arr << "[" << op.b << "] = a_ - b_;\n";
    else
      o << "  " << arr << "[" << op.a << "] = " << arr << "[" << op.a << "] * "
        << lit(std::pow(2.0, 0.5 * op.m), dtype) << ";  // equalise deferred scale\n";
  };
  if (!reverse) for (const Op& op : P.ops) one(op);
  else for (auto it = P.ops.rbegin(); it != P.ops.rend(); ++it) one(*it);
  o << "  (void)a_; (void)b_; }\n";
}

// Approximate leaf (NEXT-4): U_hat_l = G_1...G_J Pi applied as register
// rotations in "scaled" (fast-Givens) form: each position carries a plan-time scale d_c with
// value = d_c * register, so a rotation (c, s) on (p, q) is two FFMAs
//   r_p <- r_p - (s d_q / (c d_p)) r_q,   r_q <- r_q + (s d_p / (c d_q)) r_p(old),
//   d_p <- c d_p,  d_q <- c d_q
// (|s/c| <= 1 for Jacobi angles).  The 2^(-d/2) Haar scale starts d (forward) or ends it
// (inverse); one multiply per output applies d.  Forward: G_1^T ... G_J^T then
// y[slot[r]] = x[pos[perm[r]]]; inverse: the transpose in reverse order.
void emit_leaf_givens(std::ostringstream& o, const Leaf& lf, size_t l, Dir d, int dtype) {
  const std::string fma = dtype == GFT_F64 ? "__fma_rn" : "__fmaf_rn";
  const std::string mul = dtype == GFT_F64 ? "__dmul_rn" : "__fmul_rn";
  size_t nrot = 0;
  for (const auto& layer : lf.layers) nrot += layer.size();
  o << "  // ---- leaf " << l << " (k=" << lf.k << ", approximate: " << lf.layers.size() << " Givens layers, "
    << nrot << " rotations, scaled form)\n  { elem_t a_;\n";
  const char* arr = d == DIR_FWD ? "x" : "y";
  auto X = [&](int c) { return std::string(arr) + "[" + std::to_string(lf.pos[c]) + "]"; };
  std::vector<double> ds(lf.k, 1.0);
  if (d == DIR_FWD) ds = lf.scale;
  auto rot = [&](const Givens& g, bool transpose) {
    // G^T: (p, q) <- (c a - s b, s a + c b);  G: (p, q) <- (c a + s b, -s a + c b)
    const double sg = transpose ? g.s : -g.s;
    const double t1 = sg * ds[g.q] / (g.c * ds[g.p]), t2 = sg * ds[g.p] / (g.c * ds[g.q]);
    o << "  a_ = " << X(g.p) << "; " << X(g.p) << " = " << fma << "(" << lit(-t1, dtype) << ", " << X(g.q) << ", a_); "
      << X(g.q) << " = " << fma << "(" << lit(t2, dtype) << ", a_, " << X(g.q) << ");\n";
    ds[g.p] *= g.c;
    ds[g.q] *= g.c;
    for (int c : {g.p, g.q})
      if (ds[c] < 0x1p-30) {   // keep registers far from overflow (after ~60 layers)
        o << "  " << X(c) << " = " << mul << "(" << X(c) << ", " << lit(ds[c], dtype) << ");\n";
        ds[c] = 1.0;
      }
  };
  auto apply = [&](int c, double f, const std::string& dst, const std::string& src) {
    if (f == 1.0) o << "  " << dst << " = " << src << ";\n";
    else o << "  " << dst << " = " << mul << "(" << src << ", " << lit(f, dtype) << ");\n";
  };
  if (d == DIR_FWD) {
    for (const auto& layer : lf.layers)
      for (const Givens& g : layer) rot(g, true);
    for (int r = 0; r < lf.k; ++r)
      apply(lf.perm[r], ds[lf.perm[r]], "y[" + std::to_string(lf.slot[r]) + "]", X(lf.perm[r]));
  } else {
    for (int r = 0; r < lf.k; ++r) o << "  " << X(lf.perm[r]) << " = x[" << lf.slot[r] << "];\n";
    for (auto it = lf.layers.rbegin(); it != lf.layers.rend(); ++it)
      for (const Givens& g : *it) rot(g, false);
    for (int c = 0; c < lf.k; ++c) apply(c, ds[c] * lf.scale[c], X(c), X(c));
  }
  o << "  (void)a_; }\n";
}

// stream: every leaf output goes straight to this thread's SMEM row (SOUT) instead of a y
// register, so only the input row is live during the leaves (wide rows, see generate_kernel)
std::string sout(int idx) { return "SOUT(" + std::to_string(idx) + ")"; }

void emit_leaf_fma(std::ostringstream& o, const Leaf& lf, size_t l, Dir d, int dtype, bool stream = false) {
  if (lf.approx && d != DIR_FILTER) {   // the fused filter keeps F = M^T diag(h) M dense
    emit_leaf_givens(o, lf, l, d, dtype);
    if (stream)
      for (int r = 0; r < lf.k; ++r) {
        const int oi = out_idx(lf, d, r);
        o << "  " << sout(oi) << " = y[" << oi << "];\n";
      }
    return;
  }
  o << "  // ---- leaf " << l << " (k=" << lf.k << ")\n";
  std::vector<std::string> in(lf.k);
  for (int i = 0; i < lf.k; ++i) in[i] = xs("x", in_idx(lf, d, i));
  for (int r = 0; r < lf.k; ++r) {
    std::vector<double> coef(lf.k);
    for (int i = 0; i < lf.k; ++i) coef[i] = leaf_coef(lf, d, r, i);
    const int oi = out_idx(lf, d, r);
    emit_dot(o, stream ? sout(oi) : xs("y", oi), coef, in, dtype);
  }
}

// Right Haar stages on the coefficients, type T of the array:
//   forward (after the leaves):  y_p <- a + b,  y_q <- s (a - b)
//   inverse (before the leaves): x_p <- y_p + s y_q,  x_q <- y_p - s y_q   (transpose)
void emit_post_units(std::ostringstream& o, const Plan& P, const char* arr, bool inverse, const char* T,
                     bool f32 = true) {
  if (P.post.empty()) return;
  o << "  // ---- right Haar stage (" << P.post.size() << " coefficient pairs)\n  { " << T << " a_, b_;\n";
  for (const PostUnit& u : P.post) {
    if (f32 && ffma2_units()) {
      const std::string A = xs(arr, u.p), B = xs(arr, u.q);
      // forward (a+b, s(a-b)); inverse (a + s b, a - s b)
      if (!inverse) o << "  " << (u.s > 0 ? unit2(A, B, B, A, false) : unit2(A, B, A, B, false)) << "\n";
      else o << "  " << (u.s > 0 ? unit2(A, B, B, A, false) : unit2(A, B, B, A, true)) << "\n";
      continue;
    }
    o << "  a_ = " << arr << "[" << u.p << "]; b_ = " << arr << "[" << u.q << "]; ";
    if (!inverse)
      o << arr << "[" << u.p << "] = a_ + b_; " << arr << "[" << u.q << "] = "
        << (u.s > 0 ? "a_ - b_" : "b_ - a_") << ";\n";
    else
      o << arr << "[" << u.p << "] = " << (u.s > 0 ? "a_ + b_" : "a_ - b_") << "; " << arr << "[" << u.q
        << "] = " << (u.s > 0 ? "a_ - b_" : "a_ + b_") << ";\n";
  }
  o << "  (void)a_; (void)b_; }\n";
}

void emit_fast(std::ostringstream& o, const Plan& P, int dtype, Dir d, bool stream = false) {
  if (d == DIR_FILTER && !P.post.empty()) fail(GFT_ERR_COMPILE, "filter plan with right Haar stages");
  if (stream) o << "  elem_t y[GFT_N];\n";
  if (d != DIR_INV) emit_units_elem(o, P, "x", false, dtype);
  if (d == DIR_INV) emit_post_units(o, P, "x", true, "elem_t", false);
  for (size_t l = 0; l < P.leaves.size(); ++l) emit_leaf_fma(o, P.leaves[l], l, d, dtype, stream);
  const bool after = (d == DIR_FWD && !P.post.empty()) || (d != DIR_FWD && !P.ops.empty());
  if (stream && after) o << "  load_row(buf_, row_, y);   // leaf outputs back for the stages after the leaves\n";
  if (d == DIR_FWD) emit_post_units(o, P, "y", false, "elem_t", false);
  if (d != DIR_FWD) emit_units_elem(o, P, "y", true, dtype);
  if (stream && after) o << "  store_row(buf_, row_, y);\n";
}

void emit_dense(std::ostringstream& o, const Plan& P, int dtype, bool forward, bool stream = false) {
  const int n = P.n;
  std::vector<std::string> in(n);
  for (int i = 0; i < n; ++i) in[i] = xs("x", i);
  for (int k = 0; k < n; ++k) {
    std::vector<double> coef(n);
    for (int i = 0; i < n; ++i)
      coef[i] = forward ? P.U[(size_t)i * n + k] : P.U[(size_t)k * n + i];
    emit_dot(o, stream ? sout(k) : xs("y", k), coef, in, dtype);
  }
}

// ------------------------------------------------------------------------------------
// Tensor-core (tcgen05, 3xTF32) variant for plans with large leaves
// ------------------------------------------------------------------------------------
struct TcLeaf {
  int leaf, k, kp8, kp32, np;
  int hi_col, lo_col, d_col;     // TMEM columns
  int bhi_off, blo_off;          // byte offsets in the SMEM B region
};

int ru(int v, int m) { return (v + m - 1) / m * m; }

// host-side cvt.rna.tf32.f32: round to nearest (ties away) on the low 13 mantissa bits
float tf32_rna_host(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  if ((u & 0x7f800000u) == 0x7f800000u) return v;
  u = (u + 0x1000u) & ~0x1fffu;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Approximate leaves (J Givens layers) are cheap in FFMAs but the straight-line rotation code
// costs one issue slot per FFMA: past ~32 n instructions per signal the CUDA-core kernel is
// issue-bound (n = 64: J = 20, ~22 n, runs at 0.93 of HBM; J = 40, ~42 n, at 0.52 --
// ncu: issue active 60%, no_instruction stalls on the 2600-instruction body).  Such plans
// multiply each approximate leaf out (M = the folded U_hat_l^T, the same linear map) and run
// it as a tcgen05 leaf, which is HBM-bound at any k.  GFT_APPROX_TC=0/1 forces the choice.
static bool approx_on_tc(const Plan& P, int dtype) {
  if (P.n_approx_leaves == 0 || dtype != GFT_F32) return false;
  const char* e = getenv("GFT_APPROX_TC");
  if (e && *e) return e[0] != '0';
  const int64_t instr = 2 * (int64_t)P.n_units + P.sum_k2 + 2 * (int64_t)P.n_givens + P.n_approx_scale +
                        2 * (int64_t)P.n_post;
  return instr > 32 * (int64_t)P.n;
}

// leaves that go to the tensor core when they fit: exact leaves of k >= 32 (below that the
// k^2 FFMAs are cheaper than the MMA chain), approximate leaves of k >= 16 when densified
static bool tc_candidate(const Plan& P, const Leaf& lf, bool approx_tc) {
  return lf.approx ? (approx_tc && lf.k >= 16) : lf.k >= 32;
}

// pair: CTA-pair (cta_group::2) variant -- each CTA stores half of every B operand.
bool plan_tc(const Plan& P, int dtype, int stages, bool pair, std::vector<TcLeaf>& out, int& tmem_cols,
             int& b_bytes) {
  out.clear();
  if (dtype != GFT_F32 || P.n % 4 != 0 || P.n > 256) return false;   // 16-byte rows for TMA
  const bool atc = approx_on_tc(P, dtype);
  std::vector<int> order;
  for (int l = 0; l < (int)P.leaves.size(); ++l)
    if (tc_candidate(P, P.leaves[l], atc)) order.push_back(l);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return P.leaves[a].k > P.leaves[b].k; });
  const int tile = 128 * ((P.n + 31) / 32 * 32) * 4;   // padded to whole TMA boxes
  int cols = 0, bytes = 0;
  for (int l : order) {
    TcLeaf t;
    t.leaf = l;
    t.k = P.leaves[l].k;
    t.kp8 = ru(t.k, 8);
    t.kp32 = ru(t.k, 32);
    t.np = ru(t.k, 16);
    const int need = 2 * ru(t.kp8, 32) + ru(t.np, 32);
    const int bsz = 2 * t.np * t.kp32 * 4 / (pair ? 2 : 1);
    if (cols + need > 512 || stages * tile + bytes + bsz + 2048 > 227 * 1024 || t.np > 256) continue;
    t.hi_col = cols;
    t.lo_col = cols + ru(t.kp8, 32);
    t.d_col = cols + 2 * ru(t.kp8, 32);
    cols += need;
    t.bhi_off = bytes;
    t.blo_off = bytes + bsz / 2;
    bytes += bsz;
    out.push_back(t);
  }
  if (out.empty()) return false;
  tmem_cols = 32;
  while (tmem_cols < cols) tmem_cols *= 2;
  b_bytes = bytes;
  return true;
}

void emit_tmem_st(std::ostringstream& o, const std::string& arr, int col0, int count) {
  // split into power-of-two chunks <= 128 columns
  int c = 0;
  while (c < count) {
    int w = 128;
    while (w > count - c) w /= 2;
    o << "  asm volatile(\"tcgen05.st.sync.aligned.32x32b.x" << w << ".b32 [%0], {";
    for (int i = 0; i < w; ++i) o << (i ? ", " : "") << "%" << (i + 1);
    o << "};\" :: \"r\"(tm + " << (col0 + c) << "u)";
    for (int i = 0; i < w; ++i) o << ", \"r\"(" << arr << "[" << (c + i) << "])";
    o << " : \"memory\");\n";
    c += w;
  }
}

void emit_tmem_ld(std::ostringstream& o, const std::string& arr, int col0, int count) {
  int c = 0;
  while (c < count) {
    int w = 128;
    while (w > count - c) w /= 2;
    o << "  asm volatile(\"tcgen05.ld.sync.aligned.32x32b.x" << w << ".b32 {";
    for (int i = 0; i < w; ++i) o << (i ? ", " : "") << "%" << i;
    o << "}, [%" << w << "];\\n\\ttcgen05.wait::ld.sync.aligned;\" : ";
    for (int i = 0; i < w; ++i) o << (i ? ", " : "") << "\"=r\"(" << arr << "[" << (c + i) << "])";
    o << " : \"r\"(tm + " << (col0 + c) << "u) : \"memory\");\n";
    c += w;
  }
}

// hi/lo split of a 3xTF32 A operand (x = hi + lo exactly).  Default: hi = x with its 13 low
// mantissa bits cleared (one LOP3; the tensor core reads only the TF32 bits of the container
// anyway), lo = x - hi.  cvt.rna.tf32.f32 compiles to FSETP + IADD3 + SEL + LOP3 -- four ALU
// instructions per element on the staging critical path; the truncated hi leaves |lo| <= 2^-10
// |x| instead of 2^-11 (lo keeps 11 of its <= 13 bits: ~2^-21 |x| per element, well inside
// the 1e-5 per-signal bound).  GFT_TC_SPLIT=rna restores the rounded split (ablation).
std::string split_line(int i, const std::string& src) {
  static const bool rna = [] {
    const char* e = getenv("GFT_TC_SPLIT");
    return e && std::strcmp(e, "rna") == 0;
  }();
  const std::string h = "h[" + std::to_string(i) + "]", l = "l[" + std::to_string(i) + "]";
  if (rna)
    return "  " + h + " = tf32_rna(" + src + "); " + l + " = __float_as_uint(" + src + " - __uint_as_float(" + h +
           "));\n";
  return "  " + h + " = __float_as_uint(" + src + ") & 0xffffe000u; " + l + " = __float_as_uint(" + src +
         " - __uint_as_float(" + h + "));\n";
}

void emit_units(std::ostringstream& o, const Plan& P, const char* arr, bool reverse, int dtype) {
  o << "  { float a_, b_;\n";
  auto one = [&](const Op& op) {
    if (op.kind == Op::UNIT && ffma2_units())
      o << "  " << unit_ab(arr, op.a, op.b) << "\n";
    else if (op.kind == Op::UNIT)
      o << "  a_ = " << arr << "[" << op.a << "]; b_ = " << arr << "[" << op.b << "]; " << arr << "["
        << op.a << "] = a_ + b_; " << arr << "[" << op.b << "] = a_ - b_;\n";
    else
      o << "  " << arr << "[" << op.a << "] = " << arr << "[" << op.a << "] * "
        << lit(std::pow(2.0, 0.5 * op.m), dtype) << ";\n";
  };
  if (!reverse) for (const Op& op : P.ops) one(op);
  else for (auto it = P.ops.rbegin(); it != P.ops.rend(); ++it) one(*it);
  o << "  (void)a_; (void)b_; }\n";
}

void generate_tc(const Plan& P, Dir d, const std::vector<TcLeaf>& T, bool pair, std::ostringstream& o) {
  const int dtype = GFT_F32;
  std::vector<char> is_tc(P.leaves.size(), 0);
  for (const auto& t : T) is_tc[t.leaf] = 1;
  // ---- B operands, atom order (CTA half, leaf, hi|lo, k-atom, row n, 32 k) ----
  // single CTA: all Np rows; CTA pair: rank r keeps rows [r*Np/2, (r+1)*Np/2)
  std::vector<float> B;
  const int halves = pair ? 2 : 1;
  for (int r = 0; r < halves; ++r)
    for (const auto& t : T) {
      const Leaf& lf = P.leaves[t.leaf];
      const int rows = t.np / halves;
      for (int part = 0; part < 2; ++part)
        for (int a = 0; a < t.kp32 / 32; ++a)
          for (int n = r * rows; n < (r + 1) * rows; ++n)
            for (int kk = 32 * a; kk < 32 * a + 32; ++kk) {
              float v = 0.f;
              if (n < t.k && kk < t.k)   // B[n = output][k = input]
                v = (float)leaf_coef(lf, d, n, kk);
              const float hi = tf32_rna_host(v);
              B.push_back(part == 0 ? hi : v - hi);
            }
    }
  const size_t per_cta = B.size() / halves;
  o << "#define GFT_B_FLOATS " << per_cta << "\n";
  if (pair)
    o << "__device__ __align__(16) const float gft_tcB[2][" << per_cta << "] = {\n";
  else
    o << "__device__ __align__(16) const float gft_tcB[" << per_cta << "] = {\n";
  for (size_t i = 0; i < B.size(); ++i) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%af,", (double)B[i]);
    o << buf << ((i % 8 == 7) ? "\n" : "");
  }
  o << "};\n";
  // pair kernel: one `staged` mbarrier per 32-column staging chunk of every tensor-core leaf
  // (the issuer starts a chunk's MMAs while the next chunk is staged); single CTA: one
  // MMA-completion mbarrier per leaf
  const bool stage_per_leaf = getenv("GFT_TC_STAGED_LEAF") != nullptr;
  const bool stage_once = getenv("GFT_TC_STAGED_ONCE") != nullptr;
  int nstaged = 0;
  for (const auto& t : T) nstaged += stage_per_leaf ? 1 : (t.kp8 + 31) / 32;
  if (stage_once) nstaged = 1;
  o << "#define GFT_NTC " << (pair ? nstaged : (int)T.size()) << "\n";
  int si = 0;   // running staged-barrier index (pair)
  if (pair)
    o << "static __device__ __forceinline__ void gft_tile(float (&x)[GFT_N], float (&y)[GFT_N], u32 tm,\n"
         "    u32 tmem, u32 bsm, u32 mbar, u32 staged0, u32 staged_local, u32 par, int tid, u32 rank) {\n";
  else
    o << "static __device__ __forceinline__ void gft_tile(float (&x)[GFT_N], float (&y)[GFT_N], u32 tm,\n"
         "    u32 tmem, u32 bsm, u32 mbar, u32 par, int tid) {\n";
  // ---- front: butterflies (forward) ----
  if (d != DIR_INV) emit_units(o, P, "x", false, dtype);
  if (d == DIR_FILTER && !P.post.empty()) fail(GFT_ERR_COMPILE, "filter plan with right Haar stages");
  if (d == DIR_INV) emit_post_units(o, P, "x", true, "float");
  std::ostringstream iss;   // body of gft_issue_pair (CTA-pair variant)
  for (size_t ti = 0; ti < T.size(); ++ti) {
    const TcLeaf& t = T[ti];
    const Leaf& lf = P.leaves[t.leaf];
    // ---- stage A: hi/lo split of the leaf inputs -> TMEM (this thread's lane) ----
    for (int c0 = 0; c0 < t.kp8; c0 += 32) {   // 32-column chunks keep register pressure low
      const int w = std::min(32, t.kp8 - c0);
      o << "  { u32 h[" << w << "], l[" << w << "];\n";
      for (int c = c0; c < c0 + w; ++c) {
        if (c < t.k) {
          const int src = in_idx(lf, d, c);
          o << split_line(c - c0, "x[" + std::to_string(src) + "]");
        } else {
          o << "  h[" << c - c0 << "] = 0u; l[" << c - c0 << "] = 0u;\n";
        }
      }
      emit_tmem_st(o, "h", t.hi_col + c0, w);
      emit_tmem_st(o, "l", t.lo_col + c0, w);
      o << "  }\n";
      if (pair && !stage_per_leaf && !stage_once) {
        // this chunk's k-steps, all three 3xTF32 passes, as soon as the chunk is staged
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(t.np >> 3) << 17) | (16u << 24);
        const int atom_bytes = (t.np / 2) * 128;
        o << "  signal_staged(staged0 + " << 8 * si << "u);\n";
        iss << "  mbar_wait_acq_cluster(staged_local + " << 8 * si << "u, par); tc_fence_after();\n";
        for (int pass = 0; pass < 3; ++pass) {
          const int acol = pass == 2 ? t.lo_col : t.hi_col;
          const int boff = pass == 1 ? t.blo_off : t.bhi_off;
          for (int j = c0 / 8; j < (c0 + w) / 8; ++j) {
            const int bo = boff + (j / 4) * atom_bytes + (j % 4) * 32;
            iss << "  mma_ts2(tmem + " << t.d_col << "u, tmem + " << (acol + 8 * j) << "u, smem_desc_sw128(bsm + "
                << bo << "u), " << idesc << "u, " << ((pass == 0 && j == 0) ? 0 : 1) << "u);\n";
          }
        }
        ++si;
      }
    }
    if (pair && !stage_per_leaf && !stage_once) {
      if (ti + 1 == T.size()) iss << "  tc_commit_pair(mbar);\n";
      continue;
    }
    // ---- this leaf's MMAs (issued by one thread once all lanes are staged) ----
    std::ostringstream mm;
    const uint32_t mdim = pair ? 16u : 8u;   // M = 256 (pair) or 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(t.np >> 3) << 17) | (mdim << 24);
    const int ksteps = t.kp8 / 8;
    const int atom_bytes = (t.np / (pair ? 2 : 1)) * 128;
    for (int pass = 0; pass < 3; ++pass) {
      // pass 0: A_hi B_hi, pass 1: A_hi B_lo, pass 2: A_lo B_hi
      const int acol = pass == 2 ? t.lo_col : t.hi_col;
      const int boff = pass == 1 ? t.blo_off : t.bhi_off;
      for (int j = 0; j < ksteps; ++j) {
        const int bo = boff + (j / 4) * atom_bytes + (j % 4) * 32;
        mm << (pair ? "  mma_ts2(" : "  mma_ts(") << "tmem + " << t.d_col << "u, tmem + " << (acol + 8 * j)
           << "u, smem_desc_sw128(bsm + " << bo << "u), " << idesc << "u, " << ((pass == 0 && j == 0) ? 0 : 1)
           << "u);\n";
      }
    }
    if (pair) {
      // 8 warps of the pair arrive on the leader's `staged` barrier of this leaf; the leader's
      // issuer warp (gft_issue_pair) waits for it and issues the leaf's MMAs while the next
      // leaf is being staged -- compute warps never block on the issue
      // (GFT_TC_STAGED_LEAF=1: one signal per leaf; GFT_TC_STAGED_ONCE=1: one per tile)
      const bool once = stage_once;
      if (!once || ti + 1 == T.size())
        o << "  signal_staged(staged0 + " << (once ? 0 : 8 * ti) << "u);\n";
      if (!once || ti == 0)
        iss << "  mbar_wait_acq_cluster(staged_local + " << (once ? 0 : 8 * ti) << "u, par); tc_fence_after();\n";
      iss << mm.str();
      if (ti + 1 == T.size()) iss << "  tc_commit_pair(mbar);\n";   // tracks all MMAs issued before it
    } else {
      o << "  tc_wait_st(); tc_fence_before(); named_bar(1, 128);\n";
      o << "  if (tid == 0) {\n  tc_fence_after();\n" << mm.str();
      o << "  tc_commit(mbar + " << 8 * ti << "u);\n  }\n";
    }
  }
  // ---- small leaves on CUDA cores (overlap the tensor-core work) ----
  for (size_t l = 0; l < P.leaves.size(); ++l)
    if (!is_tc[l]) emit_leaf_fma(o, P.leaves[l], l, d, dtype);
  // ---- epilogue: per leaf, wait for its MMAs, accumulators -> registers ----
  if (pair) o << "  mbar_wait(mbar, par); tc_fence_after();\n";
  for (size_t ti = 0; ti < T.size(); ++ti) {
    const TcLeaf& t = T[ti];
    const Leaf& lf = P.leaves[t.leaf];
    if (!pair) o << "  mbar_wait(mbar + " << 8 * ti << "u, par); tc_fence_after();\n";
    for (int r0 = 0; r0 < t.k; r0 += 32) {
      const int w = std::min(32, t.np - r0);
      o << "  { u32 d[" << w << "];\n";
      emit_tmem_ld(o, "d", t.d_col + r0, w);
      for (int r = r0; r < std::min(t.k, r0 + w); ++r)
        o << "  y[" << out_idx(lf, d, r) << "] = __uint_as_float(d[" << r - r0 << "]);\n";
      o << "  }\n";
    }
  }
  if (d == DIR_FWD) emit_post_units(o, P, "y", false, "float");
  // ---- back: reverse butterflies (inverse) ----
  if (d != DIR_FWD) emit_units(o, P, "y", true, dtype);
  o << "}\n";
  if (pair) {
    o << "static __device__ __forceinline__ void gft_issue_pair(u32 tmem, u32 bsm, u32 mbar, u32 staged_local,\n"
         "    u32 par) {\n" << iss.str() << "}\n";
  }
}

// Warp-specialised CTA-pair variant (kernel_tc3_skeleton.cuh): the tile chain split into a
// stager (front butterflies, hi/lo -> TMEM A, small leaves -> SMEM row) and a drainer
// (TMEM D -> registers, back / coefficient butterflies); D double-buffered in TMEM.
// Returns false if the TMEM layout (A + 2 D) does not fit in 512 columns.
bool ws_layout(std::vector<TcLeaf>& T, int& a_cols, int& d_cols, int& tmem_cols) {
  a_cols = d_cols = 0;
  for (auto& t : T) {
    t.hi_col = a_cols;
    t.lo_col = a_cols + ru(t.kp8, 32);
    a_cols += 2 * ru(t.kp8, 32);
  }
  for (auto& t : T) {
    t.d_col = d_cols;            // relative to the D buffer base
    d_cols += ru(t.np, 32);
  }
  if (a_cols + 2 * d_cols > 512) return false;
  tmem_cols = 32;
  while (tmem_cols < a_cols + 2 * d_cols) tmem_cols *= 2;
  return true;
}

void generate_tc_ws(const Plan& P, Dir d, const std::vector<TcLeaf>& T, int a_cols, int d_cols,
                    std::ostringstream& o) {
  const int dtype = GFT_F32;
  std::vector<char> is_tc(P.leaves.size(), 0);
  for (const auto& t : T) is_tc[t.leaf] = 1;
  // ---- B operands: identical layout to the CTA-pair kernel (N/2 rows per CTA) ----
  std::vector<float> B;
  for (int r = 0; r < 2; ++r)
    for (const auto& t : T) {
      const Leaf& lf = P.leaves[t.leaf];
      const int rows = t.np / 2;
      for (int part = 0; part < 2; ++part)
        for (int a = 0; a < t.kp32 / 32; ++a)
          for (int n = r * rows; n < (r + 1) * rows; ++n)
            for (int kk = 32 * a; kk < 32 * a + 32; ++kk) {
              float v = 0.f;
              if (n < t.k && kk < t.k) v = (float)leaf_coef(lf, d, n, kk);
              const float hi = tf32_rna_host(v);
              B.push_back(part == 0 ? hi : v - hi);
            }
    }
  const size_t per_cta = B.size() / 2;
  int nch = 0;   // 32-column A chunks over all tensor-core leaves (staged / released one by one)
  for (const TcLeaf& t : T) nch += (t.kp8 + 31) / 32;
  o << "#define GFT_B_FLOATS " << per_cta << "\n#define GFT_A_COLS " << a_cols << "\n#define GFT_NCH " << nch
    << "\n#define GFT_D_BASE " << a_cols << "\n#define GFT_D_COLS " << d_cols << "\n#define GFT_SMALL "
    << (T.size() < P.leaves.size() ? 1 : 0) << "\n";
  o << "__device__ __align__(16) const float gft_tcB[2][" << per_cta << "] = {\n";
  for (size_t i = 0; i < B.size(); ++i) {
    char buf[48];
    std::snprintf(buf, sizeof buf, "%af,", (double)B[i]);
    o << buf << ((i % 8 == 7) ? "\n" : "");
  }
  o << "};\n";
  o << "static __device__ __forceinline__ void st_elem(unsigned char* buf, int row, int col, float v) {\n"
       "  *reinterpret_cast<float*>(buf + tile_off(row, col)) = v;\n}\n"
       "static __device__ __forceinline__ float ld_elem(const unsigned char* buf, int row, int col) {\n"
       "  return *reinterpret_cast<const float*>(buf + tile_off(row, col));\n}\n";
  // ---- stager: per 32-column A chunk c, wait until the MMAs of the previous tile on it are
  // done (a_free[c]), write hi/lo, signal staged[c] on the leader ----
  o << "static __device__ __forceinline__ void gft_stage(float (&x)[GFT_N], u32 tm, u32 staged0,\n"
       "    unsigned char* buf, int row, u32 afree, u32 apar, bool await_a, long long it) {\n";
  if (d != DIR_INV) emit_units(o, P, "x", false, dtype);
  if (d == DIR_FILTER && !P.post.empty()) fail(GFT_ERR_COMPILE, "filter plan with right Haar stages");
  if (d == DIR_INV) emit_post_units(o, P, "x", true, "float");
  int ch = 0;
  for (const TcLeaf& t : T) {
    const Leaf& lf = P.leaves[t.leaf];
    for (int c0 = 0; c0 < t.kp8; c0 += 32, ++ch) {
      const int w = std::min(32, t.kp8 - c0);
      o << "  if (await_a) { mbar_wait(afree + " << 8 * ch << "u, apar); tc_fence_after(); }\n";
      o << "  if (row == 0) TR(" << 14 + std::min(ch, 3) << ", it);\n";
      o << "  { u32 h[" << w << "], l[" << w << "];\n";
      for (int c = c0; c < c0 + w; ++c) {
        if (c < t.k) {
          const int src = in_idx(lf, d, c);
          o << split_line(c - c0, "x[" + std::to_string(src) + "]");
        } else {
          o << "  h[" << c - c0 << "] = 0u; l[" << c - c0 << "] = 0u;\n";
        }
      }
      emit_tmem_st(o, "h", t.hi_col + c0, w);
      emit_tmem_st(o, "l", t.lo_col + c0, w);
      o << "  }\n";
      o << "  signal_staged(staged0 + " << 8 * ch << "u);\n";
    }
  }
  if (T.size() < P.leaves.size()) {
    o << "  { float y[GFT_N];\n";
    for (size_t l = 0; l < P.leaves.size(); ++l)
      if (!is_tc[l]) emit_leaf_fma(o, P.leaves[l], l, d, dtype);
    for (size_t l = 0; l < P.leaves.size(); ++l)
      if (!is_tc[l])
        for (int r = 0; r < P.leaves[l].k; ++r) {
          const int oi = out_idx(P.leaves[l], d, r);
          o << "  st_elem(buf, row, " << oi << ", y[" << oi << "]);\n";
        }
    o << "  }\n";
  }
  o << "}\n";
  // ---- drainer: small-leaf outputs from SMEM, TC outputs from TMEM ----
  o << "static __device__ __forceinline__ void gft_drain(float (&y)[GFT_N], u32 tm, const unsigned char* buf, int row) {\n";
  for (size_t l = 0; l < P.leaves.size(); ++l)
    if (!is_tc[l])
      for (int r = 0; r < P.leaves[l].k; ++r) {
        const int oi = out_idx(P.leaves[l], d, r);
        o << "  y[" << oi << "] = ld_elem(buf, row, " << oi << ");\n";
      }
  for (const TcLeaf& t : T) {
    const Leaf& lf = P.leaves[t.leaf];
    for (int r0 = 0; r0 < t.k; r0 += 32) {
      const int w = std::min(32, t.np - r0);
      o << "  { u32 d[" << w << "];\n";
      emit_tmem_ld(o, "d", t.d_col + r0, w);
      for (int r = r0; r < std::min(t.k, r0 + w); ++r)
        o << "  y[" << out_idx(lf, d, r) << "] = __uint_as_float(d[" << r - r0 << "]);\n";
      o << "  }\n";
    }
  }
  o << "}\n";
  o << "static __device__ __forceinline__ void gft_finish(float (&y)[GFT_N]) {\n";
  if (d == DIR_FWD) emit_post_units(o, P, "y", false, "float");
  if (d != DIR_FWD) emit_units(o, P, "y", true, dtype);
  o << "}\n";
  // ---- issuer: chunk by chunk (all three passes of the chunk's k-steps), each chunk's MMAs
  // committed to a_free[c] so the stager can refill it ----
  o << "static __device__ __forceinline__ void gft_issue_ws(u32 tA, u32 tD, u32 bsm, u32 staged, u32 spar, u32 afree,\n"
       "    long long it) {\n";
  ch = 0;
  for (const TcLeaf& t : T) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(t.np >> 3) << 17) | (16u << 24);
    const int atom_bytes = (t.np / 2) * 128;
    for (int c0 = 0; c0 < t.kp8; c0 += 32, ++ch) {
      const int w = std::min(32, t.kp8 - c0);
      o << "  mbar_wait_acq_cluster(staged + " << 8 * ch << "u, spar); tc_fence_after();\n";
      o << "  TR(" << 10 + std::min(ch, 3) << ", it);\n";
      for (int pass = 0; pass < 3; ++pass) {
        const int acol = pass == 2 ? t.lo_col : t.hi_col;
        const int boff = pass == 1 ? t.blo_off : t.bhi_off;
        for (int j = c0 / 8; j < (c0 + w) / 8; ++j) {
          const int bo = boff + (j / 4) * atom_bytes + (j % 4) * 32;
          o << "  mma_ts2(tD + " << t.d_col << "u, tA + " << (acol + 8 * j) << "u, smem_desc_sw128(bsm + " << bo
            << "u), " << idesc << "u, " << ((pass == 0 && j == 0) ? 0 : 1) << "u);\n";
        }
      }
      o << "  tc_commit_pair(afree + " << 8 * ch << "u);\n";
    }
  }
  o << "}\n";
}

// host float -> IEEE half (round to nearest even, subnormals, overflow to inf)
uint16_t f32_to_f16_host(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  const uint32_t sign = (x >> 16) & 0x8000u;
  const int32_t e = (int32_t)((x >> 23) & 0xff) - 127 + 15;
  uint32_t m = x & 0x7fffffu;
  if (((x >> 23) & 0xff) == 0xff) return (uint16_t)(sign | 0x7c00u | (m ? 0x200u : 0u));
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {   // subnormal half (or zero)
    if (e < -10) return (uint16_t)sign;
    m |= 0x800000u;
    const int shift = 14 - e;
    uint32_t hm = m >> shift;
    const uint32_t rem = m & ((1u << shift) - 1), half = 1u << (shift - 1);
    if (rem > half || (rem == half && (hm & 1u))) ++hm;
    return (uint16_t)(sign | hm);
  }
  uint32_t hm = m >> 13;
  const uint32_t rem = m & 0x1fffu;
  uint32_t h = sign | ((uint32_t)e << 10) | hm;
  if (rem > 0x1000u || (rem == 0x1000u && (hm & 1u))) ++h;   // may carry into the exponent: correct
  return (uint16_t)h;
}
float f16_to_f32_host(uint16_t h) {
  const uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  const uint32_t e = (h >> 10) & 0x1f, m = h & 0x3ffu;
  float v;
  if (e == 0) v = std::ldexp((float)m, -24);
  else if (e == 31) v = m ? NAN : INFINITY;
  else v = std::ldexp((float)(m | 0x400u), (int)e - 25);
  uint32_t b;
  std::memcpy(&b, &v, 4);
  b |= sign;
  std::memcpy(&v, &b, 4);
  return v;
}

// Warp-specialised IO-split kernel with an fp16x2 split instead of 3xTF32 (GFT_TC_F16=1): every
// row is scaled by a power of two s = 2^-e that brings its largest tensor-core input into [1, 2)
// (exact; fp16 range), then x' = h + l with h = x' truncated to 11 significant bits (exactly an
// fp16) and l = fp16(x' - h); the leaf matrix likewise B = B_h + B_l in fp16.  D = h.B_h + h.B_l
// + l.B_h as kind::f16 MMAs (K = 16 per instruction, twice the tf32 MAC rate) accumulating in
// fp32; the drainer multiplies by 2^e.  Half the TMEM bytes of the staged A operand (16-bit
// h and l), half the B bytes, half the MMA instructions.  Error: |x' - h - l| <= 2^-11 |l| <=
// 2^-22 |x'| per element, B likewise; the dropped l.B_l term is ~2^-22 relative.
void generate_tc_ws_f16(const Plan& P, Dir d, const std::vector<TcLeaf>& T, int a_cols, int d_cols,
                        int a_bufs, std::ostringstream& o) {
  // ---- B operands: per CTA half (N/2 rows), per leaf, parts h then l; K-major, 128B-swizzled
  // atoms of 64 fp16 (128 B) x 8 rows; K padded to whole 32-element chunks ----
  std::vector<uint16_t> B;
  std::vector<int> boff_h(T.size()), boff_l(T.size()), atom_bytes(T.size());
  for (int r = 0; r < 2; ++r) {
    int off = 0;
    for (size_t ti = 0; ti < T.size(); ++ti) {
      const TcLeaf& t = T[ti];
      const Leaf& lf = P.leaves[t.leaf];
      const int rows = t.np / 2, atoms = (t.kp32 + 63) / 64;
      atom_bytes[ti] = rows * 128;
      for (int part = 0; part < 2; ++part) {
        (part == 0 ? boff_h : boff_l)[ti] = off;
        for (int a = 0; a < atoms; ++a)
          for (int n = r * rows; n < (r + 1) * rows; ++n)
            for (int kk = 64 * a; kk < 64 * a + 64; ++kk) {
              float v = 0.f;
              if (n < t.k && kk < t.k) v = (float)leaf_coef(lf, d, n, kk);
              const uint16_t h = f32_to_f16_host(v);
              B.push_back(part == 0 ? h : f32_to_f16_host(v - f16_to_f32_host(h)));
            }
        off += atoms * rows * 128;
      }
    }
  }
  const size_t per_cta = B.size() / 2;   // fp16 elements per CTA (even: whole 128 B rows)
  int nch = 0;
  for (const TcLeaf& t : T) nch += t.kp32 / 32;
  o << "#define GFT_F16X2 1\n#define GFT_B_FLOATS " << per_cta / 2 << "\n#define GFT_A_COLS " << a_cols
    << "\n#define GFT_A_BUFS " << a_bufs << "\n#define GFT_NCH " << nch << "\n#define GFT_D_BASE " << a_bufs * a_cols
    << "\n#define GFT_D_COLS " << d_cols << "\n#define GFT_SMALL 0\n";
  o << "__device__ __align__(16) const unsigned int gft_tcB[2][" << per_cta / 2 << "] = {\n";
  for (size_t i = 0; i < B.size(); i += 2) {
    char buf[24];
    std::snprintf(buf, sizeof buf, "0x%08xu,", (unsigned)B[i] | ((unsigned)B[i + 1] << 16));
    o << buf << ((i % 16 == 14) ? "\n" : "");
  }
  o << "};\n";
  o << "static __device__ __forceinline__ void st_elem(unsigned char* buf, int row, int col, float v) {\n"
       "  *reinterpret_cast<float*>(buf + tile_off(row, col)) = v;\n}\n";
  // ---- stager ----
  o << "static __device__ __forceinline__ void gft_stage(float (&x)[GFT_N], u32 tm, u32 staged0,\n"
       "    unsigned char* buf, int row, u32 afree, u32 apar, bool await_a, long long it, int* row_e) {\n";
  if (d != DIR_INV) emit_units(o, P, "x", false, GFT_F32);
  if (d == DIR_FILTER && !P.post.empty()) fail(GFT_ERR_COMPILE, "filter plan with right Haar stages");
  if (d == DIR_INV) emit_post_units(o, P, "x", true, "float");
  // row scale: e = exponent of the largest |input| of the tensor-core leaves
  o << "  float m_ = 0.f;\n";
  for (const TcLeaf& t : T)
    for (int c = 0; c < t.k; ++c) o << "  m_ = fmaxf(m_, fabsf(x[" << in_idx(P.leaves[t.leaf], d, c) << "]));\n";
  o << "  const int e_ = row_exponent(m_);\n  *row_e = e_;\n  const float sc_ = exp2_int(-e_);\n";
  int ch = 0;
  for (const TcLeaf& t : T) {
    const Leaf& lf = P.leaves[t.leaf];
    for (int c0 = 0; c0 < t.kp32; c0 += 32, ++ch) {
      o << "  if (await_a) { mbar_wait(afree + " << 8 * ch << "u, apar); tc_fence_after(); }\n";
      o << "  if (row == 0) TR(" << 14 + std::min(ch, 3) << ", it);\n";
      o << "  { u32 h[16], l[16];\n";
      for (int q = 0; q < 16; ++q) {
        const int c = c0 + 2 * q;
        auto v = [&](int cc) {
          return cc < t.k ? "x[" + std::to_string(in_idx(lf, d, cc)) + "] * sc_" : std::string("0.f");
        };
        o << "  split_f16x2(" << v(c) << ", " << v(c + 1) << ", h[" << q << "], l[" << q << "]);\n";
      }
      emit_tmem_st(o, "h", t.hi_col + c0 / 2, 16);
      emit_tmem_st(o, "l", t.lo_col + c0 / 2, 16);
      o << "  }\n";
      o << "  signal_staged(staged0 + " << 8 * ch << "u);\n";
    }
  }
  o << "}\n";
  // ---- drainer: y = 2^e D ----
  o << "static __device__ __forceinline__ void gft_drain(float (&y)[GFT_N], u32 tm, const unsigned char* buf, int row,\n"
       "    int e_) {\n  const float u_ = exp2_int(e_);\n";
  for (const TcLeaf& t : T) {
    const Leaf& lf = P.leaves[t.leaf];
    for (int r0 = 0; r0 < t.k; r0 += 32) {
      const int w = std::min(32, t.np - r0);
      o << "  { u32 d[" << w << "];\n";
      emit_tmem_ld(o, "d", t.d_col + r0, w);
      const int r1 = std::min(t.k, r0 + w);
      int r = r0;
      for (; r < r1; ++r)
        o << "  y[" << out_idx(lf, d, r) << "] = __uint_as_float(d[" << r - r0 << "]) * u_;\n";
      o << "  }\n";
    }
  }
  o << "}\n";
  o << "static __device__ __forceinline__ void gft_finish(float (&y)[GFT_N]) {\n";
  if (d == DIR_FWD) emit_post_units(o, P, "y", false, "float");
  if (d != DIR_FWD) emit_units(o, P, "y", true, GFT_F32);
  o << "}\n";
  // ---- issuer: per chunk (two K = 16 steps), passes h.B_h, h.B_l, l.B_h ----
  o << "static __device__ __forceinline__ void gft_issue_ws(u32 tA, u32 tD, u32 bsm, u32 staged, u32 spar, u32 afree,\n"
       "    long long it) {\n";
  ch = 0;
  for (size_t ti = 0; ti < T.size(); ++ti) {
    const TcLeaf& t = T[ti];
    // kind::f16: D f32 (bit 4), A / B f16 (format 0), N >> 3 at bit 17, M >> 4 at bit 24
    const uint32_t idesc = (1u << 4) | ((uint32_t)(t.np >> 3) << 17) | (16u << 24);
    for (int c0 = 0; c0 < t.kp32; c0 += 32, ++ch) {
      o << "  mbar_wait_acq_cluster(staged + " << 8 * ch << "u, spar); tc_fence_after();\n";
      o << "  TR(" << 10 + std::min(ch, 3) << ", it);\n";
      for (int pass = 0; pass < 3; ++pass) {
        const int acol = pass == 2 ? t.lo_col : t.hi_col;
        const int boff = pass == 1 ? boff_l[ti] : boff_h[ti];
        for (int j = c0 / 16; j < c0 / 16 + 2; ++j) {
          const int bo = boff + (j / 4) * atom_bytes[ti] + (j % 4) * 32;
          o << "  mma_ts2_f16(tD + " << t.d_col << "u, tA + " << (acol + 8 * j) << "u, smem_desc_sw128(bsm + " << bo
            << "u), " << idesc << "u, " << ((pass == 0 && j == 0) ? 0 : 1) << "u);\n";
        }
      }
      o << "  tc_commit_pair(afree + " << 8 * ch << "u);\n";
    }
  }
  o << "}\n";
}

// Dense comparison kernel Y = X W (H7) as a register-tiled GEMM with W in SMEM
// (kernel_dense_skeleton.cuh), for n = 64 / 128 when a tile ring of >= 2 buffers fits beside
// W.  Thread tile GFT_TM x 8 (TM = 6 fp32, 4 fp64), 256 compute threads: GFT_BM = 256 TM 8 / n.
bool dense_gemm_geometry(int n, int dtype, KernelCfg& c) {
  if (n != 64 && n != 128) return false;
  if (const char* e = getenv("GFT_NO_DENSE_GEMM")) if (e[0] == '1') return false;   // ablation
  auto env_int = [](const char* k, int v) { const char* e = getenv(k); return (e && *e) ? atoi(e) : v; };
  const int elem = dtype == GFT_F64 ? 8 : 4;
  const int tm = env_int("GFT_DG_TM", dtype == GFT_F64 ? 4 : 6), tn = env_int("GFT_DG_TN", 8);
  const int threads = env_int("GFT_DG_THREADS", 256);
  if (tm < 1 || tn < 16 / elem || tn % (16 / elem) || n % tn || (threads != 128 && threads != 256)) return false;
  const int bm = threads * tm * tn / n;
  if (bm > 256 || bm % 8 || (bm / tm) < 8 || (bm / tm) * (n / tn) != threads) return false;
  // a warp owns whole rows (all n / tn column threads, kernel_dense_skeleton.cuh)
  if (n / tn > 32 || 32 % (n / tn) || (bm / tm) % (32 / (n / tn))) return false;
  KernelCfg g;
  g.n = n;
  g.elem = elem;
  g.dgemm = 1;
  g.bm = bm;
  g.R = tm;       // thread tile rows
  g.pack = tn;    // thread tile columns
  g.warps = threads / 32;
  g.mode = 0;
  g.boxc = 128 / elem;
  g.swz_mask = 7;
  g.vec = 16 / elem;
  for (g.stages = 4; g.stages >= 2 && g.smem_bytes() > 227 * 1024; --g.stages) {}
  if (g.stages < 2) return false;
  c = g;
  return true;
}

void generate_dense_gemm(const Plan& P, int kind, int dtype, Kernel& k) {
  const KernelCfg& c = k.cfg;
  const int n = P.n;
  std::ostringstream gen;
  gen << "__device__ __align__(16) const elem_t gft_W[" << n * n << "] = {\n";
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      // forward y_j = sum_i x_i U[i][j]; inverse x_j = sum_i y_i U[j][i]
      const double v = kind == K_DENSE_FWD ? P.U[(size_t)i * n + j] : P.U[(size_t)j * n + i];
      char buf[48];
      if (dtype == GFT_F64) std::snprintf(buf, sizeof buf, "%a,", v);
      else std::snprintf(buf, sizeof buf, "%af,", (double)(float)v);
      gen << buf << ((j % 8 == 7) ? "\n" : "");
    }
  gen << "};\n";
  std::ostringstream pre;
  pre << "#define GFT_ELEM " << (dtype == GFT_F64 ? "double" : "float") << "\n";
  if (dtype == GFT_F64) pre << "#define GFT_ELEM_IS_DOUBLE 1\n";
  pre << "#define GFT_N " << n << "\n#define GFT_BM " << c.bm << "\n#define GFT_TM " << c.R << "\n#define GFT_TN " << c.pack
      << "\n#define GFT_THREADS " << 32 * c.warps << "\n#define GFT_STAGES " << c.stages << "\n";
  if (const char* e = getenv("GFT_DG_PREFETCH")) pre << "#define GFT_DG_PREFETCH " << atoi(e) << "\n";   // experiment
  {   // k-loop unroll 8 (measured, profiles/r02/r02_dense_probe8.log)
    const char* e = getenv("GFT_DG_UNROLL");
    pre << "#define GFT_DG_UNROLL " << ((e && *e) ? atoi(e) : 8) << "\n";
  }
  if (const char* e = getenv("GFT_DG_WY")) pre << "#define GFT_DG_WY " << atoi(e) << "\n";   // experiment
  if (const char* e = getenv("GFT_DG_FFMA2")) pre << "#define GFT_DG_FFMA2 " << atoi(e) << "\n";   // ablation
  const std::string skel(kSkeletonDense);
  const std::string marker = "// @@GFT_GENERATED@@";
  const size_t at = skel.find(marker);
  if (at == std::string::npos) fail(GFT_ERR_COMPILE, "dense skeleton marker missing");
  const std::string key = pre.str() + gen.str() + skel;
  char hbuf[32];
  std::snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)fnv1a(key));
  k.name = std::string("gft_") + (kind == K_DENSE_FWD ? "dgfwd" : "dginv") + "_" + (dtype == GFT_F64 ? "f64" : "f32") +
           "_n" + std::to_string(n) + "_" + hbuf;
  std::ostringstream src;
  src << "// generated by paper_1907_07875_b200 codegen.cpp — dense comparison GEMM (W in SMEM)\n"
      << pre.str() << "#define GFT_KNAME " << k.name << "\n" << skel.substr(0, at) << gen.str() << skel.substr(at);
  k.source = src.str();
}

}  // namespace

void generate_kernel(const Plan& P, int kind, int dtype, Kernel& k, bool allow_tc, bool dense_tc,
                     const CfgOverride* ov) {
  if (dense_tc && allow_tc && (kind == K_DENSE_FWD || kind == K_DENSE_INV)) {
    // dense U^T x on tensor cores: the whole basis as ONE leaf (no butterflies), generated by
    // the same tcgen05 path -- the strongest dense comparison for n >= 32
    Plan D;
    D.n = P.n;
    Leaf lf;
    lf.k = P.n;
    for (int i = 0; i < P.n; ++i) { lf.pos.push_back(i); lf.slot.push_back(i); }
    lf.M.assign((size_t)P.n * P.n, 0.0);
    for (int r = 0; r < P.n; ++r)
      for (int c = 0; c < P.n; ++c) lf.M[(size_t)r * P.n + c] = P.U[(size_t)c * P.n + r];   // M = U^T
    D.leaves.push_back(lf);
    generate_kernel(D, kind == K_DENSE_FWD ? K_FAST_FWD : K_FAST_INV, dtype, k, true, false);
    if (k.cfg.tc) {
      k.kind = kind;
      const std::string old = k.name;
      k.name = "gft_d" + old.substr(4);                      // gft_fwdtc... -> gft_dfwdtc...
      size_t at;
      while ((at = k.source.find(old)) != std::string::npos) k.source.replace(at, old.size(), k.name);
      return;
    }
  }
  k.kind = kind;
  k.dtype = dtype;
  if ((kind == K_DENSE_FWD || kind == K_DENSE_INV) && dense_gemm_geometry(P.n, dtype, k.cfg)) {
    generate_dense_gemm(P, kind, dtype, k);
    return;
  }
  k.cfg = choose_cfg(P.n, dtype, (kind == K_DENSE_FWD || kind == K_DENSE_INV) ? (int64_t)P.n * P.n : P.sum_k2,
                     ov, kind);
  static const char* kKindNameTC[] = {"fwdtc", "invtc", "", "", "filttc"};
  const Dir dir = kind == K_FAST_INV ? DIR_INV : kind == K_FILTER ? DIR_FILTER : DIR_FWD;
  if (allow_tc && (kind == K_FAST_FWD || kind == K_FAST_INV || kind == K_FILTER)) {
    std::vector<TcLeaf> T;
    int tmem_cols = 0, b_bytes = 0, stages = 3;
    bool pair = false, ok = false;
    // CTA pair first (3 tile buffers if they fit, else 2), then the single-CTA variant;
    // every big leaf must land on the tensor core for the pair variant to be chosen
    int nbig = 0;
    for (const auto& lf : P.leaves) nbig += tc_candidate(P, lf, approx_on_tc(P, dtype));
    // up to 4 tile buffers when they fit (n <= 96: +5% over 3 at n = 80 / 96; cfg5b's 64 KiB
    // tiles fit 3; tools/gpu_pair_stages.sh); GFT_TC_PAIR_MAXSTAGES overrides
    const char* pst = getenv("GFT_TC_PAIR_MAXSTAGES");
    for (int st = (pst && *pst) ? atoi(pst) : 4; st >= 2 && !ok; --st)
      if (plan_tc(P, dtype, st, true, T, tmem_cols, b_bytes) && (int)T.size() == nbig &&
          getenv("GFT_NO_CTA_PAIR") == nullptr && !(ov && ov->tc_variant == 3)) {
        ok = pair = true;
        stages = st;
      }
    if (!ok) {
      stages = 2;
      ok = plan_tc(P, dtype, stages, false, T, tmem_cols, b_bytes);
    }
    // two compute warpgroups on the CTA pair for small n: the per-tile MMA chain of one
    // warpgroup hides behind the other's staging.  320 threads leave 168 registers per
    // thread, so only plans whose every leaf is on the tensor core (no FMA leaf registers)
    // and n <= 80 qualify (measured: +4-5% at n = 64 with two 32-leaves, -6% with an FMA
    // leaf beside them; tools/tc_vs_fma.py)
    int wgs = 1, wg_cols = 0;
    const bool no_2wg = getenv("GFT_NO_TC_2WG") != nullptr || (ov && ov->tc_variant == 0);
    const bool no_ws = getenv("GFT_NO_TC_WS") != nullptr || (ov && (ov->tc_variant == 0 || ov->tc_variant == 1));
    if (ok && pair && P.n <= 80 && T.size() == P.leaves.size() && !no_2wg) {
      for (const auto& t : T) wg_cols = std::max(wg_cols, t.d_col + ru(t.np, 32));
      if (2 * wg_cols <= 512) {
        std::vector<TcLeaf> T2;
        int tc2 = 0, bb2 = 0;
        for (int st = 6; st >= 4; --st)
          if (plan_tc(P, dtype, st, true, T2, tc2, bb2) && T2.size() == T.size()) {
            wgs = 2;
            stages = st;
            tmem_cols = 32;
            while (tmem_cols < 2 * wg_cols) tmem_cols *= 2;
            break;
          }
      }
    }
    // warp-specialised pair kernel (stager / drainer, D double-buffered) for n <= 64 when its
    // TMEM layout and FOUR tile buffers fit: a buffer is held from TMA load through staging to
    // the drain, so with 3 buffers only one tile of prefetch remains and the stager waits on
    // HBM.  Measured back to back (tools/gpu_ws_cmp.sh, gpu_ws_stages.sh): n = 64 +9-16% over
    // the pair kernels; n = 80 a tie; n = 96 -5%; n = 128 (3 buffers) -7%; 5-6 buffers are
    // slower than 4 at n = 64.  GFT_NO_TC_WS=1 keeps the plain pair kernel (ablation).
    bool ws = false;
    int ws_a = 0, ws_d = 0, ws_tmem = 0;
    std::vector<TcLeaf> Tws;
    if (ok && pair && P.n <= 64 && !no_ws) {
      Tws = T;
      if (ws_layout(Tws, ws_a, ws_d, ws_tmem)) {
        const int tile = 128 * ((P.n + 31) / 32 * 32) * 4;
        const char* es = getenv("GFT_TC_WS_STAGES");   // experiment knob (default: measured 4)
        int st = (es && *es) ? atoi(es) : 4;
        while (st >= 4 && st * tile + b_bytes + 2048 > 227 * 1024) --st;
        if (st >= 4) {
          ws = true;
          stages = st;
          wgs = 1;
          tmem_cols = ws_tmem;
        }
      }
    }
    // n > 64 (tiles too big for four in-place buffers): the IO-split warp-specialised kernel --
    // two input buffers released by the stager right after reading its rows, one output buffer
    // written and stored box by box (plans without CUDA-core leaves).  With load pacing and
    // per-chunk A release it beats the plain pair kernel in a burst (cfg5b forward 6.30 vs
    // 6.13 TB/s) and under sustained load (6.00 vs 5.25 TB/s at the power-capped clock,
    // tools/r02/gpu_tc_probe7.sh).  GFT_TC_IOSPLIT=0 keeps the plain pair kernel (ablation).
    bool io_split = false;
    const char* eio = getenv("GFT_TC_IOSPLIT");
    if (ok && pair && !ws && !no_ws && P.n > 64 && T.size() == P.leaves.size() && !(eio && eio[0] == '0')) {
      Tws = T;
      // the fp16x2 layout (below) needs half the B bytes of 3xTF32: a single 128-node leaf (the
      // n = 128 dense comparison on tcgen05) fits the IO-split kernel only that way
      const char* e16 = getenv("GFT_TC_F16");
      int ac16 = 0, dc16 = 0, bb16 = 1024;
      for (const auto& t : T) { ac16 += t.kp32; dc16 += ru(t.np, 32); bb16 += 2 * ((t.kp32 + 63) / 64) * (t.np / 2) * 128; }
      const bool fit16 = !(e16 && e16[0] == '0') && ac16 + 2 * dc16 <= 512;
      const bool fit32 = ws_layout(Tws, ws_a, ws_d, ws_tmem);
      const int tile = 128 * ((P.n + 31) / 32 * 32) * 4;
      if ((fit32 && 3 * tile + b_bytes + 2048 <= 227 * 1024) || (fit16 && 3 * tile + bb16 + 2048 <= 227 * 1024)) {
        {
          ws = io_split = true;
          stages = 2;
          wgs = 1;
          tmem_cols = ws_tmem;
        }
      }
    }
    if (ok) {
      KernelCfg& c = k.cfg;
      c.tc = 1;
      c.tc_pair = pair ? 1 : 0;
      c.tc_wgs = wgs;
      c.tc_ws = ws ? 1 : 0;
      c.tc_io_split = io_split ? 1 : 0;
      c.stages = stages;
      c.mode = 0;
      c.boxc = 32;
      c.swz_mask = 7;
      c.vec = 4;
      c.R = 4;
      c.warps = 5;
      c.tc_b_bytes = b_bytes;
      c.tc_tmem_cols = tmem_cols;
      std::ostringstream gen;
      // warp-specialised kernels whose every leaf is on the tensor core: the fp16x2 split
      // (generate_tc_ws_f16) instead of 3xTF32 -- half the TMEM bytes and MMA instructions;
      // cfg5b forward 6.46 -> 6.50 TB/s burst and 5.93 -> 6.32 sustained at the power cap, max
      // per-signal error 9.9e-7 -> 7.2e-7 (tools/r02/gpu_f16_probe.sh).  GFT_TC_F16=0: 3xTF32
      bool f16 = false;
      int a_bufs = 1;
      if (ws && Tws.size() == P.leaves.size()) {
        const char* e16 = getenv("GFT_TC_F16");
        if (!(e16 && e16[0] == '0')) {
          int ac = 0, dc = 0;
          for (auto& t : Tws) { t.hi_col = ac; t.lo_col = ac + t.kp32 / 2; ac += t.kp32; }
          for (auto& t : Tws) { t.d_col = dc; dc += ru(t.np, 32); }
          int bb = 0;
          for (auto& t : Tws) bb += 2 * ((t.kp32 + 63) / 64) * (t.np / 2) * 128;
          if (ac + 2 * dc <= 512) {
            f16 = true;
            ws_a = ac;
            ws_d = dc;
            // IO-split kernels: two A buffers when they fit TMEM beside the double-buffered D, so
            // staging tile t+1 never waits for the MMAs of tile t (cfg5b 0.999 -> 1.010 of the copy
            // peak in a burst, sustained unchanged; in-place n <= 64 kernels mixed: right-Haar 32|32
            // +0.5%, z-grid 64 -2%, so they keep one; profiles/r02/r02_a2.log).  GFT_TC_A2=0 / 1
            // forces one / two (ablation)
            const char* ea2 = getenv("GFT_TC_A2");
            const bool want2 = ea2 && *ea2 ? ea2[0] == '1' : io_split;
            a_bufs = (2 * ac + 2 * dc <= 512 && want2) ? 2 : 1;
            tmem_cols = 32;
            while (tmem_cols < a_bufs * ac + 2 * dc) tmem_cols *= 2;
            c.tc_tmem_cols = tmem_cols;
            c.tc_b_bytes = bb + 1024;   // + the per-row exponents (2 tiles x 128 ints)
          }
        }
      }
      if (f16) generate_tc_ws_f16(P, dir, Tws, ws_a, ws_d, a_bufs, gen);
      else if (ws) generate_tc_ws(P, dir, Tws, ws_a, ws_d, gen);
      else generate_tc(P, dir, T, pair, gen);
      std::ostringstream pre;
      pre << "#define GFT_N " << c.n << "\n#define GFT_STAGES " << c.stages << "\n#define GFT_TMEM_COLS "
          << tmem_cols << "\n";
      if (wgs == 2) pre << "#define GFT_WGS 2\n#define GFT_WG_COLS " << wg_cols << "\n";
      if (io_split) pre << "#define GFT_IO_SPLIT 1\n";
      // in-place warp-specialised kernel: a separate storer warp stores each tile as soon as it is
      // drained and hands the buffer to the loader once the store has read it (before: one
      // thread issued store, wait-read, load in turn, so a drained tile's store waited behind
      // the previous store's read and the load pacing).  Right-Haar 32|32 0.968 -> 0.977,
      // z-grid 64 (two 32-leaves) 0.930 -> 0.970 of the copy peak (profiles/r02/r02_split_store.log).
      // GFT_TC_SPLIT_STORE=0 restores the single producer / storer thread (ablation).
      {
        const char* e = getenv("GFT_TC_SPLIT_STORE");
        if (ws && !io_split && !(e && e[0] == '0')) pre << "#define GFT_SPLIT_STORE 1\n";
      }
      if (const char* e = getenv("GFT_TC_TRACE")) if (e[0] == '1') pre << "#define GFT_TRACE 1\n";   // experiments
      if (ws) {
        // load pacing (kernel_tc3_skeleton.cuh pace_load): a fraction of the CTA's fair share of
        // HBM time per tile (read + write of its 128 rows at 6455 GB/s over 148 SMs, the
        // measured copy roof) -- 0.9 for the IO-split kernel (64 KiB tiles), 0.83 for the
        // in-place one (32 KiB tiles at n = 64).  The optimum is sharp: cfg5b 2704 ns 6.31 TB/s
        // vs 5.94 at 2550 and 6.03 at 2850; right-Haar 32|32 1250 ns 6.34 vs 6.12 at 1352
        // (tools/r02/pace_confirm.py, profiles/r02/r02_pace_confirm.log).
        // GFT_TC_LOAD_PACE_NS overrides (0 disables)
        int pace = (int)((io_split ? 0.9 : 0.83) * 2.0 * c.tile_bytes() / (6455.0 / 148.0));
        if (const char* lp = getenv("GFT_TC_LOAD_PACE_NS")) pace = atoi(lp);
        if (pace > 0) pre << "#define GFT_LOAD_PACE_NS " << pace << "\n";
      }
      const std::string skel(ws ? kSkeletonTC3 : pair ? kSkeletonTC2 : kSkeletonTC);
      const std::string marker = "// @@GFT_GENERATED@@";
      const size_t at = skel.find(marker);
      if (at == std::string::npos) fail(GFT_ERR_COMPILE, "TC skeleton marker missing");
      const std::string key = pre.str() + gen.str() + skel;
      char hbuf[32];
      std::snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)fnv1a(key));
      k.name = std::string("gft_") + kKindNameTC[kind] + (ws ? (io_split ? "3s" : "3") : pair ? (wgs == 2 ? "2w" : "2") : "") + "_f32_n" + std::to_string(c.n) + "_" + hbuf;
      std::ostringstream src;
      src << "// generated by paper_1907_07875_b200 codegen.cpp — plan-specialised GFT kernel with\n"
          << "// tcgen05 3xTF32 leaves (" << T.size() << " tensor-core leaves)\n"
          << pre.str() << "#define GFT_KNAME " << k.name << "\n"
          << skel.substr(0, at) << gen.str() << skel.substr(at);
      k.source = src.str();
      return;
    }
  }
  const KernelCfg& c = k.cfg;
  std::ostringstream body;
  // wide rows stream their leaf outputs to SMEM instead of holding a y row in registers:
  // only when x + y would be far beyond the register file (2 n words > 320, e.g. f64 n > 80:
  // a 96-node f64 leaf spills 692 B/thread otherwise, none streamed); at 2 n words = 256
  // (cfg4 f64, cfg5b dense) the register version is faster (6.31 vs 6.10 TB/s, cfg4 f64
  // forward; tools/gpu_stream_cmp.sh).  GFT_STREAM=0/1 forces it (experiments)
  const int words = c.elem / 4;
  bool stream = 2 * c.n * words > 320;
  if (const char* e = getenv("GFT_STREAM")) stream = e[0] == '1';
  if (stream)
    body << "#define GFT_STREAM 1\n"
            "static __device__ __forceinline__ unsigned int tile_off(int row, int col);\n"
            "static __device__ __forceinline__ void load_row(const unsigned char* buf, int row, elem_t (&x)[GFT_N]);\n"
            "static __device__ __forceinline__ void store_row(unsigned char* buf, int row, const elem_t (&y)[GFT_N]);\n"
            "#define SOUT(c) (*reinterpret_cast<elem_t*>(buf_ + tile_off(row_, (c))))\n"
            "static __device__ __forceinline__ void gft_body(elem_t (&x)[GFT_N], unsigned char* buf_, int row_) {\n";
  else
    body << "static __device__ __forceinline__ void gft_body(elem_t (&x)[GFT_N], elem_t (&y)[GFT_N]) {\n";
  switch (kind) {
    case K_FAST_FWD:
    case K_FAST_INV:
    case K_FILTER: emit_fast(body, P, dtype, dir, stream); break;
    case K_DENSE_FWD: emit_dense(body, P, dtype, true, stream); break;
    case K_DENSE_INV: emit_dense(body, P, dtype, false, stream); break;
    default: fail(GFT_ERR_INVALID_ARG, "bad kernel kind");
  }
  body << "}\n";
  static const char* kKindName[] = {"fwd", "inv", "dfwd", "dinv", "filt"};
  std::ostringstream pre;
  pre << "#define GFT_ELEM " << (dtype == GFT_F64 ? "double" : "float") << "\n";
  if (dtype == GFT_F64) pre << "#define GFT_ELEM_IS_DOUBLE 1\n";
  pre << "#define GFT_N " << c.n << "\n#define GFT_R " << c.R << "\n#define GFT_WARPS " << c.warps
      << "\n#define GFT_STAGES " << c.stages << "\n#define GFT_MODE " << c.mode << "\n#define GFT_BOXC "
      << c.boxc << "\n#define GFT_SWZ_MASK " << c.swz_mask << "\n#define GFT_VEC " << c.vec << "\n#define GFT_PACK " << c.pack << "\n";
  if (c.pace_ns > 0) pre << "#define GFT_PACE_NS " << c.pace_ns << "\n";
  if (c.obuf > 0) pre << "#define GFT_OBUF " << c.obuf << "\n";
  // name = kind/dtype/n + hash of everything that determines the code
  std::string key = pre.str() + body.str() + kSkeleton;
  char hbuf[32];
  std::snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)fnv1a(key));
  k.name = std::string("gft_") + kKindName[kind] + "_" + (dtype == GFT_F64 ? "f64" : "f32") + "_n" +
           std::to_string(c.n) + "_" + hbuf;
  std::ostringstream src;
  src << "// generated by paper_1907_07875_b200 codegen.cpp — plan-specialised GFT kernel\n"
      << "// kind=" << kKindName[kind] << " n=" << c.n << " leaves=" << P.leaves.size()
      << " units=" << P.n_units << "\n"
      << pre.str() << "#define GFT_KNAME " << k.name << "\n"
      << "typedef GFT_ELEM elem_t;\n"
      << body.str() << kSkeleton;
  k.source = src.str();
}

}  // namespace gft
