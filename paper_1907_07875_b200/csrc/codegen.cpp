// codegen.cpp — per-plan CUDA source generation.
//
// Every graph-dependent quantity of the fast GFT becomes code: the Haar units
// (eq:B_phi) become register add/sub pairs, the folded sub-GFT
// coefficients (Theorem 4 leaves, 1/sqrt2 absorbed as PAPER.md:158
// suggests) become FFMA/DFMA immediates, and the ascending-eigenvalue permutation
// becomes the register index the result is written to.  There are no
// tables to fetch on the device: per signal the kernel executes exactly
// 2*units + sum_k k^2 arithmetic instructions (+ explicit scale fixes, if any).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <sstream>

#include "../../include/gft.h"
#include "kernels.hpp"

namespace gft {

// The device skeleton, embedded at build time (build.py writes skeleton_inc.h).
static const char* kSkeleton =
#include "skeleton_inc.h"
    ;

KernelCfg choose_cfg(int n, int dtype) {
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
  } else {
    c.mode = 1;
    c.boxc = n;
    c.swz_mask = 0;
    // odd row pitch in vector units makes thread-per-row accesses conflict-free
    c.vec = (c.elem == 4 && n % 2 == 0) ? 2 : 1;
  }
  c.R = 1;
  while (c.R < 8 && c.tile_bytes() < 4096) c.R *= 2;
  c.warps = 4;
  c.stages = 4;
  while (c.stages > 2 && c.warps * c.stages * c.tile_bytes() > 100 * 1024) --c.stages;
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

void emit_fast_forward(std::ostringstream& o, const Plan& P, int dtype) {
  o << "  elem_t a_, b_;\n";
  int lvl = -1;
  for (const Op& op : P.ops) {
    if (op.level != lvl) { lvl = op.level; o << "  // ---- butterfly level " << lvl << "\n"; }
    if (op.kind == Op::UNIT) {
      o << "  a_ = x[" << op.a << "]; b_ = x[" << op.b << "]; x[" << op.a << "] = a_ + b_; x["
        << op.b << "] = a_ - b_;\n";
    } else {
      o << "  x[" << op.a << "] = x[" << op.a << "] * " << lit(std::pow(2.0, 0.5 * op.m), dtype)
        << ";  // equalise deferred scale\n";
    }
  }
  for (size_t l = 0; l < P.leaves.size(); ++l) {
    const Leaf& lf = P.leaves[l];
    o << "  // ---- leaf " << l << " (k=" << lf.k << ")\n";
    std::vector<std::string> in(lf.k);
    for (int c = 0; c < lf.k; ++c) in[c] = xs("x", lf.pos[c]);
    for (int r = 0; r < lf.k; ++r) {
      std::vector<double> coef(lf.M.begin() + (size_t)r * lf.k, lf.M.begin() + (size_t)(r + 1) * lf.k);
      emit_dot(o, xs("y", lf.slot[r]), coef, in, dtype);
    }
  }
}

void emit_fast_inverse(std::ostringstream& o, const Plan& P, int dtype) {
  // x holds coefficients (ascending eigenvalue order); y receives the signal.
  for (size_t l = 0; l < P.leaves.size(); ++l) {
    const Leaf& lf = P.leaves[l];
    o << "  // ---- leaf " << l << " (k=" << lf.k << ", transposed)\n";
    std::vector<std::string> in(lf.k);
    for (int r = 0; r < lf.k; ++r) in[r] = xs("x", lf.slot[r]);
    for (int c = 0; c < lf.k; ++c) {
      std::vector<double> coef(lf.k);
      for (int r = 0; r < lf.k; ++r) coef[r] = lf.M[(size_t)r * lf.k + c];
      emit_dot(o, xs("y", lf.pos[c]), coef, in, dtype);
    }
  }
  o << "  elem_t a_, b_;\n";
  int lvl = -1;
  for (auto it = P.ops.rbegin(); it != P.ops.rend(); ++it) {
    const Op& op = *it;
    if (op.level != lvl) { lvl = op.level; o << "  // ---- butterfly level " << lvl << " (reverse)\n"; }
    if (op.kind == Op::UNIT) {
      o << "  a_ = y[" << op.a << "]; b_ = y[" << op.b << "]; y[" << op.a << "] = a_ + b_; y["
        << op.b << "] = a_ - b_;\n";
    } else {
      o << "  y[" << op.a << "] = y[" << op.a << "] * " << lit(std::pow(2.0, 0.5 * op.m), dtype) << ";\n";
    }
  }
}

void emit_dense(std::ostringstream& o, const Plan& P, int dtype, bool forward) {
  const int n = P.n;
  std::vector<std::string> in(n);
  for (int i = 0; i < n; ++i) in[i] = xs("x", i);
  for (int k = 0; k < n; ++k) {
    std::vector<double> coef(n);
    for (int i = 0; i < n; ++i)
      coef[i] = forward ? P.U[(size_t)i * n + k] : P.U[(size_t)k * n + i];
    emit_dot(o, xs("y", k), coef, in, dtype);
  }
}

}  // namespace

void generate_kernel(const Plan& P, int kind, int dtype, Kernel& k) {
  k.kind = kind;
  k.dtype = dtype;
  k.cfg = choose_cfg(P.n, dtype);
  const KernelCfg& c = k.cfg;
  std::ostringstream body;
  body << "static __device__ __forceinline__ void gft_body(elem_t (&x)[GFT_N], elem_t (&y)[GFT_N]) {\n";
  switch (kind) {
    case K_FAST_FWD: emit_fast_forward(body, P, dtype); break;
    case K_FAST_INV: emit_fast_inverse(body, P, dtype); break;
    case K_DENSE_FWD: emit_dense(body, P, dtype, true); break;
    case K_DENSE_INV: emit_dense(body, P, dtype, false); break;
    default: fail(GFT_ERR_INVALID_ARG, "bad kernel kind");
  }
  body << "}\n";
  static const char* kKindName[] = {"fwd", "inv", "dfwd", "dinv"};
  std::ostringstream pre;
  pre << "#define GFT_ELEM " << (dtype == GFT_F64 ? "double" : "float") << "\n";
  if (dtype == GFT_F64) pre << "#define GFT_ELEM_IS_DOUBLE 1\n";
  pre << "#define GFT_N " << c.n << "\n#define GFT_R " << c.R << "\n#define GFT_WARPS " << c.warps
      << "\n#define GFT_STAGES " << c.stages << "\n#define GFT_MODE " << c.mode << "\n#define GFT_BOXC "
      << c.boxc << "\n#define GFT_SWZ_MASK " << c.swz_mask << "\n#define GFT_VEC " << c.vec << "\n";
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
