// kernels.hpp — per-plan CUDA code generation and the device runtime (NVRTC + driver API).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "plan.hpp"

namespace gft {

// K_NUM kinds per plan; K_FILTER kernels belong to a gft_filter (fused U diag(h) U^T)
enum KernelKind { K_FAST_FWD = 0, K_FAST_INV = 1, K_DENSE_FWD = 2, K_DENSE_INV = 3, K_NUM = 4, K_FILTER = 4 };

// Launch/layout geometry of one generated kernel (see kernel_skeleton.cuh).
struct KernelCfg {
  int n = 0, elem = 4;          // signal length, bytes per element
  int R = 1, warps = 4, stages = 3;
  int mode = 0;                 // 0 TMA tensor 2-D + swizzle, 1 bulk 1-D, 2 packed view
  int pack = 1;                 // signals per TMA row of the packed view (mode 2)
  int boxc = 0, swz_mask = 0;   // TMA box columns, swizzle mask (7/3/1/0)
  int vec = 1;                  // elements per SMEM vector access
  int pace_ns = 0;              // FMA skeleton: per-tile __nanosleep before the store (tuning.tsv pace=)
  int obuf = 0;                 // FMA skeleton IO split: output tiles per warp (0 = in place)
  // tensor-core variant (kernel_tc_skeleton.cuh): one 128-row tile per CTA iteration,
  // 4 compute warps + 1 TMA warp, big leaves as tcgen05 3xTF32 micro-GEMMs
  int tc = 0;
  int tc_pair = 0;              // CTA-pair (cta_group::2, cluster of 2) variant, grid must be even
  int tc_b_bytes = 0;           // SMEM bytes of the B operands
  int tc_tmem_cols = 0;         // TMEM columns allocated
  int tc_wgs = 1;               // compute warpgroups of the CTA-pair kernel (1 or 2)
  int tc_ws = 0;                // warp-specialised pair kernel (kernel_tc3_skeleton.cuh, 384 threads)
  int tc_io_split = 0;          // ... with separate input ring and one output buffer
  // dense comparison GEMM (kernel_dense_skeleton.cuh): tiles of `bm` rows, 32*warps compute
  // threads + 1 TMA warp, thread tile R x pack outputs, W = U or U^T resident in SMEM
  int dgemm = 0;
  int bm = 0;
  int tile_rows() const { return dgemm ? bm : tc ? 128 : 32 * R; }
  // tensor-core tiles pad each row to whole 32-float TMA boxes (kernel_tc*_skeleton.cuh)
  int tile_bytes() const { return tile_rows() * (tc ? (n + 31) / 32 * 32 : n) * elem; }
  int threads() const {
    return dgemm ? 32 * warps + 32 : tc ? (tc_ws ? 384 : tc_pair ? 32 * (4 * tc_wgs + 2) : 160) : warps * 32;
  }
  int tiles_per_cta() const { return (tc || dgemm) ? 1 : warps; }   // tiles processed concurrently per CTA
  int smem_bytes() const {
    if (dgemm) return stages * tile_bytes() + n * n * elem + 2 * stages * 8 + 1024;
    if (tc) return (stages + tc_io_split) * tile_bytes() + tc_b_bytes + (4 * stages + 48) * 8 + 16 + 1024;
    return warps * (stages + obuf) * tile_bytes() + warps * stages * 8 + 1024;
  }
  int swizzle_bytes() const { return swz_mask == 7 ? 128 : swz_mask == 3 ? 64 : swz_mask == 1 ? 32 : 0; }
};

// work = FMAs per signal of the kernel body (selects plan-specific tuning entries)
// Geometry / pacing overrides of the FMA skeleton (gft_plan_tune candidates); -1 = keep.
// tc_variant (tensor-core plans): -1 rule-based default, 0 plain CTA pair, 1 CTA pair with two
// compute warpgroups, 2 warp-specialised pair, 3 single CTA (each where it applies).
struct CfgOverride { int R = -1, stages = -1, warps = -1, pace_ns = -1, tc_variant = -1; };
KernelCfg choose_cfg(int n, int dtype, int64_t work = -1, const CfgOverride* ov = nullptr, int kind = -1);

struct LoadedFn {
  void* module = nullptr;   // CUmodule
  void* fn = nullptr;       // CUfunction
  int grid_max = 0;         // SMs * resident CTAs
  int regs = 0;
};

struct Kernel {
  Kernel();
  uint64_t uid;             // process-unique id (keys the per-thread tensor-map cache)
  int kind = 0, dtype = 0;
  KernelCfg cfg;
  std::string name, source;
  std::string cubin;        // filled by compile()
  std::string cubin_origin; // "aot-cache" | "nvrtc"
  std::mutex mu;
  std::map<void*, LoadedFn> loaded;   // per CUcontext
};

// Emits the full CUDA source (prelude + gft_body + skeleton) for a plan.
// allow_tc: fast kernels of fp32 plans with leaves >= 32 use the tcgen05 3xTF32 skeleton.
// dense_tc: the dense comparison kernels use the tcgen05 path (whole basis as one leaf).
// ov: geometry / pacing overrides of the FMA skeleton (gft_plan_tune candidates).
void generate_kernel(const Plan& P, int kind, int dtype, Kernel& k, bool allow_tc, bool dense_tc = false,
                     const CfgOverride* ov = nullptr);

// Compiles k.source to an sm_100a cubin (AOT cache lookup first unless disabled).
void compile_kernel(Kernel& k, bool allow_cache);

// Launches `k` on `stream` (a CUstream / cudaStream_t) over `batch` rows.
void launch_kernel(Kernel& k, const void* in, void* out, int64_t batch, void* stream, bool allow_cache);
void kernel_launch_config(Kernel& k, int64_t batch, int* grid, int* block, int* smem, int* regs,
                          bool allow_cache);
void unload_kernel(Kernel& k);
// Mean ms of `reps` back-to-back launches of `k` (after `warm` untimed ones), timed with
// driver events on `stream`; synchronous (gft_plan_tune).
double time_kernel_ms(Kernel& k, const void* in, void* out, int64_t batch, void* stream, int warm,
                      int reps, bool allow_cache);

// Host<->device pipelined execution (gft_execute_host).
struct HostExec;
void execute_host(Kernel& k, const void* in_host, void* out_host, int64_t batch, void* workspace,
                  size_t workspace_bytes, int64_t chunk_rows, void* stream, bool allow_cache);

std::string cubin_cache_dir();

// Measured geometry table (paper_1907_07875_b200/tuning.tsv, written from geometry sweeps on
// a B200): lines "fma <n> <f32|f64> <R> <S> <W> [work= kind= pace= obuf=]".  Returns false
// if (n, dtype) has no entry.  GFT_TUNING_FILE overrides the path ("none" disables).
bool tuned_geometry(int n, int dtype, int64_t work, int kind, int& R, int& S, int& W, int& pace_ns, int& obuf);

}  // namespace gft
