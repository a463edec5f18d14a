// cuda_rt.cpp — device runtime: driver API + NVRTC loaded with dlopen (so the library
// loads on a CPU-only host), cubin cache / NVRTC compilation, module loading per
// CUDA context, TMA tensor-map encoding and kernel launch.
#include <cuda.h>
#include <dlfcn.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>

#include "../../include/gft.h"
#include "kernels.hpp"

namespace gft {
namespace {

struct Driver {
  bool tried = false, ok = false;
  std::string err;
  CUresult (*cuInit)(unsigned);
  CUresult (*cuGetErrorString)(CUresult, const char**);
  CUresult (*cuCtxGetCurrent)(CUcontext*);
  CUresult (*cuCtxSetCurrent)(CUcontext);
  CUresult (*cuCtxGetDevice)(CUdevice*);
  CUresult (*cuStreamGetCtx)(CUstream, CUcontext*);
  CUresult (*cuDeviceGet)(CUdevice*, int);
  CUresult (*cuDeviceGetCount)(int*);
  CUresult (*cuDeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*cuDevicePrimaryCtxRetain)(CUcontext*, CUdevice);
  CUresult (*cuModuleLoadData)(CUmodule*, const void*);
  CUresult (*cuModuleUnload)(CUmodule);
  CUresult (*cuModuleGetFunction)(CUfunction*, CUmodule, const char*);
  CUresult (*cuFuncSetAttribute)(CUfunction, CUfunction_attribute, int);
  CUresult (*cuFuncGetAttribute)(int*, CUfunction_attribute, CUfunction);
  CUresult (*cuOccupancyMaxActiveBlocksPerMultiprocessor)(int*, CUfunction, int, size_t);
  CUresult (*cuLaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                             unsigned, CUstream, void**, void**);
  CUresult (*cuLaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**);
  CUresult (*cuTensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUresult (*cuMemcpyHtoDAsync)(CUdeviceptr, const void*, size_t, CUstream);
  CUresult (*cuMemcpyDtoHAsync)(void*, CUdeviceptr, size_t, CUstream);
  CUresult (*cuStreamCreate)(CUstream*, unsigned);
  CUresult (*cuEventCreate)(CUevent*, unsigned);
  CUresult (*cuEventRecord)(CUevent, CUstream);
  CUresult (*cuStreamWaitEvent)(CUstream, CUevent, unsigned);
  CUresult (*cuEventSynchronize)(CUevent);
  CUresult (*cuEventElapsedTime)(float*, CUevent, CUevent);
  CUresult (*cuEventDestroy)(CUevent);
};

struct Nvrtc {
  bool tried = false, ok = false;
  std::string err;
  nvrtcResult (*create)(nvrtcProgram*, const char*, const char*, int, const char* const*, const char* const*);
  nvrtcResult (*compile)(nvrtcProgram, int, const char* const*);
  nvrtcResult (*log_size)(nvrtcProgram, size_t*);
  nvrtcResult (*log)(nvrtcProgram, char*);
  nvrtcResult (*cubin_size)(nvrtcProgram, size_t*);
  nvrtcResult (*cubin)(nvrtcProgram, char*);
  nvrtcResult (*destroy)(nvrtcProgram*);
  const char* (*errstr)(nvrtcResult);
};

std::mutex g_init_mu;

Driver& drv() {
  static Driver d;
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (d.tried) return d;
  d.tried = true;
  void* h = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { d.err = std::string("cannot load libcuda.so.1: ") + dlerror(); return d; }
  typedef CUresult (*GetProc)(const char*, void**, int, cuuint64_t, CUdriverProcAddressQueryResult*);
  GetProc gp = (GetProc)dlsym(h, "cuGetProcAddress_v2");
  if (!gp) { d.err = "libcuda has no cuGetProcAddress_v2"; return d; }
  bool ok = true;
  auto get = [&](const char* name, void** slot) {
    CUdriverProcAddressQueryResult q;
    if (gp(name, slot, 12000, CU_GET_PROC_ADDRESS_DEFAULT, &q) != CUDA_SUCCESS || !*slot) {
      ok = false;
      d.err = std::string("driver symbol missing: ") + name;
    }
  };
#define GFT_GET(fn) get(#fn, reinterpret_cast<void**>(&d.fn))
  GFT_GET(cuInit); GFT_GET(cuGetErrorString); GFT_GET(cuCtxGetCurrent); GFT_GET(cuCtxSetCurrent);
  GFT_GET(cuCtxGetDevice); GFT_GET(cuStreamGetCtx); GFT_GET(cuDeviceGet); GFT_GET(cuDeviceGetCount);
  GFT_GET(cuDeviceGetAttribute); GFT_GET(cuDevicePrimaryCtxRetain); GFT_GET(cuModuleLoadData);
  GFT_GET(cuModuleUnload); GFT_GET(cuModuleGetFunction); GFT_GET(cuFuncSetAttribute);
  GFT_GET(cuFuncGetAttribute); GFT_GET(cuOccupancyMaxActiveBlocksPerMultiprocessor);
  GFT_GET(cuLaunchKernel); GFT_GET(cuLaunchKernelEx); GFT_GET(cuTensorMapEncodeTiled); GFT_GET(cuMemcpyHtoDAsync);
  GFT_GET(cuMemcpyDtoHAsync); GFT_GET(cuStreamCreate); GFT_GET(cuEventCreate);
  GFT_GET(cuEventRecord); GFT_GET(cuStreamWaitEvent); GFT_GET(cuEventSynchronize);
  GFT_GET(cuEventElapsedTime); GFT_GET(cuEventDestroy);
#undef GFT_GET
  if (!ok) return d;
  CUresult r = d.cuInit(0);
  if (r != CUDA_SUCCESS) { d.err = "cuInit failed (" + std::to_string((int)r) + ")"; return d; }
  int cnt = 0;
  if (d.cuDeviceGetCount(&cnt) != CUDA_SUCCESS || cnt == 0) { d.err = "no CUDA device"; return d; }
  d.ok = true;
  return d;
}

Nvrtc& rtc() {
  static Nvrtc n;
  std::lock_guard<std::mutex> lk(g_init_mu);
  if (n.tried) return n;
  n.tried = true;
  const char* cands[] = {getenv("GFT_NVRTC_LIB"), "/usr/local/cuda/lib64/libnvrtc.so.12",
                         "libnvrtc.so.12", "libnvrtc.so"};
  void* h = nullptr;
  for (const char* c : cands)
    if (c && (h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
  if (!h) { n.err = "cannot load libnvrtc.so.12"; return n; }
  bool ok = true;
  auto get = [&](const char* name, void** slot) {
    *slot = dlsym(h, name);
    if (!*slot) { ok = false; n.err = std::string("nvrtc symbol missing: ") + name; }
  };
  get("nvrtcCreateProgram", reinterpret_cast<void**>(&n.create));
  get("nvrtcCompileProgram", reinterpret_cast<void**>(&n.compile));
  get("nvrtcGetProgramLogSize", reinterpret_cast<void**>(&n.log_size));
  get("nvrtcGetProgramLog", reinterpret_cast<void**>(&n.log));
  get("nvrtcGetCUBINSize", reinterpret_cast<void**>(&n.cubin_size));
  get("nvrtcGetCUBIN", reinterpret_cast<void**>(&n.cubin));
  get("nvrtcDestroyProgram", reinterpret_cast<void**>(&n.destroy));
  get("nvrtcGetErrorString", reinterpret_cast<void**>(&n.errstr));
  n.ok = ok;
  return n;
}

void ck(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  const char* s = nullptr;
  drv().cuGetErrorString(r, &s);
  fail(GFT_ERR_CUDA, std::string(what) + ": " + (s ? s : "unknown CUDA error") + " (" +
                         std::to_string((int)r) + ")");
}

Driver& need_driver() {
  Driver& d = drv();
  if (!d.ok) fail(GFT_ERR_NO_DEVICE, d.err);
  return d;
}

std::string lib_dir() {
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&lib_dir), &info) && info.dli_fname) {
    std::string p(info.dli_fname);
    size_t s = p.rfind('/');
    if (s != std::string::npos) return p.substr(0, s);
  }
  return ".";
}

bool read_file(const std::string& path, std::string& out) {
  std::ifstream f(path, std::ios::binary);
  if (!f) return false;
  std::ostringstream ss;
  ss << f.rdbuf();
  out = ss.str();
  return !out.empty();
}

CUcontext current_ctx(void* stream) {
  Driver& d = need_driver();
  CUcontext ctx = nullptr;
  if (stream) ck(d.cuStreamGetCtx((CUstream)stream, &ctx), "cuStreamGetCtx");
  else ck(d.cuCtxGetCurrent(&ctx), "cuCtxGetCurrent");
  if (!ctx) {
    CUdevice dev;
    ck(d.cuDeviceGet(&dev, 0), "cuDeviceGet");
    ck(d.cuDevicePrimaryCtxRetain(&ctx, dev), "cuDevicePrimaryCtxRetain");
  }
  CUcontext cur = nullptr;
  d.cuCtxGetCurrent(&cur);
  if (cur != ctx) ck(d.cuCtxSetCurrent(ctx), "cuCtxSetCurrent");
  return ctx;
}

LoadedFn& ensure_loaded(Kernel& k, CUcontext ctx, bool allow_cache) {
  std::lock_guard<std::mutex> lk(k.mu);
  auto it = k.loaded.find(ctx);
  if (it != k.loaded.end()) return it->second;
  if (k.cubin.empty()) compile_kernel(k, allow_cache);
  Driver& d = need_driver();
  LoadedFn L;
  CUmodule mod;
  ck(d.cuModuleLoadData(&mod, k.cubin.data()), "cuModuleLoadData");
  CUfunction fn;
  ck(d.cuModuleGetFunction(&fn, mod, k.name.c_str()), "cuModuleGetFunction");
  const int smem = k.cfg.smem_bytes();
  ck(d.cuFuncSetAttribute(fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem),
     "cuFuncSetAttribute(max dynamic smem)");
  int occ = 1;
  if (!k.cfg.tc_pair) {   // (cluster kernels: one CTA per SM by construction)
    ck(d.cuOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, k.cfg.threads(), smem), "occupancy");
    if (occ < 1) fail(GFT_ERR_CUDA, "kernel " + k.name + " cannot be resident (occupancy 0)");
  }
  CUdevice dev;
  ck(d.cuCtxGetDevice(&dev), "cuCtxGetDevice");
  int sms = 0;
  ck(d.cuDeviceGetAttribute(&sms, CU_DEVICE_ATTRIBUTE_MULTIPROCESSOR_COUNT, dev), "SM count");
  d.cuFuncGetAttribute(&L.regs, CU_FUNC_ATTRIBUTE_NUM_REGS, fn);
  L.module = mod;
  L.fn = fn;
  L.grid_max = sms * occ;
  if (k.cfg.tc_pair) L.grid_max &= ~1;
  return k.loaded.emplace(ctx, L).first->second;
}

std::atomic<uint64_t> g_kernel_uid{1};

// Per-thread cache of the last tensor maps built for a (kernel, in, out, rows) launch: a
// serving loop that re-launches on the same buffers skips two cuTensorMapEncodeTiled calls.
struct MapCacheEntry {
  uint64_t uid = 0;
  const void* in = nullptr;
  void* out = nullptr;
  int64_t rows = -1;
  CUtensorMap tin, tout;
};
constexpr int kMapCacheWays = 4;
thread_local MapCacheEntry t_map_cache[kMapCacheWays];
thread_local int t_map_next = 0;

// L2 sector promotion of the signal tensor maps (256 B default; GFT_L2PROMO=0/64/128/256
// for experiments)
CUtensorMapL2promotion l2_promotion() {
  static const CUtensorMapL2promotion p = [] {
    const char* e = getenv("GFT_L2PROMO");
    const int v = (e && *e) ? atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return p;
}

void encode_map(CUtensorMap* m, const Kernel& k, const void* ptr, int64_t rows) {
  Driver& d = need_driver();
  const KernelCfg& c = k.cfg;
  // mode 2: the packed view [rows / g, g*n] (g = c.pack signals per TMA row)
  const int64_t g = c.mode == 2 ? c.pack : 1;
  cuuint64_t dims[2] = {(cuuint64_t)(c.n * g), (cuuint64_t)(rows / g)};
  cuuint64_t strides[1] = {(cuuint64_t)(c.n * c.elem * g)};
  cuuint32_t box[2] = {(cuuint32_t)(c.mode == 2 ? g * c.n : c.boxc), (cuuint32_t)(c.tile_rows() / g)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = c.swz_mask == 7 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : c.swz_mask == 3 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : c.swz_mask == 1 ? CU_TENSOR_MAP_SWIZZLE_32B
                                            : CU_TENSOR_MAP_SWIZZLE_NONE;
  ck(d.cuTensorMapEncodeTiled(m, c.elem == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                              2, const_cast<void*>(ptr), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, l2_promotion(),
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE),
     "cuTensorMapEncodeTiled");
}

// PDL on by default; GFT_PDL=0 disables it (ablation)
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("GFT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// max rows per launch: TMA coordinates are int32
constexpr int64_t kMaxRowsPerLaunch = (int64_t)1 << 30;

}  // namespace

bool tuned_geometry(int n, int dtype, int64_t work, int kind, int& R, int& S, int& W, int& pace_ns, int& obuf) {
  // lines: "fma <n> <f32|f64> <R> <S> <W> [work=<FMAs per signal>] [kind=fwd|inv|dfwd|dinv|filter]
  // [pace=<ns>] [obuf=<0|1|2>]"; an entry with a work / kind key applies only to kernels with
  // exactly that leaf work / of that kind (plan-specific measurements); the most specific match
  // wins (work and kind > work > kind > plain).  pace = per-tile __nanosleep of the FMA
  // skeleton; obuf = output tiles per warp (IO split, kernel_skeleton.cuh).
  struct Entry { int n, dt, R, S, W, pace, kind, obuf; int64_t work; };
  static const std::vector<Entry> table = [] {
    std::vector<Entry> t;
    const char* e = getenv("GFT_TUNING_FILE");
    std::string path = (e && *e) ? std::string(e) : lib_dir() + "/../tuning.tsv";
    if (path == "none") return t;
    std::ifstream f(path);
    std::string line;
    static const char* kKinds[] = {"fwd", "inv", "dfwd", "dinv", "filter"};
    while (std::getline(f, line)) {
      std::istringstream ss(line);
      std::string mode, dt, extra;
      Entry x;
      if (!(ss >> mode >> x.n >> dt >> x.R >> x.S >> x.W) || mode != "fma") continue;
      x.dt = dt == "f64" ? GFT_F64 : GFT_F32;
      x.work = -1;
      x.pace = 0;
      x.kind = -1;
      x.obuf = 0;
      while ((ss >> extra) && extra[0] != '#') {
        if (extra.rfind("work=", 0) == 0) x.work = std::atoll(extra.c_str() + 5);
        else if (extra.rfind("pace=", 0) == 0) x.pace = std::atoi(extra.c_str() + 5);
        else if (extra.rfind("obuf=", 0) == 0) x.obuf = std::atoi(extra.c_str() + 5);
        else if (extra.rfind("kind=", 0) == 0)
          for (int k = 0; k < 5; ++k)
            if (extra.substr(5) == kKinds[k]) x.kind = k;
      }
      t.push_back(x);
    }
    return t;
  }();
  const Entry* hit = nullptr;
  int best = -1;
  for (const Entry& x : table) {
    if (x.n != n || x.dt != dtype) continue;
    if (x.work >= 0 && x.work != work) continue;
    if (x.kind >= 0 && x.kind != kind) continue;
    const int score = (x.work >= 0 ? 2 : 0) + (x.kind >= 0 ? 1 : 0);
    if (score > best) { best = score; hit = &x; }
  }
  if (!hit) return false;
  R = hit->R; S = hit->S; W = hit->W; pace_ns = hit->pace; obuf = hit->obuf;
  return true;
}

std::string cubin_cache_dir() {
  const char* e = getenv("GFT_CUBIN_DIR");
  if (e && *e) return e;
  return lib_dir() + "/kernels";
}

void compile_kernel(Kernel& k, bool allow_cache) {
  if (!k.cubin.empty()) return;
  if (allow_cache) {
    std::string path = cubin_cache_dir() + "/" + k.name + ".cubin";
    if (read_file(path, k.cubin)) { k.cubin_origin = "aot-cache"; return; }
  }
  Nvrtc& n = rtc();
  if (!n.ok) fail(GFT_ERR_COMPILE, n.err);
  nvrtcProgram prog;
  nvrtcResult r = n.create(&prog, k.source.c_str(), (k.name + ".cu").c_str(), 0, nullptr, nullptr);
  if (r != NVRTC_SUCCESS) fail(GFT_ERR_COMPILE, std::string("nvrtcCreateProgram: ") + n.errstr(r));
  const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo", "-DNDEBUG", "--fmad=true"};
  r = n.compile(prog, 5, opts);
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    if (ls) n.log(prog, &log[0]);
    n.destroy(&prog);
    fail(GFT_ERR_COMPILE, "NVRTC failed for " + k.name + ": " + log.substr(0, 2000));
  }
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  k.cubin.assign(cs, '\0');
  n.cubin(prog, &k.cubin[0]);
  n.destroy(&prog);
  k.cubin_origin = "nvrtc";
}

void kernel_launch_config(Kernel& k, int64_t batch, int* grid, int* block, int* smem, int* regs,
                          bool allow_cache) {
  CUcontext ctx = current_ctx(nullptr);
  LoadedFn& L = ensure_loaded(k, ctx, allow_cache);
  const int64_t rows = std::min<int64_t>(batch, kMaxRowsPerLaunch);
  const int64_t tiles = (rows + k.cfg.tile_rows() - 1) / k.cfg.tile_rows();
  const int64_t ctas = (tiles + k.cfg.tiles_per_cta() - 1) / k.cfg.tiles_per_cta();
  if (grid) *grid = (int)std::max<int64_t>(1, std::min<int64_t>(ctas, L.grid_max));
  if (block) *block = k.cfg.threads();
  if (smem) *smem = k.cfg.smem_bytes();
  if (regs) *regs = L.regs;
}

void launch_kernel(Kernel& k, const void* in, void* out, int64_t batch, void* stream,
                   bool allow_cache) {
  if (batch <= 0) return;
  Driver& d = need_driver();
  CUcontext ctx = current_ctx(stream);
  LoadedFn& L = ensure_loaded(k, ctx, allow_cache);
  const KernelCfg& c = k.cfg;
  const size_t row_bytes = (size_t)c.n * c.elem;
  for (int64_t off = 0; off < batch; off += kMaxRowsPerLaunch) {
    const int64_t rows = std::min<int64_t>(batch - off, kMaxRowsPerLaunch);
    const unsigned char* pin = static_cast<const unsigned char*>(in) + off * row_bytes;
    unsigned char* pout = static_cast<unsigned char*>(out) + off * row_bytes;
    alignas(64) CUtensorMap tin, tout;
    std::memset(&tin, 0, sizeof tin);
    std::memset(&tout, 0, sizeof tout);
    if (c.mode == 0 || (c.mode == 2 && rows >= c.pack)) {
      MapCacheEntry* hit = nullptr;
      for (auto& e : t_map_cache)
        if (e.uid == k.uid && e.in == pin && e.out == pout && e.rows == rows) { hit = &e; break; }
      if (!hit) {
        hit = &t_map_cache[t_map_next];
        t_map_next = (t_map_next + 1) % kMapCacheWays;
        hit->uid = 0;   // invalid until both maps are encoded
        encode_map(&hit->tin, k, pin, rows);
        encode_map(&hit->tout, k, pout, rows);
        hit->uid = k.uid;
        hit->in = pin;
        hit->out = pout;
        hit->rows = rows;
      }
      std::memcpy(&tin, &hit->tin, sizeof tin);
      std::memcpy(&tout, &hit->tout, sizeof tout);
    }
    const int64_t tiles = (rows + c.tile_rows() - 1) / c.tile_rows();
    int64_t ctas = (tiles + c.tiles_per_cta() - 1) / c.tiles_per_cta();
    if (c.tc_pair) ctas = (ctas + 1) & ~int64_t(1);
    const unsigned grid = (unsigned)std::max<int64_t>(c.tc_pair ? 2 : 1, std::min<int64_t>(ctas, L.grid_max));
    long long nrows = rows;
    const void* xin = pin;
    void* xout = pout;
    void* args[] = {&tin, &tout, &xin, &xout, &nrows};
    // Programmatic dependent launch: the kernel may be scheduled while the previous kernel
    // in the stream drains; it executes griddepcontrol.wait before its first global read.
    CUlaunchAttribute attr[1];
    attr[0].id = CU_LAUNCH_ATTRIBUTE_PROGRAMMATIC_STREAM_SERIALIZATION;
    attr[0].value.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    CUlaunchConfig lc;
    std::memset(&lc, 0, sizeof lc);
    lc.gridDimX = grid; lc.gridDimY = 1; lc.gridDimZ = 1;
    lc.blockDimX = c.threads(); lc.blockDimY = 1; lc.blockDimZ = 1;
    lc.sharedMemBytes = c.smem_bytes();
    lc.hStream = (CUstream)stream;
    lc.attrs = attr;
    lc.numAttrs = 1;
    ck(d.cuLaunchKernelEx(&lc, (CUfunction)L.fn, args, nullptr), "cuLaunchKernelEx");
  }
}

double time_kernel_ms(Kernel& k, const void* in, void* out, int64_t batch, void* stream, int warm,
                      int reps, bool allow_cache) {
  Driver& d = need_driver();
  current_ctx(stream);
  for (int i = 0; i < warm; ++i) launch_kernel(k, in, out, batch, stream, allow_cache);
  CUevent a, b;
  ck(d.cuEventCreate(&a, CU_EVENT_DEFAULT), "cuEventCreate");
  if (d.cuEventCreate(&b, CU_EVENT_DEFAULT) != CUDA_SUCCESS) {
    d.cuEventDestroy(a);
    fail(GFT_ERR_CUDA, "cuEventCreate");
  }
  float ms = 0.f;
  CUresult r = d.cuEventRecord(a, (CUstream)stream);
  try {
    for (int i = 0; i < reps && r == CUDA_SUCCESS; ++i) launch_kernel(k, in, out, batch, stream, allow_cache);
  } catch (...) {
    d.cuEventDestroy(a);
    d.cuEventDestroy(b);
    throw;
  }
  if (r == CUDA_SUCCESS) r = d.cuEventRecord(b, (CUstream)stream);
  if (r == CUDA_SUCCESS) r = d.cuEventSynchronize(b);
  if (r == CUDA_SUCCESS) r = d.cuEventElapsedTime(&ms, a, b);
  d.cuEventDestroy(a);
  d.cuEventDestroy(b);
  ck(r, "timing events");
  return (double)ms / std::max(1, reps);
}

void unload_kernel(Kernel& k) {
  Driver& d = drv();
  if (!d.ok) return;
  std::lock_guard<std::mutex> lk(k.mu);
  for (auto& kv : k.loaded) {
    CUcontext cur = nullptr;
    d.cuCtxGetCurrent(&cur);
    if (cur != (CUcontext)kv.first) d.cuCtxSetCurrent((CUcontext)kv.first);
    d.cuModuleUnload((CUmodule)kv.second.module);
    if (cur && cur != (CUcontext)kv.first) d.cuCtxSetCurrent(cur);
  }
  k.loaded.clear();
}

namespace {
constexpr int kMaxHostSlots = 4;
struct HostStreams {
  CUstream s[kMaxHostSlots];        // stage streams: s[0] H2D, s[1] kernels, s[2] D2H
  CUevent start, done[kMaxHostSlots];
  CUevent h2d[kMaxHostSlots], kdone[kMaxHostSlots], d2h[kMaxHostSlots];   // per workspace slot
  std::mutex mu;                    // one enqueue at a time (events are reused across calls)
};
std::mutex g_hs_mu;
std::map<CUcontext, HostStreams*> g_hs;
HostStreams& host_streams(CUcontext ctx) {
  std::lock_guard<std::mutex> lk(g_hs_mu);
  auto it = g_hs.find(ctx);
  if (it != g_hs.end()) return *it->second;
  Driver& d = need_driver();
  HostStreams* h = new HostStreams();   // lives as long as the process (like the context's modules)
  for (int i = 0; i < kMaxHostSlots; ++i) ck(d.cuStreamCreate(&h->s[i], CU_STREAM_NON_BLOCKING), "cuStreamCreate");
  ck(d.cuEventCreate(&h->start, CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  for (int i = 0; i < kMaxHostSlots; ++i) {
    ck(d.cuEventCreate(&h->done[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    ck(d.cuEventCreate(&h->h2d[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    ck(d.cuEventCreate(&h->kdone[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
    ck(d.cuEventCreate(&h->d2h[i], CU_EVENT_DISABLE_TIMING), "cuEventCreate");
  }
  g_hs.emplace(ctx, h);
  return *h;
}

}  // namespace

void execute_host(Kernel& k, const void* in_host, void* out_host, int64_t batch, void* workspace,
                  size_t workspace_bytes, int64_t chunk_rows, void* stream, bool allow_cache) {
  if (batch <= 0) return;
  if (chunk_rows <= 0) fail(GFT_ERR_INVALID_ARG, "chunk_rows must be > 0");
  const size_t row_bytes = (size_t)k.cfg.n * k.cfg.elem;
  const size_t chunk_bytes = (size_t)chunk_rows * row_bytes;
  if (!workspace || workspace_bytes < 2 * chunk_bytes)
    fail(GFT_ERR_INVALID_ARG, "workspace smaller than 2 * chunk_rows * n * sizeof(dtype)");
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) || (chunk_bytes & 15))
    fail(GFT_ERR_ALIGNMENT, "workspace / chunk not 16-byte aligned");
  Driver& d = need_driver();
  CUcontext ctx = current_ctx(stream);
  HostStreams& hs = host_streams(ctx);
  std::lock_guard<std::mutex> lk(hs.mu);
  const int slots = (int)std::min<size_t>(kMaxHostSlots, workspace_bytes / chunk_bytes);
  // (a geometric ramp of small first / last chunks to shorten the pipeline fill and drain
  // measured no gain on cfg2, 44.9 GB/s each way either way -- tools/e2e_probe.py)
  std::vector<int64_t> chunks;
  for (int64_t off = 0; off < batch; off += chunk_rows) chunks.push_back(std::min(chunk_rows, batch - off));
  // Three stage streams: every H2D on one stream (the H2D copy engine runs back to back),
  // every kernel on a second, every D2H on a third; per workspace slot, events order
  // H2D -> kernel -> D2H and the slot's next H2D after its previous D2H.  Per-slot streams
  // (H2D, kernel, D2H of one chunk on one stream) stall the next H2D behind the kernel.
  CUstream sh = hs.s[0], sk = hs.s[1], sd = hs.s[2];
  ck(d.cuEventRecord(hs.start, (CUstream)stream), "cuEventRecord");
  for (int i = 0; i < 3; ++i) ck(d.cuStreamWaitEvent(hs.s[i], hs.start, 0), "cuStreamWaitEvent");
  int64_t off = 0;
  for (size_t c = 0; c < chunks.size(); ++c) {
    const int slot = (int)(c % slots);
    const int64_t rows = chunks[c];
    unsigned char* buf = static_cast<unsigned char*>(workspace) + slot * chunk_bytes;
    if ((int)c >= slots) ck(d.cuStreamWaitEvent(sh, hs.d2h[slot], 0), "cuStreamWaitEvent");
    ck(d.cuMemcpyHtoDAsync((CUdeviceptr)buf, static_cast<const unsigned char*>(in_host) + off * row_bytes,
                           rows * row_bytes, sh),
       "cuMemcpyHtoDAsync");
    ck(d.cuEventRecord(hs.h2d[slot], sh), "cuEventRecord");
    ck(d.cuStreamWaitEvent(sk, hs.h2d[slot], 0), "cuStreamWaitEvent");
    launch_kernel(k, buf, buf, rows, sk, allow_cache);
    ck(d.cuEventRecord(hs.kdone[slot], sk), "cuEventRecord");
    ck(d.cuStreamWaitEvent(sd, hs.kdone[slot], 0), "cuStreamWaitEvent");
    ck(d.cuMemcpyDtoHAsync(static_cast<unsigned char*>(out_host) + off * row_bytes, (CUdeviceptr)buf,
                           rows * row_bytes, sd),
       "cuMemcpyDtoHAsync");
    ck(d.cuEventRecord(hs.d2h[slot], sd), "cuEventRecord");
    off += rows;
  }
  // the D2H stream's last copy follows every kernel and H2D of this call
  ck(d.cuEventRecord(hs.done[0], sd), "cuEventRecord");
  ck(d.cuStreamWaitEvent((CUstream)stream, hs.done[0], 0), "cuStreamWaitEvent");
}

Kernel::Kernel() : uid(g_kernel_uid.fetch_add(1)) {}

}  // namespace gft
