// odd_pitch_probe2.cu -- second odd-pitch experiment: TMA 2-D tensor copies of a flat
// 128-byte-row view of the 2^21 x 25 f32 batch (6400-B tiles = 50 box rows) vs 1-D bulk
// copies, varying swizzle, L2 promotion and an artificial per-row FMA load ("spin") that
// stands in for the transform's arithmetic.  Pure copies (the bytes are moved unchanged).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o p2 tools/odd_pitch_probe2.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
typedef unsigned int u32;
typedef unsigned long long u64;
struct __align__(64) TmaDesc { CUtensorMap m; };

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(u32 bar, u32 par) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(par) : "memory");
  } while (!done);
}

template <int MODE, int TILE, int S, int W, int SPIN>   // MODE 0: TMA 2-D flat view, 1: 1-D bulk
__global__ void __launch_bounds__(W * 32) k_copy(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
                                                 const unsigned char* X, unsigned char* Y, long long nbytes, float* sink) {
  extern __shared__ unsigned char sm_raw[];
  unsigned char* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sm + warp * S * TILE;
  u64* bars = reinterpret_cast<u64*>(sm + W * S * TILE) + warp * S;
  const long long ntiles = nbytes / TILE;
  const long long gw = (long long)blockIdx.x * W + warp, nw = (long long)gridDim.x * W;
  if (gw >= ntiles) return;
  auto load = [&](long long t, int s) {
    u32 bar = smem_u32(&bars[s]), dst = smem_u32(wb + s * TILE);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(TILE) : "memory");
    if (MODE == 0)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"((u64)&tin), "r"(0), "r"((int)(t * (TILE / 128))), "r"(bar) : "memory");
    else
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(X + t * TILE), "r"(TILE), "r"(bar) : "memory");
  };
  auto store = [&](long long t, int s) {
    u32 src = smem_u32(wb + s * TILE);
    if (MODE == 0)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                   ::"l"((u64)&tout), "r"(0), "r"((int)(t * (TILE / 128))), "r"(src) : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(Y + t * TILE), "r"(src), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < S; ++s)
      if (gw + s * nw < ntiles) load(gw + s * nw, s);
  }
  __syncwarp();
  float acc = lane;
  for (long long it = 0;; ++it) {
    long long t = gw + it * nw;
    if (t >= ntiles) break;
    int s = (int)(it % S);
    mbar_wait(smem_u32(&bars[s]), (u32)((it / S) & 1));
#pragma unroll 1
    for (int i = 0; i < SPIN; ++i) acc = __fmaf_rn(acc, 1.000001f, 0.5f);
    __syncwarp();
    if (lane == 0) {
      store(t, s);
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (it >= 1 && gw + (it - 1 + S) * nw < ntiles) load(gw + (it - 1 + S) * nw, (int)((it - 1) % S));
    }
    __syncwarp();
  }
  if (acc == 12345.f) sink[0] = acc;
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename F>
float timeit(F f, int iters = 50) {
  for (int i = 0; i < 5; ++i) f();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < iters; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / iters;
}

void encode(TmaDesc* d, void* p, long long nbytes, int box_rows, CUtensorMapSwizzle sw, CUtensorMapL2promotion pr) {
  cuuint64_t dims[2] = {32, (cuuint64_t)(nbytes / 128)};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows}, es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&d->m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, p, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, sw, pr, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
}

template <int MODE, int TILE, int S, int W, int SPIN>
void run(const char* name, unsigned char* X, unsigned char* Y, long long nbytes, int cps, CUtensorMapSwizzle sw,
         CUtensorMapL2promotion pr, float* sink) {
  TmaDesc a, b;
  encode(&a, X, nbytes, TILE / 128, sw, pr);
  encode(&b, Y, nbytes, TILE / 128, sw, pr);
  auto k = k_copy<MODE, TILE, S, W, SPIN>;
  int smem = W * S * TILE + W * S * 8 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  float ms = timeit([&] { k<<<148 * cps, W * 32, smem>>>(a, b, X, Y, nbytes, sink); });
  printf("{\"variant\": \"%s\", \"mode\": \"%s\", \"tile\": %d, \"S\": %d, \"W\": %d, \"cps\": %d, \"spin\": %d, \"swz\": %d, \"promo\": %d, \"gbs\": %.1f, \"err\": \"%s\"}\n",
         name, MODE == 0 ? "tma2d" : "bulk1d", TILE, S, W, cps, SPIN, (int)sw, (int)pr, 2.0 * nbytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  cuInit(0);
  const long long nbytes = (1ll << 21) * 25 * 4;
  unsigned char *X, *Y;
  float* sink;
  cudaMalloc(&X, nbytes);
  cudaMalloc(&Y, nbytes);
  cudaMalloc(&sink, 4);
  cudaMemset(X, 1, nbytes);
  const auto N0 = CU_TENSOR_MAP_SWIZZLE_NONE, S128 = CU_TENSOR_MAP_SWIZZLE_128B;
  const auto P0 = CU_TENSOR_MAP_L2_PROMOTION_NONE, P256 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             P128 = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  for (int rep = 0; rep < 2; ++rep) {
    run<1, 6400, 2, 8, 0>("bulk", X, Y, nbytes, 1, N0, P0, sink);
    run<1, 6400, 2, 8, 200>("bulk", X, Y, nbytes, 1, N0, P0, sink);
    run<1, 6400, 3, 4, 200>("bulk", X, Y, nbytes, 2, N0, P0, sink);
    run<0, 6400, 2, 8, 0>("tma", X, Y, nbytes, 1, N0, P256, sink);
    run<0, 6400, 2, 8, 200>("tma", X, Y, nbytes, 1, N0, P256, sink);
    run<0, 6400, 2, 8, 0>("tma", X, Y, nbytes, 1, N0, P0, sink);
    run<0, 6400, 2, 8, 200>("tma", X, Y, nbytes, 1, N0, P0, sink);
    run<0, 6400, 2, 8, 200>("tma", X, Y, nbytes, 1, N0, P128, sink);
    run<0, 8192, 2, 8, 0>("tma 8K", X, Y, nbytes, 1, S128, P256, sink);
    run<0, 8192, 2, 8, 200>("tma 8K", X, Y, nbytes, 1, S128, P256, sink);
    run<0, 8192, 2, 8, 200>("tma 8K noswz", X, Y, nbytes, 1, N0, P256, sink);
    run<0, 6400, 3, 4, 200>("tma", X, Y, nbytes, 2, N0, P256, sink);
    run<0, 6400, 2, 8, 400>("tma", X, Y, nbytes, 1, N0, P256, sink);
    run<0, 6400, 3, 8, 200>("tma", X, Y, nbytes, 1, N0, P256, sink);
  }
  return 0;
}
