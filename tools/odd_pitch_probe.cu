// odd_pitch_probe.cu -- copy-ceiling experiment for the odd-pitch (n = 25 f32, 100-byte rows)
// data path: which HBM -> SMEM -> HBM mechanism moves a 2^21 x 25 f32 batch fastest?
//   v1: per-warp 1-D bulk copies of 64-row tiles (6400 B), like the mode-1 skeleton
//   v2: v1 with an L2 evict_first cache hint on loads and stores
//   v3: per-warp 1-D bulk copies of 8192-B chunks (ignores row boundaries: ceiling only)
//   v4: LDG.128 / STG.128 grid-stride copy (no SMEM), the torch-copy pattern
//   v5: v1 with per-thread row reads/writes through SMEM (25 LDS + 25 STS per row)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o odd_pitch_probe tools/odd_pitch_probe.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned int u32;
typedef unsigned long long u64;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u32 bar, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 par) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(par) : "memory");
  } while (!done);
}
template <bool HINT>
__device__ __forceinline__ void bulk_load(u32 dst, const void* src, u32 bytes, u32 bar, u64 pol) {
  if (HINT)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
template <bool HINT>
__device__ __forceinline__ void bulk_store(void* dst, u32 src, u32 bytes, u64 pol) {
  if (HINT)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
                 ::"l"(dst), "r"(src), "r"(bytes), "l"(pol) : "memory");
  else
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// TILE bytes per warp tile, S stages, W warps; ROWS > 0: touch rows of N floats through SMEM
template <int TILE, int S, int W, bool HINT, int ROWS, int N>
__global__ void __launch_bounds__(W * 32) bulk_copy(const unsigned char* X, unsigned char* Y, long long nbytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wb = sm + warp * S * TILE;
  u64* bars = reinterpret_cast<u64*>(sm + W * S * TILE) + warp * S;
  const long long ntiles = nbytes / TILE;
  const long long gw = (long long)blockIdx.x * W + warp, nw = (long long)gridDim.x * W;
  if (gw >= ntiles) return;
  u64 pol = 0;
  if (HINT) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < S; ++s) {
      long long t = gw + s * nw;
      if (t < ntiles) {
        mbar_expect_tx(smem_u32(&bars[s]), TILE);
        bulk_load<HINT>(smem_u32(wb + s * TILE), X + t * TILE, TILE, smem_u32(&bars[s]), pol);
      }
    }
  }
  __syncwarp();
  for (long long it = 0;; ++it) {
    long long t = gw + it * nw;
    if (t >= ntiles) break;
    int s = (int)(it % S);
    mbar_wait(smem_u32(&bars[s]), (u32)((it / S) & 1));
    unsigned char* buf = wb + s * TILE;
    if (ROWS > 0) {
      for (int r = lane; r < ROWS; r += 32) {
        float x[N];
#pragma unroll
        for (int c = 0; c < N; ++c) x[c] = reinterpret_cast<float*>(buf)[r * N + c];
#pragma unroll
        for (int c = 0; c < N; ++c) reinterpret_cast<float*>(buf)[r * N + c] = x[N - 1 - c] * 1.0001f;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
    if (lane == 0) {
      bulk_store<HINT>(Y + t * TILE, smem_u32(buf), TILE, pol);
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      if (it >= 1) {
        long long tn = gw + (it - 1 + S) * nw;
        int sp = (int)((it - 1) % S);
        if (tn < ntiles) {
          mbar_expect_tx(smem_u32(&bars[sp]), TILE);
          bulk_load<HINT>(smem_u32(wb + sp * TILE), X + tn * TILE, TILE, smem_u32(&bars[sp]), pol);
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void vec_copy(const float4* X, float4* Y, long long n4) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x, st = (long long)gridDim.x * blockDim.x;
  for (; i < n4; i += st) Y[i] = X[i];
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

template <int TILE, int S, int W, bool HINT, int ROWS, int N>
void run(const char* name, const unsigned char* X, unsigned char* Y, long long nbytes, int ctas_per_sm) {
  auto k = bulk_copy<TILE, S, W, HINT, ROWS, N>;
  int smem = W * S * TILE + W * S * 8 + 128;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int grid = 148 * ctas_per_sm;
  float ms = timeit([&] { k<<<grid, W * 32, smem>>>(X, Y, nbytes); });
  cudaError_t e = cudaGetLastError();
  printf("{\"variant\": \"%s\", \"tile\": %d, \"S\": %d, \"W\": %d, \"ctas_per_sm\": %d, \"ms\": %.5f, \"gbs\": %.1f, \"err\": \"%s\"}\n",
         name, TILE, S, W, ctas_per_sm, ms, 2.0 * nbytes / ms / 1e6, cudaGetErrorString(e));
}

int main() {
  const long long rows = 1ll << 21, n = 25;
  const long long nbytes = rows * n * 4;   // 209715200 = 32768 * 6400 = 25600 * 8192
  unsigned char *X, *Y;
  cudaMalloc(&X, nbytes);
  cudaMalloc(&Y, nbytes);
  cudaMemset(X, 1, nbytes);
  float ms = timeit([&] { cudaMemcpyAsync(Y, X, nbytes, cudaMemcpyDeviceToDevice); });
  printf("{\"variant\": \"cudaMemcpy d2d\", \"ms\": %.5f, \"gbs\": %.1f}\n", ms, 2.0 * nbytes / ms / 1e6);
  for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
    ms = timeit([&] { vec_copy<<<blocks, 256>>>((const float4*)X, (float4*)Y, nbytes / 16); });
    printf("{\"variant\": \"v4 LDG.128 grid-stride\", \"blocks\": %d, \"ms\": %.5f, \"gbs\": %.1f}\n", blocks, ms, 2.0 * nbytes / ms / 1e6);
  }
  run<6400, 3, 4, false, 0, 25>("v1 bulk 64-row tiles", X, Y, nbytes, 2);
  run<6400, 2, 8, false, 0, 25>("v1 bulk 64-row tiles", X, Y, nbytes, 1);
  run<6400, 2, 12, false, 0, 25>("v1 bulk 64-row tiles", X, Y, nbytes, 1);
  run<6400, 3, 4, true, 0, 25>("v2 bulk 64-row tiles evict_first", X, Y, nbytes, 2);
  run<6400, 2, 12, true, 0, 25>("v2 bulk 64-row tiles evict_first", X, Y, nbytes, 1);
  run<8192, 2, 8, false, 0, 25>("v3 bulk 8192-B chunks", X, Y, nbytes, 1);
  run<8192, 3, 4, false, 0, 25>("v3 bulk 8192-B chunks", X, Y, nbytes, 2);
  run<12800, 2, 4, false, 0, 25>("v1 bulk 128-row tiles", X, Y, nbytes, 2);
  run<3200, 4, 8, false, 0, 25>("v1 bulk 32-row tiles", X, Y, nbytes, 2);
  run<3200, 3, 16, false, 0, 25>("v1 bulk 32-row tiles", X, Y, nbytes, 1);
  run<6400, 3, 4, false, 64, 25>("v5 rows through SMEM", X, Y, nbytes, 2);
  run<6400, 3, 4, true, 64, 25>("v5 rows through SMEM evict_first", X, Y, nbytes, 2);
  run<6400, 2, 12, false, 64, 25>("v5 rows through SMEM", X, Y, nbytes, 1);
  // the cfg2 shape for comparison: 128 rows x 64 B = 8192-B tiles, n = 16
  {
    const long long nb16 = (1ll << 22) * 16 * 4;
    unsigned char *X2, *Y2;
    cudaMalloc(&X2, nb16);
    cudaMalloc(&Y2, nb16);
    cudaMemset(X2, 1, nb16);
    run<8192, 2, 8, false, 128, 16>("cfg2-shape rows through SMEM (1-D bulk)", X2, Y2, nb16, 1);
    run<8192, 2, 8, false, 0, 16>("cfg2-shape bulk copy only", X2, Y2, nb16, 1);
    ms = timeit([&] { vec_copy<<<148 * 8, 256>>>((const float4*)X2, (float4*)Y2, nb16 / 16); });
    printf("{\"variant\": \"cfg2-shape LDG.128\", \"ms\": %.5f, \"gbs\": %.1f}\n", ms, 2.0 * nb16 / ms / 1e6);
  }
  return 0;
}
