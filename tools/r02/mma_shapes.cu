// tcgen05.mma kind::tf32 throughput by shape (TS form: A in TMEM, B in SMEM): cycles per
// instruction issued back to back into one accumulator, cta_group::1 (M=128) and
// cta_group::2 (M=256, cluster of 2), N = 32 .. 256.  One CTA (pair) per SM (pair of SMs),
// all SMs busy.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_shapes mma_shapes.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned int u32;
typedef unsigned long long u64;
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

template <int CG, int N>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cyc) {
  __shared__ __align__(1024) unsigned char bsm[256 * 128];
  __shared__ __align__(8) u64 bar;
  __shared__ u32 tslot;
  const int warp = threadIdx.x >> 5;
  u32 rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<u32*>(bsm)[i] = 0x3f800000u;
  if (warp == 0) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tslot;
  if (threadIdx.x == 0 && rank == 0) {
    const u32 mdim = CG == 2 ? 16u : 8u;
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((u32)(N >> 3) << 17) | (mdim << 24);
    const u32 sb = smem_u32(bsm);
    const u64 bdesc = (u64)((sb >> 4) & 0x3FFFu) | ((u64)(16u >> 4) << 16) | ((u64)(1024u >> 4) << 32) |
                      (1ull << 46) | (2ull << 61);
    const u64 t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const u64 bd = bdesc + (u64)((j & 3) * 2);
        if (CG == 2)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p; }"
                       :: "r"(tmem), "r"(tmem + 256u), "l"(bd), "r"(idesc), "r"(it | j) : "memory");
        else
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
                       :: "r"(tmem), "r"(tmem + 256u), "l"(bd), "r"(idesc), "r"(it | j) : "memory");
      }
    }
    if (CG == 2)
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                   :: "r"(smem_u32(&bar)), "h"((unsigned short)3) : "memory");
    else
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                   :: "r"(smem_u32(&bar)) : "memory");
    u32 done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    } while (!done);
    cyc[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 0 && CG == 2) {
    u32 done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    } while (!done);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else __syncthreads();
  if (warp == 0) {
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" :: "r"(tmem) : "memory");
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem) : "memory");
  }
}

template <int CG, int N>
void run(int sms) {
  const int iters = 256;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaMemset(d, 0, sms * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms);
  cfg.blockDim = dim3(128);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, probe<CG, N>, iters, d);
  cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0; int cnt = 0;
  for (int i = 0; i < sms; i += CG) { sum += h[i]; cnt++; if (h[i] > mx) mx = h[i]; }
  const double per = sum / cnt / (iters * 16.0);
  const double macs_per_sm = 128.0 * N * 8;   // per SM per instruction (M/CG rows = 128)
  printf("cta_group::%d M=%d N=%3d: %.1f cycles/instr (mean over CTAs), %.0f MAC/clk/SM, err=%s\n", CG, 128 * CG, N,
         per, macs_per_sm / per, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<1, 32>(sms); run<1, 64>(sms); run<1, 128>(sms); run<1, 256>(sms);
  run<2, 32>(sms); run<2, 64>(sms); run<2, 128>(sms); run<2, 256>(sms);
  return 0;
}
