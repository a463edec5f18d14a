// peaks.cu — same-run compute-peak microbenchmarks for bench.py's roofline denominators
// ("FP32 FMA, FP64 and TF32 peaks ... measure them with a microbenchmark in
// the same run").  Not part of the GFT product path: libgftpeaks.so is a measurement tool
// loaded only by bench.py (and its GPU test).
//
// Each probe runs a persistent grid (a multiple of the SM count) of independent work and
// returns the elapsed device time of one launch measured with CUDA events on the caller's
// stream, plus the number of floating-point operations that launch performed:
//   FFMA : 16 independent fp32 FMA chains per thread (multiplier / addend are kernel
//          parameters: the constant-bank operand form the generated kernels' immediates use),
//          1 FMA = 2 flop
//   FFMA_REG : the same with every operand in a register
//   FFMA2 : packed fma.rn.f32x2 with register operands, one multiplicand a scalar broadcast to
//          both halves (the register-tiled dense GEMM's form), 1 FFMA2 = 4 flop
//   DFMA : the same in fp64
//   TF32 : tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 256, K = 8, A from TMEM, B from
//          SMEM (the TS form the GFT's tensor-core leaves use), one issuing thread per SM,
//          back to back into one TMEM accumulator; 1 MAC = 2 flop.
// C ABI (plain pointers; 0 = ok, otherwise a cudaError_t value):
//   int gft_peak_run(int which /*0 ffma, 1 dfma, 2 tf32, 3 ffma_reg, 4 ffma2*/, int sms, void* stream,
//                    double* flops, double* ms);
#include <cuda_runtime.h>
#include <stdint.h>

typedef unsigned int u32;
typedef unsigned long long u64;

#define CHAINS 16

template <typename T>
__global__ void __launch_bounds__(256) fma_probe(T* out, int iters, T a, T b) {
  T acc[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) acc[i] = acc[i] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == (T)-12345.0) out[blockIdx.x] = s;   // never true; keeps the chains live
}

// 3-register FFMA (every operand in a register, as in a register-tiled GEMM): a[] and b are
// runtime values, so no immediate / constant-bank operand form can be used
__global__ void __launch_bounds__(256) ffma_reg_probe(float* out, const float* coef, int iters) {
  float acc[CHAINS], a[4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = (float)(threadIdx.x + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = coef[i];
  const float b = coef[4];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], a[(i + k) & 3], b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += acc[i];
  if (s == -12345.0f) out[blockIdx.x] = s;
}

// packed FFMA2 (fma.rn.f32x2, sm_100) in the dense GEMM's outer-product form: a register-pair
// accumulator, a register-pair multiplicand and a scalar register broadcast to both halves;
// 1 FFMA2 = 2 FMA = 4 flop
__global__ void __launch_bounds__(256) ffma2_probe(float* out, const float* coef, int iters) {
  u64 acc[CHAINS], b[4];
  float a[4];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) acc[i] = ((u64)(threadIdx.x + i) << 32) | (u64)(threadIdx.x * 3 + i);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    a[i] = coef[i];
    b[i] = reinterpret_cast<const u64*>(coef)[4 + i];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int i = 0; i < CHAINS; ++i)
        asm("{ .reg .b64 t; mov.b64 t, {%1, %1}; fma.rn.f32x2 %0, t, %2, %0; }"
            : "+l"(acc[i]) : "f"(a[(i + k) & 3]), "l"(b[(i >> 2) & 3]));
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s ^= acc[i];
  if (s == 0x123456789ull) out[blockIdx.x] = (float)s;
}

static __device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) tf32_probe(int iters, u32* sink) {
  // B operand: 256 rows (N) x 128 B (32 fp32 of K), K-major, 128B swizzle: 32 KiB
  __shared__ __align__(1024) unsigned char bsm[256 * 128];
  __shared__ __align__(8) u64 bar;
  __shared__ u32 tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 256 * 128 / 4; i += blockDim.x) reinterpret_cast<u32*>(bsm)[i] = 0x3f800000u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const u32 tmem = tslot;
  if (threadIdx.x == 0) {
    // D: columns 0..255, A: columns 256..263 (M = 128 lanes x K = 8)
    const u32 idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    const u32 sb = smem_u32(bsm);
    const u64 bdesc = (u64)((sb >> 4) & 0x3FFFu) | ((u64)(16u >> 4) << 16) | ((u64)(1024u >> 4) << 32) |
                      (1ull << 46) | (2ull << 61);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const u64 bd = bdesc + (u64)((j & 3) * 2);   // +32 B within the atom per K step
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
                     :: "r"(tmem), "r"(tmem + 256u), "l"(bd), "r"(idesc), "r"(it | j) : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(smem_u32(&bar)) : "memory");
    u32 done = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
    } while (!done);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    u32 v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n\ttcgen05.wait::ld.sync.aligned;"
                 : "=r"(v) : "r"(tmem) : "memory");
    if (v == 0x7fc00001u) sink[blockIdx.x] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(tmem) : "memory");
  }
}

extern "C" __attribute__((visibility("default"))) int gft_peak_run(int which, int sms, void* stream, double* flops,
                                                                    double* ms) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  void* buf = nullptr;
  cudaError_t err = cudaEventCreate(&e0);
  if (err == cudaSuccess) err = cudaEventCreate(&e1);
  if (err == cudaSuccess) err = cudaMalloc(&buf, 1 << 16);
  if (err == cudaSuccess) err = cudaMemsetAsync(buf, 0, 1 << 16, s);
  if (err != cudaSuccess) {   // release whatever was created
    if (buf) cudaFree(buf);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    return (int)err;
  }
  double f = 0.0;
  auto launch = [&](bool count) {
    if (which == 0) {
      const int blocks = sms * 8, iters = 2048;   // 8 x 256 threads per SM: 2048 resident
      fma_probe<float><<<blocks, 256, 0, s>>>((float*)buf, iters, 0.999999f, 1e-7f);
      if (count) f = 2.0 * blocks * 256.0 * iters * 16.0 * CHAINS;
    } else if (which == 1) {
      const int blocks = sms * 8, iters = 256;
      fma_probe<double><<<blocks, 256, 0, s>>>((double*)buf, iters, 0.999999, 1e-7);
      if (count) f = 2.0 * blocks * 256.0 * iters * 16.0 * CHAINS;
    } else if (which == 3) {
      const int blocks = sms * 8, iters = 2048;
      ffma_reg_probe<<<blocks, 256, 0, s>>>((float*)buf, (const float*)buf + 1024, iters);
      if (count) f = 2.0 * blocks * 256.0 * iters * 16.0 * CHAINS;
    } else if (which == 4) {
      const int blocks = sms * 8, iters = 2048;
      ffma2_probe<<<blocks, 256, 0, s>>>((float*)buf, (const float*)buf + 1024, iters);
      if (count) f = 4.0 * blocks * 256.0 * iters * 16.0 * CHAINS;
    } else {
      const int iters = 2048;
      tf32_probe<<<sms, 128, 0, s>>>(iters, (u32*)buf);
      if (count) f = 2.0 * sms * (double)iters * 16.0 * 128.0 * 256.0 * 8.0;
    }
  };
  launch(false);   // warm-up
  cudaEventRecord(e0, s);
  launch(true);
  cudaEventRecord(e1, s);
  err = cudaEventSynchronize(e1);
  float t = 0.f;
  if (err == cudaSuccess) err = cudaEventElapsedTime(&t, e0, e1);
  if (err == cudaSuccess) err = cudaGetLastError();
  cudaFree(buf);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *flops = f;
  *ms = (double)t;
  return (int)err;
}
