// kernel_tc_skeleton.cuh — fused fast-GFT kernel with tensor-core (tcgen05, 3xTF32) leaves.
//
// Used when a plan has large dense sub-GFT blocks (e.g. the two 64x64 leaves of cfg5b),
// which on CUDA cores would make the kernel FMA-bound (16 flop/B > the FP32 ridge).
// Each large leaf is a micro-GEMM over the tile: D[128 x Np] = A[128 x Kp] . B^T with
// A = the tile's leaf inputs (one TMEM lane per signal), B = the folded leaf matrix in
// SMEM.  fp32 accuracy is kept with the 3xTF32 split
//     A B ~= A_hi B_hi + A_hi B_lo + A_lo B_hi,   hi = rna_tf32(v), lo = v - hi,
// accumulated in fp32 in TMEM.  Small leaves and all Haar units stay on CUDA cores and
// run while the tensor core works.
//
// Warp roles (160 threads): warps 0-3 = compute, thread t owns tile row t and TMEM lane t;
// warp 4 = TMA producer/storer.  Per tile (128 signals):
//   producer: TMA load (mbarrier full[s]) ... waits done[s] -> TMA store -> reload
//   compute : SMEM row -> registers -> butterflies -> hi/lo of big-leaf inputs -> tcgen05.st
//             -> bar(128) -> thread 0 issues tcgen05.mma (TS form: A in TMEM, B in SMEM)
//             -> small leaves on FMA -> wait tcgen05.commit -> tcgen05.ld D -> SMEM row
// The generated prelude defines GFT_N, GFT_STAGES, GFT_TMEM_COLS, GFT_B_FLOATS, GFT_KNAME,
// GFT_NTC (number of tensor-core leaves, one MMA-completion mbarrier each), gft_tcB[]
// and gft_tile() (the per-tile compute sequence).
typedef unsigned int u32;
typedef unsigned long long u64;
typedef float elem_t;

struct __align__(64) TmaDesc { u64 d[16]; };

#define GFT_TILE_ROWS 128
// tile rows are padded to whole 32-float (128 B) TMA boxes; TMA zero-fills the columns
// beyond n on load and clips them on store, so any n % 4 == 0 works
#define GFT_NP ((GFT_N + 31) / 32 * 32)
#define GFT_ROW_BYTES (GFT_NP * 4)
#define GFT_TILE_BYTES (GFT_TILE_ROWS * GFT_ROW_BYTES)
#define GFT_BOXC 32
#define GFT_BOX_BYTES (GFT_TILE_ROWS * 128)
#define GFT_NBOX (GFT_NP / GFT_BOXC)

static __device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
static __device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
static __device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_arrive(u32 bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(bar) : "memory");
}
static __device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
static __device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
static __device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
static __device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
static __device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
static __device__ __forceinline__ void tma_load_2d(u32 dst, const TmaDesc* desc, int c0, int c1, u32 bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"((u64)desc), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
static __device__ __forceinline__ void tma_store_2d(const TmaDesc* desc, int c0, int c1, u32 src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               :: "l"((u64)desc), "r"(c0), "r"(c1), "r"(src) : "memory");
}
static __device__ __forceinline__ void named_bar(u32 id, u32 n) {
  asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}
// ---- tcgen05 ----
static __device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
static __device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
static __device__ __forceinline__ void tc_commit(u32 bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(bar) : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem desc]^T   (kind::tf32, M=128, K=8)
static __device__ __forceinline__ void mma_ts(u32 d, u32 a, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p; }"
               :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
// K-major, 128B-swizzled operand: 8-row core-matrix groups 1024 B apart (SBO)
static __device__ __forceinline__ u64 smem_desc_sw128(u32 saddr) {
  return (u64)((saddr >> 4) & 0x3FFFu) | ((u64)(16u >> 4) << 16) | ((u64)(1024u >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
static __device__ __forceinline__ u32 tf32_rna(float v) {
  u32 r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}
// byte offset of (row, col) in a stage buffer: NBOX boxes [128 rows x 128 B], 128B swizzle
static __device__ __forceinline__ u32 tile_off(int row, int col) {
  const u32 lin = (u32)((col >> 5) * GFT_BOX_BYTES + row * 128 + (col & 31) * 4);
  return lin ^ (((lin >> 7) & 7u) << 4);
}
static __device__ __forceinline__ void load_row(const unsigned char* buf, int row, float (&x)[GFT_N]) {
#pragma unroll
  for (int c = 0; c < GFT_N; c += 4) {
    float4 v = *reinterpret_cast<const float4*>(buf + tile_off(row, c));
    x[c] = v.x; x[c + 1] = v.y; x[c + 2] = v.z; x[c + 3] = v.w;
  }
}
static __device__ __forceinline__ void store_row(unsigned char* buf, int row, const float (&y)[GFT_N]) {
#pragma unroll
  for (int c = 0; c < GFT_N; c += 4)
    *reinterpret_cast<float4*>(buf + tile_off(row, c)) = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
}

// @@GFT_GENERATED@@  (codegen.cpp inserts gft_tcB[] and the gft_* phase functions here)

extern "C" __global__ void __launch_bounds__(160, 1)
GFT_KNAME(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
          const float* X, float* Y, long long batch) {
  extern __shared__ unsigned char smem_raw[];
  const u32 raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  unsigned char* stages = smem;
  unsigned char* bsm = smem + GFT_STAGES * GFT_TILE_BYTES;            // B operands (1024-aligned)
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bsm + GFT_B_FLOATS * 4);
  // bars: full[S], done[S], mma
  u32* tmem_slot = reinterpret_cast<u32*>(bars + 2 * GFT_STAGES + GFT_NTC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const long long ntiles = (batch + GFT_TILE_ROWS - 1) / GFT_TILE_ROWS;
  // programmatic dependent launch: wait for the previous grid before touching global memory
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {   // TMEM allocation (whole warp), then release the permit
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_slot)), "n"(GFT_TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 128) {
    for (int s = 0; s < GFT_STAGES; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[GFT_STAGES + s]), 4);
    }
    for (int i = 0; i < GFT_NTC; ++i) mbar_init(smem_u32(&bars[2 * GFT_STAGES + i]), 1);
    fence_mbar_init();
  }
  // B operands (plan constants) -> SMEM, K-major 128B-swizzled atoms of [Np rows x 32 k]
  for (int i = tid; i < GFT_B_FLOATS / 4; i += blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(gft_tcB)[i];
    const u32 lin = (u32)i * 16u;
    *reinterpret_cast<float4*>(bsm + (lin ^ (((lin >> 7) & 7u) << 4))) = v;
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const u32 tmem = *tmem_slot;

  if (warp == 4) {
    // ---------------- producer / storer ----------------
    if (lane == 0) {
      long long it = 0;
      for (;; ++it) {
        const long long t = blockIdx.x + it * (long long)gridDim.x;
        if (t >= ntiles) break;
        const int s = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) {
          const long long tp = t - GFT_STAGES * (long long)gridDim.x;
          mbar_wait(smem_u32(&bars[GFT_STAGES + s]), (u32)(((it / GFT_STAGES) - 1) & 1));
          const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
          for (int b = 0; b < GFT_NBOX; ++b)
            tma_store_2d(&tout, b * GFT_BOXC, (int)(tp * GFT_TILE_ROWS), src + b * GFT_BOX_BYTES);
          bulk_commit();
          bulk_wait_read0();
        }
        const u32 bar = smem_u32(&bars[s]);
        const u32 dst = smem_u32(stages + s * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)(t * GFT_TILE_ROWS), bar);
      }
      // drain: store the last min(it, STAGES) tiles
      const long long first = it > GFT_STAGES ? it - GFT_STAGES : 0;
      for (long long j = first; j < it; ++j) {
        const int s = (int)(j % GFT_STAGES);
        const long long t = blockIdx.x + j * (long long)gridDim.x;
        mbar_wait(smem_u32(&bars[GFT_STAGES + s]), (u32)((j / GFT_STAGES) & 1));
        const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_store_2d(&tout, b * GFT_BOXC, (int)(t * GFT_TILE_ROWS), src + b * GFT_BOX_BYTES);
        bulk_commit();
      }
      bulk_wait_all();
    }
  } else {
    // ---------------- compute (thread tid = tile row tid = TMEM lane tid) ----------------
    const u32 tm_lane = tmem + ((u32)(warp * 32) << 16);
    const u32 bsm_s = smem_u32(bsm);
    for (long long it = 0;; ++it) {
      const long long t = blockIdx.x + it * (long long)gridDim.x;
      if (t >= ntiles) break;
      const int s = (int)(it % GFT_STAGES);
      mbar_wait(smem_u32(&bars[s]), (u32)((it / GFT_STAGES) & 1));
      unsigned char* buf = stages + s * GFT_TILE_BYTES;
      float x[GFT_N], y[GFT_N];
      load_row(buf, tid, x);
      // generated: butterflies; per big leaf: hi/lo -> TMEM, bar(128), thread 0 issues the
      // leaf's MMAs + commit (the next leaf is staged while they run); small leaves on FMA;
      // per big leaf: wait its commit, TMEM -> registers; reverse butterflies (inverse)
      gft_tile(x, y, tm_lane, tmem, bsm_s, smem_u32(&bars[2 * GFT_STAGES]), (u32)(it & 1), tid);
      store_row(buf, tid, y);
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars[GFT_STAGES + s]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(GFT_TMEM_COLS) : "memory");
  }
}
