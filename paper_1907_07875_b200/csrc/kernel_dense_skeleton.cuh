// kernel_dense_skeleton.cuh — the in-run dense comparison Y = X W on CUDA cores (row H7 of
// "GFT realized by a single n x n matrix multiplication"),
// for n = 64 / 128: a register-tiled SGEMM / DGEMM with the whole n x n matrix resident in
// shared memory.  W = U (forward, y = U^T x per row) or U^T (inverse), row-major W[i][k].
//
// Why not the FFMA-immediate straight-line code of kernel_skeleton.cuh: at n = 128 that is
// 16384 instructions per signal (256 KiB of SASS) and the kernel stalls on instruction
// fetch (ncu r01: stall_no_instruction 4.96 per issue, FMA pipe 16%).  Here the inner loop
// is a few hundred instructions and every FFMA/DFMA has both operands in registers.
//
// Per CTA (GFT_THREADS = 128 or 256 compute threads + 1 TMA warp), persistent over tiles of GFT_BM
// rows: TMA 2-D boxes of 128 B x GFT_BM rows (128B swizzle) land in a GFT_STAGES ring; thread
// (ty, tx) accumulates the GFT_TM x GFT_TN outputs rows {ty + i*(GFT_BM/GFT_TM)} x column
// groups {tx*VEC + j*(GFT_N/NG)} (VEC = 16-byte vector of elements, NG = GFT_TN/VEC groups):
// per 16-byte chunk of k, GFT_TM vector loads of X (8 consecutive rows of a quarter warp hit 8
// distinct swizzled chunks: conflict-free) and VEC x NG vector loads of W (one address per
// quarter warp: broadcast), then VEC x GFT_TM x GFT_TN FMAs.  The outputs overwrite the tile
// in place (after a barrier of the compute threads) and the TMA warp stores it.
// Generated prelude: GFT_ELEM, GFT_ELEM_IS_DOUBLE, GFT_N, GFT_BM, GFT_TM, GFT_TN, GFT_STAGES, GFT_KNAME and
// `gft_W[GFT_N * GFT_N]`.
typedef unsigned int u32;
typedef unsigned long long u64;
typedef GFT_ELEM elem_t;

struct __align__(64) TmaDesc { u64 d[16]; };

#if GFT_ELEM_IS_DOUBLE
#define GFT_VEC 2
typedef double2 vec_t;
static __device__ __forceinline__ double fma_(double a, double b, double c) { return fma(a, b, c); }
#else
#define GFT_VEC 4
typedef float4 vec_t;
static __device__ __forceinline__ float fma_(float a, float b, float c) { return fmaf(a, b, c); }
#endif
// fp32: the outer product runs on the packed FFMA2 (fma.rn.f32x2, sm_100): one instruction does
// acc[i][j..j+1] += a[i] * b[j..j+1] with a[i] broadcast to both halves (ptxas folds the
// {a, a} pack into a .F32 scalar operand) -- half the issue slots of per-lane FFMAs for the same
// register operands; each lane is the same IEEE fma.rn, so results are bit-identical.
#ifndef GFT_DG_FFMA2
#if GFT_ELEM_IS_DOUBLE
#define GFT_DG_FFMA2 0
#else
#define GFT_DG_FFMA2 1
#endif
#endif
static __device__ __forceinline__ void ffma2_bcast(u64& d, float a, u64 b) {
  asm("{ .reg .b64 t; mov.b64 t, {%1, %1}; fma.rn.f32x2 %0, t, %2, %0; }" : "+l"(d) : "f"(a), "l"(b));
}
#define GFT_NG (GFT_TN / GFT_VEC)
#define GFT_BOXC (GFT_VEC * 8)
#define GFT_BOX_BYTES (GFT_BM * 128)
#define GFT_NBOX (GFT_N / GFT_BOXC)
#define GFT_TILE_BYTES (GFT_BM * GFT_N * (int)sizeof(elem_t))
#define GFT_TY (GFT_BM / GFT_TM)
#if GFT_TY * (GFT_N / GFT_TN) != GFT_THREADS || GFT_TY % 8 != 0
#error "dense tile geometry must match GFT_THREADS (and GFT_BM / GFT_TM % 8 == 0)"
#endif
#ifndef GFT_DG_WY   // default: a warp owns whole rows (all GFT_N / GFT_TN column threads)
#define GFT_DG_WY (32 / (GFT_N / GFT_TN))
#endif
#define GFT_DG_WX (32 / GFT_DG_WY)
#if GFT_TY % GFT_DG_WY != 0 || (GFT_N / GFT_TN) % GFT_DG_WX != 0 || GFT_DG_WY * GFT_DG_WX != 32
#error "dense warp shape must tile the thread grid"
#endif

static __device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
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
static __device__ __forceinline__ void compute_bar() {   // the GFT_THREADS compute threads only
  asm volatile("bar.sync 1, %0;" :: "n"(GFT_THREADS) : "memory");
}
// byte offset of the 16-byte chunk holding element (row, col) of a tile (128B swizzle)
static __device__ __forceinline__ u32 tile_off(int row, int col) {
  const u32 lin = (u32)((col / GFT_BOXC) * GFT_BOX_BYTES + row * 128 + (col % GFT_BOXC) * (int)sizeof(elem_t));
  return lin ^ (((lin >> 7) & 7u) << 4);
}

// @@GFT_GENERATED@@  (codegen.cpp inserts gft_W[] here)

extern "C" __global__ void __launch_bounds__(GFT_THREADS + 32, 1)
GFT_KNAME(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
          const elem_t* X, elem_t* Y, long long batch) {
  extern __shared__ unsigned char smem_raw[];
  const u32 raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  unsigned char* stages = smem;
  elem_t* wsm = reinterpret_cast<elem_t*>(smem + GFT_STAGES * GFT_TILE_BYTES);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(wsm + GFT_N * GFT_N);
  unsigned long long* full = bars;                 // TMA load landed
  unsigned long long* empty = bars + GFT_STAGES;   // outputs written (compute warps)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const long long ntiles = (batch + GFT_BM - 1) / GFT_BM;
  const long long t0 = blockIdx.x, nt = gridDim.x;

  if (tid == GFT_THREADS) {
    for (int st = 0; st < GFT_STAGES; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&empty[st]), GFT_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // W -> SMEM (row-major, unswizzled: every quarter warp reads one address = broadcast)
  {
    const vec_t* src = reinterpret_cast<const vec_t*>(gft_W);
    vec_t* dst = reinterpret_cast<vec_t*>(wsm);
    for (int i = tid; i < GFT_N * GFT_N / GFT_VEC; i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == GFT_THREADS / 32) {
    // ---------------- TMA producer / storer (one extra warp) ----------------
    if (lane == 0) {
      long long it = 0;
      for (;; ++it) {
        const long long t = t0 + it * nt;
        if (t >= ntiles) break;
        const int st = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) {
          mbar_wait(smem_u32(&empty[st]), (u32)(((it / GFT_STAGES) - 1) & 1));
          const long long prow = (t - GFT_STAGES * nt) * GFT_BM;
          const u32 src = smem_u32(stages + st * GFT_TILE_BYTES);
          for (int b = 0; b < GFT_NBOX; ++b) tma_store_2d(&tout, b * GFT_BOXC, (int)prow, src + b * GFT_BOX_BYTES);
          bulk_commit();
          bulk_wait_read0();
        }
        const u32 bar = smem_u32(&full[st]);
        const u32 dst = smem_u32(stages + st * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b) tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)(t * GFT_BM), bar);
      }
      const long long first = it > GFT_STAGES ? it - GFT_STAGES : 0;
      for (long long j = first; j < it; ++j) {
        const int st = (int)(j % GFT_STAGES);
        mbar_wait(smem_u32(&empty[st]), (u32)((j / GFT_STAGES) & 1));
        const long long row0 = (t0 + j * nt) * GFT_BM;
        const u32 src = smem_u32(stages + st * GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b) tma_store_2d(&tout, b * GFT_BOXC, (int)row0, src + b * GFT_BOX_BYTES);
        bulk_commit();
      }
      bulk_wait_all();
    }
    return;
  }

  // ---------------- compute: GFT_TM x GFT_TN outputs per thread ----------------
  // warp shape: GFT_DG_WY row-threads x GFT_DG_WX column-threads.  WY = 8 makes each X load one
  // 128-B wavefront (8 swizzled rows, broadcast to the WX column threads) and each W load WX
  // distinct 16-B chunks (one wavefront) instead of 32 rows x 1 column (4 wavefronts per X load)
  const int ty = (warp % (GFT_TY / GFT_DG_WY)) * GFT_DG_WY + lane % GFT_DG_WY;
  const int tx = (warp / (GFT_TY / GFT_DG_WY)) * GFT_DG_WX + lane / GFT_DG_WY;
  // rows ty + i*GFT_TY share (row & 7) (GFT_TY % 8 == 0), so the 128B-swizzle term of every X
  // address is one per-thread constant: addr = row_i * 128 + box(kc) + ((kc*elem % 128) ^ sw)
  const u32 sw = (u32)(ty & 7) << 4;
  const elem_t* wrow = wsm + tx * GFT_VEC;
  for (long long it = 0;; ++it) {
    const long long t = t0 + it * nt;
    if (t >= ntiles) break;
    const int s = (int)(it % GFT_STAGES);
    mbar_wait(smem_u32(&full[s]), (u32)((it / GFT_STAGES) & 1));
    unsigned char* buf = stages + s * GFT_TILE_BYTES;
    const unsigned char* xrow = buf + ty * 128;
#if GFT_DG_FFMA2
    u64 acc2[GFT_TM][GFT_TN / 2];   // column pairs (j, j+1) as one f32x2 register pair
#pragma unroll
    for (int i = 0; i < GFT_TM; ++i)
#pragma unroll
      for (int j = 0; j < GFT_TN / 2; ++j) acc2[i][j] = 0ull;
#else
    elem_t acc[GFT_TM][GFT_TN];
#pragma unroll
    for (int i = 0; i < GFT_TM; ++i)
#pragma unroll
      for (int j = 0; j < GFT_TN; ++j) acc[i][j] = (elem_t)0;
#endif
#ifndef GFT_DG_PREFETCH
#define GFT_DG_PREFETCH 0
#endif
#if GFT_DG_PREFETCH
    vec_t an[GFT_TM];   // next chunk's X vectors (software prefetch)
#pragma unroll
    for (int i = 0; i < GFT_TM; ++i)
      an[i] = *reinterpret_cast<const vec_t*>(xrow + sw + i * GFT_TY * 128);
#endif
#ifndef GFT_DG_UNROLL
#define GFT_DG_UNROLL 2
#endif
    constexpr int kUnroll = GFT_DG_UNROLL;   // (#pragma unroll does not macro-expand under nvcc)
#pragma unroll kUnroll
    for (int kc = 0; kc < GFT_N; kc += GFT_VEC) {
      elem_t a[GFT_TM][GFT_VEC];
#if GFT_DG_PREFETCH
#pragma unroll
      for (int i = 0; i < GFT_TM; ++i) {
        const elem_t* pv = reinterpret_cast<const elem_t*>(&an[i]);
#pragma unroll
        for (int q = 0; q < GFT_VEC; ++q) a[i][q] = pv[q];
      }
      if (kc + GFT_VEC < GFT_N) {
        const int kn = kc + GFT_VEC;
        const u32 koff = (u32)(kn / GFT_BOXC) * GFT_BOX_BYTES + ((u32)((kn % GFT_BOXC) * (int)sizeof(elem_t)) ^ sw);
#pragma unroll
        for (int i = 0; i < GFT_TM; ++i)
          an[i] = *reinterpret_cast<const vec_t*>(xrow + koff + i * GFT_TY * 128);
      }
#else
      const u32 koff = (u32)(kc / GFT_BOXC) * GFT_BOX_BYTES + ((u32)((kc % GFT_BOXC) * (int)sizeof(elem_t)) ^ sw);
#pragma unroll
      for (int i = 0; i < GFT_TM; ++i) {
        const vec_t v = *reinterpret_cast<const vec_t*>(xrow + koff + i * GFT_TY * 128);
        const elem_t* pv = reinterpret_cast<const elem_t*>(&v);
#pragma unroll
        for (int q = 0; q < GFT_VEC; ++q) a[i][q] = pv[q];
      }
#endif
#pragma unroll
      for (int q = 0; q < GFT_VEC; ++q) {
#if GFT_DG_FFMA2
        u64 b2[GFT_TN / 2];
#pragma unroll
        for (int j = 0; j < GFT_NG; ++j) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(wrow + (kc + q) * GFT_N + j * (GFT_N / GFT_NG));
          b2[2 * j] = v.x;
          b2[2 * j + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < GFT_TM; ++i)
#pragma unroll
          for (int j = 0; j < GFT_TN / 2; ++j) ffma2_bcast(acc2[i][j], a[i][q], b2[j]);
#else
        elem_t b[GFT_TN];
#pragma unroll
        for (int j = 0; j < GFT_NG; ++j) {
          const vec_t v = *reinterpret_cast<const vec_t*>(wrow + (kc + q) * GFT_N + j * (GFT_N / GFT_NG));
          const elem_t* pv = reinterpret_cast<const elem_t*>(&v);
#pragma unroll
          for (int e = 0; e < GFT_VEC; ++e) b[j * GFT_VEC + e] = pv[e];
        }
#pragma unroll
        for (int i = 0; i < GFT_TM; ++i)
#pragma unroll
          for (int j = 0; j < GFT_TN; ++j) acc[i][j] = fma_(a[i][q], b[j], acc[i][j]);
#endif
      }
    }
#if GFT_DG_WX == GFT_N / GFT_TN
    __syncwarp();    // this warp owns whole rows (all column threads): overwrite them in place
#else
    compute_bar();   // every compute thread is done reading this tile: overwrite it in place
#endif
#pragma unroll
    for (int i = 0; i < GFT_TM; ++i)
#pragma unroll
      for (int j = 0; j < GFT_NG; ++j) {
#if GFT_DG_FFMA2
        *reinterpret_cast<ulonglong2*>(buf + tile_off(ty + i * GFT_TY, tx * GFT_VEC + j * (GFT_N / GFT_NG))) =
            make_ulonglong2(acc2[i][j * 2], acc2[i][j * 2 + 1]);
#else
        vec_t v;
        elem_t* pv = reinterpret_cast<elem_t*>(&v);
#pragma unroll
        for (int e = 0; e < GFT_VEC; ++e) pv[e] = acc[i][j * GFT_VEC + e];
        *reinterpret_cast<vec_t*>(buf + tile_off(ty + i * GFT_TY, tx * GFT_VEC + j * (GFT_N / GFT_NG))) = v;
#endif
      }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
  }
}
