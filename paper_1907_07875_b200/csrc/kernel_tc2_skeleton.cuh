// kernel_tc2_skeleton.cuh — fused fast-GFT kernel with CTA-pair (cta_group::2) tensor-core
// leaves.
//
// Same math as kernel_tc_skeleton.cuh (3xTF32 tcgen05 micro-GEMMs for the big leaves, the
// Haar butterflies and small leaves on CUDA cores), but two CTAs of a cluster on two SMs
// form one M = 256 MMA: each CTA stages its own 128-row tile into its own TMEM lanes, and
// each holds only HALF of every B operand (N/2 output rows) in SMEM — the tensor core of
// the pair reads the other half from the peer.  That halves the per-SM B footprint, which
// frees room for a third tile buffer (deeper TMA prefetch), and the pair issues half as
// many MMA instructions per signal.
//
// Per CTA (192 threads): warps 0-3 compute (thread t = tile row t = TMEM lane t), warp 4 =
// TMA producer/storer for this CTA's rows, warp 5 = MMA issuer (leader CTA only).  Per pair
// tile p (rows 256p .. 256p+255; CTA rank r owns rows 256p + 128r ..):
//   compute: rows -> registers -> butterflies -> per big leaf: hi/lo -> TMEM, then one lane
//            per warp arrives on the leader's `staged` mbarrier (remote arrive for rank 1);
//   issuer : waits for all 8 warps, issues the leaf's cta_group::2 MMAs; after the last leaf
//            one tcgen05.commit multicasts to both CTAs' `mma` mbarrier;
//   compute: small leaves on FMA meanwhile; wait -> tcgen05.ld -> SMEM row.
// Generated prelude: GFT_N, GFT_STAGES, GFT_TMEM_COLS, GFT_B_FLOATS (per CTA), GFT_KNAME,
// gft_tcB[2][GFT_B_FLOATS] and gft_tile().
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
// arrive on the mbarrier at shared::cluster address `cbar` (may live in the peer CTA)
static __device__ __forceinline__ void mbar_arrive_cluster(u32 cbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(cbar) : "memory");
}
static __device__ __forceinline__ u32 map_to_cta(u32 saddr, u32 rank) {
  u32 r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
static __device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
static __device__ __forceinline__ void mbar_wait_acq_cluster(u32 bar, u32 parity) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
static __device__ __forceinline__ u32 cluster_rank() {
  u32 r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ u32 cluster_id_x() {
  u32 r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ u32 nclusters_x() {
  u32 r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
static __device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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
// ---- tcgen05 ----
static __device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
static __device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// commit all prior MMAs of this thread; arrive on the mbarrier at the same offset in both CTAs
static __device__ __forceinline__ void tc_commit_pair(u32 bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               :: "r"(bar), "h"((unsigned short)3) : "memory");
}
// D[tmem, both CTAs] (+)= A[tmem, both CTAs] . B[smem desc, N/2 rows per CTA]^T  (M=256, K=8)
static __device__ __forceinline__ void mma_ts2(u32 d, u32 a, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p; }"
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
// one elected lane per warp signals "my 32 lanes are staged" to the leader CTA
static __device__ __forceinline__ void signal_staged(u32 staged_cluster_addr) {
  tc_wait_st();
  tc_fence_before();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive_cluster(staged_cluster_addr);
}

// @@GFT_GENERATED@@  (codegen.cpp inserts gft_tcB[][] and gft_tile() here)

// GFT_WGS compute warpgroups (1 or 2): with 2, consecutive pair tiles alternate between
// warpgroups 0 and 1, each with its own TMEM columns (GFT_WG_COLS apart) and its own
// mma / staged barriers, so one warpgroup stages and drains a tile while the tensor core
// works on the other's -- the per-tile chain is hidden for small n (registers permitting).
#ifndef GFT_WGS
#define GFT_WGS 1
#define GFT_WG_COLS 0
#endif
#define GFT_THREADS (32 * (4 * GFT_WGS + 2))

extern "C" __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GFT_THREADS, 1)
GFT_KNAME(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
          const float* X, float* Y, long long batch) {
  extern __shared__ unsigned char smem_raw[];
  const u32 raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  unsigned char* stages = smem;
  unsigned char* bsm = smem + GFT_STAGES * GFT_TILE_BYTES;            // this CTA's half of B
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bsm + GFT_B_FLOATS * 4);
  // bars: full[S], done[S], mma[GFT_WGS], staged[GFT_WGS][GFT_NTC] (one per tensor-core leaf,
  // used in the leader only: the issuer starts a leaf's MMAs while the next leaf is staged)
  u32* tmem_slot = reinterpret_cast<u32*>(bars + 2 * GFT_STAGES + GFT_WGS + GFT_WGS * GFT_NTC);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const u32 rank = cluster_rank();
  const long long npairs = (batch + 2 * GFT_TILE_ROWS - 1) / (2 * GFT_TILE_ROWS);
  const long long pid0 = cluster_id_x(), npid = nclusters_x();

  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {   // paired TMEM allocation: same warp id and smem slot in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 :: "r"(smem_u32(tmem_slot)), "n"(GFT_TMEM_COLS) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 128 * GFT_WGS) {
    for (int s = 0; s < GFT_STAGES; ++s) {
      mbar_init(smem_u32(&bars[s]), 1);
      mbar_init(smem_u32(&bars[GFT_STAGES + s]), 4);
    }
    for (int g = 0; g < GFT_WGS; ++g) {
      mbar_init(smem_u32(&bars[2 * GFT_STAGES + g]), 1);
      for (int i = 0; i < GFT_NTC; ++i) mbar_init(smem_u32(&bars[2 * GFT_STAGES + GFT_WGS + g * GFT_NTC + i]), 8);
    }
    fence_mbar_init();
  }
  // this CTA's half of every B operand -> SMEM, K-major 128B-swizzled atoms
  const float4* bsrc = reinterpret_cast<const float4*>(gft_tcB[rank]);
  for (int i = tid; i < GFT_B_FLOATS / 4; i += blockDim.x) {
    const float4 v = bsrc[i];
    const u32 lin = (u32)i * 16u;
    *reinterpret_cast<float4*>(bsm + (lin ^ (((lin >> 7) & 7u) << 4))) = v;
  }
  fence_proxy_async();
  tc_fence_before();
  cluster_sync();   // barriers initialised and B resident in both CTAs before any remote access
  tc_fence_after();
  const u32 tmem = *tmem_slot;

  if (warp == 4 * GFT_WGS) {
    // ---------------- producer / storer of this CTA's 128 rows per pair tile ----------------
    if (lane == 0) {
      long long it = 0;
      for (;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        const int s = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) {
          const long long prow = row0 - GFT_STAGES * npid * 2 * GFT_TILE_ROWS;
          mbar_wait(smem_u32(&bars[GFT_STAGES + s]), (u32)(((it / GFT_STAGES) - 1) & 1));
          const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
          for (int b = 0; b < GFT_NBOX; ++b)
            tma_store_2d(&tout, b * GFT_BOXC, (int)prow, src + b * GFT_BOX_BYTES);
          bulk_commit();
          bulk_wait_read0();
        }
        const u32 bar = smem_u32(&bars[s]);
        const u32 dst = smem_u32(stages + s * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)row0, bar);
      }
      const long long first = it > GFT_STAGES ? it - GFT_STAGES : 0;
      for (long long j = first; j < it; ++j) {
        const int s = (int)(j % GFT_STAGES);
        const long long row0 = (pid0 + j * npid) * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        mbar_wait(smem_u32(&bars[GFT_STAGES + s]), (u32)((j / GFT_STAGES) & 1));
        const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_store_2d(&tout, b * GFT_BOXC, (int)row0, src + b * GFT_BOX_BYTES);
        bulk_commit();
      }
      bulk_wait_all();
    }
  } else if (warp == 4 * GFT_WGS + 1) {
    // ---------------- MMA issuer (leader CTA only); tile it belongs to warpgroup it % WGS ----
    if (rank == 0 && lane == 0) {
      const u32 bsm_s = smem_u32(bsm);
      for (long long it = 0;; ++it) {
        if (pid0 + it * npid >= npairs) break;
        const int g = (int)(it % GFT_WGS);
        gft_issue_pair(tmem + (u32)(g * GFT_WG_COLS), bsm_s, smem_u32(&bars[2 * GFT_STAGES + g]),
                       smem_u32(&bars[2 * GFT_STAGES + GFT_WGS + g * GFT_NTC]), (u32)((it / GFT_WGS) & 1));
      }
    }
  } else {
    // ---------------- compute (row r = TMEM lane r of this warpgroup's columns) ----------------
    const int g = warp >> 2, row = tid & 127;
    const u32 tmem_g = tmem + (u32)(g * GFT_WG_COLS);
    const u32 tm_lane = tmem_g + ((u32)((warp & 3) * 32) << 16);
    const u32 bsm_s = smem_u32(bsm);
    const u32 mbar = smem_u32(&bars[2 * GFT_STAGES + g]);
    // `staged` barriers live in the leader CTA (rank 0)
    const u32 staged0 = map_to_cta(smem_u32(&bars[2 * GFT_STAGES + GFT_WGS + g * GFT_NTC]), 0);
    const u32 staged_local = smem_u32(&bars[2 * GFT_STAGES + GFT_WGS + g * GFT_NTC]);
    for (long long it = g;; it += GFT_WGS) {
      const long long p = pid0 + it * npid;
      if (p >= npairs) break;
      const int s = (int)(it % GFT_STAGES);
      mbar_wait(smem_u32(&bars[s]), (u32)((it / GFT_STAGES) & 1));
      unsigned char* buf = stages + s * GFT_TILE_BYTES;
      float x[GFT_N], y[GFT_N];
      load_row(buf, row, x);
      gft_tile(x, y, tm_lane, tmem_g, bsm_s, mbar, staged0, staged_local, (u32)((it / GFT_WGS) & 1), row, rank);
      store_row(buf, row, y);
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bars[GFT_STAGES + s]));
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();   // the peer may still be reading our B half / arriving on our barriers
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(GFT_TMEM_COLS) : "memory");
  }
}
