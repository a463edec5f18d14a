// kernel_tc3_skeleton.cuh — warp-specialised CTA-pair tensor-core GFT kernel.
//
// Same math and operand layout as kernel_tc2_skeleton.cuh (cta_group::2, M = 256, 3xTF32,
// A in TMEM, half of every B operand per CTA), but the per-tile chain
//   rows -> butterflies -> hi/lo -> TMEM -> MMA -> tcgen05.ld -> rows
// is split between two warpgroups so that consecutive tiles overlap:
//   WG0 (warps 0-3)  stager : rows -> registers -> front butterflies -> hi/lo -> TMEM A
//                             columns -> arrive on the leader's `staged`; small (CUDA-core)
//                             leaves -> their outputs written back into the SMEM row;
//   WG1 (warps 4-7)  drainer: wait for the tile's MMAs -> tcgen05.ld the D columns (double
//                             buffered in TMEM) -> free them (`d_free` on the leader) ->
//                             back butterflies / coefficient butterflies -> SMEM row;
//   warp 8           TMA producer of this CTA's rows (loads; also the stores with GFT_SPLIT_STORE=0);
//   warp 10          storer (GFT_SPLIT_STORE, the in-place default; IO-split: box-granular storer);
//   warp 9           MMA issuer (leader CTA): staged(t) and d_free(t-2) -> MMAs into
//                             D[t % 2] -> one multicast commit on mma_done[t % 2];
//   warp 11          idle (with warp 10, a full third warpgroup so that setmaxnreg can move registers:
//                             WG2 drops to 56, the stager rises to 248, the drainer to 200).
// The A columns are staged and released per 32-column chunk (GFT_NCH chunks over all
// tensor-core leaves): the issuer waits for chunk c of tile t to be staged (both CTAs), issues
// its MMAs (all three 3xTF32 passes of its k-steps) and commits them to a_free[c]; the stager
// of tile t+1 overwrites chunk c as soon as a_free[c] fires.  So staging tile t+1 runs under
// the MMAs of tile t (one A buffer suffices), and the drain of tile t-1 beside both.
// TMEM: A = all leaves' hi/lo columns, D = all leaves' D columns x 2.
// Generated part: GFT_N, GFT_STAGES, GFT_TMEM_COLS, GFT_B_FLOATS, GFT_KNAME, gft_tcB[2][],
// GFT_A_COLS, GFT_NCH, GFT_D_BASE (D buffer 0 base), GFT_D_COLS (per buffer), GFT_SMALL (1 if
// CUDA-core leaves exist), gft_stage(), gft_drain(), gft_finish(), gft_issue_ws().
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
template <int N_>
static __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N_) : "memory");
}
static __device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Load pacing: consecutive tile loads of a CTA at least GFT_LOAD_PACE_NS apart (codegen sets
// it to 0.9 x this CTA's fair share of HBM time per tile, i.e. a cap ~10% above the roof).
// Without it, at the full SM clock the CTAs issue their refills in synchronised bursts and
// the kernels move 5.5 TB/s instead of 6.3-6.45 (cfg5b IO-split, tools/r02/gpu_tc_probe7.sh);
// under sustained load (capped clock) the cap never binds.
#ifndef GFT_LOAD_PACE_NS
#define GFT_LOAD_PACE_NS 0
#endif
static __device__ __forceinline__ void pace_load(unsigned long long& t_last, long long it) {
  if (GFT_LOAD_PACE_NS > 0) {
    unsigned long long now = globaltimer_ns();
    if (it > 0)
      while (now - t_last < (unsigned long long)GFT_LOAD_PACE_NS) { __nanosleep(64); now = globaltimer_ns(); }
    t_last = now;
  }
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
// kind::f16 (fp16 A in TMEM, fp16 B in SMEM, f32 accumulate), M = 256, K = 16
static __device__ __forceinline__ void mma_ts2_f16(u32 d, u32 a, u64 bdesc, u32 idesc, u32 acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p; }"
               :: "r"(d), "r"(a), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
// fp16x2 split of two scaled inputs (GFT_F16X2): h = the 11 leading significant bits (exactly an
// fp16 for |x| >= 2^-14), l = fp16(x - h); packed low = a, high = b
static __device__ __forceinline__ void split_f16x2(float a, float b, u32& h, u32& l) {
  const float ha = __uint_as_float(__float_as_uint(a) & 0xffffe000u);
  const float hb = __uint_as_float(__float_as_uint(b) & 0xffffe000u);
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(hb), "f"(ha));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(l) : "f"(b - hb), "f"(a - ha));
}
// 2^k for k in [-149, 127]
static __device__ __forceinline__ float exp2_int(int k) {
  return k >= -126 ? __uint_as_float((u32)(k + 127) << 23) : __uint_as_float(1u << (k + 149));
}
// floor(log2 m) clamped to [-126, 127] (0 for m = 0): the row scale 2^-e brings the row's largest
// tensor-core input into [1, 2) (rows whose largest element is an fp32 subnormal keep 2^126)
static __device__ __forceinline__ int row_exponent(float m) {
  const int eb = (int)((__float_as_uint(m) >> 23) & 0xffu);
  return eb == 0 ? (m == 0.f ? 0 : -126) : (eb == 255 ? 127 : eb - 127);
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


// Phase trace (experiments only: GFT_TC_TRACE=1 adds `#define GFT_TRACE 1`): clock64 stamps of
// each role per tile for CTAs 0..7, printed by CTA 0 and 1 at exit.  Events: 0 load issued,
// 1 stager: tile landed, 2 rows in registers, 3 staged; 4 issuer: waits done, 5 committed;
// 6 drainer: MMAs done, 7 rows written; 8 storer: output ready, 9 store has read the buffer;
// 10-13 issuer: chunk 0..3 staged; 14-17 stager: chunk 0..3 free (A columns).
#ifdef GFT_TRACE
#define GFT_TR_EV 18
#define GFT_TR_TILES 48
__device__ unsigned long long gft_trace_buf[8][GFT_TR_TILES][GFT_TR_EV];
#define TR(ev, itv) do { if (blockIdx.x < 8 && (itv) < GFT_TR_TILES) gft_trace_buf[blockIdx.x][(itv)][(ev)] = clock64(); } while (0)
#else
#define TR(ev, itv) do { } while (0)
#endif

// @@GFT_GENERATED@@  (codegen.cpp inserts gft_tcB[][], gft_stage(), gft_drain(), gft_issue_ws())

// register split of the 12 warps (65536 = 32 x 4 x (248 + 200 + 56)): the stager holds a row
// plus hi/lo chunks, the drainer a row plus one D chunk, producer / issuer almost nothing
static __device__ __forceinline__ void reg_stager() { asm volatile("setmaxnreg.inc.sync.aligned.u32 248;" ::: "memory"); }
static __device__ __forceinline__ void reg_drainer() { asm volatile("setmaxnreg.inc.sync.aligned.u32 200;" ::: "memory"); }
static __device__ __forceinline__ void reg_control() { asm volatile("setmaxnreg.dec.sync.aligned.u32 56;" ::: "memory"); }

extern "C" __global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
GFT_KNAME(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
          const float* X, float* Y, long long batch) {
  extern __shared__ unsigned char smem_raw[];
  const u32 raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
#ifndef GFT_IO_SPLIT
#define GFT_IO_SPLIT 0
#endif
  // GFT_IO_SPLIT: input ring of GFT_STAGES buffers released by the stager as soon as its rows
  // are in registers, plus ONE output buffer the drainer fills box by box and a storer warp
  // drains box by box
  unsigned char* stages = smem;
  unsigned char* outbuf = smem + GFT_STAGES * GFT_TILE_BYTES;
  unsigned char* bsm = smem + (GFT_STAGES + GFT_IO_SPLIT) * GFT_TILE_BYTES;   // this CTA's half of B
#ifndef GFT_F16X2
#define GFT_F16X2 0
#endif
  // GFT_F16X2: per-row exponents of the two tiles in flight between stager and drainer
  int* row_e = reinterpret_cast<int*>(bsm + GFT_B_FLOATS * 4);
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(bsm + GFT_B_FLOATS * 4 + (GFT_F16X2 ? 1024 : 0));
  (void)row_e;
  // bars: full[S], done[S] (= input free when IO-split), rows[S], then the ones below
  // (staged alternates per tile parity, so a stager a tile ahead can never complete a phase
  // the issuer has not yet observed)
  unsigned long long* b_full = bars;
  unsigned long long* b_done = bars + GFT_STAGES;
  unsigned long long* b_rows = bars + 2 * GFT_STAGES;
  unsigned long long* b_mma = bars + 3 * GFT_STAGES;           // [2]: tile's MMAs done (D[t%2] full)
  unsigned long long* b_dfree = bars + 3 * GFT_STAGES + 2;     // [2]: D[t%2] drained
  // IO-split output ring at TMA-box granularity: box b of the output buffer is written by the
  // drainer (box_ready[b], 4 warps) and released once its store has read it (box_free[b])
  unsigned long long* b_boxrdy = bars + 3 * GFT_STAGES + 4;
  unsigned long long* b_boxfree = bars + 3 * GFT_STAGES + 4 + GFT_NBOX;
  // per A chunk: staged[t%2][c] (leader; 8 stager warps of the pair), a_free[c] (MMAs of the
  // chunk done, multicast commit)
  unsigned long long* b_staged = bars + 3 * GFT_STAGES + 4 + 2 * GFT_NBOX;
#ifndef GFT_A_BUFS
#define GFT_A_BUFS 1
#endif
  // GFT_A_BUFS == 2: tile t stages into A buffer t % 2 (GFT_A_COLS columns each), so staging
  // tile t+1 never waits for the MMAs of tile t -- only for those of tile t-1 on the same buffer
  unsigned long long* b_afree = b_staged + 2 * GFT_NCH;   // [GFT_A_BUFS][GFT_NCH]
  unsigned long long* b_erdy = b_afree + GFT_A_BUFS * GFT_NCH;    // [2] row exponents of tile t%2 written (4 stager warps)
  unsigned long long* b_efree = b_erdy + 2;          // [2] ... read (4 drainer warps)
  unsigned long long* b_sfree = b_efree + 2;         // [S] (GFT_SPLIT_STORE) in-place buffer's store has read it
  u32* tmem_slot = reinterpret_cast<u32*>(b_sfree + GFT_STAGES);
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
  if (tid == 256) {
    for (int s = 0; s < GFT_STAGES; ++s) {
      mbar_init(smem_u32(&b_full[s]), 1);
      mbar_init(smem_u32(&b_done[s]), 4);
      mbar_init(smem_u32(&b_rows[s]), 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&b_mma[b]), 1);
      mbar_init(smem_u32(&b_dfree[b]), 8);
    }
    for (int c = 0; c < 2 * GFT_NCH; ++c) mbar_init(smem_u32(&b_staged[c]), 8);
    for (int c = 0; c < GFT_A_BUFS * GFT_NCH; ++c) mbar_init(smem_u32(&b_afree[c]), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&b_erdy[b]), 4);
      mbar_init(smem_u32(&b_efree[b]), 4);
    }
    for (int b = 0; b < GFT_NBOX; ++b) {
      mbar_init(smem_u32(&b_boxrdy[b]), 4);
      mbar_init(smem_u32(&b_boxfree[b]), 1);
    }
    for (int s = 0; s < GFT_STAGES; ++s) mbar_init(smem_u32(&b_sfree[s]), 1);
    fence_mbar_init();
  }
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

  if (warp >= 8) {
    reg_control();
#if GFT_IO_SPLIT
    if (warp == 8 && lane == 0) {
      // ---------------- loader: input ring, refilled as soon as the stager has read a tile ----
      unsigned long long t_last = 0;
      for (long long it = 0;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        const int s = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) mbar_wait(smem_u32(&b_done[s]), (u32)(((it / GFT_STAGES) - 1) & 1));
        pace_load(t_last, it);
        TR(0, it);
        const u32 bar = smem_u32(&b_full[s]);
        const u32 dst = smem_u32(stages + s * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)row0, bar);
      }
    } else if (warp == 10 && lane == 0) {
      // ---------------- storer: output boxes -> HBM as soon as each is written; a box slot is
      // handed back to the drainer once the store that read it has finished reading (the
      // store of the NEXT box is already in flight then: one store group outstanding)
      int prev = -1;
      for (long long it = 0;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        for (int b = 0; b < GFT_NBOX; ++b) {
          mbar_wait(smem_u32(&b_boxrdy[b]), (u32)(it & 1));
          if (b == 0) TR(8, it);
          tma_store_2d(&tout, b * GFT_BOXC, (int)row0, smem_u32(outbuf) + b * GFT_BOX_BYTES);
          bulk_commit();
          if (prev >= 0) {
            bulk_wait_read<1>();
            mbar_arrive(smem_u32(&b_boxfree[prev]));
          }
          prev = b;
        }
        TR(9, it);
      }
      bulk_wait_all();
    } else
#endif
#ifndef GFT_SPLIT_STORE
#define GFT_SPLIT_STORE 0
#endif
#if GFT_SPLIT_STORE && !GFT_IO_SPLIT
    if (warp == 10 && lane == 0) {
      // ---------------- storer of the in-place buffers (default): stores a tile as soon as it
      // is drained and hands the buffer to the loader once the store has read it, so a store
      // never waits behind the loader's pacing
      for (long long it = 0;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        const int s = (int)(it % GFT_STAGES);
        mbar_wait(smem_u32(&b_done[s]), (u32)((it / GFT_STAGES) & 1));
        const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_store_2d(&tout, b * GFT_BOXC, (int)row0, src + b * GFT_BOX_BYTES);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(smem_u32(&b_sfree[s]));
      }
      bulk_wait_all();
    } else if (warp == 8 && lane == 0) {
      // ---------------- loader of the in-place buffers ----------------
      unsigned long long t_last = 0;
      for (long long it = 0;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        const int s = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) mbar_wait(smem_u32(&b_sfree[s]), (u32)(((it / GFT_STAGES) - 1) & 1));
        pace_load(t_last, it);
        TR(0, it);
        const u32 bar = smem_u32(&b_full[s]);
        const u32 dst = smem_u32(stages + s * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)row0, bar);
      }
    } else
#endif
    if (warp == 8 && lane == 0) {
      // ---------------- producer / storer of this CTA's 128 rows per pair tile ----------------
      unsigned long long t_last = 0;
      long long it = 0;
      for (;; ++it) {
        const long long p = pid0 + it * npid;
        if (p >= npairs) break;
        const long long row0 = p * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        const int s = (int)(it % GFT_STAGES);
        if (it >= GFT_STAGES) {
          const long long prow = row0 - GFT_STAGES * npid * 2 * GFT_TILE_ROWS;
          mbar_wait(smem_u32(&b_done[s]), (u32)(((it / GFT_STAGES) - 1) & 1));
          const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
          for (int b = 0; b < GFT_NBOX; ++b)
            tma_store_2d(&tout, b * GFT_BOXC, (int)prow, src + b * GFT_BOX_BYTES);
          bulk_commit();
          bulk_wait_read0();
        }
        pace_load(t_last, it);
        const u32 bar = smem_u32(&b_full[s]);
        const u32 dst = smem_u32(stages + s * GFT_TILE_BYTES);
        mbar_expect_tx(bar, GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)row0, bar);
      }
      const long long first = it > GFT_STAGES ? it - GFT_STAGES : 0;
      for (long long j = first; j < it; ++j) {
        const int s = (int)(j % GFT_STAGES);
        const long long row0 = (pid0 + j * npid) * 2 * GFT_TILE_ROWS + rank * GFT_TILE_ROWS;
        mbar_wait(smem_u32(&b_done[s]), (u32)((j / GFT_STAGES) & 1));
        const u32 src = smem_u32(stages + s * GFT_TILE_BYTES);
        for (int b = 0; b < GFT_NBOX; ++b)
          tma_store_2d(&tout, b * GFT_BOXC, (int)row0, src + b * GFT_BOX_BYTES);
        bulk_commit();
      }
      bulk_wait_all();
    } else if (warp == 9 && rank == 0 && lane == 0) {
      // ---------------- MMA issuer (leader CTA) ----------------
      const u32 bsm_s = smem_u32(bsm);
      for (long long it = 0;; ++it) {
        if (pid0 + it * npid >= npairs) break;
        const int b = (int)(it & 1);
        if (it >= 2) mbar_wait_acq_cluster(smem_u32(&b_dfree[b]), (u32)(((it >> 1) - 1) & 1));
        TR(4, it);
        // re-materialise the B base each tile so the ~100 MMA descriptors are not hoisted
        // out of the loop into registers (this warpgroup runs with 56 registers)
        u32 bs;
        asm volatile("mov.b32 %0, %1;" : "=r"(bs) : "r"(bsm_s));
        const int ab = GFT_A_BUFS == 2 ? b : 0;
        gft_issue_ws(tmem + (u32)(ab * GFT_A_COLS), tmem + (u32)(GFT_D_BASE + b * GFT_D_COLS), bs,
                     smem_u32(&b_staged[b * GFT_NCH]), (u32)((it >> 1) & 1), smem_u32(&b_afree[ab * GFT_NCH]), it);
        tc_commit_pair(smem_u32(&b_mma[b]));
        TR(5, it);
      }
    }
  } else if (warp < 4) {
    // ---------------- stager (row = TMEM lane = tid) ----------------
    reg_stager();
    const u32 tm_a = tmem + ((u32)(warp * 32) << 16);
    const u32 staged0[2] = {map_to_cta(smem_u32(&b_staged[0]), 0), map_to_cta(smem_u32(&b_staged[GFT_NCH]), 0)};
    for (long long it = 0;; ++it) {
      const long long p = pid0 + it * npid;
      if (p >= npairs) break;
      const int s = (int)(it % GFT_STAGES);
      mbar_wait(smem_u32(&b_full[s]), (u32)((it / GFT_STAGES) & 1));
      if (tid == 0) TR(1, it);
      unsigned char* buf = stages + s * GFT_TILE_BYTES;
      float x[GFT_N];
      load_row(buf, tid, x);
      if (tid == 0) TR(2, it);
#if GFT_IO_SPLIT
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_done[s]));   // input rows consumed: refill
#endif
      // before writing the A columns: the MMAs that last read this A buffer (tile t-1, or
      // t-2 with two buffers) are done
      // chunk c of A is rewritten once the MMAs of tile it-1 on it are done (a_free[c])
#if GFT_F16X2
      if (it >= 2) mbar_wait(smem_u32(&b_efree[it & 1]), (u32)(((it >> 1) - 1) & 1));   // drainer of it-2 read them
#if GFT_A_BUFS == 2
      // A buffer it % 2 was last read by the MMAs of tile it - 2
      gft_stage(x, tm_a + (u32)((it & 1) * GFT_A_COLS), staged0[it & 1], buf, tid,
                smem_u32(&b_afree[(it & 1) * GFT_NCH]), (u32)(((it >> 1) - 1) & 1), it >= 2, it,
                &row_e[(it & 1) * 128 + tid]);
#else
      gft_stage(x, tm_a, staged0[it & 1], buf, tid, smem_u32(b_afree), (u32)((it - 1) & 1), it >= 1, it,
                &row_e[(it & 1) * 128 + tid]);
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_erdy[it & 1]));
#else
      gft_stage(x, tm_a, staged0[it & 1], buf, tid, smem_u32(b_afree), (u32)((it - 1) & 1), it >= 1, it);
#endif
      if (tid == 0) TR(3, it);
#if GFT_SMALL
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_rows[s]));   // release: small-leaf outputs in SMEM
#endif
    }
  } else {
    // ---------------- drainer (row = TMEM lane = tid - 128) ----------------
    reg_drainer();
    const int row = tid - 128;
    const u32 lane_off = (u32)((warp - 4) * 32) << 16;
    for (long long it = 0;; ++it) {
      const long long p = pid0 + it * npid;
      if (p >= npairs) break;
      const int s = (int)(it % GFT_STAGES);
      const int b = (int)(it & 1);
      mbar_wait(smem_u32(&b_mma[b]), (u32)((it >> 1) & 1));
      tc_fence_after();
      if (row == 0) TR(6, it);
#if GFT_SMALL
      mbar_wait(smem_u32(&b_rows[s]), (u32)((it / GFT_STAGES) & 1));
#endif
#if GFT_IO_SPLIT
      unsigned char* buf = outbuf;
#else
      unsigned char* buf = stages + s * GFT_TILE_BYTES;
#endif
      float y[GFT_N];
#if GFT_F16X2
      mbar_wait(smem_u32(&b_erdy[b]), (u32)((it >> 1) & 1));
      const int e_row = row_e[b * 128 + row];
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_efree[b]));
      gft_drain(y, tmem + lane_off + (u32)(GFT_D_BASE + b * GFT_D_COLS), buf, row, e_row);
#else
      gft_drain(y, tmem + lane_off + (u32)(GFT_D_BASE + b * GFT_D_COLS), buf, row);
#endif
      // D[b] read (tcgen05.ld waited inside gft_drain): let the issuer reuse it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(map_to_cta(smem_u32(&b_dfree[b]), 0));
      gft_finish(y);
#if GFT_IO_SPLIT
#pragma unroll
      for (int b = 0; b < GFT_NBOX; ++b) {
        if (it >= 1) mbar_wait(smem_u32(&b_boxfree[b]), (u32)((it - 1) & 1));   // its last store has read it
#pragma unroll
        for (int c = 32 * b; c < 32 * b + 32 && c < GFT_N; c += 4)
          *reinterpret_cast<float4*>(buf + tile_off(row, c)) = make_float4(y[c], y[c + 1], y[c + 2], y[c + 3]);
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&b_boxrdy[b]));
      }
      if (row == 0) TR(7, it);
#else
      store_row(buf, row, y);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&b_done[s]));
#endif
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef GFT_TRACE
  if (blockIdx.x < 2 && tid == 0) {
    const long long nt = (npairs - pid0 + npid - 1) / npid;
    for (int i = 0; i < GFT_TR_TILES && i < nt; ++i) {
      const unsigned long long* e = gft_trace_buf[blockIdx.x][i];
      const unsigned long long b0 = gft_trace_buf[blockIdx.x][0][0];
      printf("TRACE cta %d tile %d: %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld %lld\n",
             (int)blockIdx.x, i,
             (long long)(e[0] - b0), (long long)(e[1] - b0), (long long)(e[2] - b0), (long long)(e[3] - b0),
             (long long)(e[4] - b0), (long long)(e[5] - b0), (long long)(e[6] - b0), (long long)(e[7] - b0),
             (long long)(e[8] - b0), (long long)(e[9] - b0), (long long)(e[10] - b0), (long long)(e[11] - b0),
             (long long)(e[12] - b0), (long long)(e[13] - b0), (long long)(e[14] - b0), (long long)(e[15] - b0),
             (long long)(e[16] - b0), (long long)(e[17] - b0));
    }
  }
#endif
  cluster_sync();   // the peer may still be reading our B half / arriving on our barriers
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" :: "r"(tmem), "n"(GFT_TMEM_COLS) : "memory");
  }
}
