// kernel_skeleton.cuh — device skeleton of every GFT kernel (sm_100a).
//
// The plan-specific part (butterfly network + dense leaves, or the dense U^T x) is the
// function gft_body() emitted by codegen.cpp in front of this file; everything else
// (HBM <-> SMEM staging, pipelining, tails) is here.  The file is compiled by NVRTC
// (or nvcc for the AOT cubin cache) together with a prelude that defines:
//   GFT_ELEM      float | double
//   GFT_N         signal length n
//   GFT_R         rows (signals) per thread per tile     -> tile = 32*GFT_R rows per warp
//   GFT_WARPS     warps per CTA (each warp is an independent pipeline)
//   GFT_STAGES    SMEM tiles per warp (loads in flight = GFT_STAGES-1)
//   GFT_MODE      0: TMA tensor 2-D copies with hardware swizzle (n*sizeof(elem) % 16 == 0)
//                 1: 1-D bulk copies of whole tiles, unpadded rows (odd n etc.)
//                 2: TMA tensor copies of a packed 2-D view [batch/GFT_PACK, GFT_PACK*n]
//                    (GFT_PACK signals per TMA row) -- rows of 16/32/64 bytes as 128-byte
//                    box rows with 128B swizzle, or (opt-in) rows whose pitch is not 16-byte
//                    aligned as 4-signal super-rows without swizzle; the SMEM tile is the
//                    unpadded row-major tile (swizzled in the first case); a tail of
//                    batch % GFT_PACK signals takes the direct path
//   GFT_BOXC      columns per TMA box (mode 0); n % GFT_BOXC == 0
//   GFT_SWZ_MASK  7 / 3 / 1 / 0 for 128B / 64B / 32B / no swizzle (modes 0 and 2)
//   GFT_PACK      signals per TMA row of the packed view (mode 2)
//   GFT_VEC       elements per SMEM vector access (16, 8 or 4/8 bytes)
//   GFT_KNAME     kernel symbol
//
// Data path per warp-tile of 32*GFT_R signals (one thread = one signal row):
//   TMA / bulk copy HBM -> SMEM (mbarrier complete_tx) -> registers (conflict-free
//   thanks to the swizzle / odd row pitch) -> gft_body() in registers -> SMEM (same
//   slot, in place) -> TMA / bulk store SMEM -> HBM.  Loads for the next GFT_STAGES-1
//   tiles are in flight while a tile is computed.  No __syncthreads anywhere.
typedef unsigned int u32;
typedef unsigned long long u64;
typedef GFT_ELEM elem_t;
#ifndef GFT_OBUF
#define GFT_OBUF 0   // output tiles per warp (IO split); 0 = outputs in place in the input tile
#endif

struct __align__(64) TmaDesc { u64 d[16]; };

#define GFT_TILE_ROWS (32 * GFT_R)
#define GFT_ROW_BYTES (GFT_N * (int)sizeof(elem_t))
#define GFT_TILE_BYTES (GFT_TILE_ROWS * GFT_ROW_BYTES)
#define GFT_BOX_ROWB (GFT_BOXC * (int)sizeof(elem_t))
#define GFT_BOX_BYTES (GFT_TILE_ROWS * GFT_BOX_ROWB)
#define GFT_NBOX (GFT_N / GFT_BOXC)

static __device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
static __device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
}
static __device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
static __device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
  u32 done = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
  } while (!done);
}
static __device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
static __device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N_>
static __device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N_) : "memory");
}
static __device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

#if GFT_MODE != 1
static __device__ __forceinline__ void tma_load_2d(u32 dst, const TmaDesc* desc, int c0, int c1, u32 bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
      :: "r"(dst), "l"((u64)desc), "r"(c0), "r"(c1), "r"(bar) : "memory");
}
static __device__ __forceinline__ void tma_store_2d(const TmaDesc* desc, int c0, int c1, u32 src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
               :: "l"((u64)desc), "r"(c0), "r"(c1), "r"(src) : "memory");
}
#endif
#if GFT_MODE == 1
static __device__ __forceinline__ void bulk_load(u32 dst, const void* src, u32 bytes, u32 bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
static __device__ __forceinline__ void bulk_store(void* dst, u32 src, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(dst), "r"(src), "r"(bytes) : "memory");
}
#endif

// Byte offset of element (row, col) inside a tile buffer.
static __device__ __forceinline__ u32 tile_off(int row, int col) {
#if GFT_MODE == 0
  const u32 lin = (u32)((col / GFT_BOXC) * GFT_BOX_BYTES + row * GFT_BOX_ROWB +
                        (col % GFT_BOXC) * (int)sizeof(elem_t));
  return lin ^ (((lin >> 7) & GFT_SWZ_MASK) << 4);   // TMA swizzle: chunk16 ^= bits[7..]
#elif GFT_MODE == 2
  const u32 lin = (u32)((row * GFT_N + col) * (int)sizeof(elem_t));
  return lin ^ (((lin >> 7) & GFT_SWZ_MASK) << 4);   // packed 128-byte box rows
#else
  return (u32)((row * GFT_N + col) * (int)sizeof(elem_t));
#endif
}

template <int V> struct VecT;
template <> struct VecT<1> { typedef elem_t T; };
#if defined(GFT_ELEM_IS_DOUBLE)
template <> struct VecT<2> { typedef double2 T; };
#else
template <> struct VecT<2> { typedef float2 T; };
template <> struct VecT<4> { typedef float4 T; };
#endif

static __device__ __forceinline__ void load_row(const unsigned char* buf, int row, elem_t (&x)[GFT_N]) {
  typedef typename VecT<GFT_VEC>::T vec_t;
#pragma unroll
  for (int c = 0; c < GFT_N; c += GFT_VEC) {
    vec_t v = *reinterpret_cast<const vec_t*>(buf + tile_off(row, c));
    const elem_t* pv = reinterpret_cast<const elem_t*>(&v);
#pragma unroll
    for (int e = 0; e < GFT_VEC; ++e) x[c + e] = pv[e];
  }
}
static __device__ __forceinline__ void store_row(unsigned char* buf, int row, const elem_t (&y)[GFT_N]) {
  typedef typename VecT<GFT_VEC>::T vec_t;
#pragma unroll
  for (int c = 0; c < GFT_N; c += GFT_VEC) {
    vec_t v;
    elem_t* pv = reinterpret_cast<elem_t*>(&v);
#pragma unroll
    for (int e = 0; e < GFT_VEC; ++e) pv[e] = y[c + e];
    *reinterpret_cast<vec_t*>(buf + tile_off(row, c)) = v;
  }
}

extern "C" __global__ void __launch_bounds__(GFT_WARPS * 32)
GFT_KNAME(const __grid_constant__ TmaDesc tin, const __grid_constant__ TmaDesc tout,
          const elem_t* X, elem_t* Y, long long batch) {  // X may alias Y (in place)
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte alignment for the 128B swizzle atom
  const u32 raw_s = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_s & 1023u)) & 1023u);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // per warp: GFT_STAGES input tiles, then (GFT_OBUF > 0) GFT_OBUF output tiles
  unsigned char* wbuf = smem + (size_t)warp * ((GFT_STAGES + GFT_OBUF) * GFT_TILE_BYTES);
  unsigned char* obase = wbuf + GFT_STAGES * GFT_TILE_BYTES;
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(smem + (size_t)GFT_WARPS * (GFT_STAGES + GFT_OBUF) * GFT_TILE_BYTES) +
      warp * GFT_STAGES;
  (void)obase;
  const long long ntiles = (batch + GFT_TILE_ROWS - 1) / GFT_TILE_ROWS;
  const long long gw = (long long)blockIdx.x * GFT_WARPS + warp;
  const long long nw = (long long)gridDim.x * GFT_WARPS;
  // programmatic dependent launch: everything above overlaps the previous kernel's tail;
  // no global memory is touched before the previous grid has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (gw >= ntiles) return;

  // partial tiles can only be handled by TMA tensor copies (OOB fill / clip); in bulk
  // mode the (single) ragged last tile takes the direct global-memory path
  auto is_direct = [&](long long t) -> bool {
#if GFT_MODE == 1
    return (t + 1) * GFT_TILE_ROWS > batch;
#elif GFT_MODE == 2
    return (batch % GFT_PACK) != 0 && (t + 1) * GFT_TILE_ROWS > batch - batch % GFT_PACK;
#else
    (void)t;
    return false;
#endif
  };
  auto issue_load = [&](long long t, int s) {
    const u32 bar = smem_u32(&bars[s]);
    const u32 dst = smem_u32(wbuf + s * GFT_TILE_BYTES);
    mbar_expect_tx(bar, GFT_TILE_BYTES);
#if GFT_MODE == 0
#pragma unroll
    for (int b = 0; b < GFT_NBOX; ++b)
      tma_load_2d(dst + b * GFT_BOX_BYTES, &tin, b * GFT_BOXC, (int)(t * GFT_TILE_ROWS), bar);
#elif GFT_MODE == 2
    tma_load_2d(dst, &tin, 0, (int)(t * (GFT_TILE_ROWS / GFT_PACK)), bar);
#else
    bulk_load(dst, reinterpret_cast<const unsigned char*>(X) + (size_t)t * GFT_TILE_BYTES,
              GFT_TILE_BYTES, bar);
#endif
  };
  auto issue_store = [&](long long t, const unsigned char* tbuf) {
    const u32 src = smem_u32(tbuf);
#if GFT_MODE == 0
#pragma unroll
    for (int b = 0; b < GFT_NBOX; ++b)
      tma_store_2d(&tout, b * GFT_BOXC, (int)(t * GFT_TILE_ROWS), src + b * GFT_BOX_BYTES);
#elif GFT_MODE == 2
    tma_store_2d(&tout, 0, (int)(t * (GFT_TILE_ROWS / GFT_PACK)), src);
#else
    bulk_store(reinterpret_cast<unsigned char*>(Y) + (size_t)t * GFT_TILE_BYTES, src, GFT_TILE_BYTES);
#endif
    bulk_commit();
  };

  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < GFT_STAGES; ++s) mbar_init(smem_u32(&bars[s]), 1);
    fence_mbar_init();
#pragma unroll 1
    for (int s = 0; s < GFT_STAGES; ++s) {
      const long long t = gw + s * nw;
      if (t < ntiles && !is_direct(t)) issue_load(t, s);
    }
  }
  __syncwarp();

#pragma unroll 1
  for (long long it = 0;; ++it) {
    const long long t = gw + it * nw;
    if (t >= ntiles) break;
    const int s = (int)(it % GFT_STAGES);
    if (!is_direct(t)) {
      mbar_wait(smem_u32(&bars[s]), (u32)((it / GFT_STAGES) & 1));
      unsigned char* buf = wbuf + s * GFT_TILE_BYTES;
#if GFT_OBUF > 0
      // IO split: outputs go to one of GFT_OBUF output tiles; the input tile is refilled with
      // tile it + GFT_STAGES as soon as the last row has been read (not after the compute and
      // the store), so GFT_STAGES - 1 .. GFT_STAGES loads stay in flight while a tile computes
      unsigned char* obuf = obase + (int)(it % GFT_OBUF) * GFT_TILE_BYTES;
      bool obuf_free = false;
#else
      unsigned char* obuf = buf;
#endif
#pragma unroll 1
      for (int r = 0; r < GFT_R; ++r) {
        const int row = lane + 32 * r;
#if defined(GFT_STREAM)
        elem_t x[GFT_N];
        load_row(buf, row, x);
#else
        elem_t x[GFT_N], y[GFT_N];
        load_row(buf, row, x);
#endif
#if GFT_OBUF > 0
        if (r == GFT_R - 1) {
          fence_proxy_async();   // generic-proxy reads of the tile before the async-proxy refill
          __syncwarp();
          if (lane == 0) {
            const long long tn = gw + (it + GFT_STAGES) * nw;
            if (tn < ntiles && !is_direct(tn)) issue_load(tn, s);
          }
        }
        if (!obuf_free) {   // the store that last read this output tile (tile it - GFT_OBUF) is done reading
          if (lane == 0) bulk_wait_read<GFT_OBUF - 1>();
          __syncwarp();
          obuf_free = true;
        }
#endif
#if defined(GFT_STREAM)
        gft_body(x, obuf, row);   // outputs written to the row by the generated code
#else
        gft_body(x, y);
        store_row(obuf, row, y);
#endif
      }
      fence_proxy_async();
      __syncwarp();
#if defined(GFT_PACE_NS)
      // request pacing (tuning.tsv pace=): with few warps per SM and little arithmetic per
      // row, warps finishing together issue their store + refill in bursts; a short sleep
      // spreads them out.  Measured on cfg3 (n = 25, 1 CTA x 4 warps x 3 stages of 96 rows):
      // 5.91 -> 6.31 TB/s for 300-500 ns, a loss on the configs already at the HBM roof
      // (profiles/r01/autotune/pace_*.log)
      __nanosleep(GFT_PACE_NS);
#endif
#if GFT_OBUF > 0
      if (lane == 0) issue_store(t, obuf);
#else
      if (lane == 0) {
        issue_store(t, buf);
        // the buffer consumed in the previous iteration is free once its store has read it
        bulk_wait_read<1>();
        if (it >= 1) {
          const long long tn = gw + (it - 1 + GFT_STAGES) * nw;
          if (tn < ntiles && !is_direct(tn)) issue_load(tn, (int)((it - 1) % GFT_STAGES));
        }
      }
#endif
      __syncwarp();
    } else {
#pragma unroll 1
      for (int r = 0; r < GFT_R; ++r) {
        const long long g = t * GFT_TILE_ROWS + lane + 32 * r;
        if (g < batch) {
#if defined(GFT_STREAM)
          // the tile's SMEM slot is unused by a direct tile: outputs go through this row
          unsigned char* sbuf = wbuf + s * GFT_TILE_BYTES;
          const int row = lane + 32 * r;
          elem_t x[GFT_N];
#pragma unroll
          for (int c = 0; c < GFT_N; ++c) x[c] = X[g * GFT_N + c];
          gft_body(x, sbuf, row);
#pragma unroll
          for (int c = 0; c < GFT_N; ++c) Y[g * GFT_N + c] = *reinterpret_cast<const elem_t*>(sbuf + tile_off(row, c));
#else
          elem_t x[GFT_N], y[GFT_N];
#pragma unroll
          for (int c = 0; c < GFT_N; ++c) x[c] = X[g * GFT_N + c];
          gft_body(x, y);
#pragma unroll
          for (int c = 0; c < GFT_N; ++c) Y[g * GFT_N + c] = y[c];
#endif
        }
      }
#if GFT_OBUF > 0
      // (IO split) this stage's buffer is refilled after a tile is read; a direct tile used it
      // as scratch, so its refill comes after the direct rows
      __syncwarp();
      if (lane == 0) {
        const long long tn = gw + (it + GFT_STAGES) * nw;
        if (tn < ntiles && !is_direct(tn)) issue_load(tn, s);
      }
      __syncwarp();
#endif
    }
  }
  if (lane == 0) bulk_wait_all();
}
