/*
 * gft.h — C ABI of the B200-native fast graph Fourier transform library.
 *
 * Method: Lu & Ortega, "Fast Graph Fourier Transforms Based on Graph Symmetry and
 * Bipartition", arXiv 1907.07875 (cited as PAPER.md:<line>, LaTeX labels in brackets).
 *
 * The GFT of a graph signal x on a fixed graph G is y = U^T x, where U holds the
 * eigenvectors of the (unnormalised) Laplacian L = D - W + S ordered by ascending
 * eigenvalue [eq:def_laplacian, PAPER.md:113-127, 136-139].  gft_plan_create() finds
 * graph symmetries (involutions phi, [def:graph_sym] PAPER.md:444-448), factors U into
 * stages of Haar butterflies followed by block-diagonal dense sub-GFTs
 * ([eq:B_phi] PAPER.md:459-469, [thm:decompose] PAPER.md:484-499, recursion PAPER.md:564),
 * solves the small sub-Laplacians once on the host in double precision, and generates
 * sm_100a kernels that apply every butterfly stage and every dense block in one HBM pass
 * per signal tile.  gft_forward()/gft_inverse() run those kernels on a caller stream.
 *
 * Conventions (all functions):
 *   - Node ids are 0-based.  Signals are row-major [batch, n], contiguous, one signal per
 *     row.  Coefficient k of row b is <u_k, x_b> with u_k the k-th eigenvector in
 *     ascending-eigenvalue order (stable by leaf emission order inside ties).
 *   - Simple eigenvalues: u_k has the canonical sign "first entry with |u_i| > 1e-8 is
 *     positive".  Repeated eigenvalues: the basis inside the eigenspace is the plan's own
 *      and is exported by gft_plan_basis().
 *   - Every function returns a gft_status; none aborts or exits.  On failure a
 *     thread-local message is available from gft_last_error().
 *   - Pointers passed in are only read during the call (nothing is retained) unless
 *     stated.  Device pointers are CUDA device addresses on the current device.
 */
#ifndef GFT_H_
#define GFT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GFT_ABI_VERSION 2
#if defined(__GNUC__)
#define GFT_API __attribute__((visibility("default")))
#else
#define GFT_API
#endif
#define GFT_MAX_LEVELS 64

typedef struct gft_plan_s* gft_plan;      /* opaque, library-owned, immutable after create */
typedef void* gft_stream;                  /* a cudaStream_t (NULL = legacy default stream) */

typedef enum { GFT_F32 = 0, GFT_F64 = 1 } gft_dtype;

typedef enum {
  GFT_OK = 0,
  GFT_ERR_INVALID_ARG = 1,     /* bad size, index out of range, self-edge, duplicate pair, NaN/Inf */
  GFT_ERR_NOT_INVOLUTION = 2,  /* phi given but phi(phi(i)) != i or not a permutation */
  GFT_ERR_NOT_SYMMETRIC = 3,   /* phi given but the graph is not phi-symmetric (Definition 2) */
  GFT_ERR_EIG_NOCONVERGE = 4,  /* host Jacobi did not converge / realised basis failed self-check */
  GFT_ERR_ALIGNMENT = 5,       /* X or Y not 16-byte aligned */
  GFT_ERR_UNSUPPORTED = 6,     /* dtype not prepared in this plan, n too large for codegen */
  GFT_ERR_CUDA = 7,            /* CUDA driver/runtime error (detail in gft_last_error) */
  GFT_ERR_NOMEM = 8,
  GFT_ERR_COMPILE = 9,         /* kernel code generation / NVRTC compilation failed */
  GFT_ERR_NO_DEVICE = 10       /* no CUDA device available for a device call */
} gft_status;

/* Plan options.  gft_plan_opts_default() fills the defaults given in brackets. */
typedef struct {
  int32_t max_depth;      /* max butterfly levels; <0 = unlimited [-1] ("until a
                             symmetry property cannot be found anymore") */
  int32_t min_leaf;       /* sub-graphs with <= min_leaf nodes are not searched further [1] */
  int64_t search_budget;  /* backtracking extensions per involution search [1000000] */
  double sym_rtol;        /* relative tolerance of the Definition-2 check of a USER phi [1e-12];
                             sub-graph searches use max(sym_rtol, 1e-10) since Theorem-4
                             weights carry rounding */
  uint32_t dtypes;        /* bitmask (1u<<GFT_F32)|(1u<<GFT_F64) of kernels to generate [both] */
  uint32_t flags;         /* GFT_FLAG_* below [0] */
  int32_t approx_layers;  /* "Haar + approximate GFT": >= 0 replaces every
                             leaf with >= approx_min_leaf nodes by at most this many layers of
                             parallel Givens rotations from the truncated Jacobi algorithm
                             (layer rule = DESIGN.md reading R-4) followed by a
                             sorting permutation.  The plan is then an orthogonal APPROXIMATE
                             GFT: gft_plan_basis() returns U_hat, gft_plan_eigenvalues() the
                             sorted diag(U_hat^T L U_hat), columns keep the rotations' signs.
                             With max_depth = 0 the whole graph is one approximate leaf (the
                             "approximate GFT" of the comparison).  -1 = exact leaves [-1] */
  int32_t approx_min_leaf;/* smallest leaf approximated [2] */
} gft_plan_opts;

#define GFT_FLAG_HOST_ONLY 1u      /* build the factorisation only; no kernel codegen (CPU use) */
#define GFT_FLAG_NO_CUBIN_CACHE 2u /* always run NVRTC even if an AOT cubin for the plan exists */
#define GFT_FLAG_NORMALIZED 8u      /* GFT of the symmetric normalised Laplacian D^-1/2 L D^-1/2
                                       (Theorem 3 holds for it);
                                       every degree d_i = l_ii must be > 0 */
#define GFT_FLAG_DENSE_TC 16u       /* the dense comparison kernels (gft_dense_*) run the whole
                                       basis as one tcgen05 leaf (fp32, n % 4 == 0, n >= 32)
                                       instead of CUDA-core FMA: the strongest dense baseline */
#define GFT_FLAG_NO_TENSOR_CORES 4u /* fp32 leaves >= 32 stay on CUDA-core FMA instead of
                                       tcgen05 micro-GEMMs (ablation / comparison).  Tensor-core
                                       leaves are fp32-accurate: the warp-specialised kernels
                                       split each row (scaled by a power of two) into fp16
                                       hi / lo parts and B into fp16 hi / lo, three kind::f16
                                       passes with fp32 accumulation; the other variants use
                                       3xTF32 */
#define GFT_FLAG_NO_RIGHT_HAAR 32u  /* do not factor right Haar stages (PAPER.md:218-269,
                                       eq:right_gft) out of symmetry-free bipartite leaves
                                       whose Laplacian diagonal is constant; such leaves then
                                       stay one dense block */

typedef struct {
  int32_t n;
  int32_t depth;                          /* number of butterfly levels D */
  int32_t n_units;                        /* total Haar units over all levels */
  int32_t units_per_level[GFT_MAX_LEVELS];
  int32_t n_leaves;                       /* dense sub-GFT blocks */
  int32_t max_leaf;                       /* largest leaf size */
  int32_t n_scale_fix;                    /* explicit sqrt(2)^m multiplies (unequal partner scales) */
  int32_t n_vz_total;                     /* V_Z pass-through nodes summed over all decompositions */
  int64_t sum_k2;                         /* sum over leaves of k^2 (leaf multiplies) */
  int64_t adds;                           /* 2*n_units + sum k(k-1) (adds incl. subtractions)
                                             over exact leaves (+ right Haar / Givens terms) */
  int64_t mults;                          /* sum k^2 + n_scale_fix (sqrt2 folded into leaves)
                                             over exact leaves (+ Givens terms) */
  int64_t paper_mults;                    /* sum k^2 + n_vz_total: tab:runtime convention (A-23) */
  int64_t dense_adds;                     /* n(n-1) */
  int64_t dense_mults;                    /* n^2 */
  int32_t n_clusters;                     /* eigenvalue clusters (tol 1e-9*max(1,lambda_max)) */
  int32_t kernels_ready;                  /* bitmask of dtypes with compiled kernels */
  double residual;                        /* max |L U_f - U_f Lambda| of the realised basis */
  double orth_error;                      /* max |U_f^T U_f - I| */
  int32_t n_right_stages;                 /* right Haar stages (bipartite leaves split E | F) */
  int32_t n_right_pairs;                  /* coefficient butterflies of those stages (2 adds
                                             each, counted in `adds`) */
  int32_t n_approx_leaves;                /* leaves realised as Givens layers (approx_layers) */
  int32_t n_givens;                       /* their rotations.  Counted as executed: 2 FFMA each
                                             (scaled "fast Givens" form) = 2 adds + 2 mults, plus
                                             one multiply per approximate-leaf output; the
                                             paper convention (paper_mults) counts 4 mults */
} gft_plan_info;

/* ---- plan lifecycle -------------------------------------------------------------- */

GFT_API void gft_plan_opts_default(gft_plan_opts* opts);

/* Build a plan for the graph with n nodes, n_edges undirected edges (src[e], dst[e], w[e])
 * and optional self-loops s[n] (NULL = none) [eq:def_laplacian PAPER.md:113-124].
 * An edge may be given as (i,j) or (j,i); i == j is rejected (self-loops go in
 * self_loops); a repeated unordered pair is rejected; w == 0 edges are dropped;
 * non-finite values are rejected; negative weights are accepted.
 * phi (NULL = auto-detect) is an optional top-level involution [Def. 1-2,
 * PAPER.md:440-448]; it must be an involution (else GFT_ERR_NOT_INVOLUTION) and the
 * graph must be phi-symmetric within opts->sym_rtol (else GFT_ERR_NOT_SYMMETRIC).
 * opts NULL = defaults.  On success *out owns host tables, the generated kernels and
 * device tables; release with gft_plan_destroy().  Kernel generation needs no GPU;
 * module loading happens on first device use. */
GFT_API gft_status gft_plan_create(gft_plan* out, int32_t n, int64_t n_edges,
                           const int32_t* src, const int32_t* dst, const double* w,
                           const double* self_loops, const int32_t* phi,
                           const gft_plan_opts* opts);

GFT_API gft_status gft_plan_destroy(gft_plan plan);   /* caller must have synchronised its streams */

/* Plan persistence: the complete factorisation (butterfly units, leaf matrices / Givens
 * layers, right Haar stages, realised basis and eigenvalues, statistics) as a versioned
 * little-endian byte string -- no involution search or eigensolve when it is loaded.
 * gft_plan_serialize: buf == NULL -> *size_out = required bytes, GFT_OK; otherwise cap must
 * be >= that size (else GFT_ERR_INVALID_ARG, *size_out set).
 * gft_plan_deserialize: rebuilds a plan from such bytes (every index and size is validated:
 * GFT_ERR_INVALID_ARG on malformed input, GFT_ERR_UNSUPPORTED on another format version);
 * opts supplies only dtypes and flags for kernel generation (the planning options are part
 * of the serialized plan).  Kernels are regenerated deterministically, so they carry the same
 * names as the original plan's and reuse its AOT / NVRTC cubins.
 * Tuning: kernels that differ from the generator's own choice (measured by gft_plan_tune or
 * set by gft_plan_tuning_set) are recorded in an optional trailer ({dtype, kind, rec5} per
 * kernel, see gft_plan_tuning_get) and
 * re-applied on load, so a tuned plan needs no re-measuring; a malformed trailer is
 * GFT_ERR_INVALID_ARG.  Records for a dtype not prepared on load are ignored. */
GFT_API gft_status gft_plan_serialize(gft_plan plan, void* buf, size_t cap, size_t* size_out);
GFT_API gft_status gft_plan_deserialize(gft_plan* out, const void* buf, size_t size,
                                        const gft_plan_opts* opts);

/* ---- hot path (device memory, asynchronous on `stream`) ----------------------------- */

/* Y[b,:] = U^T X[b,:] for b < batch using the fused fast kernel (butterflies + dense
 * leaves + ascending-eigenvalue output order, one pass).  X, Y: device, row-major
 * [batch, n], 16-byte aligned; X == Y (in place) allowed, other overlap undefined.
 * batch == 0 returns GFT_OK without a launch.  No host synchronisation, no allocation. */
GFT_API gft_status gft_forward(gft_plan plan, const void* X, void* Y, int64_t batch,
                       gft_dtype dtype, gft_stream stream);

/* X[b,:] = U Y[b,:] (exact transpose of gft_forward; B_phi^T = B_phi). */
GFT_API gft_status gft_inverse(gft_plan plan, const void* Y, void* X, int64_t batch,
                       gft_dtype dtype, gft_stream stream);

/* In-run comparison: the plain dense "matrix GFT" Y = X U with the
 * plan's realised basis U_f, same I/O layout and staging as gft_forward. */
GFT_API gft_status gft_dense_forward(gft_plan plan, const void* X, void* Y, int64_t batch,
                             gft_dtype dtype, gft_stream stream);
GFT_API gft_status gft_dense_inverse(gft_plan plan, const void* Y, void* X, int64_t batch,
                             gft_dtype dtype, gft_stream stream);

/* End-to-end variant with HOST buffers: copies X_host -> device, runs the fast transform,
 * copies the result back to Y_host, chunked over S = min(4, workspace_bytes / chunk bytes)
 * workspace slots (chunk c uses slot c mod S) on three library-owned stage streams (all
 * H2D copies, all kernels, all D2H copies; events order each chunk and the reuse of a slot),
 * so H2D, compute and D2H of neighbouring chunks overlap on both copy directions.
 * `workspace` is a device buffer of `workspace_bytes` >= 2 * chunk_rows * n * sizeof(dtype)
 * (chunk_rows > 0; 3-4 slots of 2^18 rows measured best on PCIe Gen5).
 * Concurrent calls from several host threads are serialised while they enqueue.  The caller
 * owns `workspace`; calls that may be in flight together (issued on different streams) need
 * distinct workspaces -- consecutive calls on ONE stream may share it (stream order).  Work is
 * ordered after prior work on `stream` and `stream` is made to wait for completion;
 * host buffers must stay valid until `stream` completes (use pinned memory for overlap).
 * direction: 0 = forward, 1 = inverse. */
GFT_API gft_status gft_execute_host(gft_plan plan, int32_t direction, const void* in_host,
                            void* out_host, int64_t batch, gft_dtype dtype,
                            void* workspace, size_t workspace_bytes, int64_t chunk_rows,
                            gft_stream stream);

/* ---- fused graph spectral filter ("graph spectral filtering",
 *      PAPER.md:32) ------------------------------------------------------------------------
 * y = U diag(h) U^T x in ONE HBM pass per tile: the plan's butterflies, then per leaf the
 * k x k matrix F_l = M_l^T diag(h_l) M_l (M_l = folded leaf matrix), then the butterflies
 * in reverse order — the cost of one transform instead of forward + inverse.
 * h[n]: response per coefficient in the plan's ascending-eigenvalue order (e.g. h = g(lambda)
 * from gft_plan_eigenvalues).  If h is not constant on a repeated eigenvalue the result
 * depends on the plan's basis inside that eigenspace (it is still U_f diag(h) U_f^T).
 * The filter copies what it needs: it stays valid after gft_plan_destroy(plan).
 * dtypes: bitmask as in gft_plan_opts; flags: GFT_FLAG_NO_CUBIN_CACHE / _NO_TENSOR_CORES. */
typedef struct gft_filter_s* gft_filter;
GFT_API gft_status gft_filter_create(gft_filter* out, gft_plan plan, const double* h, uint32_t dtypes,
                                     uint32_t flags);
/* Y = filter(X), device pointers [batch, n], same rules as gft_forward (in place allowed). */
GFT_API gft_status gft_filter_apply(gft_filter f, const void* X, void* Y, int64_t batch,
                                    gft_dtype dtype, gft_stream stream);
GFT_API gft_status gft_filter_kernel_name(gft_filter f, gft_dtype dtype, char* buf, size_t cap);
GFT_API gft_status gft_filter_kernel_source(gft_filter f, gft_dtype dtype, char* buf, size_t cap,
                                            size_t* len);
GFT_API gft_status gft_filter_destroy(gft_filter f);

/* Compile (NVRTC, or load from the AOT cubin cache built by build()) the kernels of `dtype`
 * selected by kinds_mask (bit k = kind k: 0 fast-fwd, 1 fast-inv, 2 dense-fwd, 3 dense-inv;
 * 0 = all) now instead of at first launch, one host thread per kernel.  Needs no GPU. */
GFT_API gft_status gft_plan_compile(gft_plan plan, gft_dtype dtype, uint32_t kinds_mask);

/* Measured tuning of the FMA-skeleton kernels of a plan (DESIGN.md §4 "Request pacing" and
 * "Measured tuning"; the analogue of FFTW_MEASURE — not part of the paper's method, which
 * fixes only the arithmetic).  For every kernel kind in kinds_mask (bits as in
 * gft_plan_compile; 0 = fast-fwd | fast-inv) that runs on the FMA skeleton:
 *   1. with GFT_TUNE_GEOMETRY in flags, the kernel is regenerated for every warp-tile geometry
 *      (rows per thread R in {1,2,4,8}, stages {2,3,4}, warps {1,2,3,4,8,12}; 1-32 KiB tiles that
 *      fit shared memory) and the fastest geometry is kept for step 2;
 *   2. the kernel is regenerated with each per-tile pacing in {0, 150, 300, 450} ns;
 * candidates are compiled in parallel (NVRTC) and timed twice over `reps` back-to-back
 * launches (after 2 untimed ones) on X -> Y with driver events on `stream`; the fastest
 * replaces the plan's kernel if it beats the current one by more than 1%.  For a kernel on
 * the tensor cores the candidates are instead the tcgen05 kernel variants that apply (plain
 * CTA pair, pair with two compute warpgroups, warp-specialised pair, single CTA), same rule;
 * the choice is recorded like a geometry (gft_plan_tuning_get).  FMA-skeleton
 * candidates change no arithmetic, so they compute bit-identical outputs; tcgen05 variants
 * compute the same split products (fp16x2 or 3xTF32; fp32-accurate, not guaranteed
 * bit-identical).
 * With GFT_TUNE_SUSTAINED in flags the current kernel first runs back to back for >= 1 s and
 * every timing pass is 10 x reps launches, so candidates are compared in the state a long
 * stream of transforms sees: on a GPU that reaches its power cap the ranking differs from the
 * burst ranking (1-3 warp, paced geometries lost 7-12% there and won on an uncapped GPU;
 * DESIGN.md §4 "Burst vs sustained").  Tune in the regime the plan will serve.
 * X, Y: caller-owned device buffers of >= batch x n elements of `dtype` (16-byte aligned,
 *   distinct); X is read, Y is overwritten.  batch should exceed L2 (e.g. >= 256 MiB of rows)
 *   for the timing to reflect HBM streaming.  reps <= 0 selects 10.
 * choice_out: NULL or int32_t[16]; for kind k, choice_out[4k..4k+3] = {R, stages, warps,
 *   pace_ns} of the kernel kept (-1s: kind not tuned / tensor-core kernel, whose variant is
 *   visible in gft_plan_kernel_name: tc / tc2 / tc2w / tc3).
 * Synchronous on `stream`.  Not thread-safe with respect to concurrent calls on the same plan
 * (it replaces kernels); gft_plan_serialize records the choice (tuning trailer).
 * Errors: GFT_ERR_INVALID_ARG (NULL / bad sizes / unknown flags), GFT_ERR_ALIGNMENT,
 * GFT_ERR_UNSUPPORTED (dtype not prepared), GFT_ERR_COMPILE, GFT_ERR_NO_DEVICE / GFT_ERR_CUDA. */
#define GFT_TUNE_GEOMETRY 1u
#define GFT_TUNE_SUSTAINED 2u
GFT_API gft_status gft_plan_tune(gft_plan plan, gft_dtype dtype, uint32_t kinds_mask, uint32_t flags,
                                 const void* X, void* Y, int64_t batch, int32_t reps, gft_stream stream,
                                 int32_t* choice_out);
/* Tuning records ("wisdom") of one kernel of a plan: rec5 = {R rows per thread, stages,
 * warps, pace_ns, tc_variant}.  An FMA-skeleton kernel has tc_variant -1; a tcgen05 kernel
 * has -1 in the first four and its variant (0 plain CTA pair, 1 pair with two compute
 * warpgroups, 2 warp-specialised pair, 3 single CTA; -1 for the opt-in IO-split kernel).
 * gft_plan_serialize stores the records of every kernel that differs from the generator's own
 * choice and gft_plan_deserialize re-applies them; set can also apply one by hand.
 * set: regenerates the kernel (compiled at its next launch or gft_plan_compile);
 * GFT_ERR_INVALID_ARG for values outside R in {1,2,4,8}, stages 2..8, warps 1..16,
 * pace 0..100000 (FMA kernels, tc_variant -1), tc_variant outside 0..3 (tcgen05 kernels), or
 * a record the kernel cannot realise (shared memory, variant not applicable).  Needs no GPU.
 * Not thread-safe with respect to concurrent calls on the same plan. */
GFT_API gft_status gft_plan_tuning_get(gft_plan plan, gft_dtype dtype, int32_t kind, int32_t* rec5);
GFT_API gft_status gft_plan_tuning_set(gft_plan plan, gft_dtype dtype, int32_t kind, const int32_t* rec5);

/* The same measured tuning for a filter's kernel (gft_filter_apply): X, Y, batch, reps,
 * flags, stream as above; choice_out: NULL or int32_t[4] = {R, stages, warps, pace_ns}
 * (-1s for a tensor-core filter kernel). */
GFT_API gft_status gft_filter_tune(gft_filter f, gft_dtype dtype, uint32_t flags, const void* X, void* Y,
                                   int64_t batch, int32_t reps, gft_stream stream, int32_t* choice_out);

/* ---- introspection (host) ------------------------------------------------------------ */

GFT_API gft_status gft_plan_info_get(gft_plan plan, gft_plan_info* info);
/* ascending eigenvalues, lambda[n] */
GFT_API gft_status gft_plan_eigenvalues(gft_plan plan, double* lambda);
/* realised basis, row-major U[i*n+k] = u_k(i) (node i, coefficient k) */
GFT_API gft_status gft_plan_basis(gft_plan plan, double* U);
/* leaf sizes in emission order; *count = number of leaves (sizes written up to cap) */
GFT_API gft_status gft_plan_leaf_sizes(gft_plan plan, int32_t* sizes, int32_t cap, int32_t* count);
/* Generated CUDA source for (kind 0 fast-fwd, 1 fast-inv, 2 dense-fwd, 3 dense-inv) and
 * dtype; writes up to cap bytes (NUL-terminated) and the full length to *len. */
GFT_API gft_status gft_plan_kernel_source(gft_plan plan, int32_t kind, gft_dtype dtype,
                                  char* buf, size_t cap, size_t* len);
/* Symbol name of a generated kernel (as shown by ncu / cuobjdump). */
GFT_API gft_status gft_plan_kernel_name(gft_plan plan, int32_t kind, gft_dtype dtype, char* buf, size_t cap);
/* Launch geometry of a kernel kind: grid, block, dynamic smem bytes, registers/thread. */
GFT_API gft_status gft_plan_launch_config(gft_plan plan, int32_t kind, gft_dtype dtype,
                                  int64_t batch, int32_t* grid, int32_t* block,
                                  int32_t* smem_bytes, int32_t* regs);

/* ---- building blocks of the decomposition (host, double) ------------------------------ */

/* Dense Laplacian L[n*n] (row-major) [eq:l_from_sw PAPER.md:122-123], same input rules
 * as gft_plan_create. */
GFT_API gft_status gft_laplacian(int32_t n, int64_t n_edges, const int32_t* src, const int32_t* dst,
                         const double* w, const double* self_loops, double* L);

/* Theorem 4 [thm:decompose PAPER.md:484-499]: given a phi-symmetric graph as a Laplacian
 * L[n*n] and an involution phi, write the Laplacians of G+ (order: V_X ascending, then
 * V_Z ascending; size n-p) into Lplus[(n-p)^2] and of G- (order: phi(V_X); size p) into
 * Lminus[p^2]; *p_out = p_phi [eq:p_phi].  V_X = smaller index of each pair (A-6). */
GFT_API gft_status gft_decompose(int32_t n, const double* L, const int32_t* phi, double sym_rtol,
                         double* Lplus, double* Lminus, int32_t* p_out);

/* Involution search: the involution phi maximising p_phi (ties: the
 * lexicographically smallest phi) such that the graph with Laplacian L is phi-symmetric
 * within rtol; identity if none.  *p_out = p_phi; *complete = 1 if the search finished
 * within budget (else the best found so far is returned). */
GFT_API gft_status gft_find_involution(int32_t n, const double* L, double rtol, int64_t budget,
                               int32_t* phi, int32_t* p_out, int32_t* complete);

/* ---- errors ------------------------------------------------------------------------- */
GFT_API const char* gft_status_str(gft_status s);
GFT_API const char* gft_last_error(void);              /* thread-local detail of the last failure */
GFT_API int32_t gft_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GFT_H_ */
