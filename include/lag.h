/*
 * lag.h — C ABI of liblag, the B200-native in situ Lagrangian flow-map
 * extraction hot path of arXiv 2004.02003 (Sane, Childs, Bujack:
 * "Scalable in situ Lagrangian flow map extraction: demonstrating the
 * viability of a communication-free model").
 *
 * Citations: P:nnn = the paper text line nnn.
 *
 * What the library computes, per rank block (one context per block):
 *   - lag_seed:  uniform seeding of basis-flow particles on the grid nodes
 *                (§2.3: "particles are seeded along a uniform grid";
 *                data reduction 1:X, X = stride^dim).
 *   - lag_advect_cycle: one RK4 step of every active particle per simulation
 *                cycle (§3.1, §2.2) through the velocity field,
 *                multilinear in space on the uniform grid and linear in time
 *                between the cycle's two slices v_t and v_{t+1}; particles
 *                leaving the block are terminated in place (BTO, P:190-196
 *                §3.1) or handed to the owning rank (COMM, the paper's
 *                Lagrangian-MPI baseline after Agranovsky et al., P:153,
 *                P:206-208).  Particle management (validity tracking and
 *                compaction so invalid particles are not launched) is
 *                fused into the same kernel.
 *   - lag_extract: at the end of an interval ("write cycle")
 *                returns the basis flows (start, end, validity) in the block's
 *                seed order, after returning particles to their origin rank in
 *                COMM mode, and reseeds for the next interval.
 *
 * Conventions
 *   - Every call returns lag_status: 0 = LAG_OK, negative = error.  No C++
 *     exception or abort crosses the ABI.  lag_last_error() gives a message.
 *   - Grid: nodes n in [0, N_a), position x(n) = origin + n * spacing.
 *     Domain Omega = prod_a [origin_a, origin_a + (N_a - 1) spacing_a], closed.
 *   - Block: owned nodes [block_lo, block_hi) per axis, half-open; a block
 *     whose block_hi == N owns the closed upper face.  Rank = x-fastest block
 *     index in `layout`.
 *   - Velocity slice arrays (borrowed, read-only in BTO mode): fp32, AoS
 *     (vx, vy[, vz]) per node, x fastest; rows dense or padded to
 *     lag_config.row_pitch_bytes (a padded pitch that is a multiple of 16 B
 *     makes the rows legal TMA strides).  Extent per axis =
 *     (min(block_hi + 1, N) - block_lo) + 2 * ghost nodes: the owned nodes,
 *     the neighbour's first (shared) node plane when block_hi < N, and `ghost`
 *     layers on every side (allocated even at global faces, never read there).
 *     Element (0,0,0) is global node block_lo - ghost.
 *   - Pointers passed to lag_advect_cycle / lag_extract may be device pointers
 *     (used in place, stream-ordered on cfg.stream) or host pointers (the
 *     library stages them through three device buffers with cudaMemcpyAsync on
 *     its own copy stream, so the next cycle's copy overlaps this cycle's
 *     kernels; pinned host memory makes the copy asynchronous; this is the
 *     end-to-end path).  The previous call's host v_t1 passed again as v_t is
 *     not copied twice, so it must not change between those two calls.
 *   - Not thread-safe per context.  Several contexts may share a device.
 */
#ifndef LAG_H
#define LAG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAG_ABI_VERSION 3   /* 3: lag_extract interval_index, row_pitch_bytes,
                               LAG_XCHG_LOCAL + lag_local_group */

#if defined(__GNUC__)
#define LAG_API __attribute__((visibility("default")))
#else
#define LAG_API
#endif

typedef struct lag_ctx_s* lag_ctx;

typedef enum {
    LAG_OK = 0,
    LAG_EINVAL = -1,      /* bad argument / configuration                      */
    LAG_ESTATE = -2,      /* call out of order (advect before seed, ...)       */
    LAG_EEMPTY = -3,      /* the block holds no seed at this stride            */
    LAG_ENOMEM = -4,      /* device allocation failed                          */
    LAG_ECUDA = -5,       /* CUDA runtime error                                */
    LAG_ENCCL = -6,       /* NCCL error (COMM mode)                            */
    LAG_EOVERFLOW = -7,   /* latched: an exchange slot or the particle list overflowed */
    LAG_EGHOST = -8,      /* latched: a stage sample fell outside the ghost layers (CFL >= 1) */
    LAG_ENONFINITE = -9   /* latched: non-finite velocity reached a particle   */
} lag_status;

typedef enum { LAG_BTO = 0, LAG_COMM = 1 } lag_mode;
typedef enum {
    LAG_XCHG_NCCL = 0,          /* grouped NCCL send/recv before the advect kernel            */
    LAG_XCHG_PEER = 1,          /* the kernels pull ghosts and hand-offs from the neighbours' memory (CUDA IPC) */
    LAG_XCHG_PEER_OVERLAP = 2,  /* LAG_XCHG_PEER fused with the advection: the first CTAs of
                                   the advect kernel run the exchange while the others
                                   advect the tiles whose stage samples cannot reach a ghost
                                   node; the rest (and the particles received this cycle)
                                   advect in a second pass.  Bitwise equal to the others.  */
    LAG_XCHG_LOCAL = 3          /* several blocks on ONE device, driven by one host thread
                                   (lag_local_group): ghost layers are copied straight from
                                   the neighbours' slice arrays and hand-offs are appended
                                   from the neighbours' slots, ordered by stream events
                                   (no NCCL, no flags, no spinning).  Bitwise equal to the
                                   other transports.                                          */
} lag_exchange;

/* Per-basis-flow status returned by lag_extract. */
typedef enum {
    LAG_VALID = 0,          /* stayed in the block (BTO) / domain (COMM) for the whole interval */
    LAG_TERM_BOUNDARY = 1,  /* BTO: a stage sample or the update left the block; end = pre-step position */
    LAG_EXIT_DOMAIN = 2     /* a stage sample or the update left the global domain; end = pre-step position */
} lag_flow_status;

/* lag_extract flags */
#define LAG_NO_RESEED 1u    /* do not reseed after extracting */
#define LAG_ASYNC     2u    /* do not synchronise: outputs must be device pointers of the
                               ctx's device, page-locked host memory, or NULL; complete
                               when ctx->stream passes this call's work; latched errors
                               are reported by the next synchronous lag_extract (or seen
                               in lag_stats) */

typedef struct {
    int32_t dim;                 /* 2 or 3                                                */
    int32_t mode;                /* lag_mode                                              */
    int64_t global_nodes[3];     /* N_a >= 2 on used axes; unused axis = 1                */
    double  origin[3];           /* o_a, finite                                           */
    double  spacing[3];          /* h_a > 0, finite                                       */
    int64_t block_lo[3];         /* owned node range [lo, hi), 0 <= lo < hi <= N          */
    int64_t block_hi[3];
    int32_t ghost;               /* G ghost node layers per side in the slice arrays;
                                    COMM with nranks > 1 requires G >= 1; BTO (and a
                                    single-block COMM run) reads none                     */
    int32_t device;              /* CUDA device ordinal                                   */
    int32_t rank;                /* COMM: this block's rank (x-fastest in layout)         */
    int32_t nranks;              /* COMM: number of ranks = prod(layout)                  */
    int32_t layout[3];           /* COMM: blocks per axis                                 */
    int32_t exchange;            /* COMM transport: lag_exchange                          */
    int64_t row_pitch_bytes;     /* bytes between consecutive x-rows of the slice arrays;
                                    0 = dense (dim * 4 * extent_x); else a multiple of
                                    dim * 4 and >= dim * 4 * extent_x (padding nodes are
                                    never read).  Plane pitch = row pitch * extent_y.    */
    const void* nccl_id;         /* COMM: 128-byte ncclUniqueId shared by all ranks (from
                                    lag_nccl_unique_id on one rank); NULL for BTO         */
    void*   stream;              /* cudaStream_t the library enqueues on (borrowed);
                                    NULL = the legacy default stream                     */
} lag_config;

typedef struct {
    int64_t seeded;          /* seeds placed at the last lag_seed                           */
    int64_t active;          /* particles currently advancing on this rank                  */
    int64_t term_boundary;   /* this interval: BTO terminations at the block boundary       */
    int64_t exit_domain;     /* this interval: global-domain exits                          */
    int64_t sent;            /* this interval: particles handed to other ranks (COMM)       */
    int64_t received;        /* this interval: particles received from other ranks (COMM)   */
    int64_t particle_steps;  /* cumulative RK4 particle-steps since lag_init                */
    int64_t cycles;          /* cumulative lag_advect_cycle calls since lag_init            */
    int32_t device_error;    /* latched async condition as a lag_status (0 = none)          */
    int32_t pad_;
    double  phase_ms[3];     /* with env LAG_PHASE_TIMING=1: cumulative device time of the
                                pre-advect exchange, the advect kernel, the post-advect step  */
} lag_stats_t;

/*
 * lag_init — one context per rank block.  The decomposition is the
 * simulation's (§2.2: the Lagrangian analysis runs on the data each
 * rank already holds), so the caller states the block; the library validates
 * the configuration, allocates every device buffer the context needs
 * (particle list, exchange slots, staging) and, in COMM mode over NCCL or
 * peer memory, joins the communicator.  Collective in COMM mode (all ranks
 * must call; LAG_XCHG_LOCAL contexts are connected by lag_local_group).
 * Errors: LAG_EINVAL (dims, spacing, bounds, layout, ghost, packed seed-node
 * width > 32 bits), LAG_ECUDA, LAG_ENCCL, LAG_ENOMEM.  *out is NULL on error.
 */
LAG_API lag_status lag_init(const lag_config* cfg, lag_ctx* out);

/*
 * lag_seed — start a new interval: place one particle on every global lattice
 * node g with g_a = 0 (mod stride) and block_lo_a <= g_a < block_hi_a (x-fastest
 * seed order), discarding any previous particles (reading R4 in
 * DESIGN.md).  *n_seeds_out = number of seeds.  COMM: every rank of the
 * decomposition reseeds at the same cycle (a reseed in the middle of an
 * interval drops the hand-offs in flight on every rank alike).
 * Errors: LAG_EINVAL (stride < 1), LAG_EEMPTY (no lattice node in the block),
 * LAG_ESTATE (a LAG_XCHG_LOCAL context not yet in a lag_local_group).
 */
LAG_API lag_status lag_seed(lag_ctx ctx, int32_t stride, int64_t* n_seeds_out);

/*
 * lag_advect_cycle — advance every active particle by one RK4 step of size dt
 * (physical time units) through v(x, t) = (1 - a) Tri(v_t, x) + a Tri(v_t1, x),
 * a = 0, 1/2, 1/2, 1 for the four stages.
 * BTO: no communication, no host synchronisation; particles with any stage
 * sample or updated position outside the block terminate at their pre-step
 * position (status LAG_TERM_BOUNDARY).  COMM (collective): fills the ghost
 * layers of v_t1 (and of v_t unless it is the previous call's v_t1) from the
 * neighbours, advances, and hands particles whose updated position lies in
 * another block to its owner.  In COMM mode the ghost layers of the slice
 * arrays are written; interior nodes never are.
 * v_t, v_t1: slice arrays (see Conventions), device or host memory.  Passing
 * the same array twice is the frozen-snapshot regime (one accessible time
 * step per cycle): identical results, corners gathered once.
 * LAG_XCHG_LOCAL: collective over the group in the same sense: each block's
 * call records its (device) slices; the call that completes the group's cycle
 * enqueues the whole cycle of every block (one exchange launch for the ghost
 * copies and appends on block 0's stream, then each block's advection on its
 * own stream, joined by events).  The slices must stay unmodified until then.
 * Errors: LAG_ESTATE (no lag_seed; LOCAL: a block called twice in one group
 * cycle, or before every block extracted), LAG_EINVAL (dt <= 0 or
 * non-finite, NULL slice; LOCAL: host slice), LAG_ECUDA, LAG_ENCCL (an NCCL
 * call failed or the communicator reports an asynchronous error).  Async
 * conditions are latched (see lag_stats).
 */
LAG_API lag_status lag_advect_cycle(lag_ctx ctx, void* v_t, void* v_t1, double dt);

/*
 * lag_extract — end of interval (write cycle, "at the end of an
 * interval ... the particle end locations are saved").  interval_index
 * is the 0-based index of the interval being extracted, counted per context
 * from lag_init: each call must pass the next one (the write cycles of one
 * block follow one another); out of order -> LAG_ESTATE.  COMM:
 * first returns every particle to its origin rank (collective; LAG_XCHG_LOCAL:
 * each block gathers its basis flows from every block of the group, and the
 * reseed of the group waits for the last block's extract).  Writes, for each of the n seeds
 * of the last lag_seed in seed order: start[i][dim] = x(g_i), end[i][dim] =
 * o + (g_i + d_i) h in fp64, status[i] = lag_flow_status.  Any of start, end,
 * status may be NULL (skipped); each may be a host or device pointer with
 * room for `capacity` entries.  Synchronises the stream and reports latched
 * asynchronous errors (LAG_EOVERFLOW, LAG_EGHOST, LAG_ENONFINITE) after
 * writing the outputs; a reported error is cleared.  Then reseeds with the
 * same stride unless flags & LAG_NO_RESEED.  With flags & LAG_ASYNC the call
 * only enqueues (no host synchronisation, for a simulation that must not
 * stall on the write cycle): outputs in device or page-locked host memory;
 * errors stay latched across the reseed until a synchronous lag_extract
 * reports them.
 * Errors: LAG_ESTATE (no lag_seed; interval_index out of order),
 * LAG_EINVAL (capacity < n; LAG_ASYNC with a pageable host output), LAG_ENCCL
 * (NCCL failure or asynchronous communicator error).
 */
LAG_API lag_status lag_extract(lag_ctx ctx, int64_t interval_index, double* start, double* end,
                               uint8_t* status, int64_t capacity, int64_t* n_out, uint32_t flags);

/*
 * lag_extract_ex — lag_extract plus, when term_cycle is not NULL, the cycle
 * (0-based within the interval) at which each non-valid basis flow
 * terminated, -1 for valid ones: with `end` this is the termination location
 * on the block boundary the paper names as future work.  Same
 * conventions and errors as lag_extract.
 */
LAG_API lag_status lag_extract_ex(lag_ctx ctx, int64_t interval_index, double* start, double* end,
                                  uint8_t* status, int32_t* term_cycle, int64_t capacity,
                                  int64_t* n_out, uint32_t flags);

/*
 * lag_local_group — connect n COMM contexts created with exchange =
 * LAG_XCHG_LOCAL into one group: ctxs[r] must hold rank r of the same layout
 * (nranks = n <= 64) on the same device; each may have its own stream (the
 * blocks then advance concurrently; the group joins the streams with events
 * around each exchange and write cycle, block 0's stream carries the
 * exchange kernels).  Call once, after every lag_init and before the first
 * lag_seed.  The group lives until its last context is destroyed.  Not
 * collective across processes: the whole group is in this process (the
 * single-GPU form of the COMM baseline, used to run several blocks of a
 * decomposition on one B200).
 * Errors: LAG_EINVAL (mismatched contexts, wrong transport, n out of range),
 * LAG_ESTATE (already grouped, set up by an earlier failed call, or seeded),
 * LAG_ENOMEM, LAG_ECUDA.
 */
LAG_API lag_status lag_local_group(lag_ctx* ctxs, int32_t n);

/* lag_stats — synchronise the stream and report counters (see lag_stats_t):
 * particle-steps are the unit of the paper's per-cycle timing (P:363-367
 * §4.2), terminations/exits and hand-offs are the particle-management and
 * communication counts of P:205-207 §3.1;
 * COMM over NCCL also polls the communicator's asynchronous error
 * (ncclCommGetAsyncError): a failure returns LAG_ENCCL. */
LAG_API lag_status lag_stats(lag_ctx ctx, lag_stats_t* out);

/* lag_destroy — free every resource of the context (NULL is a no-op). */
LAG_API lag_status lag_destroy(lag_ctx ctx);

/* lag_last_error — message of the last failing call on ctx (ctx may be NULL
 * for lag_init failures; thread-local).  Never NULL. */
LAG_API const char* lag_last_error(lag_ctx ctx);

/* lag_nccl_unique_id — write a fresh 128-byte ncclUniqueId into out (call on
 * one rank, broadcast to the others, pass as lag_config.nccl_id). */
LAG_API lag_status lag_nccl_unique_id(void* out, int64_t out_bytes);

/* lag_kernel_launches — number of kernels the context has launched since
 * lag_init (instrumentation for the benchmark's gpu_launches claim). */
LAG_API int64_t lag_kernel_launches(lag_ctx ctx);

/* lag_gridfill — post hoc reconstruction of BTO holes on a dense seed
 * lattice (paper P:229-233 §3.1 "interpolated ... post hoc"; Eq. 2,
 * P:289-303 §3.3; GridFill; reading R18 in DESIGN.md).
 *   dim      2 or 3.
 *   dims     [dim] host array: lattice extent per axis (x fastest), each >= 1.
 *   k        components per node (1..3), e.g. k = dim for end positions.
 *   values   DEVICE [n][k] f64, n = prod(dims); entries of invalid nodes are
 *            ignored (may hold anything, including NaN).
 *   valid    DEVICE [n] u8, nonzero = the node's value is known.
 *   out      DEVICE [n][k] f64 (caller-owned, must not alias values):
 *            valid nodes copy their value; an invalid node gets the linear
 *            interpolant (Eq. 1) between the nearest valid nodes on both
 *            sides along the lattice axis with the shortest such bracket
 *            (brackets of equal length averaged); NaN if no axis brackets it.
 *   filled   DEVICE [n] u8: 1 where an invalid node was filled, else 0.
 *   stream   cudaStream_t (NULL = legacy default); the call synchronises it.
 * Arithmetic is round-to-nearest f64 without contraction, so results are
 * bitwise reproducible.  Errors: LAG_EINVAL (bad sizes, NULL or non-device
 * pointers), LAG_ECUDA (launch failure); message in lag_last_error(NULL). */
LAG_API lag_status lag_gridfill(int32_t dim, const int64_t* dims, int32_t k, const double* values,
                                const uint8_t* valid, double* out, uint8_t* filled, void* stream);

/* lag_ftle — finite-time Lyapunov exponent of a flow map on a dense seed
 * lattice (paper P:415-416 §4.3, FTLE fields from basis flows post hoc;
 * operation as SPEC.md:460-468 states it).
 *   dim        2 or 3.
 *   dims       [dim] host array: lattice extent per axis (x fastest), each >= 1.
 *   spacing    [dim] host array: seed spacing per axis (stride * h), > 0.
 *   T          integration time of the flow map (nonzero, finite; |T| is used).
 *   ends       DEVICE [n][dim] f64 end positions, n = prod(dims) (complete
 *              lattice, e.g. after lag_gridfill).
 *   ftle       DEVICE [n] f64 out: ln(sqrt(lambda_max(J^T J))) / |T| with J
 *              the flow-map gradient by central differences (one-sided at
 *              lattice faces; an axis of extent 1 contributes 0); 0 where
 *              lambda_max <= 0; NaN where the stencil holds non-finite ends.
 *   n_degenerate  host out (may be NULL): nodes with lambda_max <= 0.
 *   stream     cudaStream_t (NULL = legacy default); the call synchronises it.
 * Errors: LAG_EINVAL (bad sizes, spacing, T, NULL or non-device pointers),
 * LAG_ENOMEM, LAG_ECUDA; message in lag_last_error(NULL). */
LAG_API lag_status lag_ftle(int32_t dim, const int64_t* dims, const double* spacing, double T,
                            const double* ends, double* ftle, int64_t* n_degenerate, void* stream);

/* lag_stitch — pathlines stitched from the basis flows of K successive
 * intervals (§3.2 "a trajectory can be stitched together by using basis
 * flows of successive nonoverlapping intervals"; barycentric interpolation of
 * end positions).  Reading R16: on the
 * seed lattice the Delaunay ties are broken by the fixed Kuhn template (cube
 * split along the descending order of the local coordinates).
 *   dim, dims      2 or 3; [dim] host array, lattice extent per axis (>= 2).
 *   origin, spacing [dim] host arrays: lattice node 0 and seed spacing (> 0).
 *   K              number of intervals (>= 0).
 *   ends           DEVICE [K][n][dim] f64 end positions per interval, x fastest.
 *   valid          DEVICE [K][n] u8 (nonzero = valid basis flow) or NULL = all.
 *   m, starts      number of pathlines; DEVICE [m][dim] f64 start points.
 *   path           DEVICE [m][K+1][dim] f64 out: path[q][0] = start, then one
 *                  sample per interval; NaN after a truncation.
 *   status         DEVICE [m] u8 out: 0 complete, 1 left the lattice hull (no
 *                  clamping), 2 needed an invalid basis flow
 *                  (fill holes first, lag_gridfill).
 *   stream         cudaStream_t (NULL = legacy default); the call synchronises it.
 * Errors: LAG_EINVAL (sizes, spacing, NULL or non-device pointers), LAG_ECUDA. */
LAG_API lag_status lag_stitch(int32_t dim, const int64_t* dims, const double* origin, const double* spacing,
                              int32_t K, const double* ends, const uint8_t* valid, int64_t m,
                              const double* starts, double* path, uint8_t* status, void* stream);

/* lag_abi_version — LAG_ABI_VERSION the library was built with. */
LAG_API int32_t lag_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LAG_H */
