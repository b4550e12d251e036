// lag_brick.cuh — stride-1 3-D advect kernel with the velocity box of a seed
// brick staged in shared memory (DESIGN.md §6 "advect_brick_kernel").
//
// Same method as advect_kernel (one RK4 step per particle per cycle, P:204
// §3.1; trilinear in space, linear in time, P:138 + north star; BTO
// termination or COMM hand-off) and the same particle records,
// tiles, termination records and counters.  What differs is where the
// corners come from and how many registers that costs:
//
// * One CTA (8 warps) per seed brick: 16 tiles = 32 x 4 x 4 seeds (the seed
//   order of seed_kernel with by = bz = 4).  At stride 1 these particles stay
//   within a few cells of each other over an interval, so the nodes their
//   stage samples touch form a small box.
// * The box = the brick's cell bounding box (written by the previous cycle,
//   or by brick_bbox_kernel after seeding) + one cell of margin for the stage
//   samples (CFL < 1), clipped to the fast range (block interior in BTO,
//   gather range in COMM).  Warp 0 stages both slices' boxes with bulk async
//   copies (cp.async.bulk, one per node row, completion on an mbarrier) while
//   every warp loads its particle records.
// * Every stage gathers its 8 corners from shared memory (LDS, no L1/L2
//   round trip, conflict-free for an x-run of particles): stage 1 v_t,
//   stage 2 v_t + v_t1 (kept for stage 3 unless a sample moved cell),
//   stage 4 v_t1.  No corner cache lives across stages 1 -> 2 or 3 -> 4, so
//   the kernel fits 85 registers (3 CTAs = 24 warps per SM) and has no
//   reload branches.
// * A sample outside the box's fast range takes the slow path: the full
//   boundary classification (classify_slow) and, if still valid (closed top
//   face, COMM ghost cells, a box that did not fit), corners from global
//   memory.
// * The epilogue also reduces the survivors' cells into the brick's bounding
//   box for the next cycle.
#pragma once
#include "lag_kernels.cuh"

namespace lag {

constexpr int kBrickThreads = 512;          // 16 warps, one tile each per brick
constexpr int kBrickTiles = 16;             // tiles per brick (4 x 4 rows of 32 seeds)
constexpr int kBrickRows = 4;               // seed brick rows per axis (y, z)
constexpr int kBrickMinBlocks = 1;          // one persistent CTA per SM
constexpr int kBoxBytes = 32 * 1024;        // shared-memory box per slice (x 2 slices x 2 buffers)
constexpr int kBBoxInts = 8;                // per brick: min xyz, max xyz, known, pad

struct BrickArgs {
    AdvectArgs a;
    int32_t* bbox;                  // [brick][kBBoxInts] global cells of the live particles
    int32_t n_seed_bricks;          // bricks holding seeded tiles (COMM appends come after)
    int64_t slice_bytes;            // bytes of one slice array (bulk copies stay inside)
};

struct BoxParams {
    int32_t o[3];                   // global cell of box offset 0 (fast range origin)
    int32_t span[3];                // fast cells: 0 <= c - o <= span
    uint32_t off0, off1;            // smem byte offset of node o in the v_t / v_t1 box
    int32_t P, Q;                   // smem row / plane pitch (bytes)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Pairs of x-neighbour corners (see gather_pairs) from a staged box.
__device__ __forceinline__ void gather_pairs_sm(const unsigned char* sm, uint32_t off, int P, int Q,
                                                f2_t* Pc) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const float* q = reinterpret_cast<const float*>(sm + off + (r & 1) * P + (r >> 1) * Q);
        float e[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) e[k] = q[k];
#pragma unroll
        for (int c = 0; c < 3; ++c) Pc[r * 3 + c] = f2_pack(e[c], e[3 + c]);
    }
}

// Cell of a stage sample at fs (cell units from the stage-1 cell origin, whose
// offsets from the box origin are v1): offsets v, fractions f; true = fast.
__device__ __forceinline__ bool brick_cell(const int v1[3], const float fs[3], const int32_t span[3],
                                           int v[3], float f[3]) {
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        int tb;
        const float fl = floor_fma(fs[ax], tb);
        f[ax] = fs[ax] - fl;                                             // exact
        v[ax] = v1[ax] + (tb - kMagicBits);
        ok &= (unsigned)v[ax] <= (unsigned)span[ax];
    }
    return ok;
}

// Slow path of one stage sample: classify (BTO: TERM/EXIT; COMM: EXIT or a
// ghost cell) and return the slice-local node index of a valid cell.
// v is updated to the offsets of the classified cell (the closed top face
// moves to the last cell, f = 1).
template <bool BTO>
__device__ __forceinline__ int brick_slow(const AdvectArgs& a, const int32_t o[3], int v[3],
                                          float f[3], uint8_t& st, bool& ghost_bad) {
    int c[3] = {v[0] + o[0], v[1] + o[1], v[2] + o[2]};
    st = classify_slow<3, BTO>(a, c, f, ghost_bad);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) v[ax] = c[ax] - o[ax];
    return node_index<3>(a, c);
}

// Warp 0: stage the box of `brick` into buffer `buf` (params -> bp) and arm
// the buffer's mbarrier with the bytes in flight (0 when not staged, so the
// barrier phase always completes once per use).
__device__ __forceinline__ void stage_box(const BrickArgs& B, int brick, unsigned char* smb,
                                          BoxParams& bp, unsigned long long* mbar, int lane) {
    const AdvectArgs& a = B.a;
    int32_t o[3], span[3], P = 0, Q = 0, io = 0;
    int dx = 0, dy = 0, dz = 0;
    bool staged = brick < B.n_seed_bricks && B.bbox[brick * kBBoxInts + 6] == 1;
    if (staged) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int lo_c = max(B.bbox[brick * kBBoxInts + ax] - 1, a.gmin[ax]);
            const int hi_c = min(B.bbox[brick * kBBoxInts + 3 + ax] + 1, a.gmin[ax] + a.gspan[ax]);
            o[ax] = lo_c;
            span[ax] = hi_c - lo_c;
            staged &= hi_c >= lo_c;
        }
    }
    if (staged) {
        dx = span[0] + 2; dy = span[1] + 2; dz = span[2] + 2;          // box nodes
        const int rowb = 12 * dx;
        const int gy = 12 * a.sx, gz = 12 * a.sxy;                     // global pitches (bytes)
        P = rowb + 32; P += (gy - P) & 15;                             // P == gy (mod 16)
        Q = P * (dy - 1) + rowb + 32; Q += (gz - Q) & 15;              // Q == gz (mod 16)
        const int need = 64 + Q * (dz - 1) + P * (dy - 1) + rowb;
        staged = need <= kBoxBytes;
        io = (o[0] - a.base[0]) + a.sx * (o[1] - a.base[1]) + a.sxy * (o[2] - a.base[2]);
    }
    if (!staged) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) { o[ax] = 1 << 29; span[ax] = 0; }   // nothing fast
    }
    const uintptr_t g0 = reinterpret_cast<uintptr_t>(a.v0) + 12 * (uintptr_t)io;
    const uintptr_t g1 = reinterpret_cast<uintptr_t>(a.v1) + 12 * (uintptr_t)io;
    const uint32_t off0 = 16 + (uint32_t)(g0 & 15);                    // smem == global (mod 16)
    const uint32_t off1 = kBoxBytes + 16 + (uint32_t)(g1 & 15);
    const int rows = dy * dz;
    // one bulk copy per node row and slice: the 16 B-aligned span of the
    // row, clipped to the slice array; clipped ends are copied by hand
    uint32_t bytes = 0;
    if (staged) {
        const uintptr_t base0 = reinterpret_cast<uintptr_t>(a.v0), base1 = reinterpret_cast<uintptr_t>(a.v1);
        for (int k = lane; k < 2 * rows; k += 32) {
            const int s = k >= rows, row = s ? k - rows : k;
            const int zl = row / dy, yl = row - zl * dy;
            const uintptr_t gb = s ? base1 : base0;
            const uintptr_t gs = (s ? g1 : g0) + (uintptr_t)(12 * a.sx) * yl + (uintptr_t)(12 * a.sxy) * zl;
            const uintptr_t ge = gs + 12 * dx;
            const uintptr_t bs = max(gs & ~(uintptr_t)15, (gb + 15) & ~(uintptr_t)15);
            const uintptr_t be = min((ge + 15) & ~(uintptr_t)15, (gb + B.slice_bytes) & ~(uintptr_t)15);
            if (be > bs) bytes += (uint32_t)(be - bs);
        }
        bytes = __reduce_add_sync(0xffffffffu, bytes);
    }
    if (lane == 0) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) { bp.o[ax] = o[ax]; bp.span[ax] = span[ax]; }
        bp.off0 = off0; bp.off1 = off1; bp.P = P; bp.Q = Q;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                     :: "r"(smem_u32(mbar)), "r"(bytes) : "memory");
    }
    __syncwarp();
    if (!staged) return;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const uintptr_t base0 = reinterpret_cast<uintptr_t>(a.v0), base1 = reinterpret_cast<uintptr_t>(a.v1);
    for (int k = lane; k < 2 * rows; k += 32) {
        const int s = k >= rows, row = s ? k - rows : k;
        const int zl = row / dy, yl = row - zl * dy;
        const uintptr_t gb = s ? base1 : base0;
        const uintptr_t gs = (s ? g1 : g0) + (uintptr_t)(12 * a.sx) * yl + (uintptr_t)(12 * a.sxy) * zl;
        const uintptr_t ge = gs + 12 * dx;
        const uintptr_t bs = max(gs & ~(uintptr_t)15, (gb + 15) & ~(uintptr_t)15);
        const uintptr_t be = min((ge + 15) & ~(uintptr_t)15, (gb + B.slice_bytes) & ~(uintptr_t)15);
        const uint32_t ss = (s ? off1 : off0) + (uint32_t)(P * yl + Q * zl);   // smem of gs
        if (be > bs)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                :: "r"(smem_u32(smb) + ss + (uint32_t)(bs - gs)), "l"(bs), "r"((uint32_t)(be - bs)),
                   "r"(smem_u32(mbar)) : "memory");
        // row ends outside the 16 B-aligned part of the array (by hand)
        const uintptr_t h1 = be > bs ? min(bs, ge) : ge;
        for (uintptr_t p = gs; p < h1; p += 4)
            *reinterpret_cast<float*>(smb + ss + (uint32_t)(p - gs)) = __ldg(reinterpret_cast<const float*>(p));
        if (be > bs)
            for (uintptr_t p = max(be, gs); p < ge; p += 4)
                *reinterpret_cast<float*>(smb + ss + (uint32_t)(p - gs)) = __ldg(reinterpret_cast<const float*>(p));
    }
}

// Persistent: CTA c advects bricks c, c + G, ... (one tile per warp).  Box k+1
// is staged into the other buffer while brick k computes (double buffering).
template <bool BTO>
__global__ void __launch_bounds__(kBrickThreads, kBrickMinBlocks)
advect_brick_kernel(const BrickArgs B) {
    extern __shared__ __align__(128) unsigned char sm[];        // [2][v_t box | v_t1 box]
    __shared__ BoxParams bps[2];
    __shared__ __align__(8) unsigned long long mbar[2];
    __shared__ int32_t nbb[2][6];
    const AdvectArgs& a = B.a;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int n_tiles = a.n_tiles_dev ? *a.n_tiles_dev : a.n_tiles;
    const int n_bricks = (n_tiles + kBrickTiles - 1) / kBrickTiles;
    const int G = gridDim.x;

    unsigned long long steps = 0, nterm = 0, nexit = 0, nsent = 0;
    uint32_t errbits = 0;
    bool did_remote = false;

    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&mbar[1])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 2; ++i) {
            nbb[i][0] = nbb[i][1] = nbb[i][2] = 0x7fffffff;
            nbb[i][3] = nbb[i][4] = nbb[i][5] = -0x7fffffff;
        }
    }
    __syncthreads();
    int brick = blockIdx.x;
    if (warp == 0 && brick < n_bricks) stage_box(B, brick, sm, bps[0], &mbar[0], lane);
    int tile = brick * kBrickTiles + warp;
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    int cnt = brick < n_bricks && tile < n_tiles ? a.tile_count[tile] : 0;
    float4 r = lane < cnt ? a.state[(size_t)tile * kTile + lane] : z4;
    __syncthreads();

#pragma unroll 1
    for (int it = 0; brick < n_bricks; brick += G, ++it) {
        const int buf = it & 1;
        const int nbrick = brick + G;
        if (warp == 0 && nbrick < n_bricks)
            stage_box(B, nbrick, sm + (buf ^ 1) * 2 * kBoxBytes, bps[buf ^ 1], &mbar[buf ^ 1], lane);
        const int ntile = nbrick * kBrickTiles + warp;
        const int ncnt = nbrick < n_bricks && ntile < n_tiles ? a.tile_count[ntile] : 0;
        const float4 nr = lane < ncnt ? a.state[(size_t)ntile * kTile + lane] : z4;
        if (threadIdx.x == 0) {                                  // next use of the other accumulator
            nbb[buf ^ 1][0] = nbb[buf ^ 1][1] = nbb[buf ^ 1][2] = 0x7fffffff;
            nbb[buf ^ 1][3] = nbb[buf ^ 1][4] = nbb[buf ^ 1][5] = -0x7fffffff;
        }
        {
            uint32_t done = 0;
            const uint32_t par = (uint32_t)(it >> 1) & 1u;
            while (!done)
                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                             : "=r"(done) : "r"(smem_u32(&mbar[buf])), "r"(par) : "memory");
        }
        const unsigned char* smb = sm + buf * 2 * kBoxBytes;
        const BoxParams& bp = bps[buf];
        const int32_t o[3] = {bp.o[0], bp.o[1], bp.o[2]};
        const int32_t span[3] = {bp.span[0], bp.span[1], bp.span[2]};
        const uint32_t off0 = bp.off0, off1 = bp.off1;
        const int P = bp.P, Q = bp.Q;
        int bbmin[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff};
        int bbmax[3] = {-0x7fffffff, -0x7fffffff, -0x7fffffff};
        do {
            if (cnt == 0) break;                                 // warp-uniform
        const bool live = lane < cnt;
        float4* trec = a.state + (size_t)tile * kTile;
        int g[3];
        unpack_g(__float_as_uint(r.w), a, g);
        const float d[3] = {r.x, r.y, r.z};
        uint8_t st = ST_VALID;
        bool ghost_bad = false;
        f2_t S[12];

        // ---- stage 1: q1 = x, v_t only ----
        int v1[3];
        float f1[3];
        {
            int gbo[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) gbo[ax] = g[ax] - o[ax] - kMagicBits;
            const bool fast = cells_b<3>(gbo, d, span, v1, f1);
            if (fast) {
                gather_pairs_sm(smb, off0 + 12 * v1[0] + P * v1[1] + Q * v1[2], P, Q, S);
            } else if (live) {                               // committed: clamp only
                uint8_t st1;
                const int idx = brick_slow<BTO>(a, o, v1, f1, st1, ghost_bad);
                LAG_CHECK_GATHER(a, idx, true);
                gather_pairs<3>(a.v0, idx, a.sx, a.sxy, S);
            }
        }
        float k1[3];
        interp_pairs<3>(S, f1, k1);

        // ---- stage 2: q2 = x + dt/2 k1, alpha = 1/2: v_t + v_t1 ----
        float e[3], f[3];
        int v[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = fmaf(a.hdth[ax], k1[ax], f1[ax]);
        int cur2[3];
        {
            const bool fast = brick_cell(v1, e, span, v, f);
            if (fast) {
                const uint32_t off = 12 * v[0] + P * v[1] + Q * v[2];
                f2_t T[12];
                gather_pairs_sm(smb, off0 + off, P, Q, S);
                gather_pairs_sm(smb, off1 + off, P, Q, T);
#pragma unroll
                for (int i = 0; i < 12; ++i) S[i] = f2_add(S[i], T[i]);
            } else if (live) {
                const int idx = brick_slow<BTO>(a, o, v, f, st, ghost_bad);
                if (st == ST_VALID) {
                    f2_t T[12];
                    LAG_CHECK_GATHER(a, idx, true);
                    gather_pairs<3>(a.v0, idx, a.sx, a.sxy, S);
                    gather_pairs<3>(a.v1, idx, a.sx, a.sxy, T);
#pragma unroll
                    for (int i = 0; i < 12; ++i) S[i] = f2_add(S[i], T[i]);
                }
                v[0] = -(1 << 30);                           // slow: never equal below
            }
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) cur2[ax] = v[ax];
        }
        float T2[3];
        interp_pairs<3>(S, f, T2);                           // T2 = 2 k2

        // ---- stage 3: q3 = x + dt/4 T2, alpha = 1/2 (same cell: keep S) ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = fmaf(a.qdth[ax], T2[ax], f1[ax]);
        {
            const bool fast = brick_cell(v1, e, span, v, f);
            const bool same = fast && v[0] == cur2[0] && v[1] == cur2[1] && v[2] == cur2[2];
            if (!same && live && st == ST_VALID) {
                if (fast) {
                    const uint32_t off = 12 * v[0] + P * v[1] + Q * v[2];
                    f2_t T[12];
                    gather_pairs_sm(smb, off0 + off, P, Q, S);
                    gather_pairs_sm(smb, off1 + off, P, Q, T);
#pragma unroll
                    for (int i = 0; i < 12; ++i) S[i] = f2_add(S[i], T[i]);
                } else {
                    const int idx = brick_slow<BTO>(a, o, v, f, st, ghost_bad);
                    if (st == ST_VALID) {
                        f2_t T[12];
                        LAG_CHECK_GATHER(a, idx, true);
                        gather_pairs<3>(a.v0, idx, a.sx, a.sxy, S);
                        gather_pairs<3>(a.v1, idx, a.sx, a.sxy, T);
#pragma unroll
                        for (int i = 0; i < 12; ++i) S[i] = f2_add(S[i], T[i]);
                    }
                }
            }
        }
        float T3[3];
        interp_pairs<3>(S, f, T3);                           // T3 = 2 k3

        // ---- stage 4: q4 = x + dt/2 T3, alpha = 1: v_t1 ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = fmaf(a.hdth[ax], T3[ax], f1[ax]);
        {
            const bool fast = brick_cell(v1, e, span, v, f);
            if (fast) {
                gather_pairs_sm(smb, off1 + 12 * v[0] + P * v[1] + Q * v[2], P, Q, S);
            } else if (live && st == ST_VALID) {
                const int idx = brick_slow<BTO>(a, o, v, f, st, ghost_bad);
                if (st == ST_VALID) {
                    LAG_CHECK_GATHER(a, idx, true);
                    gather_pairs<3>(a.v1, idx, a.sx, a.sxy, S);
                }
            }
        }
        float k4[3];
        interp_pairs<3>(S, f, k4);

        // ---- update: x' = x + dt/6 (k1 + 2k2 + 2k3 + k4) ----
        float dn[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
            dn[ax] = fmaf(a.sdth[ax], (k1[ax] + k4[ax]) + (T2[ax] + T3[ax]), d[ax]);
        bool finite = true;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) finite &= fabsf(dn[ax]) < 4194304.f;   // 2^22 cells
        bool migrate = false;
        int nb = 0;
        int cn[3];
        {
            float fn[3];
            int gbb[3];                                      // g - bmin - magic
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) gbb[ax] = g[ax] - a.bmin[ax] - kMagicBits;
            const bool inblk = cells_b<3>(gbb, dn, a.bspan, cn, fn);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) cn[ax] += a.bmin[ax];     // global cells
            if (!inblk && live && st == ST_VALID) {
                bool gdummy = false;
                int cc[3] = {cn[0], cn[1], cn[2]};
                if constexpr (BTO) {
                    st = classify_slow<3, true>(a, cc, fn, gdummy);
                } else {
                    // COMM: in the domain but outside the block -> hand off
                    bool out_dom = false;
                    int mul = 1;
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) {
                        out_dom |= (cn[ax] < 0) | (cn[ax] > a.N[ax] - 1) |
                                   ((cn[ax] == a.N[ax] - 1) & (fn[ax] != 0.f));
                        const int oo = (cn[ax] < a.lo[ax]) ? -1
                                       : ((cn[ax] >= a.hi[ax] && a.hi[ax] < a.N[ax]) ? 1 : 0);
                        migrate |= (oo != 0);
                        nb += (oo + 1) * mul;
                        mul *= 3;
                    }
                    if (out_dom) { st = ST_EXIT; migrate = false; }
                }
            }
        }
        if (live && !finite) { errbits |= ERR_NONFINITE; st = ST_EXIT; migrate = false; }
        if (live && ghost_bad) { errbits |= ERR_GHOST; if (st == ST_VALID) st = ST_EXIT; migrate = false; }

        // ---- particle management (as advect_kernel) + next cycle's box ----
        const bool keep = live && st == ST_VALID && !migrate;
        if (keep) {
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) { bbmin[ax] = min(bbmin[ax], cn[ax]); bbmax[ax] = max(bbmax[ax], cn[ax]); }
        }
        const unsigned kmask = __ballot_sync(0xffffffffu, keep);
        const unsigned dmask = __ballot_sync(0xffffffffu, live && st != ST_VALID);
        const unsigned tmask = __ballot_sync(0xffffffffu, live && st == ST_TERM);
        __syncwarp();
        if (keep) {
            const int pos = __popc(kmask & ((1u << lane) - 1u));
            trec[pos] = make_float4(dn[0], dn[1], dn[2], r.w);
        }
        if constexpr (!BTO) {
            const unsigned mmask = __ballot_sync(0xffffffffu, migrate);
            if (migrate) {
                const unsigned peers = __match_any_sync(mmask, nb);
                const int leader = __ffs(peers) - 1;
                float4* sb = a.slot_ptr[nb];
                uint32_t base0 = 0;
                if (lane == leader) base0 = atomicAdd(reinterpret_cast<uint32_t*>(sb), (uint32_t)__popc(peers));
                base0 = __shfl_sync(peers, base0, leader);
                const uint32_t pos = base0 + __popc(peers & ((1u << lane) - 1u));
                if (pos < (uint32_t)a.slot_capv[nb])
                    sb[1 + pos] = make_float4(dn[0], dn[1], dn[2], r.w);
                else
                    errbits |= ERR_OVERFLOW;
                did_remote = true;
            }
            if (lane == 0) nsent += __popc(mmask);
        }
        if (dmask) {
            uint32_t slot0 = 0;
            if (lane == 0) slot0 = atomicAdd(a.dead_count, (uint32_t)__popc(dmask));
            slot0 = __shfl_sync(0xffffffffu, slot0, 0);
            if (live && st != ST_VALID) {
                const uint32_t s = slot0 + __popc(dmask & ((1u << lane) - 1u));
                if (s < a.dead_cap) {
                    a.dead_rec[s] = r;                       // pre-step position
                    a.dead_info[s] = ((uint32_t)st << 24) | (uint32_t)(a.cycle & 0xffffff);
                } else {
                    errbits |= ERR_OVERFLOW;
                }
            }
        }
        if (lane == 0) {
            a.tile_count[tile] = (uint8_t)__popc(kmask);
            steps += (unsigned long long)cnt;
            nterm += __popc(tmask);
            nexit += __popc(dmask) - __popc(tmask);
        }
        } while (false);

        // ---- the brick's cell box for the next cycle ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const int mn = __reduce_min_sync(0xffffffffu, bbmin[ax]);
            const int mx = __reduce_max_sync(0xffffffffu, bbmax[ax]);
            if (lane == 0) { atomicMin(&nbb[buf][ax], mn); atomicMax(&nbb[buf][3 + ax], mx); }
        }
        __syncthreads();                     // buffer `buf` free; box params of the next brick visible
        if (threadIdx.x < 8 && brick < B.n_seed_bricks) {
            const int i = threadIdx.x;
            B.bbox[brick * kBBoxInts + i] = i < 6 ? nbb[buf][i] : (i == 6 ? 1 : 0);
        }
        __syncwarp();
        tile = ntile; cnt = ncnt; r = nr;
    }

    // one atomic per warp per counter
    if (lane == 0 && steps) {
        atomicAdd(&a.counters[CNT_STEPS], steps);
        if (nterm) atomicAdd(&a.counters[CNT_TERM], nterm);
        if (nexit) atomicAdd(&a.counters[CNT_EXIT], nexit);
        if (nsent) atomicAdd(&a.counters[CNT_SENT], nsent);
    }
    errbits = __reduce_or_sync(0xffffffffu, errbits);
    if (lane == 0 && errbits) atomicOr(a.err, errbits);
    if constexpr (!BTO) {
        if (a.n_sig) {                                           // peer transport (see advect_kernel)
            if (did_remote) __threadfence_system();
            __syncwarp();
            if (lane == 0) {
                const uint32_t total = (gridDim.x * kBrickThreads) >> 5;
                if (atomicAdd(a.done_warps, 1u) == total - 1) {
                    *a.done_warps = 0u;
                    __threadfence_system();
                    for (int k = 0; k < a.n_sig; ++k)
                        *reinterpret_cast<volatile unsigned long long*>(a.sig_flag[k]) = a.sig_value;
                    __threadfence_system();
                }
            }
        }
    }
}

// Seed bricks' cell boxes (stride-s lattice nodes, d = 0: the cell of a node
// is the node itself).  One thread per brick.
struct BBoxInitArgs {
    int32_t* bbox;
    int64_t n_bricks;
    int32_t first[3], stride, ns[3];
};

static __global__ void brick_bbox_kernel(const BBoxInitArgs a) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.n_bricks) return;
    int64_t ix0, iy0, iz0;
    brick_tile(b * kBrickTiles, a.ns, kBrickRows, kBrickRows, ix0, iy0, iz0);
    const int64_t i1[3] = {min(ix0 + kTile - 1, (int64_t)a.ns[0] - 1), min(iy0 + kBrickRows - 1, (int64_t)a.ns[1] - 1),
                           min(iz0 + kBrickRows - 1, (int64_t)a.ns[2] - 1)};
    const int64_t i0[3] = {ix0, iy0, iz0};
    int32_t* q = a.bbox + b * kBBoxInts;
    for (int ax = 0; ax < 3; ++ax) {
        q[ax] = (int32_t)(a.first[ax] + a.stride * i0[ax]);
        q[3 + ax] = (int32_t)(a.first[ax] + a.stride * i1[ax]);        // min > max: empty brick
    }
    q[6] = 1;
    q[7] = 0;
}

}  // namespace lag
