// lag_kernels.cuh — sm_100a kernels of the in situ Lagrangian flow-map hot path.
//
// Paper: arXiv 2004.02003 (P:nnn = PAPER.md line).  Design: DESIGN.md.
//
// Particle record (16 B, one float4): (d_x, d_y, d_z, bits(g)) where g is the
// particle's integer global seed node packed into 32 bits (bx | by | bz bits)
// and d its displacement from g in cell units.  Position in index space is
// u = g + d; keeping d small preserves fp32 precision.
//
// Particle list = warp tiles of 32 records + one u8 live count per tile.  The
// advect kernel compacts survivors in place inside each tile (warp ballot),
// so invalid particles are never launched again ("managing memory to
// prevent invalid particles from being launched on GPU threads").  No atomics
// on the hot path; order inside a tile is stable (deterministic).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lag {

constexpr int kTile = 32;
constexpr int kThreads = 128;          // advect CTA size (4 warps; DESIGN.md §9 CTA-size sweep)
constexpr int kMinBlocks = 4;          // __launch_bounds__ min CTAs per SM
constexpr int kBrickRows = 4;          // seed tiles are ordered in 32 x 4 x 4 bricks (3-D)

enum : uint32_t { ERR_OVERFLOW = 1u, ERR_GHOST = 2u, ERR_NONFINITE = 4u, ERR_XCHG = 8u };
enum : int { CNT_STEPS = 0, CNT_TERM = 1, CNT_EXIT = 2, CNT_SENT = 3, CNT_RECV = 4, CNT_N = 8 };
enum : uint8_t { ST_VALID = 0, ST_TERM = 1, ST_EXIT = 2 };

struct AdvectArgs {
    const float* __restrict__ v0;   // slice at t   (AoS, element 0 = global node base)
    const float* __restrict__ v1;   // slice at t+dt
    float4* state;                  // particle records, tiles of 32
    uint8_t* tile_count;            // live records per tile
    const int32_t* n_tiles_dev;     // device-side tile count (COMM appends) or nullptr
    int32_t n_tiles;                // host-known tile count (used when n_tiles_dev == nullptr)
    int32_t N[3];                   // global nodes
    int32_t lo[3], hi[3];           // block [lo, hi)
    int32_t base[3];                // global node index of slice element 0 (= lo - G)
    int32_t cmax[3];                // largest local cell index a gather may use (ext - 2)
    // fast-path cell ranges (global cell index c): gathers [gmin, gmin + gspan],
    // block membership [bmin, bmin + bspan]; anything else takes the slow path
    int32_t gmin[3], gspan[3];
    int32_t bmin[3], bspan[3];
    int32_t gidx0;                  // node index of global cell gmin (local slice coordinates)
    int32_t frozen;                 // v0 == v1: one snapshot per cycle; load corners once
    int32_t slice_nodes;            // nodes in one slice array (debug bounds checks)
    int32_t sx, sxy;                // slice pitch (nodes) of a row / a plane
    float hdth[3], qdth[3], sdth[3];// dt/h * (1/2, 1/4, 1/6)
    uint32_t bx, by;                // packed seed-node bit widths (x, y)
    uint32_t mx, my;                // masks
    // termination records (both modes): appended, scattered by extract
    float4* dead_rec;
    uint32_t* dead_info;            // (status << 24) | cycle
    uint32_t* dead_count;
    uint32_t dead_cap;
    unsigned long long* counters;   // CNT_*
    uint32_t* err;
    int32_t cycle;
    // COMM: outgoing slots, one per neighbour offset (3^dim):
    // slot k = slot_rec[slot_base[k]] = header (u32 count) then slot_capv[k] records
    float4* slot_rec;
    int32_t slot_base[27];
    int32_t slot_capv[27];
    float4* slot_ptr[27];           // slot of offset k: local (NCCL, peer) or the owner's inbox (LOCAL)
    // COMM exchange overlap (LAG_XCHG_PEER_OVERLAP): pass 1 advects tiles
    // [0, *n_tiles_b) whose stage samples cannot reach a ghost node and defers
    // the others; pass 2 advects the deferred tiles and the tiles appended by
    // this cycle's exchange.  pass 0: every tile.
    int32_t pass;
    const uint32_t* n_tiles_b;      // tile count before this cycle's append
    uint32_t* next_b;               // pass 2 sets the next cycle's n_tiles_b / defer_count
    uint32_t* next_defer;           // (the other parity's words)
    uint32_t* defer_list;
    uint32_t* defer_count;
    int32_t smin[3], sspan[3];      // ghost-free cells (gather offsets): samples stay off ghost nodes
};

// Programmatic dependent launch (kernels launched with the
// programmatic-stream-serialization attribute, lag_api.cu / lag_peer.cu):
// the next kernel in the stream may be scheduled once every CTA of this one
// has called griddep_launch(); griddep_wait() blocks until the previous
// kernel has completed and its memory is visible (a no-op when the kernel
// was launched without the attribute or after a non-kernel stream item).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// floor(e) on the FMA pipe (no FRND): for |e| < 2^22, e + 1.5*2^23 rounded
// toward -inf is 1.5*2^23 + floor(e) exactly, so its bits hold floor(e) in
// the low mantissa (bits - 0x4B400000 = floor(e)) and t - 1.5*2^23 is floor(e).
constexpr int kMagicBits = 0x4B400000;    // bits of 12582912.0f = 1.5 * 2^23
__device__ __forceinline__ float floor_fma(float e, int& bits) {
    const float t = __fadd_rd(e, 12582912.0f);
    bits = __float_as_int(t);
    return t - 12582912.0f;
}

// Slow path (a sample near a block or global face): full classification with
// integer compares on the cell index.
//   EXIT : outside the closed global domain [0, N-1]
//   TERM : (BTO) outside the half-open block, closed at the global top
//   VALID: inside; the closed upper face c = N-1, f = 0 is moved to
//          c = N-2, f = 1 (same point, interpolation cell inside the grid);
//          COMM flags a gather outside the ghost layers.
template <int DIM, bool BTO>
__device__ __forceinline__ uint8_t classify_slow(const AdvectArgs& a, int c[3], float f[3],
                                                 bool& ghost_bad) {
    bool out_dom = false, out_blk = false;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        out_dom |= (c[ax] < 0) | (c[ax] > a.N[ax] - 1) | ((c[ax] == a.N[ax] - 1) & (f[ax] != 0.f));
        if constexpr (BTO)
            out_blk |= (c[ax] < a.lo[ax]) | ((c[ax] >= a.hi[ax]) & (a.hi[ax] < a.N[ax]));
    }
    if (out_dom) return ST_EXIT;
    if (out_blk) return ST_TERM;
    bool gb = false;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        if (c[ax] == a.N[ax] - 1) { c[ax] = a.N[ax] - 2; f[ax] = 1.f; }
        const int l = c[ax] - a.base[ax];
        gb |= (l < 0) | (l > a.cmax[ax]);
    }
    if (gb) {                                            // COMM only: CFL >= 1 in a stage
        ghost_bad = true;
        return ST_EXIT;
    }
    return ST_VALID;
}

// Slow path on gather offsets v = c - gmin: convert to cells, classify, convert back.
template <int DIM, bool BTO>
__device__ __forceinline__ uint8_t classify_slow_v(const AdvectArgs& a, int v[3], float f[3],
                                                bool& ghost_bad) {
    int c[3];
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) c[ax] = v[ax] + a.gmin[ax];
    const uint8_t st = classify_slow<DIM, BTO>(a, c, f, ghost_bad);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) v[ax] = c[ax] - a.gmin[ax];
    return st;
}

// Node index (local slice coordinates) of the cell with gather offsets v.
template <int DIM>
__device__ __forceinline__ int vindex(const AdvectArgs& a, const int v[3]) {
    if constexpr (DIM == 3) return v[0] + a.sx * v[1] + a.sxy * v[2] + a.gidx0;
    else return v[0] + a.sx * v[1] + a.gidx0;
}

// ---------------------------------------------------------------------------
// Packed fp32x2 (Blackwell FFMA2 / FMUL2 / FADD2): the corner cache holds, per
// corner row (dy, dz) and component c, the pair {V(x0).c, V(x0+1).c} of the
// row's two x-neighbour nodes in one 64-bit register pair, so one packed
// instruction serves two corners (half the FP issue slots of scalar code).
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2_pack(float lo, float hi) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(f2_t r, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
}
__device__ __forceinline__ f2_t f2_fma(f2_t a, f2_t b, f2_t c) {
    f2_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2_t f2_mul(f2_t a, f2_t b) {
    f2_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2_t f2_add(f2_t a, f2_t b) {
    f2_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}

// Debug build (-DLAG_DEBUG_BOUNDS): trap if a corner gather of cell origin
// `idx` would leave the slice array (compute-sanitizer is unavailable here).
#ifdef LAG_DEBUG_BOUNDS
#define LAG_CHECK_GATHER(a, idx, live)                                                    \
    do {                                                                                  \
        const long long far_ = (long long)(idx) + 1 + (a).sx + (DIM == 3 ? (a).sxy : 0);  \
        if ((live) && ((idx) < 0 || far_ >= (a).slice_nodes)) __trap();                  \
    } while (0)
#else
#define LAG_CHECK_GATHER(a, idx, live) do { } while (0)
#endif

// number of corner pairs per slice: rows (2^(DIM-1)) x components (DIM)
template <int DIM> struct Pairs { static constexpr int n = (1 << (DIM - 1)) * DIM; };

// Gather the 2^DIM corners of local node idx (cell origin) into pairs:
// P[row * DIM + c] = {V(row, x0).c, V(row, x0 + 1).c}, row = dy + 2 dz.
template <int DIM>
__device__ __forceinline__ void gather_pairs(const float* __restrict__ v, int idx, int sx, int sxy,
                                             f2_t* P) {
    const float* p = v + DIM * idx;
#pragma unroll
    for (int r = 0; r < (1 << (DIM - 1)); ++r) {
        const int dy = r & 1, dz = r >> 1;
        const float* q = p + DIM * (dy * sx + dz * sxy);
        float e[2 * DIM];
#pragma unroll
        for (int k = 0; k < 2 * DIM; ++k) e[k] = __ldg(q + k);
#pragma unroll
        for (int c = 0; c < DIM; ++c) P[r * DIM + c] = f2_pack(e[c], e[DIM + c]);
    }
}

// Trilinear (bilinear) interpolation from the pair cache at fractions f.
template <int DIM>
__device__ __forceinline__ void interp_pairs(const f2_t* P, const float f[3], float out[3]) {
    const f2_t U = f2_pack(1.f - f[0], f[0]);            // x weights {1-fx, fx}
    constexpr int R = 1 << (DIM - 1);
    float wr[R];                                          // row weights
    if constexpr (DIM == 3) {
        const float uy = 1.f - f[1], uz = 1.f - f[2];
        wr[0] = uy * uz; wr[1] = f[1] * uz; wr[2] = uy * f[2]; wr[3] = f[1] * f[2];
    } else {
        wr[0] = 1.f - f[1]; wr[1] = f[1];
    }
    f2_t W[R];
#pragma unroll
    for (int r = 0; r < R; ++r) W[r] = f2_mul(U, f2_pack(wr[r], wr[r]));   // broadcast operand
#pragma unroll
    for (int c = 0; c < DIM; ++c) {
        f2_t acc = f2_mul(W[0], P[c]);
#pragma unroll
        for (int r = 1; r < R; ++r) acc = f2_fma(W[r], P[r * DIM + c], acc);
        float lo, hi;
        f2_unpack(acc, lo, hi);
        out[c] = lo + hi;
    }
    if constexpr (DIM == 2) out[2] = 0.f;
}

// "in the stage-1 cell": fs in [0, 1) on every axis.  Non-negative floats
// order like their bits and negatives have the sign bit, so one unsigned
// compare of the largest bit pattern decides (NaN and inf fail it too).
template <int DIM>
__device__ __forceinline__ bool in_unit_cell(const float fs[3]) {
    uint32_t m = max(__float_as_uint(fs[0]), __float_as_uint(fs[1]));
    if constexpr (DIM == 3) m = max(m, __float_as_uint(fs[2]));
    return m < 0x3F800000u;
}

// A stage sample that left the stage-1 cell (rare): its cell v1 + floor(fs),
// fractions, the fast-range test and, outside it, the full classification.
// Latches non-finite samples (non-finite velocity reached the particle).
template <int DIM, bool BTO, bool PASSES>
__device__ __forceinline__ int stage_moved(const AdvectArgs& a, const int v1[3], const float fs[3],
                                        uint8_t& st, bool& ghost_bad, uint32_t& errbits, float f[3],
                                        int shifted = 0) {
    int v[3] = {0, 0, 0};
    bool ok = true, finite = true;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        int tb;
        const float fl = floor_fma(fs[ax], tb);
        f[ax] = fs[ax] - fl;                                   // exact
        v[ax] = v1[ax] + (tb - kMagicBits);
        ok &= (unsigned)v[ax] <= (unsigned)a.gspan[ax];
        finite &= fabsf(fs[ax]) < 4194304.f;                   // 2^22 cells
    }
    if constexpr (DIM == 2) f[2] = 0.f;
    if (!finite) {
        errbits |= ERR_NONFINITE;
        st = ST_EXIT;
        return 0;
    }
    if (!ok) st = classify_slow_v<DIM, BTO>(a, v, f, ghost_bad);
    if constexpr (!BTO && PASSES) {
        // overlap pass 1 (LAG_XCHG_PEER_OVERLAP): the tile was judged
        // ghost-free from its stage-1 cells, which holds while samples stay
        // within one cell of them (CFL < 1); a farther sample may read ghost
        // nodes the exchange CTAs are writing: latched as a ghost error
        if (a.pass == 1) {
            // within one cell of the stage-1 cell the tile was judged by (the
            // frame is one cell below it on the axes of `shifted`, first cycle)
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) ghost_bad |= (unsigned)(v[ax] - v1[ax] + 1 - ((shifted >> ax) & 1)) > 2u;
        }
    }
    return vindex<DIM>(a, v);
}

// One stage s >= 2 of the RK4 step for the lane's particle: the sample
// fs = f1 + beta dt k (cell units from the stage-1 cell origin).  In the
// common case every lane's sample lies in its stage-1 cell and the corner
// cache holds that cell: nothing to do (one vote).  Otherwise the lanes that
// left the cell, or whose cache holds another cell, locate their sample and
// reload the cache (both slices for stages 2-3, v_t1 only for stage 4).
template <int DIM, bool BTO, bool FROZEN, bool PASSES, int SLICES>
__device__ __forceinline__ void stage_locate(const AdvectArgs& a, bool active, const int v1[3], int idx1,
                                             const float fs[3], int& cur, uint8_t& st, bool& ghost_bad,
                                             uint32_t& errbits, float f[3], f2_t* S, f2_t* B,
                                             int shifted = 0) {
    constexpr int NP = Pairs<DIM>::n;
    const bool same = in_unit_cell<DIM>(fs);
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) f[ax] = fs[ax];
    const bool need = active && st == ST_VALID && (!same || cur != idx1);
    if (__any_sync(0xffffffffu, need)) {
        if (need) {
            int idx = idx1;
            if (!same) idx = stage_moved<DIM, BTO, PASSES>(a, v1, fs, st, ghost_bad, errbits, f, shifted);
            LAG_CHECK_GATHER(a, idx, st == ST_VALID);
            if (st == ST_VALID && idx != cur) {
                if constexpr (SLICES == 2) {
                    gather_pairs<DIM>(a.v0, idx, a.sx, a.sxy, S);
                    if constexpr (FROZEN) {
#pragma unroll
                        for (int i = 0; i < NP; ++i) B[i] = S[i];
                    } else {
                        gather_pairs<DIM>(a.v1, idx, a.sx, a.sxy, B);
                    }
#pragma unroll
                    for (int i = 0; i < NP; ++i) S[i] = f2_add(S[i], B[i]);
                } else {
                    gather_pairs<DIM>(a.v1, idx, a.sx, a.sxy, B);
                }
                cur = idx;
            }
        }
    }
}

// Rare per-tile work after the update (warp-uniform branch): membership of
// the updated position for lanes outside the fast block range (BTO: TERM or
// EXIT; COMM: hand-off or EXIT), non-finite updates, compaction with holes,
// termination records and COMM hand-offs.  Returns the new live count.
template <int DIM, bool BTO>
__device__ __forceinline__ int tile_slow(const AdvectArgs& a, float4* trec, int lane, bool live, bool inblk,
                                      const int g[3], const float4 r, const float dn[3], uint8_t st,
                                      bool ghost_bad, uint32_t& errbits, uint32_t& nterm,
                                      uint32_t& nexit, uint32_t& nsent) {
    bool migrate = false;
    int nb = 0;
    if (live && st == ST_VALID) {
        bool finite = true;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) finite &= fabsf(dn[ax]) < 4194304.f;   // 2^22 cells
        if (!finite) {
            errbits |= ERR_NONFINITE;
            st = ST_EXIT;
        } else if (!inblk) {
            int cn[3] = {0, 0, 0};
            float fn[3] = {0.f, 0.f, 0.f};
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                int tb;
                const float fl = floor_fma(dn[ax], tb);
                fn[ax] = dn[ax] - fl;
                cn[ax] = g[ax] + (tb - kMagicBits);
            }
            bool gdummy = false;
            if constexpr (BTO) {
                st = classify_slow<DIM, true>(a, cn, fn, gdummy);
            } else {
                // COMM: in the domain but outside the block -> hand off
                bool out_dom = false;
                int mul = 1;
#pragma unroll
                for (int ax = 0; ax < DIM; ++ax) {
                    out_dom |= (cn[ax] < 0) | (cn[ax] > a.N[ax] - 1) |
                               ((cn[ax] == a.N[ax] - 1) & (fn[ax] != 0.f));
                    const int o = (cn[ax] < a.lo[ax]) ? -1
                                  : ((cn[ax] >= a.hi[ax] && a.hi[ax] < a.N[ax]) ? 1 : 0);
                    migrate |= (o != 0);
                    nb += (o + 1) * mul;
                    mul *= 3;
                }
                if constexpr (DIM == 2) nb += 9;     // offset index (ox+1) + 3(oy+1) + 9(oz+1), oz = 0
                if (out_dom) { st = ST_EXIT; migrate = false; }
            }
        }
    }
    if (live && ghost_bad) { errbits |= ERR_GHOST; if (st == ST_VALID) st = ST_EXIT; migrate = false; }

    const bool keep = live && st == ST_VALID && !migrate;
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
                a.dead_rec[s] = r;                   // pre-step position
                a.dead_info[s] = ((uint32_t)st << 24) | (uint32_t)(a.cycle & 0xffffff);
            } else {
                errbits |= ERR_OVERFLOW;
            }
        }
    }
    if (lane == 0) {
        nterm += __popc(tmask);
        nexit += __popc(dmask) - __popc(tmask);
    }
    return __popc(kmask);
}

// The advect loop over a virtual grid of `ncta` CTAs (this CTA = `cta`):
// advect_kernel runs it on the whole grid; the COMM overlap pass 1
// (advect_xchg_kernel, lag_api.cu) on the CTAs after its exchange CTAs.
// Persistent: warp w owns tiles w, w + W, w + 2W, ... (W = all warps), so the
// GPU sweeps the particle list as one compact window (L2-friendly).
//
// The common path is straight-line: every sample in its stage-1 cell, the
// updated position inside the block, every live particle kept.  Anything
// else (a cell change, a face, a termination, a hand-off) is detected by one
// warp vote and handled out of line (stage_locate, tile_slow).
// PASSES: the overlapped COMM transport's two passes (a.pass 1 / 2); every
// other launch advances every tile in one pass and compiles without them.
template <int DIM, bool BTO, bool FROZEN, bool PASSES = false>
__device__ __forceinline__ void advect_body(const AdvectArgs& a, const int cta, const int ncta) {
    constexpr int NP = Pairs<DIM>::n;
    const int lane = threadIdx.x & 31;
    const int warp = (cta * kThreads + threadIdx.x) >> 5;
    int n_tiles = a.n_tiles_dev ? *a.n_tiles_dev : a.n_tiles;
    // overlap passes (COMM): loop over virtual tile indices, map to real tiles
    int n_def = 0, n_b = 0;
    if constexpr (!BTO && PASSES) {
        if (a.pass == 1) {
            n_tiles = (int)*a.n_tiles_b;
        } else if (a.pass == 2) {
            n_def = (int)*a.defer_count;
            n_b = (int)*a.n_tiles_b;
            // the tile count is final for this cycle: the next cycle's pass 1
            // starts from it with an empty deferral list
            if (cta == 0 && threadIdx.x == 0) { *a.next_b = (uint32_t)n_tiles; *a.next_defer = 0u; }
            n_tiles = n_def + (n_tiles - n_b);
        }
    }
    auto real_tile = [&](int v) -> int {
        if constexpr (!BTO && PASSES) {
            if (a.pass == 2) return v < n_def ? (int)a.defer_list[v] : n_b + (v - n_def);
            // pass 1: the tiles next to a face come in runs (one x-run of a
            // brick: 16 consecutive tiles in 64), and the grid's warp count is
            // a multiple of 64, so a plain stride hands some warps only tiles
            // that are deferred; rotating each full chunk of 64 tiles by its
            // chunk index spreads them over all warps (a bijection; locality
            // stays within the chunk)
            if ((v | 63) < n_tiles) return (v & ~63) | (((v & 63) + (v >> 6)) & 63);
        }
        return v;
    };
    const int tstride = (ncta * kThreads) >> 5;

    uint32_t steps = 0, nterm = 0, nexit = 0, nsent = 0;  // per warp and launch: < 2^32
    uint32_t errbits = 0;

    // software pipeline: the next tile's count and record are in flight while
    // the current tile computes
    int tile = warp;                          // virtual index (== real outside overlap pass 2)
    int rtile = tile < n_tiles ? real_tile(tile) : 0;
    int cnt = tile < n_tiles ? a.tile_count[rtile] : 0;
    float4 r = tile < n_tiles ? a.state[(size_t)rtile * kTile + lane] : make_float4(0.f, 0.f, 0.f, 0.f);

    while (tile < n_tiles) {
        const int ntile = tile + tstride;
        const int nrtile = ntile < n_tiles ? real_tile(ntile) : 0;
        const int ncnt = ntile < n_tiles ? a.tile_count[nrtile] : 0;
        const float4 nr = ntile < n_tiles ? a.state[(size_t)nrtile * kTile + lane]
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        if (cnt == 0) { tile = ntile; rtile = nrtile; cnt = ncnt; r = nr; continue; }
        const bool live = lane < cnt;
        float4* trec = a.state + (size_t)rtile * kTile;
        const uint32_t w = __float_as_uint(r.w);
        const int g[3] = {(int)(w & a.mx), (int)((w >> a.bx) & a.my), DIM == 3 ? (int)(w >> (a.bx + a.by)) : 0};
        const float d[3] = {r.x, r.y, DIM == 3 ? r.z : 0.f};

        f2_t S[NP], B[NP];
        bool ghost_bad = false;
        uint8_t st = ST_VALID;

        // ---- stage 1: q1 = x (validated when committed) ----
        // gather offsets v = g + floor(d) - gmin; one unsigned compare per axis
        int v1c[3] = {0, 0, 0};
        float f1[3] = {0.f, 0.f, 0.f};
        bool ok1 = true;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
            int tb;
            const float fl = floor_fma(d[ax], tb);
            f1[ax] = d[ax] - fl;                             // exact
            v1c[ax] = g[ax] + tb - (a.gmin[ax] + kMagicBits);
            ok1 &= (unsigned)v1c[ax] <= (unsigned)a.gspan[ax];
        }
        if (__any_sync(0xffffffffu, live && !ok1)) {         // closed top face: clamp (rare)
            if (live && !ok1) classify_slow_v<DIM, BTO>(a, v1c, f1, ghost_bad);
        }
        if constexpr (!BTO && PASSES) {
            if (a.pass == 1) {                // a sample could reach a ghost node: after the exchange
                bool safe = true;
#pragma unroll
                for (int ax = 0; ax < DIM; ++ax) safe &= (unsigned)(v1c[ax] - a.smin[ax]) <= (unsigned)a.sspan[ax];
                if (__any_sync(0xffffffffu, live && !safe)) {
                    if (lane == 0) a.defer_list[atomicAdd(a.defer_count, 1u)] = (uint32_t)rtile;
                    tile = ntile; rtile = nrtile; cnt = ncnt; r = nr;
                    continue;
                }
            }
        }
        int idx1 = live ? vindex<DIM>(a, v1c) : 0;           // stage-1 cell origin (node index)
        LAG_CHECK_GATHER(a, idx1, live);
        int cur = idx1;                                      // cell held by the corner cache
        int shifted = 0;                                     // first cycle: axes framed one cell below
        float k1[3];
        if (a.cycle == 0 && __all_sync(0xffffffffu, !live || ((d[0] == 0.f) & (d[1] == 0.f) & (d[2] == 0.f)))) {
            // every particle sits on its seed node (first cycle of an interval;
            // later cycles do not test it: a particle at rest on a node takes
            // the general path, which handles f = 0 as well):
            // the trilinear value at a node is the node value (f = 0, or f = 1
            // on a clamped top face) — 3 loads; stage 2 gathers its own cell
            // (cur = -1 forces it)
            int node[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) node[ax] = v1c[ax] + (f1[ax] != 0.f ? 1 : 0);
            const float* pv = a.v0 + DIM * (live ? vindex<DIM>(a, node) : 0);
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) k1[ax] = __ldg(pv + ax);
            if constexpr (DIM == 2) k1[2] = 0.f;
            // the stage samples move along k1: on an axis where it is
            // negative they fall into the cell below the node, so take that
            // cell as the frame (f = 1, the same point) when it is a gather
            // cell; the samples then stay in one cell and no lane relocates
            // (overlap pass 1 still judges them against the unshifted cell)
            bool moved = false;
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                const bool down = (f1[ax] == 0.f) & (k1[ax] < 0.f) & (v1c[ax] > 0);
                v1c[ax] -= down ? 1 : 0;
                f1[ax] = down ? 1.f : f1[ax];
                moved |= down;
                shifted |= (down ? 1 : 0) << ax;
            }
            if (moved && live) idx1 = vindex<DIM>(a, v1c);
            cur = -1;
        } else {
            gather_pairs<DIM>(a.v0, idx1, a.sx, a.sxy, S);
            if constexpr (FROZEN) {
#pragma unroll
                for (int i = 0; i < NP; ++i) B[i] = S[i];
            } else {
                gather_pairs<DIM>(a.v1, idx1, a.sx, a.sxy, B);
            }
            interp_pairs<DIM>(S, f1, k1);
#pragma unroll
            for (int i = 0; i < NP; ++i) S[i] = f2_add(S[i], B[i]);   // S = v0 + v1 (stages 2, 3)
        }

        float e[3], f[3];
        // ---- stage 2: q2 = x + dt/2 k1, alpha = 1/2 ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = ax < DIM ? fmaf(a.hdth[ax], k1[ax], f1[ax]) : 0.f;
        stage_locate<DIM, BTO, FROZEN, PASSES, 2>(a, live, v1c, idx1, e, cur, st, ghost_bad, errbits, f, S, B, shifted);
        float T2[3];
        interp_pairs<DIM>(S, f, T2);                          // T2 = 2 k2

        // ---- stage 3: q3 = x + dt/2 k2 = x + dt/4 T2, alpha = 1/2 ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = ax < DIM ? fmaf(a.qdth[ax], T2[ax], f1[ax]) : 0.f;
        stage_locate<DIM, BTO, FROZEN, PASSES, 2>(a, live, v1c, idx1, e, cur, st, ghost_bad, errbits, f, S, B, shifted);
        float T3[3];
        interp_pairs<DIM>(S, f, T3);                          // T3 = 2 k3

        // ---- stage 4: q4 = x + dt k3 = x + dt/2 T3, alpha = 1 ----
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) e[ax] = ax < DIM ? fmaf(a.hdth[ax], T3[ax], f1[ax]) : 0.f;
        stage_locate<DIM, BTO, FROZEN, PASSES, 1>(a, live, v1c, idx1, e, cur, st, ghost_bad, errbits, f, S, B, shifted);
        float k4[3];
        interp_pairs<DIM>(B, f, k4);

        // ---- update: x' = x + dt/6 (k1 + 2k2 + 2k3 + k4) ----
        float dn[3];
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax)
            dn[ax] = fmaf(a.sdth[ax], (k1[ax] + k4[ax]) + (T2[ax] + T3[ax]), d[ax]);
        if constexpr (DIM == 2) dn[2] = 0.f;
        // membership of the updated position: g + floor(dn) in the fast block
        // range (non-finite or huge dn fails the compare too)
        bool inblk = true;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
            int tb;
            floor_fma(dn[ax], tb);
            inblk &= (unsigned)(g[ax] + tb - (a.bmin[ax] + kMagicBits)) <= (unsigned)a.bspan[ax];
        }

        // ---- particle management: compact survivors, record terminations ----
        const bool fast = live && st == ST_VALID && inblk && !ghost_bad;
        if (__all_sync(0xffffffffu, fast || !live)) {
            // every live particle kept: in place, the tile count is unchanged
            if (live) trec[lane] = make_float4(dn[0], dn[1], dn[2], r.w);
        } else {
            const int kept = tile_slow<DIM, BTO>(a, trec, lane, live, inblk, g, r, dn, st, ghost_bad, errbits,
                                                 nterm, nexit, nsent);
            if (lane == 0) a.tile_count[rtile] = (uint8_t)kept;
        }
        steps += (uint32_t)cnt;
        tile = ntile; rtile = nrtile; cnt = ncnt; r = nr;
    }

    // one atomic per warp per counter (no CTA barrier: finished warps retire)
    if (lane == 0 && steps) {
        atomicAdd(&a.counters[CNT_STEPS], (unsigned long long)steps);
        if (nterm) atomicAdd(&a.counters[CNT_TERM], (unsigned long long)nterm);
        if (nexit) atomicAdd(&a.counters[CNT_EXIT], (unsigned long long)nexit);
        if (nsent) atomicAdd(&a.counters[CNT_SENT], (unsigned long long)nsent);
    }
    errbits = __reduce_or_sync(0xffffffffu, errbits);
    if (lane == 0 && errbits) atomicOr(a.err, errbits);
}

template <int DIM, bool BTO, bool FROZEN, bool PASSES = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
advect_kernel(const AdvectArgs a) {
    // wait for the previous kernel (the exchange that appended to the lists),
    // then let the next one be scheduled: it takes the SMs this persistent
    // grid leaves in its tail.  Triggering only after the wait keeps every
    // kernel after the one two places before it (the next exchange must not
    // pack into the outbox parity the neighbour may still be pulling until
    // this cycle's exchange has seen the neighbour's signal).
    griddep_wait();
    griddep_launch();
    advect_body<DIM, BTO, FROZEN, PASSES>(a, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// seeding: lattice nodes g = first + stride * (ix, iy, iz).
// Tile order: bricks of (32 x by x bz) seeds, x fastest inside a tile, tiles
// of a brick consecutive (rows ry fastest, then rz), bricks x-fastest, so
// the warps sweeping consecutive tiles share node rows in L1/L2 (a row of
// nodes serves the particle rows on both sides of it).  Tiles past a ragged
// edge are partial or empty (count 0).  by = bz = 1 is plain x-fastest row
// order (2-D).
struct SeedArgs {
    float4* state;
    uint8_t* tile_count;
    uint32_t* n_tiles_word;         // COMM: device-side tile count to initialise (or nullptr)
    uint32_t* snap_b;               // COMM: the overlap transport's two tile-count snapshots
    uint32_t* snap_defer;           //       and two deferral counts (cycle parity)
    int64_t n_tiles;                // tiles of the brick layout (>= ceil(n / 32))
    int32_t first[3], stride, ns[3];
    int32_t by, bz;                 // brick rows (y, z) of 32-seed tiles
    uint32_t bx, by_bits;
};

// tile t -> seed lattice coordinates of its lane 0 (ix0, iy, iz)
__host__ __device__ inline void brick_tile(int64_t t, const int32_t ns[3], int by, int bz,
                                           int64_t& ix0, int64_t& iy, int64_t& iz) {
    const int64_t tb = (int64_t)by * bz;
    const int64_t brick = t / tb, j = t % tb;
    const int64_t nbx = (ns[0] + kTile - 1) / kTile, nby = (ns[1] + by - 1) / by;
    ix0 = (brick % nbx) * kTile;
    const int64_t r = brick / nbx;
    iy = (r % nby) * by + j % by;
    iz = (r / nby) * bz + j / by;
}

__host__ __device__ inline int64_t brick_tiles(const int32_t ns[3], int by, int bz) {
    const int64_t nbx = (ns[0] + kTile - 1) / kTile, nby = (ns[1] + by - 1) / by, nbz = (ns[2] + bz - 1) / bz;
    return nbx * nby * nbz * by * bz;
}

// One CTA per brick: grid (bricks in x, y, z), block (32 lanes, by rows,
// bz rows), so the tile and its lattice row follow from the indices without
// a division.
static __global__ void seed_kernel(const SeedArgs a) {
    const int lane = threadIdx.x, ry = threadIdx.y, rz = threadIdx.z;
    const int nbx = gridDim.x, nby = gridDim.y;
    const int brick = blockIdx.x + nbx * (blockIdx.y + nby * blockIdx.z);
    const int t = brick * (a.by * a.bz) + ry + a.by * rz;
    const int i = t * kTile + lane;              // 32-bit: tiles * 32 < 2^31 (lag_init bounds the slice)
    if (i == 0 && a.n_tiles_word) *a.n_tiles_word = (uint32_t)a.n_tiles;
    if (i == 0 && a.snap_b) {                  // overlap transport: either parity may come first
        a.snap_b[0] = a.snap_b[1] = (uint32_t)a.n_tiles;
        a.snap_defer[0] = a.snap_defer[1] = 0u;
    }
    const int ix0 = blockIdx.x * kTile;
    const int iy = blockIdx.y * a.by + ry;
    const int iz = blockIdx.z * a.bz + rz;
    const bool row = iy < a.ns[1] && iz < a.ns[2];
    const int cnt = row ? min(a.ns[0] - ix0, kTile) : 0;
    if (lane < cnt) {
        const uint32_t gx = (uint32_t)(a.first[0] + a.stride * (ix0 + lane));
        const uint32_t gy = (uint32_t)(a.first[1] + a.stride * iy);
        const uint32_t gz = (uint32_t)(a.first[2] + a.stride * iz);
        const uint32_t w = gx | (gy << a.bx) | (gz << (a.bx + a.by_bits));
        a.state[i] = make_float4(0.f, 0.f, 0.f, __uint_as_float(w));
    }
    if (lane == 0) a.tile_count[t] = (uint8_t)cnt;
}

// ---------------------------------------------------------------------------
// extraction: scatter live and terminated records to seed order (fp64 output)
struct ExtractArgs {
    const float4* state;
    const uint8_t* tile_count;
    int32_t n_tiles;
    const float4* dead_rec;
    const uint32_t* dead_info;
    const uint32_t* n_dead_dev;     // device-side count of termination records
    uint32_t dead_cap;
    const int32_t* n_tiles_dev;     // COMM: device-side tile count (nullptr: n_tiles)
    int64_t n;                      // seeds
    int32_t dim;
    int32_t first[3], stride, ns[3];
    uint32_t bx, by, mx, my;
    double o[3], h[3];
    int32_t lo[3], hi[3];           // own block: records seeded elsewhere are skipped (COMM)
    const float4* ret;              // COMM: records returned to this origin (32 B each:
    uint32_t n_ret;                 //        float4 record, u32 info, pad)
    double* start;                  // [n][dim]
    double* end;                    // [n][dim]
    uint8_t* status;                // [n]
    int32_t* term_cycle;            // [n] or nullptr: cycle of termination, -1 if valid
    int32_t write_start;            // scatter kernels write start (BTO); else extract_start_kernel
};

__device__ __forceinline__ bool own_seed(const ExtractArgs& a, uint32_t w) {
    const int g[3] = {(int)(w & a.mx), (int)((w >> a.bx) & a.my), (int)(w >> (a.bx + a.by))};
    bool in = true;
    for (int ax = 0; ax < 3; ++ax) in &= (g[ax] >= a.lo[ax]) & (g[ax] < a.hi[ax]);
    return in;
}

// Seed index (x fastest) of packed seed node w; 32-bit: n < 2^31 (lag_init).
__device__ __forceinline__ int seed_index(const ExtractArgs& a, uint32_t w, int g[3]) {
    g[0] = (int)(w & a.mx);
    g[1] = (int)((w >> a.bx) & a.my);
    g[2] = (int)(w >> (a.bx + a.by));
    int ix = g[0] - a.first[0], iy = g[1] - a.first[1], iz = g[2] - a.first[2];
    if (a.stride != 1) { ix /= a.stride; iy /= a.stride; iz /= a.stride; }
    return ix + a.ns[0] * (iy + a.ns[1] * iz);
}

// One basis flow in seed order: end = o + (g + d) h in fp64; start = o + g h
// when the scatter kernels cover every seed (BTO: each seed is live or dead);
// COMM writes starts with extract_start_kernel (hand-offs may be in flight
// on another rank when a slot overflowed).
template <int DIM>
__device__ __forceinline__ void write_flow(const ExtractArgs& a, int s, const int g[3], const float4 r,
                                           uint8_t status, int32_t tc) {
    const float d[3] = {r.x, r.y, r.z};
    const int64_t o = (int64_t)s * DIM;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        a.end[o + ax] = a.o[ax] + ((double)g[ax] + (double)d[ax]) * a.h[ax];
        if (a.write_start) a.start[o + ax] = a.o[ax] + (double)g[ax] * a.h[ax];
    }
    a.status[s] = status;
    if (a.term_cycle) a.term_cycle[s] = tc;
}

template <int DIM>
static __global__ void extract_start_kernel(const ExtractArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n) return;
    const int64_t idx[3] = {i % a.ns[0], (i / a.ns[0]) % a.ns[1], i / ((int64_t)a.ns[0] * a.ns[1])};
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax)
        a.start[i * DIM + ax] = a.o[ax] + (double)(a.first[ax] + a.stride * idx[ax]) * a.h[ax];
    if (a.term_cycle) a.term_cycle[i] = -1;
}

template <int DIM>
static __global__ void extract_live_kernel(const ExtractArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t tile = i / kTile;
    const int n_tiles = a.n_tiles_dev ? *a.n_tiles_dev : a.n_tiles;
    if (tile >= n_tiles) return;
    if ((int)(i % kTile) >= a.tile_count[tile]) return;
    const float4 r = a.state[i];
    if (!own_seed(a, __float_as_uint(r.w))) return;
    int g[3];
    const int s = seed_index(a, __float_as_uint(r.w), g);
    write_flow<DIM>(a, s, g, r, ST_VALID, -1);
}

template <int DIM>
static __global__ void extract_dead_kernel(const ExtractArgs a) {
    const uint32_t n_dead = min(*a.n_dead_dev, a.dead_cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_dead;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float4 r = a.dead_rec[i];
        if (!own_seed(a, __float_as_uint(r.w))) continue;
        int g[3];
        const int s = seed_index(a, __float_as_uint(r.w), g);
        const uint32_t info = a.dead_info[i];
        write_flow<DIM>(a, s, g, r, (uint8_t)(info >> 24), (int32_t)(info & 0xffffffu));
    }
}

template <int DIM>
static __global__ void extract_returned_kernel(const ExtractArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= a.n_ret) return;
    const float4 r = a.ret[2 * i];
    const uint32_t info = __float_as_uint(a.ret[2 * i + 1].x);
    int g[3];
    const int s = seed_index(a, __float_as_uint(r.w), g);
    const uint8_t st = (uint8_t)(info >> 24);
    write_flow<DIM>(a, s, g, r, st, st != ST_VALID ? (int32_t)(info & 0xffffffu) : -1);
}

}  // namespace lag
