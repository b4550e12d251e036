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
#ifndef LAG_ADV_THREADS
#define LAG_ADV_THREADS 128
#endif
#ifndef LAG_ADV_MINB
#define LAG_ADV_MINB 4
#endif
#ifndef LAG_ADV_TPW
#define LAG_ADV_TPW 4
#endif
constexpr int kThreads = LAG_ADV_THREADS;     // advect CTA size
constexpr int kMinBlocks = LAG_ADV_MINB;      // __launch_bounds__ min CTAs per SM
constexpr int kTilesPerWarp = LAG_ADV_TPW;    // contiguous 32-particle tiles per warp
#ifndef LAG_ADV_PERSIST
#define LAG_ADV_PERSIST 1
#endif
#ifndef LAG_PREFETCH
#define LAG_PREFETCH 0   // 1: L2, 2: L1 prefetch of the next tile's stage-1 corner rows
#endif
#ifndef LAG_POLY
#define LAG_POLY 0       // 1: polynomial-form trilinear (coefficients per corner set)
#endif

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
    int32_t tiles_per_warp;         // contiguous tiles per warp (non-persistent grid)
    // COMM: outgoing slots, one per neighbour offset (3^dim):
    // slot k = slot_rec[slot_base[k]] = header (u32 count) then slot_capv[k] records
    float4* slot_rec;
    int32_t slot_base[27];
    int32_t slot_capv[27];
    float4* slot_ptr[27];           // slot of offset k: local (NCCL) or the owner's inbox (peer)
    // peer transport: the last warp to retire signals "particles of cycle
    // sig_value ready" into each neighbour's flag word
    unsigned long long* sig_flag[26];
    int32_t n_sig;
    unsigned long long sig_value;
    uint32_t* done_warps;
    // COMM exchange overlap (LAG_XCHG_PEER_OVERLAP): pass 1 advects tiles
    // [0, *n_tiles_b) whose stage samples cannot reach a ghost node and defers
    // the others; pass 2 advects the deferred tiles and the tiles appended by
    // this cycle's exchange.  pass 0: every tile.
    int32_t pass;
    const uint32_t* n_tiles_b;      // tile count before this cycle's append
    uint32_t* defer_list;
    uint32_t* defer_count;
    int32_t smin[3], sspan[3];      // ghost-free cells (gather offsets): samples stay off ghost nodes
#ifdef LAG_EXP_TIMELINE
    unsigned long long* tl;         // experiment: per-cycle globaltimer stamps [64][8]
#endif
};

#ifdef LAG_EXP_TIMELINE
__device__ __forceinline__ unsigned long long lag_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

__device__ __forceinline__ void unpack_g(uint32_t w, const AdvectArgs& a, int g[3]) {
    g[0] = (int)(w & a.mx);
    g[1] = (int)((w >> a.bx) & a.my);
    g[2] = (int)(w >> (a.bx + a.by));
}

// Corner gather: the 2^DIM corners of local cell li, DIM components each, AoS.
// C layout: [(dz*2 + dy)*2 + dx][comp].
template <int DIM>
__device__ __forceinline__ void gather(const float* __restrict__ v, const int li[3],
                                       int sx, int sxy, float* C) {
    if constexpr (DIM == 3) {
        const float* p = v + 3 * (li[0] + sx * li[1] + sxy * li[2]);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int dy = r & 1, dz = r >> 1;
            const float* q = p + 3 * (dy * sx + dz * sxy);
#pragma unroll
            for (int e = 0; e < 6; ++e) C[r * 6 + e] = __ldg(q + e);
        }
    } else {
        const float* p = v + 2 * (li[0] + sx * li[1]);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float* q = p + 2 * (r * sx);
#pragma unroll
            for (int e = 0; e < 4; ++e) C[r * 4 + e] = __ldg(q + e);
        }
    }
}

// Multilinear interpolation inside one cell with fractional offsets f
// (two partial sums per component for ILP).
template <int DIM>
__device__ __forceinline__ void interp(const float* C, const float f[3], float out[3]) {
    if constexpr (DIM == 3) {
        const float ux = 1.f - f[0], uy = 1.f - f[1], uz = 1.f - f[2];
        float w[8];
        const float w00 = uy * uz, w10 = f[1] * uz, w01 = uy * f[2], w11 = f[1] * f[2];
        w[0] = ux * w00; w[1] = f[0] * w00;
        w[2] = ux * w10; w[3] = f[0] * w10;
        w[4] = ux * w01; w[5] = f[0] * w01;
        w[6] = ux * w11; w[7] = f[0] * w11;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            float s0 = w[0] * C[c], s1 = w[1] * C[3 + c];
#pragma unroll
            for (int k = 2; k < 8; k += 2) {
                s0 = fmaf(w[k], C[k * 3 + c], s0);
                s1 = fmaf(w[k + 1], C[(k + 1) * 3 + c], s1);
            }
            out[c] = s0 + s1;
        }
    } else {
        const float ux = 1.f - f[0], uy = 1.f - f[1];
        float w[4] = {ux * uy, f[0] * uy, ux * f[1], f[0] * f[1]};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            float s = w[0] * C[c];
#pragma unroll
            for (int k = 1; k < 4; ++k) s = fmaf(w[k], C[k * 2 + c], s);
            out[c] = s;
        }
        out[2] = 0.f;
    }
}

// Trilinear polynomial form of one cell's corners (in place, per component):
//   Tri(f) = p0 + fx (px + fy (pxy + fz pxyz) + fz pxz) + fy (py + fz pyz) + fz pz
// Built once per gathered corner set (off the stage-to-stage critical path);
// each evaluation is then 7 FFMA per component with a 4-deep chain.  Linear
// in the corner values, so coefficients of v_t + v_t1 are the sums.
template <int DIM>
__device__ __forceinline__ void to_poly(float* C) {
    if constexpr (!LAG_POLY) return;
    if constexpr (DIM == 3) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float v000 = C[0 * 3 + c], v100 = C[1 * 3 + c], v010 = C[2 * 3 + c], v110 = C[3 * 3 + c];
            const float v001 = C[4 * 3 + c], v101 = C[5 * 3 + c], v011 = C[6 * 3 + c], v111 = C[7 * 3 + c];
            const float px = v100 - v000, py = v010 - v000, pz = v001 - v000;
            const float d1 = v110 - v010, d2 = v101 - v001, d3 = v011 - v001, d4 = v111 - v011;
            const float pxy = d1 - px;
            C[0 * 3 + c] = v000;
            C[1 * 3 + c] = px;
            C[2 * 3 + c] = py;
            C[3 * 3 + c] = pxy;
            C[4 * 3 + c] = pz;
            C[5 * 3 + c] = d2 - px;              // pxz
            C[6 * 3 + c] = d3 - py;              // pyz
            C[7 * 3 + c] = (d4 - d2) - pxy;      // pxyz
        }
    } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float v00 = C[0 * 2 + c], v10 = C[1 * 2 + c], v01 = C[2 * 2 + c], v11 = C[3 * 2 + c];
            const float px = v10 - v00, py = v01 - v00;
            C[1 * 2 + c] = px;
            C[2 * 2 + c] = py;
            C[3 * 2 + c] = (v11 - v01) - px;     // pxy
        }
    }
}

template <int DIM>
__device__ __forceinline__ void interp(const float* C, const float f[3], float out[3]);

template <int DIM>
__device__ __forceinline__ void poly_eval(const float* P, const float f[3], float out[3]) {
    if constexpr (!LAG_POLY) { interp<DIM>(P, f, out); return; }
    if constexpr (DIM == 3) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float a = fmaf(f[2], P[7 * 3 + c], P[3 * 3 + c]);   // pxy + fz pxyz
            float b = fmaf(f[1], a, P[1 * 3 + c]);                    // px + fy (...)
            b = fmaf(f[2], P[5 * 3 + c], b);                          //    + fz pxz
            const float t = fmaf(f[2], P[6 * 3 + c], P[2 * 3 + c]);   // py + fz pyz
            float r = fmaf(f[2], P[4 * 3 + c], P[0 * 3 + c]);         // p0 + fz pz
            r = fmaf(f[1], t, r);
            out[c] = fmaf(f[0], b, r);
        }
    } else {
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const float b = fmaf(f[1], P[3 * 2 + c], P[1 * 2 + c]);   // px + fy pxy
            const float r = fmaf(f[1], P[2 * 2 + c], P[0 * 2 + c]);   // p0 + fy py
            out[c] = fmaf(f[0], b, r);
        }
        out[2] = 0.f;
    }
}

// Cell of a stage sample e (displacement from g, cell units):
// c = g + floor(e), f = e - floor(e) (exact).  Fast path: every axis inside
// the range [lo_, lo_ + span_] (one unsigned compare per axis).
// floor(e) on the FMA pipe (no FRND): for |e| < 2^22, e + 1.5*2^23 rounded
// toward -inf is 1.5*2^23 + floor(e) exactly, so its bits hold floor(e) in
// the low mantissa (bits - 0x4B400000 = floor(e)) and t - 1.5*2^23 is floor(e).
__device__ __forceinline__ float floor_fma(float e, int& bits) {
    const float t = __fadd_rd(e, 12582912.0f);
    bits = __float_as_int(t);
    return t - 12582912.0f;
}

template <int DIM>
__device__ __forceinline__ bool cells(const int g[3], const float e[3], const int32_t* rmin,
                                      const int32_t* rspan, int c[3], float f[3]) {
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        int tb;
        const float fl = floor_fma(e[ax], tb);
        f[ax] = e[ax] - fl;                              // exact
        c[ax] = g[ax] + (tb - 0x4B400000);
        ok &= (unsigned)(c[ax] - rmin[ax]) <= (unsigned)rspan[ax];
    }
    if constexpr (DIM == 2) { c[2] = 0; f[2] = 0.f; }
    return ok;
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

// Biased form used on the hot path: gb = g - rmin - bits(1.5*2^23) per
// axis (per particle, once), so v = c - rmin is one add of the floor's float
// bits and the range test one unsigned compare.
constexpr int kMagicBits = 0x4B400000;    // bits of 12582912.0f = 1.5 * 2^23
template <int DIM>
__device__ __forceinline__ bool cells_b(const int gb[3], const float e[3], const int32_t* rspan,
                                        int v[3], float f[3]) {
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        int tb;
        const float fl = floor_fma(e[ax], tb);
        f[ax] = e[ax] - fl;                              // exact
        v[ax] = gb[ax] + tb;                             // = c - rmin (|e| < 2^22)
        ok &= (unsigned)v[ax] <= (unsigned)rspan[ax];
    }
    if constexpr (DIM == 2) { v[2] = 0; f[2] = 0.f; }
    return ok;
}

// Node index (local slice coordinates) of the cell with gather offsets v.
template <int DIM>
__device__ __forceinline__ int vindex(const AdvectArgs& a, const int v[3]) {
    if constexpr (DIM == 3) return v[0] + a.sx * v[1] + a.sxy * v[2] + a.gidx0;
    else return v[0] + a.sx * v[1] + a.gidx0;
}

// Slow path on gather offsets: convert to cells, classify, convert back.
template <int DIM, bool BTO>
__device__ __forceinline__ uint8_t classify_slow_v(const AdvectArgs& a, int v[3], float f[3],
                                                   bool& ghost_bad);

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

// Stage sample s >= 2 relative to the stage-1 cell: fs = f1 + beta dt k (cell
// units from the stage-1 cell origin).  fs in [0, 1) on every axis (one
// unsigned compare of the float bits per axis: negatives have the sign bit)
// means the stage-1 cell, which the committed position already validated, so
// nothing else is tested.  Otherwise the sample's cell v1 + floor(fs) takes
// the fast-range test and, outside it, the full classification.  Returns the
// node index of the cell to interpolate in (f = fractions inside it).
template <int DIM, bool BTO>
__device__ __forceinline__ int stage_cell(const AdvectArgs& a, const int v1[3], int idx1,
                                          const float fs[3], bool test, uint8_t& st,
                                          bool& ghost_bad, float f[3]) {
    bool same = true;
#pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        f[ax] = fs[ax];
        same &= __float_as_uint(fs[ax]) < 0x3F800000u;
    }
    if constexpr (DIM == 2) f[2] = 0.f;
    int idx = idx1;
    if (!same && test) {
        int v[3];
        bool ok = true;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
            int tb;
            const float fl = floor_fma(fs[ax], tb);
            f[ax] = fs[ax] - fl;                                   // exact
            v[ax] = v1[ax] + (tb - 0x4B400000);
            ok &= (unsigned)v[ax] <= (unsigned)a.gspan[ax];
        }
        if constexpr (DIM == 2) v[2] = 0;
        if (!ok) st = classify_slow_v<DIM, BTO>(a, v, f, ghost_bad);
        idx = vindex<DIM>(a, v);
    }
    return idx;
}

template <int DIM>
__device__ __forceinline__ int node_index(const AdvectArgs& a, const int c[3]) {
    const int lx = c[0] - a.base[0], ly = c[1] - a.base[1];
    if constexpr (DIM == 3) return lx + a.sx * ly + a.sxy * (c[2] - a.base[2]);
    else return lx + a.sx * ly;
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
#ifdef LAG_EXP_NOLOAD   // timing experiment: synthetic corners, no velocity traffic
#pragma unroll
    for (int i = 0; i < Pairs<DIM>::n; ++i)
        P[i] = f2_pack(__int_as_float(idx + i) * 1e-30f, __int_as_float(idx - i) * 1e-30f);
    return;
#endif
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

// Corner gather by linear node index (see gather()).
template <int DIM>
__device__ __forceinline__ void gather_idx(const float* __restrict__ v, int idx, int sx, int sxy,
                                           float* C) {
#ifdef LAG_EXP_NOLOAD   // timing experiment: synthetic corners, no velocity traffic
#pragma unroll
    for (int i = 0; i < (1 << DIM) * DIM; ++i) C[i] = __int_as_float(idx + i) * 1e-30f;
    return;
#endif
    if constexpr (DIM == 3) {
        const float* p = v + 3 * idx;
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const int dy = r & 1, dz = r >> 1;
            const float* q = p + 3 * (dy * sx + dz * sxy);
#pragma unroll
            for (int e = 0; e < 6; ++e) C[r * 6 + e] = __ldg(q + e);
        }
    } else {
        const float* p = v + 2 * idx;
#pragma unroll
        for (int r = 0; r < 2; ++r) {
            const float* q = p + 2 * (r * sx);
#pragma unroll
            for (int e = 0; e < 4; ++e) C[r * 4 + e] = __ldg(q + e);
        }
    }
}

// The advect loop over a virtual grid of `ncta` CTAs (this CTA = `cta`):
// advect_kernel runs it on the whole grid; the COMM overlap pass 1
// (advect_xchg_kernel, lag_api.cu) on the CTAs after its exchange CTAs.
template <int DIM, bool BTO, bool FROZEN>
__device__ __forceinline__ void advect_body(const AdvectArgs& a, const int cta, const int ncta) {
    constexpr int NC = (1 << DIM) * DIM;             // corner floats per slice
    const int lane = threadIdx.x & 31;
    const int warp = (cta * kThreads + threadIdx.x) >> 5;
    int n_tiles_all = a.n_tiles_dev ? *a.n_tiles_dev : a.n_tiles;
    // overlap passes (COMM): loop over virtual tile indices, map to real tiles
    int n_def = 0, n_b = 0;
    if constexpr (!BTO) {
        if (a.pass == 1) {
            n_tiles_all = (int)*a.n_tiles_b;
        } else if (a.pass == 2) {
            n_def = (int)*a.defer_count;
            n_b = (int)*a.n_tiles_b;
            n_tiles_all = n_def + (n_tiles_all - n_b);
        }
    }
    auto real_tile = [&](int v) -> int {
        if constexpr (!BTO) {
            if (a.pass == 2) return v < n_def ? (int)a.defer_list[v] : n_b + (v - n_def);
        }
        return v;
    };
    // non-persistent grid: warp w owns tiles [w*tpw, (w+1)*tpw) (contiguous, so
    // a CTA's particles are spatial neighbours); the block scheduler balances
    // the load across SMs
#if LAG_ADV_PERSIST
    // persistent grid: warp w owns tiles w, w + W, w + 2W, ... (W = all warps),
    // so the GPU sweeps the particle list as one compact window
    const int tile0 = warp;
    const int tstride = (ncta * kThreads) >> 5;
    const int n_tiles = n_tiles_all;
#else
    const int tile0 = warp * a.tiles_per_warp;
    const int tstride = 1;
    const int n_tiles = min(n_tiles_all, tile0 + a.tiles_per_warp);
#endif

    uint32_t steps = 0, nterm = 0, nexit = 0, nsent = 0;  // per warp and launch: < 2^32
    uint32_t errbits = 0;
    bool did_remote = false;
#ifdef LAG_EXP_TIMELINE
    if (a.tl && cta == 0 && threadIdx.x == 0) a.tl[(a.sig_value & 63) * 8 + 6] = lag_gtimer();
#endif

    // software pipeline: the next tile's count and records are in flight while
    // the current tile computes
    int tile = tile0;                         // virtual index (== real outside overlap pass 2)
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
        int g[3];
        unpack_g(__float_as_uint(r.w), a, g);
        const float d[3] = {r.x, r.y, DIM == 3 ? r.z : 0.f};

        constexpr int NP = Pairs<DIM>::n;
        f2_t S[NP], B[NP];
        int c[3];
        float f[3], e[3];
        bool ghost_bad = false;
        uint8_t st = ST_VALID;

        // ---- stage 1: q1 = x (validated when committed) ----
        int gb[3];                            // g - gmin - magic (see cells_b)
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) gb[ax] = g[ax] - a.gmin[ax] - kMagicBits;
        if (!cells_b<DIM>(gb, d, a.gspan, c, f) && live)
            classify_slow_v<DIM, BTO>(a, c, f, ghost_bad);   // top-face clamp only
        if constexpr (!BTO) {
            if (a.pass == 1) {                // a sample could reach a ghost node: after the exchange
                bool safe = true;
#pragma unroll
                for (int ax = 0; ax < DIM; ++ax) safe &= (unsigned)(c[ax] - a.smin[ax]) <= (unsigned)a.sspan[ax];
                if (__any_sync(0xffffffffu, live && !safe)) {
                    if (lane == 0) a.defer_list[atomicAdd(a.defer_count, 1u)] = (uint32_t)rtile;
                    tile = ntile; rtile = nrtile; cnt = ncnt; r = nr;
                    continue;
                }
            }
        }
        int cur = vindex<DIM>(a, c);
        LAG_CHECK_GATHER(a, cur, live);
        if (!live) cur = 0;
        const int idx1 = cur;                 // stage-1 cell: offsets, fractions
        const int v1c[3] = {c[0], c[1], c[2]};
        const float f1[3] = {f[0], f[1], f[2]};
        float k1[3];
        if (__all_sync(0xffffffffu, !live || ((d[0] == 0.f) & (d[1] == 0.f) & (d[2] == 0.f)))) {
            // every particle sits on its seed node (first cycle of an interval):
            // the trilinear value at a node is the node value (f = 0, or f = 1
            // on a clamped top face) — 3 loads; the stage-2 sample gathers its
            // own cell (cur = -1 forces it)
            int node[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) node[ax] = c[ax] + (f[ax] != 0.f ? 1 : 0);
            const float* pv = a.v0 + DIM * (live ? vindex<DIM>(a, node) : 0);
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) k1[ax] = __ldg(pv + ax);
            if constexpr (DIM == 2) k1[2] = 0.f;
            cur = -1;
#pragma unroll
            for (int i = 0; i < NP; ++i) S[i] = B[i] = 0ull;   // lanes stopped at stage 2 stay finite
        } else {
            gather_pairs<DIM>(a.v0, cur, a.sx, a.sxy, S);
            if constexpr (FROZEN) {
#pragma unroll
                for (int i = 0; i < NP; ++i) B[i] = S[i];
            } else {
                gather_pairs<DIM>(a.v1, cur, a.sx, a.sxy, B);
            }
            interp_pairs<DIM>(S, f, k1);
#pragma unroll
            for (int i = 0; i < NP; ++i) S[i] = f2_add(S[i], B[i]);   // S = v0 + v1 (stages 2, 3)
        }

        // ---- stage 2: q2 = x + dt/2 k1, alpha = 1/2 ----
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) e[ax] = fmaf(a.hdth[ax], k1[ax], f1[ax]);
        {
            const int idx = stage_cell<DIM, BTO>(a, v1c, idx1, e, live, st, ghost_bad, f);
            LAG_CHECK_GATHER(a, idx, live && st == ST_VALID);
#ifdef LAG_EXP_NORELOAD
            if (false) {
#else
            if (live && st == ST_VALID && idx != cur) {
#endif
                gather_pairs<DIM>(a.v0, idx, a.sx, a.sxy, S);
                if constexpr (FROZEN) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) B[i] = S[i];
                } else {
                    gather_pairs<DIM>(a.v1, idx, a.sx, a.sxy, B);
                }
#pragma unroll
                for (int i = 0; i < NP; ++i) S[i] = f2_add(S[i], B[i]);
                cur = idx;
            }
        }
        float T2[3];
        interp_pairs<DIM>(S, f, T2);                          // T2 = 2 k2
#if LAG_PREFETCH
        // the next tile's stage-1 corner rows (its record arrived by now): one
        // prefetch per row and slice, so its gathers hit the cache
        if (ntile < n_tiles && lane < ncnt) {
            int gn[3];
            unpack_g(__float_as_uint(nr.w), a, gn);
            const float dn0[3] = {nr.x, nr.y, DIM == 3 ? nr.z : 0.f};
            int vn[3];
            bool okn = true;
#pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                vn[ax] = gn[ax] - a.gmin[ax] + (__float_as_int(floorf(dn0[ax]) + 12582912.0f) - kMagicBits);
                okn &= (unsigned)vn[ax] <= (unsigned)a.gspan[ax];
            }
            if constexpr (DIM == 2) vn[2] = 0;
            if (okn) {
                const int in = vindex<DIM>(a, vn);
#pragma unroll
                for (int r = 0; r < (1 << (DIM - 1)); ++r) {
                    const int o = DIM * (in + (r & 1) * a.sx + (r >> 1) * a.sxy);
#if LAG_PREFETCH == 1
                    asm volatile("prefetch.global.L2 [%0];" :: "l"(a.v0 + o));
                    if constexpr (!FROZEN) asm volatile("prefetch.global.L2 [%0];" :: "l"(a.v1 + o));
#else
                    asm volatile("prefetch.global.L1 [%0];" :: "l"(a.v0 + o));
                    if constexpr (!FROZEN) asm volatile("prefetch.global.L1 [%0];" :: "l"(a.v1 + o));
#endif
                }
            }
        }
#endif

        // ---- stage 3: q3 = x + dt/2 k2 = x + dt/4 T2, alpha = 1/2 ----
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) e[ax] = fmaf(a.qdth[ax], T2[ax], f1[ax]);
        {
            const int idx = stage_cell<DIM, BTO>(a, v1c, idx1, e, live && st == ST_VALID, st, ghost_bad, f);
            LAG_CHECK_GATHER(a, idx, live && st == ST_VALID);
#ifdef LAG_EXP_NORELOAD
            if (false) {
#else
            if (live && st == ST_VALID && idx != cur) {
#endif
                gather_pairs<DIM>(a.v0, idx, a.sx, a.sxy, S);
                if constexpr (FROZEN) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) B[i] = S[i];
                } else {
                    gather_pairs<DIM>(a.v1, idx, a.sx, a.sxy, B);
                }
#pragma unroll
                for (int i = 0; i < NP; ++i) S[i] = f2_add(S[i], B[i]);
                cur = idx;
            }
        }
        float T3[3];
        interp_pairs<DIM>(S, f, T3);                          // T3 = 2 k3

        // ---- stage 4: q4 = x + dt k3 = x + dt/2 T3, alpha = 1 ----
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) e[ax] = fmaf(a.hdth[ax], T3[ax], f1[ax]);
        {
            const int idx = stage_cell<DIM, BTO>(a, v1c, idx1, e, live && st == ST_VALID, st, ghost_bad, f);
            LAG_CHECK_GATHER(a, idx, live && st == ST_VALID);
#ifndef LAG_EXP_NORELOAD
            if (live && st == ST_VALID && idx != cur) {
                gather_pairs<DIM>(a.v1, idx, a.sx, a.sxy, B);
            }
#endif
        }
        float k4[3];
        interp_pairs<DIM>(B, f, k4);

        // ---- update: x' = x + dt/6 (k1 + 2k2 + 2k3 + k4) ----
        float dn[3];
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax)
            dn[ax] = fmaf(a.sdth[ax], (k1[ax] + k4[ax]) + (T2[ax] + T3[ax]), d[ax]);
        if constexpr (DIM == 2) dn[2] = 0.f;
        bool finite = true;
#pragma unroll
        for (int ax = 0; ax < DIM; ++ax) finite &= fabsf(dn[ax]) < 4194304.f;   // 2^22 cells
        // membership of the updated position: fast = inside the block
        bool migrate = false;
        int nb = 0;
        {
            int cn[3];
            float fn[3];
            int gbb[3];                       // g - bmin - magic
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) gbb[ax] = BTO ? gb[ax] : g[ax] - a.bmin[ax] - kMagicBits;
            const bool inblk = cells_b<DIM>(gbb, dn, a.bspan, cn, fn);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) cn[ax] += a.bmin[ax];         // back to cells (slow path)
            if (!inblk && live && st == ST_VALID) {
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
        if (live && !finite) { errbits |= ERR_NONFINITE; st = ST_EXIT; migrate = false; }
        if (live && ghost_bad) { errbits |= ERR_GHOST; if (st == ST_VALID) st = ST_EXIT; migrate = false; }

        // ---- particle management: compact survivors, record terminations ----
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
                    a.dead_rec[s] = r;                   // pre-step position
                    a.dead_info[s] = ((uint32_t)st << 24) | (uint32_t)(a.cycle & 0xffffff);
                } else {
                    errbits |= ERR_OVERFLOW;
                }
            }
        }
        if (lane == 0) {
            a.tile_count[rtile] = (uint8_t)__popc(kmask);
            steps += (uint32_t)cnt;
            nterm += __popc(tmask);
            nexit += __popc(dmask) - __popc(tmask);
        }
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
    if constexpr (!BTO) {
        if (a.n_sig) {
            if (did_remote) __threadfence_system();          // my remote hand-offs are performed
            __syncwarp();
            if (lane == 0) {
                const uint32_t total = (ncta * kThreads) >> 5;
                if (atomicAdd(a.done_warps, 1u) == total - 1) {  // last warp of the grid
                    *a.done_warps = 0u;
#ifdef LAG_EXP_TIMELINE
                    if (a.tl) a.tl[(a.sig_value & 63) * 8 + 7] = lag_gtimer();
#endif
                    __threadfence_system();
                    for (int k = 0; k < a.n_sig; ++k)
                        *reinterpret_cast<volatile unsigned long long*>(a.sig_flag[k]) = a.sig_value;
                    __threadfence_system();
                }
            }
        }
    }
}

template <int DIM, bool BTO, bool FROZEN>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
advect_kernel(const AdvectArgs a) {
    advect_body<DIM, BTO, FROZEN>(a, blockIdx.x, gridDim.x);
}

// ---------------------------------------------------------------------------
// seeding: lattice nodes g = first + stride * (ix, iy, iz).
// Tile order: bricks of (32 x by x bz) seeds, x fastest inside a tile, tiles
// of a brick consecutive (rows ry fastest, then rz), bricks x-fastest.  A CTA
// of by*bz warps then advects one brick at a time, so the node rows its
// corner gathers share stay in that SM's L1 (a row of nodes serves the
// particle rows on both sides of it).  Tiles past a ragged edge are partial
// or empty (count 0).  by = bz = 1 is plain x-fastest row order.
#ifndef LAG_BRICK_Y
#define LAG_BRICK_Y 1
#endif
#ifndef LAG_BRICK_Z
#define LAG_BRICK_Z 1
#endif
struct SeedArgs {
    float4* state;
    uint8_t* tile_count;
    uint32_t* n_tiles_word;         // COMM: device-side tile count to initialise (or nullptr)
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

static __global__ void seed_kernel(const SeedArgs a) {
    // 32-bit index math: tiles * 32 < 2^31 (lag_init bounds the slice)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && a.n_tiles_word) *a.n_tiles_word = (uint32_t)a.n_tiles;
    if (i >= (int)a.n_tiles * kTile) return;
    const int t = i >> 5, lane = i & 31;
    const int tb = a.by * a.bz;
    const int brick = t / tb, j = t - brick * tb;
    const int nbx = (a.ns[0] + kTile - 1) / kTile, nby = (a.ns[1] + a.by - 1) / a.by;
    const int bq = brick / nbx;
    const int ix0 = (brick - bq * nbx) * kTile;
    const int jz = j / a.by;
    const int iy = (bq % nby) * a.by + (j - jz * a.by);
    const int iz = (bq / nby) * a.bz + jz;
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
