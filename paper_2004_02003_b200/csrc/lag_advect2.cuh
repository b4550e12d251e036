// lag_advect2.cuh — advect_kernel with NPT tiles per warp advanced together
// (3-D, two slices).  Same method, records, compaction and counters as
// advect_kernel (lag_kernels.cuh; §3.1): every lane
// carries NPT independent particles (one from each of NPT adjacent tiles)
// through the RK4 stages in lock step, so the stage-1 gathers of all of them
// are in flight together and their interpolation chains interleave.  The
// per-thread state that does not depend on the particle (parameters,
// pointers, counters, loop state) is paid once per NPT particles, which
// is what buys more particle streams per SM than NPT separate warps.
#pragma once
#include "lag_kernels.cuh"

namespace lag {

#ifndef LAG_NPT
#define LAG_NPT 2
#endif
#ifndef LAG_ADV2_MINB
#define LAG_ADV2_MINB 3
#endif
constexpr int kNpt = LAG_NPT;
constexpr int kAdv2MinBlocks = LAG_ADV2_MINB;     // CTAs of kThreads per SM

template <bool BTO>
__global__ void __launch_bounds__(kThreads, kAdv2MinBlocks)
advect2_kernel(const AdvectArgs a) {
    constexpr int NP = Pairs<3>::n;                  // 12 corner pairs per slice
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * kThreads + threadIdx.x) >> 5;
    const int n_tiles = a.n_tiles_dev ? *a.n_tiles_dev : a.n_tiles;
    const int n_groups = (n_tiles + kNpt - 1) / kNpt;
    const int gstride = (gridDim.x * kThreads) >> 5;

    unsigned long long steps = 0, nterm = 0, nexit = 0, nsent = 0;
    uint32_t errbits = 0;
    bool did_remote = false;

    // group q = tiles q*NPT .. q*NPT + NPT-1 (adjacent rows of a seed brick)
    int grp = warp;
    int cnt[kNpt];
    float4 r[kNpt];
#pragma unroll
    for (int p = 0; p < kNpt; ++p) {
        const int t = grp * kNpt + p;
        cnt[p] = grp < n_groups && t < n_tiles ? a.tile_count[t] : 0;
        r[p] = grp < n_groups && t < n_tiles ? a.state[(size_t)t * kTile + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
    }

    while (grp < n_groups) {
        const int ngrp = grp + gstride;
        int ncnt[kNpt];
        float4 nr[kNpt];
#pragma unroll
        for (int p = 0; p < kNpt; ++p) {
            const int t = ngrp * kNpt + p;
            ncnt[p] = ngrp < n_groups && t < n_tiles ? a.tile_count[t] : 0;
            nr[p] = ngrp < n_groups && t < n_tiles ? a.state[(size_t)t * kTile + lane]
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        bool live[kNpt];
        int g[kNpt][3];
        float d[kNpt][3];
        uint8_t st[kNpt];
        bool ghost_bad[kNpt];
        f2_t S[kNpt][NP], B[kNpt][NP];
        int gb[kNpt][3], v1c[kNpt][3], idx1[kNpt], cur[kNpt];
        float f1[kNpt][3];
        float k1[kNpt][3], T2[kNpt][3], T3[kNpt][3], k4[kNpt][3];

        // ---- stage 1: q1 = x ----
#pragma unroll
        for (int p = 0; p < kNpt; ++p) {
            live[p] = lane < cnt[p];
            unpack_g(__float_as_uint(r[p].w), a, g[p]);
            d[p][0] = r[p].x; d[p][1] = r[p].y; d[p][2] = r[p].z;
            st[p] = ST_VALID;
            ghost_bad[p] = false;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) gb[p][ax] = g[p][ax] - a.gmin[ax] - kMagicBits;
            int c[3];
            float f[3];
            if (!cells_b<3>(gb[p], d[p], a.gspan, c, f) && live[p])
                classify_slow_v<3, BTO>(a, c, f, ghost_bad[p]);      // top-face clamp only
            int i = vindex<3>(a, c);
            LAG_CHECK_GATHER(a, i, live[p]);
            if (!live[p]) i = 0;
            idx1[p] = cur[p] = i;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) { v1c[p][ax] = c[ax]; f1[p][ax] = f[ax]; }
        }
#pragma unroll
        for (int p = 0; p < kNpt; ++p) {
            gather_pairs<3>(a.v0, idx1[p], a.sx, a.sxy, S[p]);
            gather_pairs<3>(a.v1, idx1[p], a.sx, a.sxy, B[p]);
        }
#pragma unroll
        for (int p = 0; p < kNpt; ++p) {
            interp_pairs<3>(S[p], f1[p], k1[p]);
#pragma unroll
            for (int i = 0; i < NP; ++i) S[p][i] = f2_add(S[p][i], B[p][i]);   // v0 + v1 (stages 2, 3)
        }

        // ---- stages 2 and 3 (alpha = 1/2: S), stage 4 (alpha = 1: B) ----
#pragma unroll
        for (int s = 2; s <= 4; ++s) {
            float f[kNpt][3];
            int idx[kNpt];
#pragma unroll
            for (int p = 0; p < kNpt; ++p) {
                float e[3];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax)
                    e[ax] = s == 2 ? fmaf(a.hdth[ax], k1[p][ax], f1[p][ax])
                          : s == 3 ? fmaf(a.qdth[ax], T2[p][ax], f1[p][ax])
                                   : fmaf(a.hdth[ax], T3[p][ax], f1[p][ax]);
                idx[p] = stage_cell<3, BTO>(a, v1c[p], idx1[p], e, live[p] && st[p] == ST_VALID,
                                            st[p], ghost_bad[p], f[p]);
            }
#pragma unroll
            for (int p = 0; p < kNpt; ++p) {
                LAG_CHECK_GATHER(a, idx[p], live[p] && st[p] == ST_VALID);
                if (live[p] && st[p] == ST_VALID && idx[p] != cur[p]) {
                    if (s < 4) {
                        gather_pairs<3>(a.v0, idx[p], a.sx, a.sxy, S[p]);
                        gather_pairs<3>(a.v1, idx[p], a.sx, a.sxy, B[p]);
#pragma unroll
                        for (int i = 0; i < NP; ++i) S[p][i] = f2_add(S[p][i], B[p][i]);
                        cur[p] = idx[p];
                    } else {
                        gather_pairs<3>(a.v1, idx[p], a.sx, a.sxy, B[p]);
                    }
                }
            }
#pragma unroll
            for (int p = 0; p < kNpt; ++p) {
                if (s == 2) interp_pairs<3>(S[p], f[p], T2[p]);       // T2 = 2 k2
                else if (s == 3) interp_pairs<3>(S[p], f[p], T3[p]);  // T3 = 2 k3
                else interp_pairs<3>(B[p], f[p], k4[p]);
            }
        }

        // ---- update, membership, particle management (as advect_kernel) ----
#pragma unroll
        for (int p = 0; p < kNpt; ++p) {
            if (cnt[p] == 0) continue;                               // warp-uniform
            const int tile = grp * kNpt + p;
            float4* trec = a.state + (size_t)tile * kTile;
            float dn[3];
#pragma unroll
            for (int ax = 0; ax < 3; ++ax)
                dn[ax] = fmaf(a.sdth[ax], (k1[p][ax] + k4[p][ax]) + (T2[p][ax] + T3[p][ax]), d[p][ax]);
            bool finite = true;
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) finite &= fabsf(dn[ax]) < 4194304.f;
            bool migrate = false;
            int nb = 0;
            uint8_t sp = st[p];
            {
                int cn[3];
                float fn[3];
                int gbb[3];
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) gbb[ax] = BTO ? gb[p][ax] : g[p][ax] - a.bmin[ax] - kMagicBits;
                const bool inblk = cells_b<3>(gbb, dn, a.bspan, cn, fn);
#pragma unroll
                for (int ax = 0; ax < 3; ++ax) cn[ax] += a.bmin[ax];
                if (!inblk && live[p] && sp == ST_VALID) {
                    bool gdummy = false;
                    if constexpr (BTO) {
                        sp = classify_slow<3, true>(a, cn, fn, gdummy);
                    } else {
                        bool out_dom = false;
                        int mul = 1;
#pragma unroll
                        for (int ax = 0; ax < 3; ++ax) {
                            out_dom |= (cn[ax] < 0) | (cn[ax] > a.N[ax] - 1) |
                                       ((cn[ax] == a.N[ax] - 1) & (fn[ax] != 0.f));
                            const int o = (cn[ax] < a.lo[ax]) ? -1
                                          : ((cn[ax] >= a.hi[ax] && a.hi[ax] < a.N[ax]) ? 1 : 0);
                            migrate |= (o != 0);
                            nb += (o + 1) * mul;
                            mul *= 3;
                        }
                        if (out_dom) { sp = ST_EXIT; migrate = false; }
                    }
                }
            }
            if (live[p] && !finite) { errbits |= ERR_NONFINITE; sp = ST_EXIT; migrate = false; }
            if (live[p] && ghost_bad[p]) { errbits |= ERR_GHOST; if (sp == ST_VALID) sp = ST_EXIT; migrate = false; }

            const bool keep = live[p] && sp == ST_VALID && !migrate;
            const unsigned kmask = __ballot_sync(0xffffffffu, keep);
            const unsigned dmask = __ballot_sync(0xffffffffu, live[p] && sp != ST_VALID);
            const unsigned tmask = __ballot_sync(0xffffffffu, live[p] && sp == ST_TERM);
            __syncwarp();
            if (keep) {
                const int pos = __popc(kmask & ((1u << lane) - 1u));
                trec[pos] = make_float4(dn[0], dn[1], dn[2], r[p].w);
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
                        sb[1 + pos] = make_float4(dn[0], dn[1], dn[2], r[p].w);
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
                if (live[p] && sp != ST_VALID) {
                    const uint32_t si = slot0 + __popc(dmask & ((1u << lane) - 1u));
                    if (si < a.dead_cap) {
                        a.dead_rec[si] = r[p];                       // pre-step position
                        a.dead_info[si] = ((uint32_t)sp << 24) | (uint32_t)(a.cycle & 0xffffff);
                    } else {
                        errbits |= ERR_OVERFLOW;
                    }
                }
            }
            if (lane == 0) {
                a.tile_count[tile] = (uint8_t)__popc(kmask);
                steps += (unsigned long long)cnt[p];
                nterm += __popc(tmask);
                nexit += __popc(dmask) - __popc(tmask);
            }
        }
        grp = ngrp;
#pragma unroll
        for (int p = 0; p < kNpt; ++p) { cnt[p] = ncnt[p]; r[p] = nr[p]; }
    }

    if (lane == 0 && steps) {
        atomicAdd(&a.counters[CNT_STEPS], steps);
        if (nterm) atomicAdd(&a.counters[CNT_TERM], nterm);
        if (nexit) atomicAdd(&a.counters[CNT_EXIT], nexit);
        if (nsent) atomicAdd(&a.counters[CNT_SENT], nsent);
    }
    errbits = __reduce_or_sync(0xffffffffu, errbits);
    if (lane == 0 && errbits) atomicOr(a.err, errbits);
    if constexpr (!BTO) {
        if (a.n_sig) {                                               // peer transport (see advect_kernel)
            if (did_remote) __threadfence_system();
            __syncwarp();
            if (lane == 0) {
                const uint32_t total = (gridDim.x * kThreads) >> 5;
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

}  // namespace lag
