// lag_append.cuh — COMM: received particles -> new tiles at the end of the
// particle list (shared by the NCCL path's append_kernel and the peer path's
// fused exchange kernel).
#pragma once
#include "lag_internal.h"

namespace lag {
constexpr int kMaxOff = 27;

struct Box {            // local slice coordinates
    int x0, y0, z0, nx, ny, nz;
    int64_t off;        // float offset in the pack buffer
    int slice;          // 0 = v_t, 1 = v_t1
};


// whose headers the append resets: the NCCL transport's outgoing slots (sent
// this cycle), the consumed inbox (LOCAL transport), or none (peer
// transport: the sender resets its own slots once the receiver has read them)
enum : int { RESET_SLOTS = 0, RESET_RECV = 1, RESET_NONE = 2 };

struct AppendArgs {
    float4* state;
    uint8_t* tile_count;
    uint32_t* words;
    unsigned long long* counters;
    int cap_tiles;
    int npeers;
    float4* recv[kMaxOff];
    uint32_t cap[kMaxOff];
    float4* slots;                  // outgoing slots: headers reset here (NCCL)
    int32_t slot_base[kMaxOff];
    int noff;
    int reset;                      // headers reset after the append: RESET_* below
    const unsigned long long* cnt[kMaxOff];   // non-null: the record count of recv[p] (peer transport)
    int discard;                    // drop the records (a reseed in the middle of an interval)
};

// Received particles become new tiles at the end of the list.  Every CTA of
// the calling grid takes a grid-stride share of the records (one latency
// round for a few thousand hand-offs instead of one per 256 records); each
// CTA reads the headers and the old tile count first, and the last CTA to
// finish resets the headers and publishes the new tile count.
__device__ __forceinline__ void append_body(const AppendArgs& a, int cta, int ncta) {
    __shared__ uint32_t pre[kMaxOff + 1];
    __shared__ uint32_t old_tiles, total_s;
    // the headers and the tile count are read in parallel (one load
    // latency, not one per neighbour), then thread 0 takes the prefix sum
    if (threadIdx.x < (unsigned)a.npeers) {
        const int p = threadIdx.x;
        uint32_t c = a.cnt[p] ? (uint32_t)*reinterpret_cast<const volatile unsigned long long*>(a.cnt[p])
                              : *reinterpret_cast<const volatile uint32_t*>(a.recv[p]);
        if (c > a.cap[p]) { c = a.cap[p]; atomicOr(a.words + W_ERR, ERR_OVERFLOW); }
        pre[p + 1] = c;
    }
    if (threadIdx.x == 32) old_tiles = *reinterpret_cast<const volatile uint32_t*>(a.words + W_NTILES);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int p = 0; p < a.npeers; ++p) {
            const uint32_t c = pre[p + 1];
            pre[p] = s;
            s += c;
        }
        if (a.discard) s = 0;
        pre[a.npeers] = s;
        const uint32_t room = (uint32_t)(a.cap_tiles - (int)old_tiles) * kTile;
        if (s > room) { atomicOr(a.words + W_ERR, ERR_OVERFLOW); s = room; }
        total_s = s;
    }
    __syncthreads();
    const uint32_t total = total_s;
    const uint32_t nthr = ncta * blockDim.x;
    for (uint32_t j = cta * blockDim.x + threadIdx.x; j < total; j += nthr) {
        int p = 0;
        while (p + 1 < a.npeers && pre[p + 1] <= j) ++p;
        a.state[(size_t)old_tiles * kTile + j] = a.recv[p][1 + (j - pre[p])];
    }
    const uint32_t new_tiles = (total + kTile - 1) / kTile;
    for (uint32_t t = cta * blockDim.x + threadIdx.x; t < new_tiles; t += nthr) {
        const uint32_t rem = total - t * kTile;
        a.tile_count[old_tiles + t] = (uint8_t)(rem >= (uint32_t)kTile ? kTile : rem);
    }
    __syncthreads();                 // this CTA read every header and wrote its share
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(a.words + W_APPEND_DONE, 1u) == (uint32_t)ncta - 1) {      // last CTA
            a.words[W_APPEND_DONE] = 0u;
            if (a.reset == RESET_RECV) {
                for (int p = 0; p < a.npeers; ++p) *reinterpret_cast<uint32_t*>(a.recv[p]) = 0u;
            } else if (a.reset == RESET_SLOTS) {
                for (int k = 0; k < a.noff; ++k) *reinterpret_cast<uint32_t*>(a.slots + a.slot_base[k]) = 0u;
            }
            a.words[W_NTILES] = old_tiles + new_tiles;
            if (total) atomicAdd(&a.counters[CNT_RECV], (unsigned long long)total);
            __threadfence();
        }
    }
}


static __global__ void __launch_bounds__(256) append_kernel(AppendArgs a) { append_body(a, blockIdx.x, gridDim.x); }

}  // namespace lag
