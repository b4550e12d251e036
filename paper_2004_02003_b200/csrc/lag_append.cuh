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
    int zero_recv;                  // peer transport: reset the consumed inbox headers instead
};

// one CTA: received particles become new tiles at the end of the list
__device__ __forceinline__ void append_body(const AppendArgs& a) {
    __shared__ uint32_t pre[kMaxOff + 1];
    __shared__ uint32_t old_tiles;
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int p = 0; p < a.npeers; ++p) {
            pre[p] = s;
            uint32_t c = *reinterpret_cast<const uint32_t*>(a.recv[p]);
            if (c > a.cap[p]) { c = a.cap[p]; atomicOr(a.words + W_ERR, ERR_OVERFLOW); }
            s += c;
        }
        pre[a.npeers] = s;
        old_tiles = a.words[W_NTILES];
    }
    __syncthreads();
    uint32_t total = pre[a.npeers];
    const uint32_t room = (uint32_t)(a.cap_tiles - (int)old_tiles) * kTile;
    if (total > room) {
        if (threadIdx.x == 0) atomicOr(a.words + W_ERR, ERR_OVERFLOW);
        total = room;
    }
    for (uint32_t j = threadIdx.x; j < total; j += blockDim.x) {
        int p = 0;
        while (p + 1 < a.npeers && pre[p + 1] <= j) ++p;
        a.state[(size_t)old_tiles * kTile + j] = a.recv[p][1 + (j - pre[p])];
    }
    const uint32_t new_tiles = (total + kTile - 1) / kTile;
    for (uint32_t t = threadIdx.x; t < new_tiles; t += blockDim.x) {
        const uint32_t rem = total - t * kTile;
        a.tile_count[old_tiles + t] = (uint8_t)(rem >= (uint32_t)kTile ? kTile : rem);
    }
    __syncthreads();                 // every count read before any header reset
    if (a.zero_recv) {
        if (threadIdx.x < (unsigned)a.npeers) *reinterpret_cast<uint32_t*>(a.recv[threadIdx.x]) = 0u;
    } else if (threadIdx.x < (unsigned)a.noff) {
        *reinterpret_cast<uint32_t*>(a.slots + a.slot_base[threadIdx.x]) = 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.words[W_NTILES] = old_tiles + new_tiles;
        if (total) atomicAdd(&a.counters[CNT_RECV], (unsigned long long)total);
    }
}


static __global__ void __launch_bounds__(1024) append_kernel(AppendArgs a) { append_body(a); }

}  // namespace lag
