// lag_xchg.cuh — the per-cycle peer-memory exchange of the COMM baseline
// (LAG_XCHG_PEER / LAG_XCHG_PEER_OVERLAP; protocol in lag_peer.cu) as device
// functions over a virtual grid of `ncta` CTAs: lag_peer.cu runs them as two
// kernels; with LAG_XCHG_PEER_OVERLAP the first CTAs of the advect kernel's
// pass 1 run them while the other CTAs advect the ghost-free tiles.
#pragma once
#include "lag_kernels.cuh"
#include "lag_append.cuh"

namespace lag {

constexpr int kOff = kMaxOff;
constexpr int kMaxPeers = 26;
struct PeerBox {            // one ghost box to fill from a remote outbox
    int x0, y0, z0, nx, ny, nz;
    int64_t off;            // float offset of this box in the flattened copy
    const float* src[2][2]; // [parity][slice 0 = v_t, 1 = v_t1] remote source
    int slice;
};

// Per-cycle exchange (the hand-offs wait in the senders' own slots):
//   A: pack my ghost sources (grid-stride); the last CTA to finish fences and
//      signals halo(seq) to every neighbour.  Launched as a programmatic
//      dependent of the previous advect kernel, the packing and the ghost
//      pull (inputs: the new slices) overlap that kernel's tail; the signal
//      and the append wait for its end (griddep_wait);
//   B: the first `npull` CTAs wait (bounded) for all neighbours' halo(seq)
//      (which implies their hand-offs of cycle seq-1 are written: stream
//      order), pull their share of the ghost layers and of those hand-offs
//      with remote loads and append them.  Few waiters: a few hundred CTAs
//      polling one flag word queue up its L2 slice and delay the neighbour's
//      remote store to it by several microseconds.
struct XchgArgs {
    float* v0;
    float* v1;
    const Box* send_boxes;
    int nsend;
    float* outbox;                                 // my outbox at parity q
    int64_t sfl;                                   // floats to pack
    int signal_halo;
    unsigned long long* halo_flag[kMaxPeers];      // neighbour's halo flag word for me
    uint32_t* done_ctas;                           // kernel A completion counter
    int npeers;
    const unsigned long long* my_flags;
    int back[kMaxPeers];
    unsigned long long need_halo, need_part;
    long long timeout_cycles;
    uint32_t* err;
    const PeerBox* recv_boxes;
    int nrecv;
    int parity;
    int64_t rtotal;                                // floats to pull
    int sx, sxy, dim;
    unsigned long long seq;
    int do_append;
    // my outgoing particle slots the advect kernel fills next cycle: reset
    // once every neighbour has signalled this cycle (it has read them)
    uint32_t* zero_slot[kMaxPeers];
    int nzero;
    // write cycle: signal "particles(seq) ready" to every neighbour first
    // (halo(seq+1) implies it on the per-cycle path)
    unsigned long long* part_flag[kMaxPeers];
    int signal_part;
    // a slice the ghost pull writes was read by the previous advect kernel
    // (the same buffer passed again): pull only after that kernel ended
    int pull_wait;
    // hand-off counts travel with the signal: the signalling thread copies my
    // slot headers (the parity the neighbours append now) into their count
    // words, so the receiver's append skips one remote round trip
    int send_cnt;
    const uint32_t* my_hdr[kMaxPeers];
    unsigned long long* cnt_word[kMaxPeers];
};

// the signalling thread: counts, then the release fence, then the flags
__device__ __forceinline__ void xchg_publish(const XchgArgs& x, unsigned long long* const* flag) {
    if (x.send_cnt)
        for (int p = 0; p < x.npeers; ++p)
            *reinterpret_cast<volatile unsigned long long*>(x.cnt_word[p]) =
                *reinterpret_cast<const volatile uint32_t*>(x.my_hdr[p]);
    __threadfence_system();
    for (int p = 0; p < x.npeers; ++p) *reinterpret_cast<volatile unsigned long long*>(flag[p]) = x.seq;
}

__device__ __forceinline__ void xchg_pack_signal(const XchgArgs& x, int cta, int ncta) {
    for (int64_t i = (int64_t)cta * blockDim.x + threadIdx.x; i < x.sfl;
         i += (int64_t)ncta * blockDim.x) {
        int k = 0;
        while (k + 1 < x.nsend && x.send_boxes[k + 1].off <= i) ++k;
        const Box& b = x.send_boxes[k];
        const int64_t j = i - b.off;
        const int comp = (int)(j % x.dim);
        const int64_t node = j / x.dim;
        const int xx = (int)(node % b.nx), yy = (int)((node / b.nx) % b.ny), zz = (int)(node / ((int64_t)b.nx * b.ny));
        const float* src = b.slice ? x.v1 : x.v0;
        x.outbox[i] = src[(int64_t)x.dim * ((b.x0 + xx) + (int64_t)x.sx * (b.y0 + yy) + (int64_t)x.sxy * (b.z0 + zz)) + comp];
    }
    __syncthreads();                                  // the CTA's packs are visible to thread 0
    if (threadIdx.x == 0 && x.signal_halo) {
        // release at GPU scope (the packs and the counter live on this GPU);
        // the last CTA's system-scope fence then releases everything it has
        // observed to the neighbours (causality is transitive), so only one
        // CTA pays the system-scope fence
        __threadfence();
        if (atomicAdd(x.done_ctas, 1u) == (uint32_t)ncta - 1) {   // last CTA: halo(seq) ready
            *x.done_ctas = 0u;
            griddep_wait();                           // and my previous advect's hand-offs (see below)
            xchg_publish(x, x.halo_flag);
        }
    }
}

__device__ __forceinline__ void xchg_wait_pull(const XchgArgs& x, const AppendArgs& ap, int cta, int ncta) {
    if (x.signal_part && cta == 0 && threadIdx.x == 0) xchg_publish(x, x.part_flag);   // write cycle
    if (threadIdx.x < x.npeers) {
        const volatile unsigned long long* fh = x.my_flags + 0 * kOff + x.back[threadIdx.x];
        const volatile unsigned long long* fp = x.my_flags + 1 * kOff + x.back[threadIdx.x];
        const long long t0 = clock64();
        while (*fh < x.need_halo || *fp < x.need_part) {
            if (clock64() - t0 > x.timeout_cycles) { atomicOr(x.err, ERR_XCHG); break; }
            __nanosleep(100);
        }
        __threadfence_system();
    }
    __syncthreads();
    if (cta == 0 && threadIdx.x < x.nzero) *x.zero_slot[threadIdx.x] = 0u;
    // the append (remote hand-off records) and the ghost pull (remote face
    // values) run side by side: a quarter of the CTAs append
    int na = x.do_append ? max(1, ncta / 4) : 0;
    if (ncta - na < 1) na = 0;                        // too few CTAs: each does both
    if (cta < na) {
        griddep_wait();                               // the previous advect kernel's particle lists
        append_body(ap, cta, na);
        return;
    }
    const int pc = cta - na, npc = ncta - na;
    if (x.pull_wait) griddep_wait();
    // remote loads: 8 in flight per thread (a few CTAs cover the ghost layers
    // when they run inside the advect kernel's pass 1)
    const int64_t step = (int64_t)npc * blockDim.x;
    for (int64_t i0 = (int64_t)pc * blockDim.x + threadIdx.x; i0 < x.rtotal; i0 += 8 * step) {
        float val[8];
        float* dst[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = i0 + u * step;
            dst[u] = nullptr;
            if (i < x.rtotal) {
                int lo = 0, hi = x.nrecv - 1;                 // box with off <= i (offsets ascending)
                while (lo < hi) {
                    const int mid = (lo + hi + 1) >> 1;
                    if (x.recv_boxes[mid].off <= i) lo = mid; else hi = mid - 1;
                }
                const PeerBox& b = x.recv_boxes[lo];
                const int j = (int)(i - b.off);
                const int comp = j % x.dim;
                const int node = j / x.dim;
                const int xx = node % b.nx, yy = (node / b.nx) % b.ny, zz = node / (b.nx * b.ny);
                dst[u] = (b.slice ? x.v1 : x.v0) +
                         (int64_t)x.dim * ((b.x0 + xx) + (int64_t)x.sx * (b.y0 + yy) + (int64_t)x.sxy * (b.z0 + zz)) + comp;
                val[u] = b.src[x.parity][b.slice][j];
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (dst[u]) *dst[u] = val[u];
    }
    if (x.do_append && na == 0) {
        griddep_wait();                               // the previous advect kernel's particle lists
        append_body(ap, cta, ncta);
    }                         // hand-offs of cycle seq-1 (all CTAs)
}

// exchange role of the advect kernel's pass 1 (LAG_XCHG_PEER_OVERLAP)
constexpr int kXchgCtas = 48;   // CTAs of kThreads running the exchange
struct XchgFused {
    int32_t ncta;                   // CTAs 0..ncta-1 run the exchange; 0 = none
    XchgArgs x;
    AppendArgs ap;
};

}  // namespace lag
