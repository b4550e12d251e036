// lag_peer.cu — COMM mode over NVLink peer memory (exchange = LAG_XCHG_PEER):
// the per-cycle exchange of the Lagrangian-MPI baseline done by
// the kernels themselves, with no NCCL call on the per-cycle path.
//
// Every rank owns one CUDA-IPC allocation, mapped by its neighbours:
//   flags  [4][27] u64  — "halo ready" / "particles ready" sequence numbers
//                         and the hand-off counts of two parities, one word
//                         per sending neighbour (its offset index)
//   pslot  [3 parities][sum over peers of (1 + cap) float4] — my outgoing
//                         particle slots (header + records), one per
//                         neighbour, filled by my advect kernel with local
//                         atomics and stores, read by the neighbour
//   outbox [2 parities][2 slices][halo floats] — my packed ghost sources, read
//                         by the neighbours with remote loads
// Per cycle (seq = 1, 2, ...; ghost parity q = seq & 1, slot parity seq % 3):
//   pack my faces -> outbox[q]; signal halo(seq) to each neighbour;
//   wait until every neighbour signalled halo >= seq (bounded spin, latched
//   error on timeout) — its exchange(seq) runs after its advect(seq-1), so
//   the flag also says that advect's hand-offs are written; reset my
//   pslot[(seq+1) % 3] headers; ghost layers <- neighbours' outbox[q] and
//   hand-offs <- neighbours' pslot[(seq-1) % 3] toward me (remote loads);
//   advect writes leaving particles into my pslot[seq % 3].
// Three slot parities: the advect of cycle seq writes parity seq % 3 while
// (overlap transport) the exchange of the same cycle reads the neighbours'
// parity (seq-1) % 3 and resets mine of parity (seq+1) % 3, last read by the
// neighbour in its exchange(seq-1), which ended before it signalled halo(seq).
// Two ghost parities suffice: a neighbour reuses outbox parity q at seq+2
// only after it waited for my halo(seq+1), which I signal after pulling.
// Write cycle: the flush kernel signals particles(seq), waits for the
// neighbours' particles(seq) and appends their pslot[seq % 3]; the first
// exchange of the next interval appends nothing.
#include "lag_internal.h"
#include "lag_append.cuh"
#include "lag_xchg.cuh"

#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <unistd.h>
#include <cstring>
#include <vector>

using namespace lag;

#define CKC(call)                                                                  \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            lag_set_error(ctx, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                          __FILE__, __LINE__);                                     \
            return LAG_ECUDA;                                                      \
        }                                                                          \
    } while (0)
#define CKN(call)                                                                  \
    do {                                                                           \
        ncclResult_t r_ = (call);                                                  \
        if (r_ != ncclSuccess) {                                                   \
            lag_set_error(ctx, "%s: %s (%s:%d)", #call, ncclGetErrorString(r_),    \
                          __FILE__, __LINE__);                                     \
            return LAG_ENCCL;                                                      \
        }                                                                          \
    } while (0)

namespace lag {

// per-rank layout table published to every rank (int64 words)
enum : int { T_PSLOT = 0, T_PSLOT_PAR = 1, T_OUTBOX = 2, T_HALO = 3, T_SLOT = 4, T_SEND = 4 + kOff,
             T_WORDS = 4 + 2 * kOff };
constexpr int kSlotParities = 3;
// flag words, one per sending neighbour (its offset index): halo(seq),
// particles(seq) (write cycle), hand-off counts (two parities: seq & 1)
enum : int { F_HALO = 0, F_PART = 1, F_CNT = 2, kFlagKinds = 4 };

// pack + signal, then wait + pull + append, in one launch: every CTA must be
// resident (a CTA waiting for the neighbours' signal must not keep one of
// ours that has not packed from running), so the grid is capped at the
// resident capacity
__global__ void __launch_bounds__(256) peer_exchange_kernel(XchgArgs x, AppendArgs ap, int npull) {
    griddep_launch();                 // the advect kernel may be scheduled (it waits for this grid)
    xchg_pack_signal(x, blockIdx.x, gridDim.x);
    if ((int)blockIdx.x < npull) xchg_wait_pull(x, ap, blockIdx.x, npull);
}

__global__ void __launch_bounds__(256) peer_wait_pull_kernel(XchgArgs x, AppendArgs ap) {
    xchg_wait_pull(x, ap, blockIdx.x, gridDim.x);
}

}  // namespace lag

// ---------------------------------------------------------------------------

struct PeerState {
    char* mem = nullptr;                      // my IPC allocation
    size_t bytes = 0;
    std::vector<char*> remote;                // per peer: mapped neighbour allocation
    std::vector<int64_t> table;               // nranks * T_WORDS
    unsigned long long* flags = nullptr;      // mine
    float4* pslot[kSlotParities] = {nullptr, nullptr, nullptr};
    float* outbox = nullptr;                  // [2][2][halo]
    std::vector<lag::PeerBox> boxes;          // v1 boxes then v0 boxes
    lag::PeerBox* d_boxes = nullptr;
    int64_t halo_recv_floats = 0;
    int64_t halo_send_floats = 0;
    std::vector<int64_t> my_table;            // my own layout words
    unsigned long long seq = 0;
    uint32_t* done_ctas = nullptr;            // pack completion counter
};

lag_status lag_peer_init(lag_ctx_s* ctx, ncclComm_t nccl, const std::vector<int>& prank,
                         const std::vector<int>& poff, const std::vector<int>& pback,
                         const std::vector<uint32_t>& cap_send, int64_t halo_send_floats,
                         const std::vector<int64_t>& send_box_off, const std::vector<int64_t>& send_box_by_off,
                         const std::vector<int>& recv_box_x0y0z0nxnynz, int64_t halo_recv_floats,
                         PeerState** out) {
    *out = nullptr;
    PeerState* ps = new PeerState();
    const int R = ctx->cfg.nranks;
    const int np = (int)prank.size();
    // my layout: flags | pslot[3] | outbox[2][2]
    int64_t slot_f4 = 0;
    std::vector<int64_t> slot_off(kOff, -1);            // my slot toward the neighbour at offset k
    for (int i = 0; i < np; ++i) { slot_off[poff[i]] = slot_f4; slot_f4 += cap_send[i] + 1; }
    const size_t pslot_off = 1024;                      // after the 4 x 27 u64 flag words (864 B)
    static_assert(kFlagKinds * kOff * sizeof(unsigned long long) <= 1024, "flags overlap the slots");
    const size_t pslot_bytes = (size_t)std::max<int64_t>(1, slot_f4) * sizeof(float4);
    const size_t outbox_off = pslot_off + kSlotParities * pslot_bytes;
    const size_t outbox_bytes = (size_t)std::max<int64_t>(1, halo_send_floats) * sizeof(float);
    ps->bytes = outbox_off + 4 * outbox_bytes;
    CKC(cudaMalloc(&ps->mem, ps->bytes));
    CKC(cudaMemset(ps->mem, 0, ps->bytes));
    ps->flags = reinterpret_cast<unsigned long long*>(ps->mem);
    for (int q = 0; q < kSlotParities; ++q)
        ps->pslot[q] = reinterpret_cast<float4*>(ps->mem + pslot_off + q * pslot_bytes);
    ps->outbox = reinterpret_cast<float*>(ps->mem + outbox_off);
    ps->halo_recv_floats = halo_recv_floats;
    ps->halo_send_floats = std::max<int64_t>(1, halo_send_floats);
    // publish layout + IPC handle
    std::vector<int64_t> mine(T_WORDS, -1);
    mine[T_PSLOT] = (int64_t)pslot_off;
    mine[T_PSLOT_PAR] = (int64_t)pslot_bytes;
    mine[T_OUTBOX] = (int64_t)outbox_off;
    mine[T_HALO] = halo_send_floats;
    for (int k = 0; k < kOff; ++k) { mine[T_SLOT + k] = slot_off[k]; mine[T_SEND + k] = send_box_by_off[k]; }
    ps->my_table = mine;
    cudaIpcMemHandle_t h;
    CKC(cudaIpcGetMemHandle(&h, ps->mem));
    const size_t rec = T_WORDS * sizeof(int64_t) + sizeof(h);
    std::vector<char> host(rec * (R + 1));
    std::memcpy(host.data(), mine.data(), T_WORDS * sizeof(int64_t));
    std::memcpy(host.data() + T_WORDS * sizeof(int64_t), &h, sizeof(h));
    char* d = nullptr;
    CKC(cudaMalloc(&d, rec * (R + 1)));
    CKC(cudaMemcpyAsync(d, host.data(), rec, cudaMemcpyHostToDevice, ctx->stream));
    CKN(ncclAllGather(d, d + rec, rec, ncclUint8, nccl, ctx->stream));
    CKC(cudaMemcpyAsync(host.data() + rec, d + rec, rec * R, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    cudaFree(d);
    ps->table.assign((size_t)R * T_WORDS, 0);
    ps->remote.assign(np, nullptr);
    for (int r = 0; r < R; ++r)
        std::memcpy(&ps->table[(size_t)r * T_WORDS], host.data() + rec * (r + 1), T_WORDS * sizeof(int64_t));
    for (int i = 0; i < np; ++i) {
        cudaIpcMemHandle_t hr;
        std::memcpy(&hr, host.data() + rec * (prank[i] + 1) + T_WORDS * sizeof(int64_t), sizeof(hr));
        void* ptr = nullptr;
        CKC(cudaIpcOpenMemHandle(&ptr, hr, cudaIpcMemLazyEnablePeerAccess));
        ps->remote[i] = (char*)ptr;
    }
    // ghost boxes to pull: for peer i, its outbox box toward me (my index at it = back)
    for (int slice = 1; slice >= 0; --slice) {
        int64_t off = 0;
        for (int i = 0; i < np; ++i) {
            const int* bx = &recv_box_x0y0z0nxnynz[6 * i];
            PeerBox b{};
            b.x0 = bx[0]; b.y0 = bx[1]; b.z0 = bx[2]; b.nx = bx[3]; b.ny = bx[4]; b.nz = bx[5];
            b.slice = slice;
            const int64_t* t = &ps->table[(size_t)prank[i] * T_WORDS];
            // peer's outbox parity q = [v_t1 boxes | v_t boxes] (the pack-buffer layout)
            for (int q = 0; q < 2; ++q)
                for (int sl = 0; sl < 2; ++sl)
                    b.src[q][sl] = reinterpret_cast<const float*>(ps->remote[i] + t[T_OUTBOX] +
                                   (size_t)(q * 2 + (sl == 1 ? 0 : 1)) * std::max<int64_t>(1, t[T_HALO]) * sizeof(float)) +
                                   t[T_SEND + pback[i]];
            b.off = off + (slice == 0 ? halo_recv_floats : 0);
            off += (int64_t)b.nx * b.ny * b.nz * ctx->cfg.dim;
            ps->boxes.push_back(b);
        }
    }
    CKC(cudaMalloc(&ps->done_ctas, sizeof(uint32_t)));
    CKC(cudaMemset(ps->done_ctas, 0, sizeof(uint32_t)));
    CKC(cudaMalloc(&ps->d_boxes, sizeof(PeerBox) * std::max<size_t>(1, ps->boxes.size())));
    if (!ps->boxes.empty())
        CKC(cudaMemcpy(ps->d_boxes, ps->boxes.data(), sizeof(PeerBox) * ps->boxes.size(), cudaMemcpyHostToDevice));
    (void)send_box_off;
    *out = ps;
    return LAG_OK;
}

void lag_peer_destroy(PeerState* ps) {
    if (!ps) return;
    for (char* p : ps->remote) if (p) cudaIpcCloseMemHandle(p);
    cudaFree(ps->d_boxes);
    cudaFree(ps->done_ctas);
    cudaFree(ps->mem);
    delete ps;
}

// my outgoing slot (parity q) toward the neighbour at offset index poff
float4* lag_peer_my_slot(PeerState* ps, int q, int poff) {
    return ps->pslot[q % kSlotParities] + ps->my_table[T_SLOT + poff];
}

// neighbour i's outgoing slot (parity q) toward me (my offset index at it = pback)
float4* lag_peer_remote_slot(PeerState* ps, int i, int prank, int pback, int q) {
    const int64_t* t = &ps->table[(size_t)prank * T_WORDS];
    return reinterpret_cast<float4*>(ps->remote[i] + t[T_PSLOT] + (size_t)(q % kSlotParities) * t[T_PSLOT_PAR]) +
           t[T_SLOT + pback];
}


unsigned long long& lag_peer_seq(PeerState* ps) { return ps->seq; }

unsigned long long* lag_peer_remote_flag(PeerState* ps, int i, int kind, int pback) {
    return reinterpret_cast<unsigned long long*>(ps->remote[i]) + kind * kOff + pback;
}

// my count word (parity par) written by the neighbour at offset index poff
const unsigned long long* lag_peer_my_count(PeerState* ps, int par, int poff) {
    return ps->flags + (F_CNT + (par & 1)) * kOff + poff;
}

// The fused exchange (see peer_exchange_kernel).  halo: this cycle's ghost
// exchange (seq = the cycle, already incremented); otherwise the write-cycle
// flush of cycle seq's hand-offs (signal particles(seq), wait for the
// neighbours' signal).  append_args: the neighbours' slots to append, or null.
lag_status lag_peer_exchange(lag_ctx_s* ctx, PeerState* ps, const void* send_boxes, int nsend,
                             int64_t sfl, float* v0, float* v1, bool with_v0, bool halo,
                             const std::vector<int>& poff, const std::vector<int>& pback,
                             const void* append_args) {
    const int np = (int)poff.size();
    cudaStream_t st = ctx->stream;
    XchgArgs x{};
    const unsigned long long seq = ps->seq;
    const int q = (int)(seq & 1);
    x.v0 = v0; x.v1 = v1;
    x.send_boxes = reinterpret_cast<const Box*>(send_boxes);
    x.nsend = halo ? (with_v0 ? 2 * nsend : nsend) : 0;
    x.outbox = ps->outbox + (size_t)q * 2 * ps->halo_send_floats;
    x.sfl = halo ? (with_v0 ? 2 : 1) * sfl : 0;
    x.signal_halo = halo ? 1 : 0;
    x.npeers = np;
    for (int i = 0; i < np; ++i) {
        x.halo_flag[i] = lag_peer_remote_flag(ps, i, F_HALO, pback[i]);
        x.back[i] = poff[i];
    }
    x.my_flags = ps->flags;
    x.need_halo = halo ? seq : 0;
    x.need_part = halo ? 0 : seq;
    // counts published with the signal: per cycle, of the slots the advect
    // filled last cycle (parity seq-1), in count parity seq; at the write
    // cycle, of this cycle's slots, in count parity seq+1
    const int slot_par = (int)((halo ? seq + kSlotParities - 1 : seq) % kSlotParities);
    const int cnt_par = (int)((halo ? seq : seq + 1) & 1);
    x.send_cnt = 1;
    for (int i = 0; i < np; ++i) {
        x.my_hdr[i] = reinterpret_cast<const uint32_t*>(lag_peer_my_slot(ps, slot_par, poff[i]));
        x.cnt_word[i] = lag_peer_remote_flag(ps, i, F_CNT + cnt_par, pback[i]);
    }
    if (halo) {                                // my slots the advect fills next cycle
        x.nzero = np;
        for (int i = 0; i < np; ++i)
            x.zero_slot[i] = reinterpret_cast<uint32_t*>(lag_peer_my_slot(ps, (int)((seq + 1) % kSlotParities), poff[i]));
    } else {
        x.signal_part = 1;
        for (int i = 0; i < np; ++i) x.part_flag[i] = lag_peer_remote_flag(ps, i, F_PART, pback[i]);
    }
    x.timeout_cycles = 8000000000LL;
    x.err = ctx->words + W_ERR;
    x.recv_boxes = ps->d_boxes;
    const int nb = (int)ps->boxes.size() / 2;
    x.nrecv = halo ? (with_v0 ? 2 * nb : nb) : 0;
    x.parity = q;
    x.rtotal = halo ? (with_v0 ? 2 : 1) * ps->halo_recv_floats : 0;
    x.sx = ctx->sx; x.sxy = ctx->sxy; x.dim = ctx->cfg.dim;
    x.seq = seq;
    x.do_append = append_args ? 1 : 0;
    for (const float* w : {halo ? v1 : nullptr, (halo && with_v0) ? v0 : nullptr})
        if (w && (w == ctx->prev_d0 || w == ctx->prev_d1)) x.pull_wait = 1;
    x.done_ctas = ps->done_ctas;
    AppendArgs ap{};
    if (append_args) ap = *reinterpret_cast<const AppendArgs*>(append_args);
    if (ctx->xchg_fused && halo) {           // overlap: the advect kernel's first CTAs run it
        XchgFused* f = reinterpret_cast<XchgFused*>(ctx->xchg_fused);
        f->x = x;
        f->ap = ap;
        return LAG_OK;
    }
    const int cap = ctx->num_sms * 2;          // resident: 2 CTAs of 256 threads per SM
    if (halo) {
        const int64_t work = std::max(x.sfl, x.rtotal);
        const int g = (int)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, cap));
        // waiters: enough for one round of remote loads (8 in flight per thread)
        const int npull = (int)std::max<int64_t>(std::min<int64_t>(8, g), std::min<int64_t>((x.rtotal + 2047) / 2048, g));
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr.val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(g); lc.blockDim = dim3(256); lc.dynamicSmemBytes = 0; lc.stream = st;
        lc.attrs = &attr; lc.numAttrs = 1;
        CKC(cudaLaunchKernelEx(&lc, peer_exchange_kernel, x, ap, npull));
    } else {
        const int gb = (int)std::max<int64_t>(1, std::min<int64_t>((x.rtotal + 255) / 256, cap));
        peer_wait_pull_kernel<<<gb, 256, 0, st>>>(x, ap);
    }
    ++ctx->launches;
    CKC(cudaGetLastError());
    return LAG_OK;
}
