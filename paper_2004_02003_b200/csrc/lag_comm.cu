// lag_comm.cu — COMM mode: the paper's communicating baseline (Lagrangian-MPI
// after Agranovsky et al., §2.3, §3.1) on NCCL over NVLink.
//
// Per lag_advect_cycle (one NCCL group per cycle, no host synchronisation):
//   1. halo_pack    : the parts of my slice interior my neighbours need as
//                     ghost layers (faces, edges, corners: all 3^d - 1 offsets
//                     go direct — NVSwitch gives every peer full bandwidth)
//   2. NCCL group   : halo boxes + the particle slots filled by the previous
//                     cycle's advect (messages sent in cycle c are advanced by
//                     the receiver from cycle c+1 on)
//   3. halo_unpack  : write the received ghost layers of v_t1 (and v_t)
//   4. append       : received particles -> new tiles at the end of the list
//   5. advect       : (lag_api.cu) writes leaving particles to per-offset slots
// Slots are fixed-capacity [header | cap records] so NCCL sizes are known on
// the host; overflow is latched as LAG_EOVERFLOW.
// lag_extract first flushes pending particles, then returns every particle
// to its origin rank ("each compute node returns its particles to
// their originating nodes"; untimed write cycle).
#include "lag_internal.h"
#include "lag_append.cuh"

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

using namespace lag;

// lag_peer.cu (LAG_XCHG_PEER transport)
struct PeerState;
lag_status lag_peer_init(lag_ctx_s* ctx, ncclComm_t nccl, const std::vector<int>& prank,
                         const std::vector<int>& poff, const std::vector<int>& pback,
                         const std::vector<uint32_t>& cap_send, int64_t halo_send_floats,
                         const std::vector<int64_t>& send_box_off, const std::vector<int64_t>& send_box_by_off,
                         const std::vector<int>& recv_box_x0y0z0nxnynz, int64_t halo_recv_floats,
                         PeerState** out);
void lag_peer_destroy(PeerState* ps);
float4* lag_peer_remote_slot(PeerState* ps, int i, int prank, int pback, int q);
float4* lag_peer_my_slot(PeerState* ps, int q, int poff);
unsigned long long& lag_peer_seq(PeerState* ps);
unsigned long long* lag_peer_remote_flag(PeerState* ps, int i, int kind, int pback);
const unsigned long long* lag_peer_my_count(PeerState* ps, int par, int poff);
lag_status lag_peer_exchange(lag_ctx_s* ctx, PeerState* ps, const void* send_boxes, int nsend,
                             int64_t sfl, float* v0, float* v1, bool with_v0, bool halo,
                             const std::vector<int>& poff, const std::vector<int>& pback,
                             const void* append_args);

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

constexpr int kMaxCuts = 65;

struct RouteRec {       // return-to-origin record (32 B)
    float4 rec;
    uint32_t info;      // (status << 24) | cycle ; 0 = valid
    uint32_t pad[3];
};

struct Peer {
    int rank;
    int off;                    // neighbour offset index (0..3^d-1)
    int back;                   // the offset index of me as seen from the peer
    int send_box, recv_box;     // indices into the box tables
    int64_t halo_floats_send, halo_floats_recv;
    uint32_t cap_send, cap_recv;   // particle slot capacities (records)
    float4* recv_slot;             // [1 + cap_recv]
};

struct Comm {
    ncclComm_t nccl = nullptr;
    int me[3] = {0, 0, 0};
    std::vector<int64_t> blocks;        // nranks * 6 (lo[3], hi[3])
    std::vector<Peer> peers;
    std::vector<Box> send_boxes, recv_boxes;    // per peer, one slice
    Box* d_send_boxes = nullptr;                // [2 * npeers]: v1 boxes then v0 boxes
    Box* d_recv_boxes = nullptr;
    float* halo_send = nullptr;                 // 2 slices worth
    float* halo_recv = nullptr;
    int64_t halo_send_floats = 0, halo_recv_floats = 0;   // one slice
    // outgoing particle slots: per offset [header | cap]
    float4* slots = nullptr;
    int32_t slot_base[kMaxOff] = {0};
    int32_t slot_capv[kMaxOff] = {0};
    int64_t slot_total = 0;
    float4* recv_slots = nullptr;
    int64_t recv_total = 0;
    bool pending = false;
    // routing
    int32_t cuts[3][kMaxCuts] = {{0}};
    int ncuts[3] = {0, 0, 0};
    int32_t* d_cuts = nullptr;
    uint32_t* d_route_count = nullptr;  // [nranks]
    RouteRec* route = nullptr;          // [cap]
    RouteRec* route_recv = nullptr;     // [cap]
    uint32_t* d_route_pos = nullptr;
    uint32_t* d_seg = nullptr;          // [nranks + 1] segment starts
    uint32_t* d_all = nullptr;          // [nranks * (nranks + 1)] count exchange
    int64_t route_cap = 0;
    uint32_t n_returned = 0;
    // LAG_XCHG_PEER transport
    PeerState* peer = nullptr;
    std::vector<int> prank, poff, pback;
};

// ---------------------------------------------------------------------------
// kernels

struct BoxArgs {
    const float* v0;
    float* v1;           // v_t1 (written by unpack)
    float* v0w;          // v_t  (written by unpack when its ghosts are stale)
    const Box* boxes;
    int nbox;
    float* buf;
    int sx, sxy, dim;
    int64_t total;       // floats over all boxes
};

// One grid row per box (blockIdx.y), the row's CTAs striding over the box's
// floats: the buffer holds box after box (Box::off), each x-fastest with the
// components innermost (32-bit index math: a box is far below 2^31 floats).
__device__ __forceinline__ int64_t box_node(const BoxArgs& a, const Box& b, int k, int& comp) {
    const int rowf = b.nx * a.dim;
    const int row = k / rowf, within = k - row * rowf;
    const int y = row % b.ny, z = row / b.ny;
    comp = within;
    return (int64_t)a.dim * (b.x0 + (int64_t)a.sx * (b.y0 + y) + (int64_t)a.sxy * (b.z0 + z));
}

__global__ void __launch_bounds__(256) halo_pack_kernel(BoxArgs a) {
    const Box& b = a.boxes[blockIdx.y];
    const int nf = b.nx * b.ny * b.nz * a.dim;
    const float* src = b.slice ? a.v1 : a.v0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x) {
        int within;
        const int64_t o = box_node(a, b, k, within);
        a.buf[b.off + k] = src[o + within];
    }
}

// the received ghost layers (grid rows [0, nbox)) and the received particles
// (grid row nbox, append_body on its first `app_ctas` CTAs) in one launch
__global__ void __launch_bounds__(256) halo_unpack_append_kernel(BoxArgs a, AppendArgs ap, int app_ctas) {
    if ((int)blockIdx.y == a.nbox) {
        if ((int)blockIdx.x < app_ctas) append_body(ap, blockIdx.x, app_ctas);
        return;
    }
    const Box& b = a.boxes[blockIdx.y];
    const int nf = b.nx * b.ny * b.nz * a.dim;
    float* dst = b.slice ? a.v1 : a.v0w;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x) {
        int within;
        const int64_t o = box_node(a, b, k, within);
        dst[o + within] = a.buf[b.off + k];
    }
}

struct RouteArgs {
    const float4* state;
    const uint8_t* tile_count;
    const uint32_t* words;
    const float4* dead_rec;
    const uint32_t* dead_info;
    uint32_t dead_cap;
    const int32_t* cuts;        // [3][kMaxCuts]
    int ncuts0, ncuts1, ncuts2;
    int lay0, lay1;
    uint32_t bx, by, mx, my;
    int me;
    uint32_t* count;            // [nranks]
    uint32_t* pos;              // [nranks] running positions (pass 2)
    const uint32_t* seg;        // [nranks] segment starts (pass 2)
    RouteRec* out;
    int pass;
};

__device__ __forceinline__ int origin_rank(const RouteArgs& a, uint32_t w) {
    const int g[3] = {(int)(w & a.mx), (int)((w >> a.bx) & a.my), (int)(w >> (a.bx + a.by))};
    const int nc[3] = {a.ncuts0, a.ncuts1, a.ncuts2};
    int c[3];
    for (int ax = 0; ax < 3; ++ax) {
        int k = 0;
        while (k + 1 < nc[ax] - 1 && a.cuts[ax * kMaxCuts + k + 1] <= g[ax]) ++k;
        c[ax] = k;
    }
    return c[0] + a.lay0 * (c[1] + a.lay1 * c[2]);
}

__global__ void route_kernel(RouteArgs a) {
    const int64_t n_live = (int64_t)a.words[W_NTILES] * kTile;
    uint32_t n_dead = a.words[W_DEAD];
    if (n_dead > a.dead_cap) n_dead = a.dead_cap;
    const int64_t total = n_live + n_dead;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        float4 r;
        uint32_t info;
        if (i < n_live) {
            if ((int)(i % kTile) >= a.tile_count[i / kTile]) continue;
            r = a.state[i];
            info = 0u;
        } else {
            r = a.dead_rec[i - n_live];
            info = a.dead_info[i - n_live];
        }
        const int o = origin_rank(a, __float_as_uint(r.w));
        if (o == a.me) continue;
        if (a.pass == 0) {
            atomicAdd(&a.count[o], 1u);
        } else {
            const uint32_t p = a.seg[o] + atomicAdd(&a.pos[o], 1u);
            RouteRec rr;
            rr.rec = r; rr.info = info; rr.pad[0] = rr.pad[1] = rr.pad[2] = 0;
            a.out[p] = rr;
        }
    }
}

}  // namespace lag

// ---------------------------------------------------------------------------
// host side

static int off_index(const int o[3]) { return (o[0] + 1) + 3 * ((o[1] + 1) + 3 * (o[2] + 1)); }
static lag_status comm_setup(lag_ctx_s* ctx);

lag_status lag_comm_init(lag_ctx_s* ctx) {
    const lag_config& c = ctx->cfg;
    Comm* cm = new Comm();
    ctx->comm = cm;
    cm->me[0] = c.rank % c.layout[0];
    cm->me[1] = (c.rank / c.layout[0]) % c.layout[1];
    cm->me[2] = c.rank / (c.layout[0] * c.layout[1]);
    cm->blocks.assign((size_t)c.nranks * 6, 0);
    int64_t mine[6] = {c.block_lo[0], c.block_lo[1], c.block_lo[2], c.block_hi[0], c.block_hi[1], c.block_hi[2]};
    if (c.exchange == LAG_XCHG_LOCAL) {
        // the other blocks are contexts of this process: lag_local_group
        // fills the block table and finishes the setup
        return LAG_OK;
    }
    if (c.nranks > 1) {
        ncclUniqueId id;
        std::memcpy(&id, c.nccl_id, sizeof(id));
        CKN(ncclCommInitRank(&cm->nccl, c.nranks, id, c.rank));
        int64_t* d = nullptr;
        CKC(cudaMalloc(&d, sizeof(int64_t) * 6 * (c.nranks + 1)));
        CKC(cudaMemcpyAsync(d, mine, sizeof(mine), cudaMemcpyHostToDevice, ctx->stream));
        CKN(ncclAllGather(d, d + 6, 6, ncclInt64, cm->nccl, ctx->stream));
        CKC(cudaMemcpyAsync(cm->blocks.data(), d + 6, sizeof(int64_t) * 6 * c.nranks, cudaMemcpyDeviceToHost, ctx->stream));
        CKC(cudaStreamSynchronize(ctx->stream));
        cudaFree(d);
    } else {
        std::copy(mine, mine + 6, cm->blocks.begin());
    }
    return comm_setup(ctx);
}

// Neighbours, ghost boxes, particle slots and routing tables from the block
// table cm->blocks (every rank's [lo, hi)).
static lag_status comm_setup(lag_ctx_s* ctx) {
    const lag_config& c = ctx->cfg;
    Comm* cm = ctx->comm;
    const int D = c.dim;
    const int G = c.ghost;
    const int64_t* mine = &cm->blocks[(size_t)c.rank * 6];
    // per-axis cut points (block lo values along each axis, plus N)
    for (int ax = 0; ax < 3; ++ax) {
        std::vector<int32_t> v;
        for (int r = 0; r < c.nranks; ++r) v.push_back((int32_t)cm->blocks[(size_t)r * 6 + ax]);
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        if ((int)v.size() != c.layout[ax] || (int)v.size() + 1 > kMaxCuts) {
            lag_set_error(ctx, "blocks do not form the declared layout on axis %d", ax);
            return LAG_EINVAL;
        }
        v.push_back((int32_t)c.global_nodes[ax]);
        cm->ncuts[ax] = (int)v.size();
        for (size_t k = 0; k < v.size(); ++k) cm->cuts[ax][k] = v[k];
    }
    // neighbours, halo boxes, slot capacities
    auto top = [&](const int64_t* b, int ax) { return std::min(b[3 + ax] + 1, c.global_nodes[ax]); };
    const int64_t* my = mine;
    int64_t send_off = 0, recv_off = 0, slot_off = 0;
    for (int oz = (D == 3 ? -1 : 0); oz <= (D == 3 ? 1 : 0); ++oz)
        for (int oy = -1; oy <= 1; ++oy)
            for (int ox = -1; ox <= 1; ++ox) {
                const int o[3] = {ox, oy, oz};
                const int k = off_index(o);
                // particle slot capacity by neighbour kind: faces get a full face of nodes
                int64_t cap = 64;
                {
                    int nz = 0;
                    int64_t area = 1;
                    for (int ax = 0; ax < D; ++ax) {
                        if (o[ax] == 0) area *= (my[3 + ax] - my[ax]);
                        else ++nz;
                    }
                    if (ox == 0 && oy == 0 && oz == 0) cap = 0;
                    else if (nz == 1) cap = area + 1024;
                    else if (nz == 2 && D == 3) cap = area + 256;
                    else cap = 64 + (D == 2 ? area : 0);
                }
                cm->slot_base[k] = (int32_t)slot_off;
                cm->slot_capv[k] = (int32_t)cap;
                slot_off += cap + 1;
                if (ox == 0 && oy == 0 && oz == 0) continue;
                int nbc[3];
                bool ok = true;
                for (int ax = 0; ax < 3; ++ax) {
                    nbc[ax] = cm->me[ax] + o[ax];
                    if (nbc[ax] < 0 || nbc[ax] >= c.layout[ax]) ok = false;
                }
                if (!ok) continue;
                const int nr = nbc[0] + c.layout[0] * (nbc[1] + c.layout[1] * nbc[2]);
                const int64_t* nb = &cm->blocks[(size_t)nr * 6];
                Box rb{}, sb{};
                int64_t rlo[3], rn[3], slo[3], sn[3];
                for (int ax = 0; ax < 3; ++ax) {
                    if (ax >= D) { rlo[ax] = 0; rn[ax] = 1; slo[ax] = 0; sn[ax] = 1; continue; }
                    // my ghost region filled by this neighbour
                    if (o[ax] < 0) { rlo[ax] = my[ax] - G; rn[ax] = G; }
                    else if (o[ax] == 0) { rlo[ax] = my[ax]; rn[ax] = top(my, ax) - my[ax]; }
                    else { rlo[ax] = top(my, ax); rn[ax] = G; }
                    // the neighbour's ghost region (offset -o) that I fill
                    if (-o[ax] < 0) { slo[ax] = nb[ax] - G; sn[ax] = G; }
                    else if (o[ax] == 0) { slo[ax] = nb[ax]; sn[ax] = top(nb, ax) - nb[ax]; }
                    else { slo[ax] = top(nb, ax); sn[ax] = G; }
                    if (slo[ax] < my[ax] || slo[ax] + sn[ax] > top(my, ax)) {
                        lag_set_error(ctx, "block too thin for %d ghost layers on axis %d", G, ax);
                        return LAG_EINVAL;
                    }
                }
                auto local = [&](const int64_t* lo3, const int64_t* n3, int64_t off) {
                    Box b{};
                    b.x0 = (int)(lo3[0] - ctx->base[0]); b.y0 = (int)(lo3[1] - ctx->base[1]); b.z0 = (int)(lo3[2] - ctx->base[2]);
                    b.nx = (int)n3[0]; b.ny = (int)n3[1]; b.nz = (int)n3[2];
                    b.off = off; b.slice = 1;
                    return b;
                };
                sb = local(slo, sn, send_off);
                rb = local(rlo, rn, recv_off);
                Peer p{};
                p.rank = nr;
                p.off = k;
                const int ob[3] = {-o[0], -o[1], -o[2]};
                p.back = off_index(ob);
                p.send_box = (int)cm->send_boxes.size();
                p.recv_box = (int)cm->recv_boxes.size();
                p.halo_floats_send = sn[0] * sn[1] * sn[2] * D;
                p.halo_floats_recv = rn[0] * rn[1] * rn[2] * D;
                send_off += p.halo_floats_send;
                recv_off += p.halo_floats_recv;
                cm->send_boxes.push_back(sb);
                cm->recv_boxes.push_back(rb);
                cm->peers.push_back(p);
            }
    cm->halo_send_floats = send_off;
    cm->halo_recv_floats = recv_off;
    cm->slot_total = slot_off;
    // the receive capacity from a peer = the peer's send capacity toward me:
    // the same formula evaluated with the peer's block
    for (Peer& p : cm->peers) {
        const int64_t* nb = &cm->blocks[(size_t)p.rank * 6];
        int o[3] = {0, 0, 0};
        {
            int k = p.back;
            o[0] = k % 3 - 1; o[1] = (k / 3) % 3 - 1; o[2] = k / 9 - 1;
        }
        int nz = 0;
        int64_t area = 1;
        for (int ax = 0; ax < D; ++ax) {
            if (o[ax] == 0) area *= (nb[3 + ax] - nb[ax]);
            else ++nz;
        }
        int64_t cap = nz == 1 ? area + 1024 : ((nz == 2 && D == 3) ? area + 256 : 64 + (D == 2 ? area : 0));
        p.cap_send = (uint32_t)cm->slot_capv[p.off];
        p.cap_recv = (uint32_t)cap;
        cm->recv_total += cap + 1;
    }
    // device buffers
    const size_t np = cm->peers.size();
    std::vector<Box> sb2(cm->send_boxes), rb2(cm->recv_boxes);
    for (size_t i = 0; i < np; ++i) {   // v0 copies of the boxes follow the v1 ones
        Box b = cm->send_boxes[i]; b.slice = 0; b.off += send_off; sb2.push_back(b);
        Box r = cm->recv_boxes[i]; r.slice = 0; r.off += recv_off; rb2.push_back(r);
    }
    CKC(cudaMalloc(&cm->d_send_boxes, sizeof(Box) * std::max<size_t>(1, sb2.size())));
    CKC(cudaMalloc(&cm->d_recv_boxes, sizeof(Box) * std::max<size_t>(1, rb2.size())));
    if (!sb2.empty()) {
        CKC(cudaMemcpy(cm->d_send_boxes, sb2.data(), sizeof(Box) * sb2.size(), cudaMemcpyHostToDevice));
        CKC(cudaMemcpy(cm->d_recv_boxes, rb2.data(), sizeof(Box) * rb2.size(), cudaMemcpyHostToDevice));
    }
    CKC(cudaMalloc(&cm->halo_send, sizeof(float) * std::max<int64_t>(1, 2 * send_off)));
    CKC(cudaMalloc(&cm->halo_recv, sizeof(float) * std::max<int64_t>(1, 2 * recv_off)));
    CKC(cudaMalloc(&cm->slots, sizeof(float4) * std::max<int64_t>(1, cm->slot_total)));
    CKC(cudaMemset(cm->slots, 0, sizeof(float4) * std::max<int64_t>(1, cm->slot_total)));
    CKC(cudaMalloc(&cm->recv_slots, sizeof(float4) * std::max<int64_t>(1, cm->recv_total)));
    {
        int64_t off = 0;
        for (Peer& p : cm->peers) { p.recv_slot = cm->recv_slots + off; off += p.cap_recv + 1; }
    }
    CKC(cudaMalloc(&cm->d_cuts, sizeof(int32_t) * 3 * kMaxCuts));
    CKC(cudaMemcpy(cm->d_cuts, cm->cuts, sizeof(int32_t) * 3 * kMaxCuts, cudaMemcpyHostToDevice));
    CKC(cudaMalloc(&cm->d_route_count, sizeof(uint32_t) * 2 * std::max(1, c.nranks)));
    cm->d_route_pos = cm->d_route_count + c.nranks;
    CKC(cudaMalloc(&cm->d_seg, sizeof(uint32_t) * (c.nranks + 1)));
    CKC(cudaMalloc(&cm->d_all, sizeof(uint32_t) * c.nranks * (c.nranks + 1)));
    // return-to-origin buffers (LAG_XCHG_LOCAL gathers from the group's lists instead)
    cm->route_cap = c.exchange == LAG_XCHG_LOCAL ? 1 : ctx->cap;
    CKC(cudaMalloc(&cm->route, sizeof(RouteRec) * std::max<int64_t>(1, cm->route_cap)));
    CKC(cudaMalloc(&cm->route_recv, sizeof(RouteRec) * std::max<int64_t>(1, cm->route_cap)));
    for (const Peer& p : cm->peers) { cm->prank.push_back(p.rank); cm->poff.push_back(p.off); cm->pback.push_back(p.back); }
    if ((c.exchange == LAG_XCHG_PEER || c.exchange == LAG_XCHG_PEER_OVERLAP) && !cm->peers.empty()) {
        std::vector<uint32_t> caps;
        std::vector<int64_t> send_off, send_by_off(kMaxOff, 0);
        std::vector<int> rbox;
        for (const Peer& p : cm->peers) {
            caps.push_back(p.cap_send);
            const Box& sb = cm->send_boxes[(size_t)p.send_box];
            send_off.push_back(sb.off);
            send_by_off[p.off] = sb.off;
            const Box& rb = cm->recv_boxes[(size_t)p.recv_box];
            rbox.insert(rbox.end(), {rb.x0, rb.y0, rb.z0, rb.nx, rb.ny, rb.nz});
        }
        lag_status st = lag_peer_init(ctx, cm->nccl, cm->prank, cm->poff, cm->pback, caps,
                                      cm->halo_send_floats, send_off, send_by_off, rbox,
                                      cm->halo_recv_floats, &cm->peer);
        if (st != LAG_OK) return st;
    }
    return LAG_OK;
}

void lag_comm_destroy(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    if (!cm) return;
    lag_peer_destroy(cm->peer);
    if (cm->nccl) ncclCommDestroy(cm->nccl);
    cudaFree(cm->d_send_boxes); cudaFree(cm->d_recv_boxes);
    cudaFree(cm->halo_send); cudaFree(cm->halo_recv);
    cudaFree(cm->slots); cudaFree(cm->recv_slots); cudaFree(cm->d_cuts);
    cudaFree(cm->d_route_count); cudaFree(cm->route); cudaFree(cm->route_recv);
    cudaFree(cm->d_seg); cudaFree(cm->d_all);
    delete cm;
    ctx->comm = nullptr;
}

static void local_unrecord(lag_ctx_s* ctx);
static AppendArgs append_args(lag_ctx_s* ctx, int peer_parity, int cnt_parity = 0);

lag_status lag_comm_reset(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    local_unrecord(ctx);
    // peer transports, reseed in the middle of an interval: the last cycle's
    // hand-offs stay in the senders' own slots and are never read (the next
    // exchange appends only while an interval is pending on this rank, and
    // lag_seed is collective); each slot is reset before it is written again.
    // Empty outgoing slots (NCCL); nothing pending (seed_kernel sets W_NTILES)
    CKC(cudaMemsetAsync(cm->slots, 0, sizeof(float4) * std::max<int64_t>(1, cm->slot_total), ctx->stream));
    cm->pending = false;
    cm->n_returned = 0;
    return LAG_OK;
}

static lag_status launch_append(lag_ctx_s* ctx, int peer_parity = -1) {
    AppendArgs a = append_args(ctx, peer_parity);
    append_kernel<<<ctx->num_sms, 256, 0, ctx->stream>>>(a);
    ++ctx->launches;
    CKC(cudaGetLastError());
    return LAG_OK;
}

// peer_parity >= 0: the neighbours' own slots of that parity (peer
// transports, read remotely; the senders reset them), with the counts they
// published in my count words of parity cnt_parity; otherwise the slots NCCL
// delivered, and my sent slots are reset
static AppendArgs append_args(lag_ctx_s* ctx, int peer_parity, int cnt_parity) {
    Comm* cm = ctx->comm;
    AppendArgs a{};
    a.state = ctx->state; a.tile_count = ctx->tile_count; a.words = ctx->words;
    a.counters = ctx->counters; a.cap_tiles = ctx->cap_tiles;
    a.npeers = (int)cm->peers.size();
    for (size_t i = 0; i < cm->peers.size(); ++i) {
        const Peer& p = cm->peers[i];
        a.recv[i] = peer_parity >= 0 ? lag_peer_remote_slot(cm->peer, (int)i, p.rank, p.back, peer_parity)
                                     : p.recv_slot;
        a.cnt[i] = peer_parity >= 0 ? lag_peer_my_count(cm->peer, cnt_parity, p.off) : nullptr;
        a.cap[i] = p.cap_recv;
    }
    a.reset = peer_parity >= 0 ? RESET_NONE : RESET_SLOTS;
    a.slots = cm->slots;
    a.noff = kMaxOff;                               // all 27 offset headers (2-D uses 9..17)
    for (int k = 0; k < kMaxOff; ++k) a.slot_base[k] = cm->slot_base[k];
    return a;
}

// One NCCL group: optional halo boxes (v1 [+ v0]) and the pending particle slots.
// CTAs per box row: enough for the largest box at one float per thread (<= 64)
static int box_ctas(const Comm* cm) {
    int64_t mx = 1;
    for (const Box& b : cm->send_boxes) mx = std::max<int64_t>(mx, (int64_t)b.nx * b.ny * b.nz);
    for (const Box& b : cm->recv_boxes) mx = std::max<int64_t>(mx, (int64_t)b.nx * b.ny * b.nz);
    return (int)std::max<int64_t>(1, std::min<int64_t>((3 * mx + 255) / 256, 64));
}

static lag_status exchange(lag_ctx_s* ctx, float* v0, float* v1, bool halo, bool halo_v0) {
    Comm* cm = ctx->comm;
    const int D = ctx->cfg.dim;
    const size_t np = cm->peers.size();
    if (np == 0) return LAG_OK;
    const int nbox = halo ? (int)(halo_v0 ? 2 * np : np) : 0;
    const int64_t sfl = halo ? (halo_v0 ? 2 : 1) * cm->halo_send_floats : 0;
    const int64_t rfl = halo ? (halo_v0 ? 2 : 1) * cm->halo_recv_floats : 0;
    if (halo && sfl > 0) {
        BoxArgs b{};
        b.v0 = v0; b.v1 = v1; b.v0w = v0; b.boxes = cm->d_send_boxes; b.nbox = nbox;
        b.buf = cm->halo_send; b.sx = ctx->sx; b.sxy = ctx->sxy; b.dim = D; b.total = sfl;
        halo_pack_kernel<<<dim3(box_ctas(cm), (unsigned)nbox), 256, 0, ctx->stream>>>(b);
        ++ctx->launches;
        CKC(cudaGetLastError());
    }
    CKN(ncclGroupStart());
    for (const Peer& p : cm->peers) {
        if (halo) {
            const Box& s = cm->send_boxes[(size_t)p.send_box];
            const Box& r = cm->recv_boxes[(size_t)p.recv_box];
            CKN(ncclSend(cm->halo_send + s.off, p.halo_floats_send, ncclFloat32, p.rank, cm->nccl, ctx->stream));
            CKN(ncclRecv(cm->halo_recv + r.off, p.halo_floats_recv, ncclFloat32, p.rank, cm->nccl, ctx->stream));
            if (halo_v0) {
                CKN(ncclSend(cm->halo_send + cm->halo_send_floats + s.off, p.halo_floats_send, ncclFloat32, p.rank, cm->nccl, ctx->stream));
                CKN(ncclRecv(cm->halo_recv + cm->halo_recv_floats + r.off, p.halo_floats_recv, ncclFloat32, p.rank, cm->nccl, ctx->stream));
            }
        }
        // particle slot toward this peer: header + cap records (float4 = 4 floats)
        CKN(ncclSend(cm->slots + cm->slot_base[p.off], (size_t)(p.cap_send + 1) * 4, ncclFloat32, p.rank, cm->nccl, ctx->stream));
        CKN(ncclRecv(p.recv_slot, (size_t)(p.cap_recv + 1) * 4, ncclFloat32, p.rank, cm->nccl, ctx->stream));
    }
    CKN(ncclGroupEnd());
    if (halo && rfl > 0) {
        BoxArgs b{};
        b.v0 = v0; b.v1 = v1; b.v0w = v0; b.boxes = cm->d_recv_boxes; b.nbox = nbox;
        b.buf = cm->halo_recv; b.sx = ctx->sx; b.sxy = ctx->sxy; b.dim = D; b.total = rfl;
        const AppendArgs ap = append_args(ctx, -1);
        const int app_ctas = 16;
        halo_unpack_append_kernel<<<dim3(std::max(app_ctas, box_ctas(cm)), (unsigned)(nbox + 1)), 256, 0, ctx->stream>>>(b, ap, app_ctas);
        ++ctx->launches;
        CKC(cudaGetLastError());
        return LAG_OK;
    }
    return launch_append(ctx);
}

// Peer transport, one cycle: one fused exchange kernel (lag_peer.cu).
static lag_status peer_pre_advect(lag_ctx_s* ctx, float* v0, float* v1, bool with_v0) {
    Comm* cm = ctx->comm;
    const unsigned long long seq = ++lag_peer_seq(cm->peer);
    // hand-offs of cycle seq-1, unless this is the first cycle of an interval
    const AppendArgs ap = append_args(ctx, (int)((seq - 1) % 3), (int)(seq & 1));
    return lag_peer_exchange(ctx, cm->peer, cm->d_send_boxes, (int)cm->peers.size(), cm->halo_send_floats,
                             v0, v1, with_v0, true, cm->poff, cm->pback, cm->pending ? &ap : nullptr);
}

bool lag_comm_overlap(lag_ctx_s* ctx) {
    return ctx->comm && ctx->comm->peer && !ctx->comm->peers.empty() &&
           ctx->cfg.exchange == LAG_XCHG_PEER_OVERLAP;
}

lag_status lag_comm_pre_advect(lag_ctx_s* ctx, float* v0, float* v1, bool v0_is_prev_v1) {
    Comm* cm = ctx->comm;
    if (cm->peers.empty()) return LAG_OK;
    lag_status st = cm->peer ? peer_pre_advect(ctx, v0, v1, !v0_is_prev_v1)
                             : exchange(ctx, v0, v1, true, !v0_is_prev_v1);
    cm->pending = false;
    return st;
}

void lag_comm_fill_args(lag_ctx_s* ctx, AdvectArgs* a) {
    Comm* cm = ctx->comm;
    a->slot_rec = cm->slots;
    for (int k = 0; k < kMaxOff; ++k) {
        a->slot_base[k] = cm->slot_base[k];
        a->slot_capv[k] = cm->slot_capv[k];
        a->slot_ptr[k] = cm->slots + cm->slot_base[k];
    }
    if (cm->peer) {                  // my own slots of this cycle's parity (read by the neighbours)
        const unsigned long long seq = lag_peer_seq(cm->peer);
        for (size_t i = 0; i < cm->peers.size(); ++i)
            a->slot_ptr[cm->peers[i].off] = lag_peer_my_slot(cm->peer, (int)(seq % 3), cm->peers[i].off);
    }
}

lag_status lag_comm_post_advect(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    cm->pending = !cm->peers.empty();       // this cycle's hand-offs wait in the slots
    return LAG_OK;
}

// Write cycle: flush pending hand-offs, then route every record whose seed
// belongs to another rank back to it (exact sizes; untimed, host syncs allowed).
lag_status lag_comm_return_to_origin(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    const lag_config& c = ctx->cfg;
    cm->n_returned = 0;
    if (c.nranks == 1) return LAG_OK;
    if (cm->pending) {
        lag_status st;
        if (cm->peer) {
            const unsigned long long seq = lag_peer_seq(cm->peer);
            const AppendArgs ap = append_args(ctx, (int)(seq % 3), (int)((seq + 1) & 1));
            st = lag_peer_exchange(ctx, cm->peer, cm->d_send_boxes, (int)cm->peers.size(), 0,
                                   nullptr, nullptr, false, false, cm->poff, cm->pback, &ap);
        } else {
            st = exchange(ctx, nullptr, nullptr, false, false);
        }
        if (st != LAG_OK) return st;
        cm->pending = false;
    }
    const int R = c.nranks;
    RouteArgs ra{};
    ra.state = ctx->state; ra.tile_count = ctx->tile_count; ra.words = ctx->words;
    ra.dead_rec = ctx->dead_rec; ra.dead_info = ctx->dead_info; ra.dead_cap = (uint32_t)ctx->cap;
    ra.cuts = cm->d_cuts; ra.ncuts0 = cm->ncuts[0]; ra.ncuts1 = cm->ncuts[1]; ra.ncuts2 = cm->ncuts[2];
    ra.lay0 = c.layout[0]; ra.lay1 = c.layout[1];
    ra.bx = ctx->bits[0]; ra.by = ctx->bits[1];
    ra.mx = (1u << ctx->bits[0]) - 1u; ra.my = (1u << ctx->bits[1]) - 1u;
    ra.me = c.rank;
    ra.count = cm->d_route_count; ra.pos = cm->d_route_pos;
    std::vector<uint32_t> seg(R + 1, 0), cnt(R, 0);
    uint32_t* d_seg = cm->d_seg;
    CKC(cudaMemsetAsync(cm->d_route_count, 0, sizeof(uint32_t) * 2 * R, ctx->stream));
    const int blocks = ctx->num_sms * 4;
    ra.pass = 0;
    route_kernel<<<blocks, 256, 0, ctx->stream>>>(ra);
    ++ctx->launches;
    CKC(cudaMemcpyAsync(cnt.data(), cm->d_route_count, sizeof(uint32_t) * R, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    for (int r = 0; r < R; ++r) seg[r + 1] = seg[r] + cnt[r];
    if (seg[R] > (uint32_t)cm->route_cap) { lag_set_error(ctx, "route buffer overflow"); return LAG_EOVERFLOW; }
    CKC(cudaMemcpyAsync(d_seg, seg.data(), sizeof(uint32_t) * (R + 1), cudaMemcpyHostToDevice, ctx->stream));
    ra.pass = 1; ra.seg = d_seg; ra.out = cm->route;
    route_kernel<<<blocks, 256, 0, ctx->stream>>>(ra);
    ++ctx->launches;
    // exchange the counts: everyone learns how much it receives from whom
    uint32_t* d_all = cm->d_all;
    CKC(cudaMemcpyAsync(d_all, cnt.data(), sizeof(uint32_t) * R, cudaMemcpyHostToDevice, ctx->stream));
    CKN(ncclAllGather(d_all, d_all + R, R, ncclUint32, cm->nccl, ctx->stream));
    std::vector<uint32_t> all((size_t)R * R);
    CKC(cudaMemcpyAsync(all.data(), d_all + R, sizeof(uint32_t) * R * R, cudaMemcpyDeviceToHost, ctx->stream));
    CKC(cudaStreamSynchronize(ctx->stream));
    std::vector<uint32_t> rseg(R + 1, 0);
    for (int r = 0; r < R; ++r) rseg[r + 1] = rseg[r] + (r == c.rank ? 0 : all[(size_t)r * R + c.rank]);
    if (rseg[R] > (uint32_t)cm->route_cap) { lag_set_error(ctx, "route receive overflow"); return LAG_EOVERFLOW; }
    CKN(ncclGroupStart());
    for (int r = 0; r < R; ++r) {
        if (r == c.rank) continue;
        if (cnt[r]) CKN(ncclSend(cm->route + seg[r], (size_t)cnt[r] * sizeof(RouteRec), ncclUint8, r, cm->nccl, ctx->stream));
        const uint32_t in = all[(size_t)r * R + c.rank];
        if (in) CKN(ncclRecv(cm->route_recv + rseg[r], (size_t)in * sizeof(RouteRec), ncclUint8, r, cm->nccl, ctx->stream));
    }
    CKN(ncclGroupEnd());
    CKC(cudaStreamSynchronize(ctx->stream));
    cm->n_returned = rseg[R];
    return LAG_OK;
}

// Returned records for extract (valid when lag_comm_return_to_origin ran).
void lag_comm_returned(lag_ctx_s* ctx, const float4** rec, int64_t* stride_f4, uint32_t* n) {
    Comm* cm = ctx->comm;
    *rec = cm ? reinterpret_cast<const float4*>(cm->route_recv) : nullptr;
    *stride_f4 = sizeof(RouteRec) / sizeof(float4);
    *n = cm ? cm->n_returned : 0;
}

extern "C" lag_status lag_nccl_unique_id(void* out, int64_t out_bytes) {
    lag_ctx_s* ctx = nullptr;
    if (!out || out_bytes < (int64_t)sizeof(ncclUniqueId)) {
        lag_set_error(nullptr, "need %zu bytes for ncclUniqueId", sizeof(ncclUniqueId));
        return LAG_EINVAL;
    }
    ncclUniqueId id;
    CKN(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
    return LAG_OK;
}

lag_status lag_comm_async_error(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    if (!cm || !cm->nccl) return LAG_OK;
    ncclResult_t res = ncclSuccess;
    CKN(ncclCommGetAsyncError(cm->nccl, &res));
    if (res != ncclSuccess && res != ncclInProgress) {
        lag_set_error(ctx, "NCCL communicator asynchronous error: %s", ncclGetErrorString(res));
        return LAG_ENCCL;
    }
    return LAG_OK;
}

// ---------------------------------------------------------------------------
// LAG_XCHG_LOCAL: the blocks of a decomposition as contexts of one process on
// one device, each on its own stream.  Per group cycle (enqueued by the call
// that completes it; events replace every flag and wait):
//   0. the group stream (block 0's) waits for every block's stream;
//   1. one kernel copies every block's ghost layers of v_t1 (and of v_t when
//      it is not the previous call's v_t1) from the neighbours' slice arrays;
//   2. one kernel (blockIdx.y = block) appends to each block the hand-offs
//      the neighbours' advect kernels left in their slots toward it (the
//      previous cycle's, as in the NCCL transport) and zeroes those headers;
//   3. every block's stream waits for that, then runs its advect kernel
//      (lag_api.cu), which writes leaving particles to its own slots; the
//      blocks advance concurrently.
// The write cycle joins the streams, appends the last hand-offs once, and
// each block gathers its basis flows from every block's lists (lag_api.cu);
// the streams join again before the group reseeds.

namespace lag {
constexpr int kLocalMax = 64;
constexpr int kLocalAppendCtas = 8;   // a block receives a few hundred hand-offs per cycle
struct LocalBox {               // ghost box of block dst filled from block src's interior
    int dst, src;
    int dx0, dy0, dz0;          // dst slice coordinates
    int sx0, sy0, sz0;          // src slice coordinates
    int nx, ny, nz;
    int64_t off;                // float offset in the flattened copy (one slice)
};
struct LocalCopyArgs {
    const LocalBox* boxes;
    int nbox;
    int nybox;                  // grid rows running ghost boxes (nbox, or 2 nbox with v_t boxes)
    const AppendArgs* app;      // [n] per-block append arguments (rows nybox .. nybox + n - 1)
    int app_ctas;               // CTAs per block's append
    int dim;
    int64_t total;              // floats over all boxes (one slice)
    unsigned long long fill_v0; // bit r: block r's v_t needs its ghosts too
    float* v0[kLocalMax];
    float* v1[kLocalMax];
    int sx[kLocalMax], sxy[kLocalMax];
};

// every block's append in one launch: blockIdx.y = block (AppendArgs are
// fixed for the group's lifetime: lists, words, the neighbours' slots)
__global__ void __launch_bounds__(256) local_append_kernel(const AppendArgs* __restrict__ app) {
    const AppendArgs& a = app[blockIdx.y];
    if (a.npeers == 0) return;
    append_body(a, blockIdx.x, gridDim.x);
}

// blockIdx.y = ghost box (v_t1 boxes, then the v_t boxes of the blocks whose
// v_t is not the previous call's v_t1); the CTAs of a row stride over the
// box's floats (32-bit index math: a box is far below 2^31 floats)
__global__ void __launch_bounds__(256) local_ghost_kernel(const LocalCopyArgs a) {
    const int y = blockIdx.y;
    if (y >= a.nybox) {                                 // grid row of a block's append
        if ((int)blockIdx.x >= a.app_ctas) return;
        const AppendArgs& ap = a.app[y - a.nybox];
        if (ap.npeers) append_body(ap, blockIdx.x, a.app_ctas);
        return;
    }
    const int slice = y < a.nbox ? 1 : 0;
    const LocalBox& b = a.boxes[slice ? y : y - a.nbox];
    if (!slice && !((a.fill_v0 >> b.dst) & 1ull)) return;
    const int dim = a.dim;
    const int nf = b.nx * b.ny * b.nz * dim;
    const int rowf = b.nx * dim;
    const float* src = slice ? a.v1[b.src] : a.v0[b.src];
    float* dst = slice ? a.v1[b.dst] : a.v0[b.dst];
    const int ssx = a.sx[b.src], ssxy = a.sxy[b.src], dsx = a.sx[b.dst], dsxy = a.sxy[b.dst];
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nf; k += gridDim.x * blockDim.x) {
        const int row = k / rowf, within = k - row * rowf;
        const int yy = row % b.ny, zz = row / b.ny;
        dst[(int64_t)dim * (b.dx0 + (int64_t)dsx * (b.dy0 + yy) + (int64_t)dsxy * (b.dz0 + zz)) + within] =
            src[(int64_t)dim * (b.sx0 + (int64_t)ssx * (b.sy0 + yy) + (int64_t)ssxy * (b.sz0 + zz)) + within];
    }
}

struct LocalGroup {
    std::vector<lag_ctx_s*> m;          // rank -> context (nullptr once destroyed)
    std::vector<lag_local_rec> rec;
    std::vector<char> has;              // recorded in the current group cycle
    int nrec = 0;
    std::vector<char> extracted;
    int nextracted = 0;
    std::vector<LocalBox> boxes;
    LocalBox* d_boxes = nullptr;
    int64_t total = 0;
    int max_box_floats = 0;
    AppendArgs* d_app = nullptr;        // [n] per-block append arguments
    std::vector<cudaEvent_t> ev;        // per block: join points
    int alive = 0;
};
}  // namespace lag

static AppendArgs local_append_args(lag_ctx_s* ctx) {
    Comm* cm = ctx->comm;
    LocalGroup* g = ctx->group;
    AppendArgs a{};
    a.state = ctx->state; a.tile_count = ctx->tile_count; a.words = ctx->words;
    a.counters = ctx->counters; a.cap_tiles = ctx->cap_tiles;
    a.npeers = (int)cm->peers.size();
    for (size_t i = 0; i < cm->peers.size(); ++i) {
        const Peer& p = cm->peers[i];
        const Comm* pc = g->m[p.rank]->comm;            // the neighbour's slot toward me
        a.recv[i] = pc->slots + pc->slot_base[p.back];
        a.cap[i] = (uint32_t)pc->slot_capv[p.back];
    }
    a.reset = RESET_RECV;                               // each slot has exactly one reader: me
    a.noff = 0;
    return a;
}

// The group stream waits for every block's stream (fan-in).
static lag_status local_join_in(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    if (!g->m[0]) { lag_set_error(ctx, "LAG_XCHG_LOCAL: block 0 of the group was destroyed"); return LAG_ESTATE; }
    cudaStream_t s0 = g->m[0]->stream;
    for (size_t r = 1; r < g->m.size(); ++r) {
        if (!g->m[r] || g->m[r]->stream == s0) continue;
        CKC(cudaEventRecord(g->ev[r], g->m[r]->stream));
        CKC(cudaStreamWaitEvent(s0, g->ev[r], 0));
    }
    return LAG_OK;
}

// Every block's stream waits for the group stream (fan-out).
static lag_status local_join_out(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    if (!g->m[0]) { lag_set_error(ctx, "LAG_XCHG_LOCAL: block 0 of the group was destroyed"); return LAG_ESTATE; }
    cudaStream_t s0 = g->m[0]->stream;
    CKC(cudaEventRecord(g->ev[0], s0));
    for (size_t r = 1; r < g->m.size(); ++r)
        if (g->m[r] && g->m[r]->stream != s0) CKC(cudaStreamWaitEvent(g->m[r]->stream, g->ev[0], 0));
    return LAG_OK;
}

// Appends of every block (one launch on the group stream).
static lag_status local_appends(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    lag_ctx_s* c0 = g->m[0];
    bool any = false;
    for (lag_ctx_s* c : g->m) any |= !c->comm->peers.empty();
    if (!any) return LAG_OK;
    local_append_kernel<<<dim3(kLocalAppendCtas, (unsigned)g->m.size()), 256, 0, c0->stream>>>(g->d_app);
    ++ctx->launches;
    CKC(cudaGetLastError());
    for (lag_ctx_s* c : g->m) c->comm->pending = false;
    return LAG_OK;
}

extern "C" lag_status lag_local_group(lag_ctx* ctxs, int32_t n) {
    lag_ctx_s* ctx = nullptr;
    if (!ctxs || n < 1 || n > kLocalMax) { lag_set_error(nullptr, "lag_local_group: need 1..%d contexts", kLocalMax); return LAG_EINVAL; }
    for (int r = 0; r < n; ++r) {
        lag_ctx_s* c = ctxs[r];
        if (!c || c->cfg.mode != LAG_COMM || c->cfg.exchange != LAG_XCHG_LOCAL || c->cfg.rank != r ||
            c->cfg.nranks != n || c->cfg.device != ctxs[0]->cfg.device ||
            c->cfg.dim != ctxs[0]->cfg.dim || (c->cfg.ghost < 1 && n > 1)) {
            lag_set_error(nullptr, "lag_local_group: context %d is not rank %d of an n = %d LAG_XCHG_LOCAL "
                          "COMM group on the same device", r, r, n);
            return LAG_EINVAL;
        }
        for (int a = 0; a < 3; ++a)
            if (c->cfg.global_nodes[a] != ctxs[0]->cfg.global_nodes[a] || c->cfg.layout[a] != ctxs[0]->cfg.layout[a]) {
                lag_set_error(nullptr, "lag_local_group: context %d has another grid or layout", r);
                return LAG_EINVAL;
            }
        if (c->group || c->seeded || c->comm->slots) {
            // (a failed earlier call may have set up some blocks: destroy the
            // contexts and create them again)
            lag_set_error(nullptr, "lag_local_group: context %d is already grouped, set up or seeded", r);
            return LAG_ESTATE;
        }
    }
    for (int r = 0; r < n; ++r) {
        ctx = ctxs[r];
        Comm* cm = ctx->comm;
        for (int q = 0; q < n; ++q)
            for (int a = 0; a < 3; ++a) {
                cm->blocks[(size_t)q * 6 + a] = ctxs[q]->cfg.block_lo[a];
                cm->blocks[(size_t)q * 6 + 3 + a] = ctxs[q]->cfg.block_hi[a];
            }
        lag_status st = comm_setup(ctx);
        if (st != LAG_OK) { lag_set_error(nullptr, "lag_local_group: block %d: %s", r, ctx->msg.c_str()); return st; }
    }
    LocalGroup* g = new LocalGroup();
    g->m.assign(ctxs, ctxs + n);
    g->rec.assign(n, lag_local_rec{});
    g->has.assign(n, 0);
    g->extracted.assign(n, 0);
    g->alive = n;
    // ghost boxes: block r's receive box from peer p <- p's send box toward r
    for (int r = 0; r < n; ++r) {
        const Comm* cr = ctxs[r]->comm;
        for (const Peer& p : cr->peers) {
            const Comm* cp = ctxs[p.rank]->comm;
            const Box* sb = nullptr;
            for (const Peer& pp : cp->peers)
                if (pp.rank == r && pp.off == p.back) sb = &cp->send_boxes[(size_t)pp.send_box];
            const Box& rb = cr->recv_boxes[(size_t)p.recv_box];
            if (!sb || sb->nx != rb.nx || sb->ny != rb.ny || sb->nz != rb.nz) {
                delete g;
                lag_set_error(nullptr, "lag_local_group: ghost boxes of blocks %d and %d do not match", r, p.rank);
                return LAG_EINVAL;
            }
            LocalBox b{};
            b.dst = r; b.src = p.rank;
            b.dx0 = rb.x0; b.dy0 = rb.y0; b.dz0 = rb.z0;
            b.sx0 = sb->x0; b.sy0 = sb->y0; b.sz0 = sb->z0;
            b.nx = rb.nx; b.ny = rb.ny; b.nz = rb.nz;
            b.off = g->total;
            g->total += (int64_t)b.nx * b.ny * b.nz * ctxs[0]->cfg.dim;
            g->max_box_floats = std::max(g->max_box_floats, b.nx * b.ny * b.nz * ctxs[0]->cfg.dim);
            g->boxes.push_back(b);
        }
    }
    ctx = ctxs[0];
    for (int r = 0; r < n; ++r) ctxs[r]->group = g;   // (local_append_args reads g->m)
    std::vector<AppendArgs> app(n);
    for (int r = 0; r < n; ++r) app[r] = local_append_args(ctxs[r]);
    g->ev.assign(n, nullptr);
    cudaError_t e = cudaSuccess;
    for (int r = 0; r < n && e == cudaSuccess; ++r) e = cudaEventCreateWithFlags(&g->ev[r], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_app, sizeof(AppendArgs) * n);
    if (e == cudaSuccess) e = cudaMemcpy(g->d_app, app.data(), sizeof(AppendArgs) * n, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !g->boxes.empty()) {
        e = cudaMalloc(&g->d_boxes, sizeof(LocalBox) * g->boxes.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(g->d_boxes, g->boxes.data(), sizeof(LocalBox) * g->boxes.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        for (int r = 0; r < n; ++r) { ctxs[r]->group = nullptr; if (g->ev[r]) cudaEventDestroy(g->ev[r]); }
        cudaFree(g->d_boxes);
        cudaFree(g->d_app);
        delete g;
        lag_set_error(nullptr, "lag_local_group: %s", cudaGetErrorString(e));
        return LAG_ECUDA;
    }
    return LAG_OK;
}

static void local_unrecord(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    if (!g) return;
    const int r = ctx->cfg.rank;
    if (g->has[r]) { g->has[r] = 0; --g->nrec; }
}

lag_status lag_local_record(lag_ctx_s* ctx, const lag_local_rec& rec, bool* complete) {
    LocalGroup* g = ctx->group;
    const int r = ctx->cfg.rank;
    *complete = false;
    if (g->has[r]) {
        lag_set_error(ctx, "LAG_XCHG_LOCAL: block %d already recorded this group cycle", r);
        return LAG_ESTATE;
    }
    for (int q = 0; q < (int)g->m.size(); ++q)
        if (!g->m[q]) { lag_set_error(ctx, "LAG_XCHG_LOCAL: block %d was destroyed", q); return LAG_ESTATE; }
    g->rec[r] = rec;
    g->has[r] = 1;
    if (++g->nrec == (int)g->m.size()) {
        for (lag_ctx_s* c : g->m)
            if (!c->seeded) { lag_set_error(ctx, "LAG_XCHG_LOCAL: block %d is not seeded", c->cfg.rank); g->has[r] = 0; --g->nrec; return LAG_ESTATE; }
        std::fill(g->has.begin(), g->has.end(), 0);
        g->nrec = 0;
        *complete = true;
    }
    return LAG_OK;
}

lag_status lag_local_run_cycle(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    const int n = (int)g->m.size();
    lag_status st = local_join_in(ctx);
    if (st != LAG_OK) return st;
    lag_ctx_s* c0 = g->m[0];
    // one launch: grid rows [0, nybox) copy ghost boxes, the next n rows
    // append each block's hand-offs
    LocalCopyArgs a{};
    a.boxes = g->d_boxes;
    a.nbox = (int)g->boxes.size();
    a.dim = ctx->cfg.dim;
    a.total = g->total;
    for (int r = 0; r < n; ++r) {
        a.v0[r] = g->rec[r].v0;
        a.v1[r] = g->rec[r].v1;
        a.sx[r] = g->m[r]->sx;
        a.sxy[r] = g->m[r]->sxy;
        if (!g->rec[r].v0_prev) a.fill_v0 |= 1ull << r;
    }
    a.nybox = a.nbox * (a.fill_v0 ? 2 : 1);
    a.app = g->d_app;
    a.app_ctas = kLocalAppendCtas;
    const int bx = std::max(kLocalAppendCtas, std::min((g->max_box_floats + 255) / 256, 64));
    local_ghost_kernel<<<dim3(bx, (unsigned)(a.nybox + n)), 256, 0, c0->stream>>>(a);
    ++ctx->launches;
    CKC(cudaGetLastError());
    for (lag_ctx_s* c : g->m) c->comm->pending = false;
    return local_join_out(ctx);
}

lag_ctx_s* lag_local_member(lag_ctx_s* ctx, int r) { return ctx->group->m[r]; }
const lag_local_rec& lag_local_recorded(lag_ctx_s* ctx, int r) { return ctx->group->rec[r]; }
int lag_local_size(lag_ctx_s* ctx) { return (int)ctx->group->m.size(); }

lag_status lag_local_flush(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    if (g->nextracted > 0) return LAG_OK;               // an earlier block of this write cycle did it
    for (lag_ctx_s* c : g->m)
        if (!c) { lag_set_error(ctx, "LAG_XCHG_LOCAL: a block of the group was destroyed"); return LAG_ESTATE; }
    bool pending = false;
    for (lag_ctx_s* c : g->m) pending |= c->comm->pending;
    // every block's last cycle is done before any block gathers from it
    lag_status st = local_join_in(ctx);
    if (st == LAG_OK && pending) st = local_appends(ctx);
    if (st == LAG_OK) st = local_join_out(ctx);
    return st;
}

lag_status lag_local_join_all(lag_ctx_s* ctx) {
    lag_status st = local_join_in(ctx);
    return st == LAG_OK ? local_join_out(ctx) : st;
}

bool lag_local_extracted(lag_ctx_s* ctx, bool* all) {
    LocalGroup* g = ctx->group;
    const int r = ctx->cfg.rank;
    if (!g->extracted[r]) { g->extracted[r] = 1; ++g->nextracted; }
    *all = g->nextracted == (int)g->m.size();
    if (*all) {
        std::fill(g->extracted.begin(), g->extracted.end(), 0);
        g->nextracted = 0;
    }
    return true;
}

bool lag_local_extracting(lag_ctx_s* ctx) { return ctx->group && ctx->group->nextracted > 0; }

void lag_local_leave(lag_ctx_s* ctx) {
    LocalGroup* g = ctx->group;
    if (!g) return;
    g->m[ctx->cfg.rank] = nullptr;
    ctx->group = nullptr;
    if (--g->alive == 0) {
        cudaFree(g->d_boxes);
        cudaFree(g->d_app);
        for (cudaEvent_t e : g->ev) if (e) cudaEventDestroy(e);
        delete g;
    }
}
