// lag_api.cu — C ABI of liblag (include/lag.h): validation, device memory,
// launches.  Kernels: lag_kernels.cuh.  COMM exchange: lag_comm.cu.
//
// The product path has no CPU fallback: every step of the hot path runs in
// the kernels below; host code only validates, allocates and enqueues.
#include "lag.h"
#include "lag_internal.h"
#include "lag_xchg.cuh"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

using namespace lag;

static thread_local std::string g_init_error = "no error";

// COMM overlap pass 1 (LAG_XCHG_PEER_OVERLAP): CTAs [0, xf.ncta) run this
// cycle's peer exchange (pack + signal, wait + ghost pull + append of the
// previous cycle's hand-offs, lag_xchg.cuh) while the other CTAs advect the
// tiles whose stage samples cannot reach a ghost node (a.pass = 1).  The grid
// is the resident capacity, so the exchange CTAs never wait for a slot.
template <int DIM, bool FROZEN>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
advect_xchg_kernel(const AdvectArgs a, const XchgFused xf) {
    // a programmatic dependent of the previous pass 2: the exchange CTAs pack
    // and pull at once and wait for it only to signal and append (lag_xchg.cuh);
    // the advect CTAs wait for it first (its tile lists, this cycle's snapshot)
    griddep_launch();
    if ((int)blockIdx.x < xf.ncta) {
        xchg_pack_signal(xf.x, blockIdx.x, xf.ncta);
        xchg_wait_pull(xf.x, xf.ap, blockIdx.x, xf.ncta);
        return;
    }
    griddep_wait();
    advect_body<DIM, false, FROZEN, true>(a, blockIdx.x - xf.ncta, gridDim.x - xf.ncta);
}

int lag_set_error(lag_ctx_s* ctx, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    if (ctx) ctx->msg = buf; else g_init_error = buf;
    return 0;
}

#define CK(call)                                                                   \
    do {                                                                           \
        cudaError_t e_ = (call);                                                   \
        if (e_ != cudaSuccess) {                                                   \
            lag_set_error(ctx, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                          __FILE__, __LINE__);                                     \
            return e_ == cudaErrorMemoryAllocation ? LAG_ENOMEM : LAG_ECUDA;      \
        }                                                                          \
    } while (0)

static int bits_for(int64_t n) {       // bits to hold values 0..n-1 (>= 1)
    int b = 1;
    while ((int64_t(1) << b) < n) ++b;
    return b;
}

template <typename T>
static lag_status dmalloc(lag_ctx_s* ctx, T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
    if (e != cudaSuccess) {
        lag_set_error(ctx, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
        return LAG_ENOMEM;
    }
    return LAG_OK;
}

static void dfree(void* p) { if (p) cudaFree(p); }

// ---------------------------------------------------------------------------

extern "C" int32_t lag_abi_version(void) { return LAG_ABI_VERSION; }

extern "C" const char* lag_last_error(lag_ctx ctx) {
    return ctx ? ctx->msg.c_str() : g_init_error.c_str();
}

extern "C" int64_t lag_kernel_launches(lag_ctx ctx) { return ctx ? ctx->launches : 0; }

static lag_status validate(const lag_config* c) {
    lag_ctx_s* ctx = nullptr;
    if (!c) { lag_set_error(ctx, "cfg is NULL"); return LAG_EINVAL; }
    if (c->dim != 2 && c->dim != 3) { lag_set_error(ctx, "dim must be 2 or 3 (got %d)", c->dim); return LAG_EINVAL; }
    if (c->mode != LAG_BTO && c->mode != LAG_COMM) { lag_set_error(ctx, "mode must be LAG_BTO or LAG_COMM"); return LAG_EINVAL; }
    int64_t total_bits = 0;
    for (int a = 0; a < 3; ++a) {
        const bool used = a < c->dim;
        const int64_t N = c->global_nodes[a];
        if (used) {
            if (N < 2 || N >= (int64_t(1) << 22)) { lag_set_error(ctx, "global_nodes[%d] = %lld must be in [2, 2^22)", a, (long long)N); return LAG_EINVAL; }
            if (!(c->spacing[a] > 0.0) || !std::isfinite(c->spacing[a])) { lag_set_error(ctx, "spacing[%d] must be finite and > 0", a); return LAG_EINVAL; }
            if (!std::isfinite(c->origin[a])) { lag_set_error(ctx, "origin[%d] must be finite", a); return LAG_EINVAL; }
            if (!(0 <= c->block_lo[a] && c->block_lo[a] < c->block_hi[a] && c->block_hi[a] <= N)) {
                lag_set_error(ctx, "block [%lld, %lld) on axis %d must satisfy 0 <= lo < hi <= N = %lld", (long long)c->block_lo[a], (long long)c->block_hi[a], a, (long long)N);
                return LAG_EINVAL;
            }
            total_bits += bits_for(N);
        } else if (N != 1 || c->block_lo[a] != 0 || c->block_hi[a] != 1) {
            lag_set_error(ctx, "unused axis %d must have global_nodes = 1 and block [0, 1)", a);
            return LAG_EINVAL;
        }
    }
    if (total_bits > 32 || (c->dim == 3 && bits_for(c->global_nodes[0]) + bits_for(c->global_nodes[1]) >= 32)) {
        lag_set_error(ctx, "grid too large: the packed seed node needs %lld > 32 bits", (long long)total_bits);
        return LAG_EINVAL;
    }
    if (c->ghost < 0 || c->ghost > 8) { lag_set_error(ctx, "ghost must be in [0, 8]"); return LAG_EINVAL; }
    if (c->mode == LAG_COMM) {
        if (c->ghost < 1 && c->nranks > 1) { lag_set_error(ctx, "COMM mode with neighbours needs ghost >= 1"); return LAG_EINVAL; }
        int64_t prod = 1;
        for (int a = 0; a < 3; ++a) {
            if (c->layout[a] < 1 || (a >= c->dim && c->layout[a] != 1)) { lag_set_error(ctx, "bad layout"); return LAG_EINVAL; }
            prod *= c->layout[a];
        }
        if (prod != c->nranks || c->rank < 0 || c->rank >= c->nranks) { lag_set_error(ctx, "rank/nranks/layout mismatch"); return LAG_EINVAL; }
        if (c->exchange != LAG_XCHG_NCCL && c->exchange != LAG_XCHG_PEER && c->exchange != LAG_XCHG_PEER_OVERLAP &&
            c->exchange != LAG_XCHG_LOCAL) {
            lag_set_error(ctx, "exchange must be LAG_XCHG_NCCL, LAG_XCHG_PEER, LAG_XCHG_PEER_OVERLAP or LAG_XCHG_LOCAL");
            return LAG_EINVAL;
        }
        if (c->exchange == LAG_XCHG_LOCAL) {
            if (c->nranks > 64) { lag_set_error(ctx, "LAG_XCHG_LOCAL groups hold at most 64 blocks"); return LAG_EINVAL; }
        } else if (c->nranks > 1 && !c->nccl_id) {
            lag_set_error(ctx, "COMM mode with nranks > 1 needs nccl_id");
            return LAG_EINVAL;
        }
    }
    const int64_t ext_x = std::min(c->block_hi[0] + 1, c->global_nodes[0]) - c->block_lo[0] + 2 * c->ghost;
    if (c->row_pitch_bytes != 0 &&
        (c->row_pitch_bytes < 0 || c->row_pitch_bytes % (4 * c->dim) != 0 || c->row_pitch_bytes < 4 * c->dim * ext_x)) {
        lag_set_error(ctx, "row_pitch_bytes = %lld must be 0 or a multiple of %d that is >= %lld",
                      (long long)c->row_pitch_bytes, 4 * c->dim, (long long)(4 * c->dim * ext_x));
        return LAG_EINVAL;
    }
    // slice extent must fit 32-bit element offsets
    int64_t nodes = c->row_pitch_bytes ? c->row_pitch_bytes / (4 * c->dim) : ext_x;
    for (int a = 1; a < c->dim; ++a)
        nodes *= (std::min(c->block_hi[a] + 1, c->global_nodes[a]) - c->block_lo[a] + 2 * c->ghost);
    if (nodes * c->dim >= (int64_t(1) << 31)) { lag_set_error(ctx, "block slice too large for 32-bit offsets"); return LAG_EINVAL; }
    return LAG_OK;
}

extern "C" lag_status lag_init(const lag_config* cfg, lag_ctx* out) {
    if (out) *out = nullptr;
    lag_ctx_s* ctx = nullptr;
    if (!out) { lag_set_error(ctx, "out is NULL"); return LAG_EINVAL; }
    lag_status st = validate(cfg);
    if (st != LAG_OK) return st;

    ctx = new (std::nothrow) lag_ctx_s();
    if (!ctx) { lag_set_error(nullptr, "out of host memory"); return LAG_ENOMEM; }
    ctx->cfg = *cfg;
    ctx->stream = (cudaStream_t)cfg->stream;
    {
        cudaError_t e = cudaSetDevice(cfg->device);
        if (e != cudaSuccess) {
            lag_set_error(nullptr, "cudaSetDevice(%d): %s", cfg->device, cudaGetErrorString(e));
            delete ctx;
            return LAG_ECUDA;
        }
    }
    const int D = cfg->dim;
    for (int a = 0; a < 3; ++a) {
        const bool used = a < D;
        ctx->ext[a] = used ? (int)(std::min(cfg->block_hi[a] + 1, cfg->global_nodes[a]) - cfg->block_lo[a] + 2 * cfg->ghost) : 1;
        ctx->base[a] = used ? (int)(cfg->block_lo[a] - cfg->ghost) : 0;
    }
    ctx->bits[0] = bits_for(cfg->global_nodes[0]);
    ctx->bits[1] = bits_for(cfg->global_nodes[1]);
    ctx->bits[2] = D == 3 ? bits_for(cfg->global_nodes[2]) : 0;
    ctx->sx = cfg->row_pitch_bytes ? (int)(cfg->row_pitch_bytes / (4 * D)) : ctx->ext[0];
    ctx->sxy = ctx->sx * ctx->ext[1];
    ctx->slice_floats = (int64_t)ctx->sxy * ctx->ext[2] * D;
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, cfg->device);
    ctx->num_sms = dev_sms;

    // max seeds at stride 1 bounds every later seeding
    int64_t owned = 1;
    for (int a = 0; a < D; ++a) owned *= (cfg->block_hi[a] - cfg->block_lo[a]);
    ctx->max_seeds = owned;
    // COMM: particles migrate in; keep room for 2x the owned nodes (+ tail tiles)
    ctx->cap = cfg->mode == LAG_COMM ? 2 * owned + 64 * kTile : owned;
    // seed tiles in brick order (ragged bricks leave partial tiles; stride 1
    // bounds every stride) + COMM room for appended tiles
    ctx->brick[0] = D == 3 ? kBrickRows : 1;
    ctx->brick[1] = D == 3 ? kBrickRows : 1;
    {
        int32_t o[3] = {1, 1, 1};
        for (int a = 0; a < D; ++a) o[a] = (int32_t)(cfg->block_hi[a] - cfg->block_lo[a]);
        const int64_t seed_tiles = brick_tiles(o, ctx->brick[0], ctx->brick[1]);
        const int64_t extra = cfg->mode == LAG_COMM ? (ctx->cap - owned + kTile - 1) / kTile : 0;
        ctx->cap_tiles = (int)(seed_tiles + extra);
    }

    auto fail = [&](lag_status s) {
        std::string m = ctx->msg;
        lag_destroy(ctx);
        g_init_error = m;
        return s;
    };
    if ((st = dmalloc(ctx, &ctx->state, (size_t)ctx->cap_tiles * kTile)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->tile_count, (size_t)ctx->cap_tiles)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->dead_rec, (size_t)ctx->cap)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->dead_info, (size_t)ctx->cap)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->words, (size_t)kWords)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->counters, (size_t)CNT_N)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->out_start, (size_t)owned * D)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->out_end, (size_t)owned * D)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->out_status, (size_t)owned)) != LAG_OK) return fail(st);
    if ((st = dmalloc(ctx, &ctx->out_cycle, (size_t)owned)) != LAG_OK) return fail(st);
    {
        cudaError_t e = cudaMemsetAsync(ctx->counters, 0, CNT_N * sizeof(unsigned long long), ctx->stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(ctx->words, 0, kWords * sizeof(uint32_t), ctx->stream);
        if (e != cudaSuccess) { lag_set_error(ctx, "memset: %s", cudaGetErrorString(e)); return fail(LAG_ECUDA); }
    }
    if (cfg->mode == LAG_COMM) {
        st = lag_comm_init(ctx);
        if (st != LAG_OK) return fail(st);
        if (lag_comm_overlap(ctx)) {
            if ((st = dmalloc(ctx, &ctx->defer_list, (size_t)ctx->cap_tiles)) != LAG_OK) return fail(st);
        }
    }
    // occupancy-sized persistent grid for the advect kernel
    int occ = 1;
    if (D == 3)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cfg->mode == LAG_BTO ? advect_kernel<3, true, false> : advect_kernel<3, false, false>, kThreads, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cfg->mode == LAG_BTO ? advect_kernel<2, true, false> : advect_kernel<2, false, false>, kThreads, 0);
    ctx->advect_blocks_per_sm = occ > 0 ? occ : 1;
    {
        const char* pt = getenv("LAG_PHASE_TIMING");
        ctx->phase_timing = pt && pt[0] == '1';
        if (ctx->phase_timing)
            for (int i = 0; i < 64; ++i)
                for (int j = 0; j < 4; ++j) cudaEventCreate(&ctx->ph_ev[i][j]);
    }
    *out = ctx;
    return LAG_OK;
}

extern "C" lag_status lag_destroy(lag_ctx ctx) {
    if (!ctx) return LAG_OK;
    cudaSetDevice(ctx->cfg.device);
    if (ctx->stream_synced_needed) cudaStreamSynchronize(ctx->stream);
    lag_local_leave(ctx);
    lag_comm_destroy(ctx);
    dfree(ctx->defer_list);
    dfree(ctx->state); dfree(ctx->tile_count); dfree(ctx->dead_rec); dfree(ctx->dead_info);
    dfree(ctx->words); dfree(ctx->counters); dfree(ctx->out_start); dfree(ctx->out_end);
    if (ctx->phase_timing)
        for (int i = 0; i < 64; ++i)
            for (int j = 0; j < 4; ++j) cudaEventDestroy(ctx->ph_ev[i][j]);
    dfree(ctx->out_status); dfree(ctx->out_cycle);
    for (int k = 0; k < lag_ctx_s::kStage; ++k) {
        dfree(ctx->stage[k]);
        if (ctx->stage_ready[k]) cudaEventDestroy(ctx->stage_ready[k]);
        if (ctx->stage_free[k]) cudaEventDestroy(ctx->stage_free[k]);
    }
    if (ctx->cstream) cudaStreamDestroy(ctx->cstream);
    delete ctx;
    return LAG_OK;
}

// ---------------------------------------------------------------------------

lag_status lag_reset_interval(lag_ctx_s* ctx) {
    // device words: [W_DEAD] dead count, [W_ERR] error bits, [W_NTILES] tile count (COMM);
    // error bits stay latched until a synchronous lag_extract reports them
    static_assert(W_DEAD == 0 && W_ERR == 1, "word layout");
    CK(cudaMemsetAsync(ctx->words + W_DEAD, 0, sizeof(uint32_t), ctx->stream));
    CK(cudaMemsetAsync(ctx->words + W_ERR + 1, 0, (kWords - W_ERR - 1) * sizeof(uint32_t), ctx->stream));
    CK(cudaMemsetAsync(ctx->counters + CNT_TERM, 0, 4 * sizeof(unsigned long long), ctx->stream));
    return LAG_OK;
}

extern "C" lag_status lag_seed(lag_ctx ctx, int32_t stride, int64_t* n_seeds_out) {
    if (n_seeds_out) *n_seeds_out = 0;
    if (!ctx) { lag_set_error(nullptr, "ctx is NULL"); return LAG_EINVAL; }
    if (stride < 1) { lag_set_error(ctx, "stride must be >= 1 (got %d)", stride); return LAG_EINVAL; }
    if (ctx->cfg.mode == LAG_COMM && ctx->cfg.exchange == LAG_XCHG_LOCAL && !ctx->group) {
        lag_set_error(ctx, "LAG_XCHG_LOCAL context without lag_local_group");
        return LAG_ESTATE;
    }
    CK(cudaSetDevice(ctx->cfg.device));
    const int D = ctx->cfg.dim;
    int64_t n = 1;
    for (int a = 0; a < 3; ++a) {
        if (a < D) {
            const int64_t lo = ctx->cfg.block_lo[a], hi = ctx->cfg.block_hi[a];
            const int64_t first = ((lo + stride - 1) / stride) * stride;
            const int64_t cnt = first < hi ? (hi - first + stride - 1) / stride : 0;
            ctx->first[a] = (int)first;
            ctx->ns[a] = (int)cnt;
        } else {
            ctx->first[a] = 0;
            ctx->ns[a] = 1;
        }
        n *= ctx->ns[a];
    }
    if (n == 0) {
        ctx->seeded = false;
        lag_set_error(ctx, "no lattice node of stride %d in the block", stride);
        return LAG_EEMPTY;
    }
    lag_status st = lag_reset_interval(ctx);
    if (st != LAG_OK) return st;
    ctx->stride = stride;
    ctx->n_seeds = n;
    ctx->n_tiles = (int)brick_tiles(ctx->ns, ctx->brick[0], ctx->brick[1]);
    if (ctx->cfg.mode == LAG_COMM) {
        // tail tiles past the seeds are empty; n_tiles lives on the device (appends)
        CK(cudaMemsetAsync(ctx->tile_count, 0, (size_t)ctx->cap_tiles, ctx->stream));
        st = lag_comm_reset(ctx);
        if (st != LAG_OK) return st;
    }
    SeedArgs sa{};
    sa.state = ctx->state; sa.tile_count = ctx->tile_count; sa.n_tiles = ctx->n_tiles; sa.stride = stride;
    sa.n_tiles_word = ctx->cfg.mode == LAG_COMM ? ctx->words + W_NTILES : nullptr;
    sa.snap_b = ctx->cfg.mode == LAG_COMM ? ctx->words + W_NTILES_B : nullptr;
    sa.snap_defer = ctx->cfg.mode == LAG_COMM ? ctx->words + W_DEFER : nullptr;
    for (int a = 0; a < 3; ++a) { sa.first[a] = ctx->first[a]; sa.ns[a] = ctx->ns[a]; }
    sa.by = ctx->brick[0]; sa.bz = ctx->brick[1];
    sa.bx = ctx->bits[0]; sa.by_bits = ctx->bits[1];
    const dim3 bricks((unsigned)((ctx->ns[0] + kTile - 1) / kTile), (unsigned)((ctx->ns[1] + sa.by - 1) / sa.by),
                      (unsigned)((ctx->ns[2] + sa.bz - 1) / sa.bz));
    if (bricks.y > 65535u || bricks.z > 65535u) {
        lag_set_error(ctx, "seed lattice too tall for the brick grid (%u x %u bricks in y, z)", bricks.y, bricks.z);
        return LAG_EINVAL;
    }
    seed_kernel<<<bricks, dim3(kTile, sa.by, sa.bz), 0, ctx->stream>>>(sa);
    ++ctx->launches;
    CK(cudaGetLastError());
    ctx->seeded = true;
    ctx->cycles_in_interval = 0;
    ctx->active_host = n;
    ctx->last_v1 = nullptr;
    if (n_seeds_out) *n_seeds_out = n;
    return LAG_OK;
}

// Device-resident velocity for a caller pointer: device memory is used in
// place; host memory is copied into one of two staging buffers (end-to-end
// path).  Only the previous call's v_t1 passed again as v_t is reused; it must
// not change between those two calls.
static lag_status resolve_slice(lag_ctx_s* ctx, void* p, int avoid, float** out, int* slot_out) {
    *slot_out = -1;
    cudaPointerAttributes at{};
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) { cudaGetLastError(); at.type = cudaMemoryTypeUnregistered; }
    if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
        if (at.type == cudaMemoryTypeDevice && at.device != ctx->cfg.device) {
            lag_set_error(ctx, "slice pointer lives on device %d, context on %d", at.device, ctx->cfg.device);
            return LAG_EINVAL;
        }
        *out = (float*)p;
        return LAG_OK;
    }
    // only the previous call's v_t1, passed again as this call's v_t, is reused
    // (the in situ sequence); any other host slice is copied afresh
    if (avoid < 0 && ctx->last_v1_slot >= 0 && ctx->stage_src[ctx->last_v1_slot] == p) {
        const int s = ctx->last_v1_slot;
        CK(cudaStreamWaitEvent(ctx->stream, ctx->stage_ready[s], 0));
        *out = ctx->stage[s]; *slot_out = s;
        return LAG_OK;
    }
    // least recently read buffer (never the one this call already uses); its
    // copy waits only for that buffer's last reader, so it overlaps the
    // kernels of the cycle in flight
    int s = -1;
    for (int k = 0; k < lag_ctx_s::kStage; ++k)
        if (k != avoid && (s < 0 || ctx->stage_use[k] < ctx->stage_use[s])) s = k;
    if (!ctx->cstream) {
        CK(cudaStreamCreateWithFlags(&ctx->cstream, cudaStreamNonBlocking));
        for (int k = 0; k < lag_ctx_s::kStage; ++k) {
            CK(cudaEventCreateWithFlags(&ctx->stage_ready[k], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->stage_free[k], cudaEventDisableTiming));
        }
    }
    if (!ctx->stage[s]) {
        lag_status st = dmalloc(ctx, &ctx->stage[s], (size_t)ctx->slice_floats);
        if (st != LAG_OK) return st;
    }
    if (ctx->stage_use[s] >= 0) CK(cudaStreamWaitEvent(ctx->cstream, ctx->stage_free[s], 0));
    CK(cudaMemcpyAsync(ctx->stage[s], p, (size_t)ctx->slice_floats * sizeof(float),
                       cudaMemcpyHostToDevice, ctx->cstream));
    CK(cudaEventRecord(ctx->stage_ready[s], ctx->cstream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->stage_ready[s], 0));
    ctx->stage_src[s] = p;
    *out = ctx->stage[s]; *slot_out = s;
    return LAG_OK;
}

// Fold recorded phase events into ph_ms (synchronises on the events).
static void fold_phases(lag_ctx_s* ctx) {
    for (int i = 0; i < ctx->ph_n; ++i) {
        float ms;
        for (int j = 0; j < 3; ++j)
            // overlap (LAG_XCHG_PEER_OVERLAP): snapshot, pass 1 (exchange CTAs +
            // ghost-free tiles), pass 2
            if (cudaEventElapsedTime(&ms, ctx->ph_ev[i][j], ctx->ph_ev[i][j + 1]) == cudaSuccess) ctx->ph_ms[j] += ms;
    }
    ctx->ph_n = 0;
}

// One cycle of one block, slices already device-resident: (COMM) the
// pre-advect exchange unless the LOCAL group ran it, the advect kernel, the
// post-advect bookkeeping.  s0/s1: staging buffers read (host slices) or -1.
static lag_status advect_enqueue(lag_ctx_s* ctx, float* d0, float* d1, double dt, bool v0_prev,
                                 int s0, int s1) {
    lag_status st;
    const int D = ctx->cfg.dim;
    if (ctx->phase_timing && ctx->ph_n == 64) fold_phases(ctx);
    cudaEvent_t* ev = ctx->phase_timing ? ctx->ph_ev[ctx->ph_n++] : nullptr;
    if (ev) cudaEventRecord(ev[0], ctx->stream);
    const bool overlap = ctx->cfg.mode == LAG_COMM && lag_comm_overlap(ctx);
    XchgFused xf{};
    if (overlap) {
        // the exchange is not launched here: pass 1's first CTAs run it
        // (the tile count before its append and the empty deferral list of
        // this cycle were set by the previous pass 2 or by the seed kernel)
        ctx->xchg_fused = &xf;
        st = lag_comm_pre_advect(ctx, d0, d1, v0_prev);
        ctx->xchg_fused = nullptr;
        if (st != LAG_OK) return st;
        xf.ncta = kXchgCtas;
    } else if (ctx->cfg.mode == LAG_COMM && !ctx->group) {      // LOCAL: the group ran it
        st = lag_comm_pre_advect(ctx, d0, d1, v0_prev);
        if (st != LAG_OK) return st;
    }
    if (ev && !overlap) cudaEventRecord(ev[1], ctx->stream);
    AdvectArgs a{};
    a.v0 = d0; a.v1 = d1;
    a.frozen = d0 == d1 ? 1 : 0;
    a.slice_nodes = (int32_t)(ctx->slice_floats / ctx->cfg.dim);
    a.state = ctx->state; a.tile_count = ctx->tile_count;
    a.n_tiles_dev = ctx->cfg.mode == LAG_COMM ? (const int32_t*)(ctx->words + W_NTILES) : nullptr;
    a.n_tiles = ctx->n_tiles;
    for (int ax = 0; ax < 3; ++ax) {
        a.N[ax] = (int)ctx->cfg.global_nodes[ax];
        a.lo[ax] = (int)ctx->cfg.block_lo[ax];
        a.hi[ax] = (int)ctx->cfg.block_hi[ax];
        a.base[ax] = ctx->base[ax];
        a.cmax[ax] = ctx->ext[ax] - 2;
        {
            // fast ranges of global cell indices
            const int N = (int)ctx->cfg.global_nodes[ax], lo = (int)ctx->cfg.block_lo[ax], hi = (int)ctx->cfg.block_hi[ax];
            const int btop = (hi < N ? hi - 1 : N - 2);                 // last valid cell in the block
            const int gmin = std::max(ctx->base[ax], 0);
            const int gtop = std::min(ctx->base[ax] + ctx->ext[ax] - 2, N - 2);
            a.bmin[ax] = lo; a.bspan[ax] = btop - lo;
            if (ctx->cfg.mode == LAG_BTO) { a.gmin[ax] = lo; a.gspan[ax] = btop - lo; }
            else { a.gmin[ax] = gmin; a.gspan[ax] = gtop - gmin; }
            if (ax >= D) { a.bmin[ax] = a.gmin[ax] = 0; a.bspan[ax] = a.gspan[ax] = 0; }
        }
        const double dth = ax < D ? dt / ctx->cfg.spacing[ax] : 0.0;
        a.hdth[ax] = (float)(0.5 * dth);
        a.qdth[ax] = (float)(0.25 * dth);
        a.sdth[ax] = (float)(dth / 6.0);
    }
    a.sx = ctx->sx;
    a.sxy = ctx->sxy;
    a.gidx0 = (a.gmin[0] - a.base[0]) + a.sx * (a.gmin[1] - a.base[1]) + a.sxy * (a.gmin[2] - a.base[2]);
    a.bx = ctx->bits[0]; a.by = ctx->bits[1];
    a.mx = (1u << ctx->bits[0]) - 1u; a.my = (1u << ctx->bits[1]) - 1u;
    a.dead_rec = ctx->dead_rec; a.dead_info = ctx->dead_info;
    a.dead_count = ctx->words + W_DEAD; a.dead_cap = (uint32_t)ctx->cap;
    a.counters = ctx->counters; a.err = ctx->words + W_ERR;
    a.cycle = ctx->cycles_in_interval;
    if (ctx->cfg.mode == LAG_COMM) lag_comm_fill_args(ctx, &a);
    if (overlap) {
        // ghost-free cells: a stage sample (within one cell of the stage-1 cell,
        // CFL < 1) never needs node lo-1 (lower neighbour) or hi+1 (upper one)
        for (int ax = 0; ax < 3; ++ax) {
            const int N = (int)ctx->cfg.global_nodes[ax], lo = (int)ctx->cfg.block_lo[ax], hi = (int)ctx->cfg.block_hi[ax];
            const int cmin = lo > 0 ? lo + 1 : a.gmin[ax];
            const int cmax = hi < N ? hi - 2 : a.gmin[ax] + a.gspan[ax];
            if (ax >= D) { a.smin[ax] = 0; a.sspan[ax] = 0; }
            else if (cmax < cmin) { a.smin[ax] = 1 << 29; a.sspan[ax] = 0; }      // nothing ghost-free
            else { a.smin[ax] = cmin - a.gmin[ax]; a.sspan[ax] = cmax - cmin; }
        }
        const int par = (int)(ctx->cycles_total & 1);
        a.n_tiles_b = ctx->words + W_NTILES_B + par;
        a.defer_list = ctx->defer_list;
        a.defer_count = ctx->words + W_DEFER + par;
        a.next_b = ctx->words + W_NTILES_B + (par ^ 1);
        a.next_defer = ctx->words + W_DEFER + (par ^ 1);
    }

    const int tiles = ctx->cfg.mode == LAG_COMM ? ctx->cap_tiles : ctx->n_tiles;
    const int warps_per_block = kThreads / 32;
    // persistent grid: at most the resident CTAs (one wave)
    int blocks = (tiles + warps_per_block - 1) / warps_per_block;
    const int max_blocks = ctx->num_sms * ctx->advect_blocks_per_sm;
    if (blocks > max_blocks) blocks = max_blocks;
    if (blocks < 1) blocks = 1;
    const bool bto = ctx->cfg.mode == LAG_BTO;
    // programmatic dependent launch: the CTAs are scheduled while the
    // previous kernel (e.g. the peer exchange) drains and wait in
    // griddep_wait() for its end, so the launch latency overlaps it
    cudaLaunchAttribute pdl{};
    pdl.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl.val.programmaticStreamSerializationAllowed = 1;
    auto launch = [&](const AdvectArgs& aa, int nb) -> cudaError_t {
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(nb); lc.blockDim = dim3(kThreads); lc.dynamicSmemBytes = 0; lc.stream = ctx->stream;
        lc.attrs = &pdl; lc.numAttrs = 1;
        if (D == 3) {
            if (aa.frozen) return bto ? cudaLaunchKernelEx(&lc, advect_kernel<3, true, true>, aa)
                                      : cudaLaunchKernelEx(&lc, advect_kernel<3, false, true>, aa);
            return bto ? cudaLaunchKernelEx(&lc, advect_kernel<3, true, false>, aa)
                       : cudaLaunchKernelEx(&lc, advect_kernel<3, false, false>, aa);
        }
        if (aa.frozen) return bto ? cudaLaunchKernelEx(&lc, advect_kernel<2, true, true>, aa)
                                  : cudaLaunchKernelEx(&lc, advect_kernel<2, false, true>, aa);
        return bto ? cudaLaunchKernelEx(&lc, advect_kernel<2, true, false>, aa)
                   : cudaLaunchKernelEx(&lc, advect_kernel<2, false, false>, aa);
    };
    if (overlap) {
        // pass 1: exchange CTAs + ghost-free tiles; pass 2 (stream-ordered after
        // it): deferred tiles and this cycle's arrivals
        AdvectArgs a1 = a;
        a1.pass = 1;
        const int nb1 = std::max(blocks, kXchgCtas + 1);
        if (ev) cudaEventRecord(ev[1], ctx->stream);
        // both passes are programmatic dependents of the kernel before them
        cudaLaunchConfig_t l1{};
        l1.gridDim = dim3(nb1); l1.blockDim = dim3(kThreads); l1.stream = ctx->stream;
        l1.attrs = &pdl; l1.numAttrs = 1;
        if (D == 3) CK(a.frozen ? cudaLaunchKernelEx(&l1, advect_xchg_kernel<3, true>, a1, xf)
                                : cudaLaunchKernelEx(&l1, advect_xchg_kernel<3, false>, a1, xf));
        else CK(a.frozen ? cudaLaunchKernelEx(&l1, advect_xchg_kernel<2, true>, a1, xf)
                         : cudaLaunchKernelEx(&l1, advect_xchg_kernel<2, false>, a1, xf));
        ++ctx->launches;
        if (ev) cudaEventRecord(ev[2], ctx->stream);
        AdvectArgs a2 = a;
        a2.pass = 2;
        cudaLaunchConfig_t l2 = l1;
        l2.gridDim = dim3(blocks);
        if (D == 3) CK(a2.frozen ? cudaLaunchKernelEx(&l2, advect_kernel<3, false, true, true>, a2)
                                 : cudaLaunchKernelEx(&l2, advect_kernel<3, false, false, true>, a2));
        else CK(a2.frozen ? cudaLaunchKernelEx(&l2, advect_kernel<2, false, true, true>, a2)
                          : cudaLaunchKernelEx(&l2, advect_kernel<2, false, false, true>, a2));
    } else {
        CK(launch(a, blocks));
    }
    ++ctx->launches;
    CK(cudaGetLastError());
    if (ev && !overlap) cudaEventRecord(ev[2], ctx->stream);
    if (ctx->cfg.mode == LAG_COMM) {
        st = lag_comm_post_advect(ctx);
        if (st != LAG_OK) return st;
    }
    if (ev) cudaEventRecord(ev[3], ctx->stream);
    for (int k : {s0, s1})                  // staged host slices: read up to here
        if (k >= 0) {
            CK(cudaEventRecord(ctx->stage_free[k], ctx->stream));
            ctx->stage_use[k] = ctx->cycles_total;
        }
    ctx->last_v1_slot = s1;
    ctx->prev_d0 = d0;
    ctx->prev_d1 = d1;
    ++ctx->cycles_in_interval;
    ++ctx->cycles_total;
    return LAG_OK;
}


extern "C" lag_status lag_advect_cycle(lag_ctx ctx, void* v_t, void* v_t1, double dt) {
    if (!ctx) { lag_set_error(nullptr, "ctx is NULL"); return LAG_EINVAL; }
    if (!ctx->seeded) { lag_set_error(ctx, "lag_advect_cycle before lag_seed"); return LAG_ESTATE; }
    if (!v_t || !v_t1) { lag_set_error(ctx, "velocity slice pointer is NULL"); return LAG_EINVAL; }
    if (!(dt > 0.0) || !std::isfinite(dt)) { lag_set_error(ctx, "dt must be finite and > 0"); return LAG_EINVAL; }
    CK(cudaSetDevice(ctx->cfg.device));
    lag_status st;
    if (ctx->cfg.mode == LAG_COMM && ctx->cfg.exchange == LAG_XCHG_LOCAL) {
        if (!ctx->group) { lag_set_error(ctx, "LAG_XCHG_LOCAL context without lag_local_group"); return LAG_ESTATE; }
        if (lag_local_extracting(ctx)) {
            lag_set_error(ctx, "LAG_XCHG_LOCAL: lag_advect_cycle while the group's write cycle is incomplete");
            return LAG_ESTATE;
        }
        for (void* p : {v_t, v_t1}) {
            cudaPointerAttributes at{};
            if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
                at.device != ctx->cfg.device) {
                cudaGetLastError();
                lag_set_error(ctx, "LAG_XCHG_LOCAL needs device slices on device %d", ctx->cfg.device);
                return LAG_EINVAL;
            }
        }
        lag_local_rec rec{(float*)v_t, (float*)v_t1, dt, v_t == ctx->last_v1};
        bool complete = false;
        if ((st = lag_local_record(ctx, rec, &complete)) != LAG_OK) return st;
        ctx->last_v1 = v_t1;
        if (!complete) return LAG_OK;            // the group's last block enqueues the cycle
        if ((st = lag_local_run_cycle(ctx)) != LAG_OK) return st;
        for (int r = 0; r < lag_local_size(ctx); ++r) {
            lag_ctx_s* m = lag_local_member(ctx, r);
            const lag_local_rec& q = lag_local_recorded(ctx, r);
            if ((st = advect_enqueue(m, q.v0, q.v1, q.dt, q.v0_prev, -1, -1)) != LAG_OK) {
                if (m != ctx) lag_set_error(ctx, "block %d: %s", r, m->msg.c_str());
                return st;
            }
        }
        return LAG_OK;
    }
    float* d0 = nullptr;
    float* d1 = nullptr;
    int s0 = -1, s1 = -1;
    if ((st = resolve_slice(ctx, v_t, -1, &d0, &s0)) != LAG_OK) return st;
    if ((st = resolve_slice(ctx, v_t1, s0, &d1, &s1)) != LAG_OK) return st;
    st = advect_enqueue(ctx, d0, d1, dt, v_t == ctx->last_v1, s0, s1);
    if (st != LAG_OK) return st;
    ctx->last_v1 = v_t1;
    return LAG_OK;
}

static lag_status latched(lag_ctx_s* ctx, uint32_t err) {
    if (err & ERR_OVERFLOW) { lag_set_error(ctx, "latched: exchange slot or particle list overflow"); return LAG_EOVERFLOW; }
    if (err & ERR_GHOST) { lag_set_error(ctx, "latched: a stage sample left the ghost layers (CFL >= 1?)"); return LAG_EGHOST; }
    if (err & ERR_NONFINITE) { lag_set_error(ctx, "latched: non-finite velocity reached a particle"); return LAG_ENONFINITE; }
    if (err & ERR_XCHG) { lag_set_error(ctx, "latched: peer exchange timed out waiting for a neighbour"); return LAG_ENCCL; }
    return LAG_OK;
}

static lag_status copy_out(lag_ctx_s* ctx, void* dst, const void* src, size_t bytes) {
    if (!dst || bytes == 0 || dst == src) return LAG_OK;
    CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
    return LAG_OK;
}

// Output written by the kernels directly when it is device memory of this
// context's device; otherwise into the context's staging buffer, copied out.
template <typename T>
static T* out_target(lag_ctx_s* ctx, T* user, T* staging) {
    if (!user) return staging;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, user) != cudaSuccess) { cudaGetLastError(); return staging; }
    if (at.type == cudaMemoryTypeDevice && at.device == ctx->cfg.device) return user;
    return staging;
}

extern "C" lag_status lag_extract(lag_ctx ctx, int64_t interval_index, double* start, double* end,
                                  uint8_t* status, int64_t capacity, int64_t* n_out, uint32_t flags) {
    return lag_extract_ex(ctx, interval_index, start, end, status, nullptr, capacity, n_out, flags);
}

extern "C" lag_status lag_extract_ex(lag_ctx ctx, int64_t interval_index, double* start, double* end,
                                     uint8_t* status, int32_t* term_cycle, int64_t capacity,
                                     int64_t* n_out, uint32_t flags) {
    if (n_out) *n_out = 0;
    if (!ctx) { lag_set_error(nullptr, "ctx is NULL"); return LAG_EINVAL; }
    if (!ctx->seeded) { lag_set_error(ctx, "lag_extract before lag_seed"); return LAG_ESTATE; }
    if (interval_index != ctx->intervals_done) {
        lag_set_error(ctx, "lag_extract of interval %lld out of order (next is %lld)",
                      (long long)interval_index, (long long)ctx->intervals_done);
        return LAG_ESTATE;
    }
    const bool local = ctx->cfg.mode == LAG_COMM && ctx->cfg.exchange == LAG_XCHG_LOCAL;
    if (local && !ctx->group) { lag_set_error(ctx, "LAG_XCHG_LOCAL context without lag_local_group"); return LAG_ESTATE; }
    if (capacity < ctx->n_seeds && (start || end || status || term_cycle)) {
        lag_set_error(ctx, "capacity %lld < %lld seeds", (long long)capacity, (long long)ctx->n_seeds);
        return LAG_EINVAL;
    }
    CK(cudaSetDevice(ctx->cfg.device));
    lag_status st;
    if (local) {
        st = lag_local_flush(ctx);                // the group's pending hand-offs, once
        if (st != LAG_OK) return st;
    } else if (ctx->cfg.mode == LAG_COMM) {
        st = lag_comm_return_to_origin(ctx);      // collective; leaves only own-origin records
        if (st != LAG_OK) return st;
    }
    const int D = ctx->cfg.dim;
    ExtractArgs e{};
    e.state = ctx->state; e.tile_count = ctx->tile_count;
    e.n_tiles = ctx->cfg.mode == LAG_COMM ? ctx->cap_tiles : ctx->n_tiles;
    e.n_tiles_dev = ctx->cfg.mode == LAG_COMM ? (const int32_t*)(ctx->words + W_NTILES) : nullptr;
    e.dead_rec = ctx->dead_rec; e.dead_info = ctx->dead_info;
    e.n_dead_dev = ctx->words + W_DEAD; e.dead_cap = (uint32_t)ctx->cap;
    e.n = ctx->n_seeds; e.dim = D; e.stride = ctx->stride;
    for (int a = 0; a < 3; ++a) {
        e.first[a] = ctx->first[a]; e.ns[a] = ctx->ns[a];
        e.o[a] = ctx->cfg.origin[a]; e.h[a] = ctx->cfg.spacing[a];
    }
    e.bx = ctx->bits[0]; e.by = ctx->bits[1];
    e.mx = (1u << ctx->bits[0]) - 1u; e.my = (1u << ctx->bits[1]) - 1u;
    for (int a = 0; a < 3; ++a) { e.lo[a] = (int)ctx->cfg.block_lo[a]; e.hi[a] = (int)ctx->cfg.block_hi[a]; }
    e.ret = nullptr; e.n_ret = 0;
    if (ctx->cfg.mode == LAG_COMM) {
        int64_t stride_f4 = 2;
        lag_comm_returned(ctx, &e.ret, &stride_f4, &e.n_ret);
    }
    e.start = out_target(ctx, start, ctx->out_start);
    e.end = out_target(ctx, end, ctx->out_end);
    e.status = out_target(ctx, status, ctx->out_status);
    e.term_cycle = term_cycle ? out_target(ctx, term_cycle, ctx->out_cycle) : nullptr;
    const bool async = (flags & LAG_ASYNC) != 0;
    if (async) {
        // device outputs of this device, or page-locked host outputs (copied
        // from the staging buffers by stream-ordered asynchronous copies)
        for (const void* p : {(const void*)start, (const void*)end, (const void*)status, (const void*)term_cycle}) {
            if (!p) continue;
            cudaPointerAttributes at{};
            const bool ok = cudaPointerGetAttributes(&at, p) == cudaSuccess &&
                            ((at.type == cudaMemoryTypeDevice && at.device == ctx->cfg.device) ||
                             at.type == cudaMemoryTypeHost);
            if (!ok) {
                cudaGetLastError();
                lag_set_error(ctx, "LAG_ASYNC needs device outputs on device %d or page-locked host outputs",
                              ctx->cfg.device);
                return LAG_EINVAL;
            }
        }
    }
    e.write_start = ctx->cfg.mode == LAG_BTO ? 1 : 0;
    const unsigned nb_seed = (unsigned)((ctx->n_seeds + 255) / 256);
    const unsigned nb_dead = (unsigned)std::max(1, ctx->num_sms * 2);
    if (!e.write_start) {
        if (D == 3) extract_start_kernel<3><<<nb_seed, 256, 0, ctx->stream>>>(e);
        else extract_start_kernel<2><<<nb_seed, 256, 0, ctx->stream>>>(e);
        ++ctx->launches;
    }
    // LOCAL: every block of the group may hold particles seeded here (the
    // group's last hand-offs were appended by lag_local_flush); the own-seed
    // filter of the scatter kernels picks this block's
    const int nsrc = local ? lag_local_size(ctx) : 1;
    for (int q = 0; q < nsrc; ++q) {
        ExtractArgs eq = e;
        if (local) {
            const lag_ctx_s* m = lag_local_member(ctx, q);
            if (!m) { lag_set_error(ctx, "LAG_XCHG_LOCAL: block %d of the group was destroyed", q); return LAG_ESTATE; }
            eq.state = m->state; eq.tile_count = m->tile_count; eq.n_tiles = m->cap_tiles;
            eq.n_tiles_dev = (const int32_t*)(m->words + W_NTILES);
            eq.dead_rec = m->dead_rec; eq.dead_info = m->dead_info;
            eq.n_dead_dev = m->words + W_DEAD; eq.dead_cap = (uint32_t)m->cap;
        }
        const unsigned nbl = (unsigned)(((int64_t)eq.n_tiles * kTile + 255) / 256);
        if (D == 3) {
            extract_live_kernel<3><<<nbl, 256, 0, ctx->stream>>>(eq);
            extract_dead_kernel<3><<<nb_dead, 256, 0, ctx->stream>>>(eq);
        } else {
            extract_live_kernel<2><<<nbl, 256, 0, ctx->stream>>>(eq);
            extract_dead_kernel<2><<<nb_dead, 256, 0, ctx->stream>>>(eq);
        }
        ctx->launches += 2;
    }
    if (e.n_ret > 0) {
        if (D == 3) extract_returned_kernel<3><<<(e.n_ret + 255) / 256, 256, 0, ctx->stream>>>(e);
        else extract_returned_kernel<2><<<(e.n_ret + 255) / 256, 256, 0, ctx->stream>>>(e);
        ++ctx->launches;
    }
    CK(cudaGetLastError());
    const size_t n = (size_t)ctx->n_seeds;
    if ((st = copy_out(ctx, start, e.start, n * D * sizeof(double))) != LAG_OK) return st;
    if ((st = copy_out(ctx, end, e.end, n * D * sizeof(double))) != LAG_OK) return st;
    if ((st = copy_out(ctx, status, e.status, n)) != LAG_OK) return st;
    if ((st = copy_out(ctx, term_cycle, e.term_cycle, n * sizeof(int32_t))) != LAG_OK) return st;
    lag_status err = LAG_OK;
    if (!async) {
        CK(cudaMemcpyAsync(&ctx->host_words[0], ctx->words, kWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));  // the only host sync of the write cycle
        if (ctx->cfg.mode == LAG_COMM) {
            lag_status ne = lag_comm_async_error(ctx);
            if (ne != LAG_OK) return ne;
        }
        err = latched(ctx, ctx->host_words[W_ERR]);
        if (ctx->host_words[W_ERR])              // reported: clear the latch
            CK(cudaMemsetAsync(ctx->words + W_ERR, 0, sizeof(uint32_t), ctx->stream));
    }
    if (n_out) *n_out = ctx->n_seeds;
    ++ctx->intervals_done;
    if (local) {
        // every block must gather its flows before any block is reseeded:
        // the last extract of the group reseeds the blocks that asked for it
        ctx->reseed_pending = !(flags & LAG_NO_RESEED);
        bool all = false;
        lag_local_extracted(ctx, &all);
        if (all) {
            // every block's gather is done before any block's list is reseeded
            if ((st = lag_local_join_all(ctx)) != LAG_OK) return st;
            for (int q = 0; q < lag_local_size(ctx); ++q) {
                lag_ctx_s* m = lag_local_member(ctx, q);
                if (!m || !m->reseed_pending) continue;
                m->reseed_pending = false;
                st = lag_seed(m, m->stride, nullptr);
                if (st != LAG_OK) {
                    if (m != ctx) lag_set_error(ctx, "block %d: %s", q, m->msg.c_str());
                    return st;
                }
            }
        }
        return err;
    }
    if (!(flags & LAG_NO_RESEED)) {
        st = lag_seed(ctx, ctx->stride, nullptr);
        if (st != LAG_OK) return st;
    } else {
        ctx->seeded = true;   // outputs stay valid; advect continues the interval
    }
    return err;
}

extern "C" lag_status lag_stats(lag_ctx ctx, lag_stats_t* out) {
    if (!ctx || !out) { lag_set_error(ctx, "NULL argument"); return LAG_EINVAL; }
    CK(cudaSetDevice(ctx->cfg.device));
    unsigned long long c[CNT_N];
    CK(cudaMemcpyAsync(c, ctx->counters, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(&ctx->host_words[0], ctx->words, kWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->cfg.mode == LAG_COMM) {
        lag_status ne = lag_comm_async_error(ctx);
        if (ne != LAG_OK) return ne;
    }
    std::memset(out, 0, sizeof(*out));
    out->seeded = ctx->seeded ? ctx->n_seeds : 0;
    out->term_boundary = (int64_t)c[CNT_TERM];
    out->exit_domain = (int64_t)c[CNT_EXIT];
    out->sent = (int64_t)c[CNT_SENT];
    out->received = (int64_t)c[CNT_RECV];
    out->particle_steps = (int64_t)c[CNT_STEPS];
    out->cycles = ctx->cycles_total;
    out->active = out->seeded + out->received - out->sent - out->term_boundary - out->exit_domain;
    out->device_error = (int32_t)latched(ctx, ctx->host_words[W_ERR]);
    if (ctx->phase_timing) {
        fold_phases(ctx);
        out->phase_ms[0] = ctx->ph_ms[0]; out->phase_ms[1] = ctx->ph_ms[1]; out->phase_ms[2] = ctx->ph_ms[2];
    }
    return LAG_OK;
}
