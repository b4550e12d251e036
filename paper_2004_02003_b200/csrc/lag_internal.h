// lag_internal.h — context layout shared by lag_api.cu and lag_comm.cu.
#pragma once
#include "lag.h"
#include "lag_kernels.cuh"

#include <cuda_runtime.h>
#include <string>

namespace lag {
// W_NTILES_B / W_DEFER: overlap transport, two words each (cycle parity)
enum : int { W_DEAD = 0, W_ERR = 1, W_NTILES = 2, W_APPEND_DONE = 3, W_NTILES_B = 4, W_DEFER = 6, kWords = 8 };
struct Comm;         // lag_comm.cu
struct LocalGroup;   // lag_comm.cu (LAG_XCHG_LOCAL)
}

struct lag_ctx_s {
    lag_config cfg{};
    cudaStream_t stream = nullptr;
    std::string msg = "no error";
    // geometry
    int ext[3] = {1, 1, 1};          // slice extent (nodes) incl. ghosts
    int base[3] = {0, 0, 0};         // global node of slice element 0
    int bits[3] = {0, 0, 0};         // packed seed-node widths
    int sx = 1, sxy = 1;             // slice row / plane pitch in nodes (row_pitch_bytes)
    int64_t slice_floats = 0;        // floats of one slice array (pitched)
    int num_sms = 148;
    int advect_blocks_per_sm = 1;
    // particles
    int64_t max_seeds = 0, cap = 0;
    int cap_tiles = 0;
    int n_tiles = 0;                 // tiles holding seeds
    int brick[2] = {1, 1};           // seed brick rows (y, z) of 32-seed tiles
    int64_t n_seeds = 0, active_host = 0;
    int first[3] = {0, 0, 0}, ns[3] = {1, 1, 1};
    int stride = 1;
    bool seeded = false;
    bool stream_synced_needed = true;
    int cycles_in_interval = 0;
    int64_t cycles_total = 0;
    int64_t intervals_done = 0;      // write cycles extracted (lag_extract interval_index)
    bool reseed_pending = false;     // LOCAL: reseed when the group's last block extracted
    int64_t launches = 0;
    float4* state = nullptr;
    uint8_t* tile_count = nullptr;
    float4* dead_rec = nullptr;
    uint32_t* dead_info = nullptr;
    uint32_t* words = nullptr;                 // W_*
    unsigned long long* counters = nullptr;    // CNT_*
    uint32_t host_words[lag::kWords] = {0};
    // extraction staging (device)
    double* out_start = nullptr;
    double* out_end = nullptr;
    uint8_t* out_status = nullptr;
    int32_t* out_cycle = nullptr;
    // host-pointer staging (end-to-end path)
    // three staging buffers on their own copy stream: the H2D copy of the
    // next cycle's slice overlaps the current cycle's kernels
    static constexpr int kStage = 3;
    float* stage[kStage] = {nullptr, nullptr, nullptr};
    const void* stage_src[kStage] = {nullptr, nullptr, nullptr};
    int64_t stage_use[kStage] = {-1, -1, -1};     // cycle that last read the buffer
    cudaEvent_t stage_ready[kStage] = {};         // copy done (copy stream)
    cudaEvent_t stage_free[kStage] = {};          // last reader done (ctx->stream)
    cudaStream_t cstream = nullptr;
    int last_v1_slot = -1;                        // buffer holding the previous call's host v_t1
    const void* last_v1 = nullptr;
    const float* prev_d0 = nullptr;            // device slices the last advect kernel read
    const float* prev_d1 = nullptr;
    // COMM
    lag::Comm* comm = nullptr;
    lag::LocalGroup* group = nullptr;          // LAG_XCHG_LOCAL
    // LAG_XCHG_PEER_OVERLAP: the exchange runs in the first CTAs of the advect
    // pass 1 while the ghost-free tiles advect; deferred tile ids in defer_list
    void* xchg_fused = nullptr;                // non-null: lag_peer_exchange fills this XchgFused, no launch
    uint32_t* defer_list = nullptr;
    // phase timing (LAG_PHASE_TIMING=1): events around pre-exchange / advect / post
    bool phase_timing = false;
    cudaEvent_t ph_ev[64][4] = {};
    int ph_n = 0;
    double ph_ms[3] = {0.0, 0.0, 0.0};
};

int lag_set_error(lag_ctx_s* ctx, const char* fmt, ...);
lag_status lag_reset_interval(lag_ctx_s* ctx);

// lag_comm.cu
lag_status lag_comm_init(lag_ctx_s* ctx);
void lag_comm_destroy(lag_ctx_s* ctx);
lag_status lag_comm_reset(lag_ctx_s* ctx);
lag_status lag_comm_pre_advect(lag_ctx_s* ctx, float* v0, float* v1, bool v0_is_prev_v1);
void lag_comm_fill_args(lag_ctx_s* ctx, lag::AdvectArgs* a);
lag_status lag_comm_post_advect(lag_ctx_s* ctx);
bool lag_comm_overlap(lag_ctx_s* ctx);        // LAG_XCHG_PEER_OVERLAP with neighbours
lag_status lag_comm_return_to_origin(lag_ctx_s* ctx);
lag_status lag_comm_async_error(lag_ctx_s* ctx);   // ncclCommGetAsyncError poll
// LAG_XCHG_LOCAL (lag_comm.cu): group cycle and write cycle
struct lag_local_rec { float* v0; float* v1; double dt; bool v0_prev; };
lag_status lag_local_record(lag_ctx_s* ctx, const lag_local_rec& r, bool* complete);
lag_status lag_local_run_cycle(lag_ctx_s* ctx);   // ghost copy + appends (group-wide)
lag_ctx_s* lag_local_member(lag_ctx_s* ctx, int r);
const lag_local_rec& lag_local_recorded(lag_ctx_s* ctx, int r);
int lag_local_size(lag_ctx_s* ctx);
lag_status lag_local_flush(lag_ctx_s* ctx);       // first extract of the group: pending hand-offs
lag_status lag_local_join_all(lag_ctx_s* ctx);    // every block's stream waits for every other
bool lag_local_extracted(lag_ctx_s* ctx, bool* all);   // mark this block extracted
bool lag_local_extracting(lag_ctx_s* ctx);        // some block extracted, not all
void lag_local_leave(lag_ctx_s* ctx);
void lag_comm_returned(lag_ctx_s* ctx, const float4** rec, int64_t* stride_f4, uint32_t* n);
