// lag_recon.cu — post hoc reconstruction of BTO holes on the GPU (GridFill).
//
// Paper: flow information lost at block boundaries "can be interpolated using
// additional information from adjacent processes post hoc" (§3.1;
// reconstruction P:262-274 §3.2).  Eq. 2 (§3.3) shows linear
// interpolation through a hole equals interpolation between its valid
// neighbours; GridFill applies Eq. 1 along lattice axes.
// Reading R18: each hole takes the axis with the shortest valid
// bracket; ties are averaged.
//
// Two passes: (1) a coalesced copy of the valid nodes that compacts the holes
// into a scratch list (one warp-aggregated atomic per warp); (2) one thread
// per hole, whose bracket search grows a radius over all axes at once and
// stops as soon as no shorter bracket can exist, so holes in bands a few
// seeds wide touch only a few nodes.  Arithmetic uses explicit
// round-to-nearest double ops (no FMA contraction) in the same order as the
// CPU version, so the result is bitwise reproducible.
#include "lag.h"
#include "lag_internal.h"

#include <climits>
#include <mutex>
#include <cstdint>

namespace {

struct FillArgs {
    const double* values;   // [n][k]
    const uint8_t* valid;   // [n]
    double* out;            // [n][k]
    uint8_t* filled;        // [n]
    int64_t dims[3];
    int dim, k;
    int64_t n;
    int64_t* holes;                 // scratch: compacted hole indices (order irrelevant)
    unsigned long long* n_holes;    // scratch: their count
};

__global__ void __launch_bounds__(256) gridfill_copy_kernel(FillArgs a) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < a.n;
    const bool hole = in && !__ldg(a.valid + i);
    if (in && !hole) {
        for (int c = 0; c < a.k; ++c) a.out[i * a.k + c] = __ldg(a.values + i * a.k + c);
        a.filled[i] = 0;
    }
    // one global atomic per CTA (not per warp): the counter is a single L2 line
    __shared__ unsigned warp_count[8], warp_off[8];
    __shared__ unsigned long long cta_base;
    const unsigned m = __ballot_sync(0xffffffffu, hole);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) warp_count[warp] = __popc(m);
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned tot = 0;
        for (int w = 0; w < 8; ++w) { warp_off[w] = tot; tot += warp_count[w]; }
        cta_base = tot ? atomicAdd(a.n_holes, (unsigned long long)tot) : 0;
    }
    __syncthreads();
    if (hole) a.holes[cta_base + warp_off[warp] + __popc(m & ((1u << lane) - 1))] = i;
}

template <int DIM>
__device__ __forceinline__ void fill_hole(const FillArgs& a, int64_t i) {
    const int dims[3] = {(int)a.dims[0], (int)a.dims[1], (int)a.dims[2]};
    const int64_t str[3] = {1, a.dims[0], a.dims[0] * a.dims[1]};
    const int pos[3] = {(int)(i % a.dims[0]), (int)((i / a.dims[0]) % a.dims[1]),
                        (int)(i / (a.dims[0] * a.dims[1]))};
    const int k = a.k;
    // Radius search: a side is found at the first valid node at distance d.
    // A bracket with sides (dl, dr) is complete once d >= max(dl, dr), and
    // its span dl + dr is at least max(dl, dr) + 1; so once d >= best - 1 no
    // unfound bracket can be as short as the best found: the search is exact.
    int dl[DIM], dr[DIM];            // distance to the valid side; 0 = not found yet, -1 = none
    #pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        dl[ax] = pos[ax] == 0 ? -1 : 0;
        dr[ax] = pos[ax] == dims[ax] - 1 ? -1 : 0;
    }
    // The radii are visited in chunks of R whose loads are all issued before
    // any is tested (a hole with no bracket walks to the lattice faces; the
    // chunking turns that dependent chain into R-wide independent loads).
    constexpr int R = 4;
    int best = INT_MAX;
    for (int d0 = 1;; d0 += R) {
        uint32_t lv[DIM], rv[DIM];   // bit j: node at distance d0 + j is valid
        #pragma unroll
        for (int ax = 0; ax < DIM; ++ax) {
            lv[ax] = rv[ax] = 0;
            #pragma unroll
            for (int j = 0; j < R; ++j) {
                const int d = d0 + j;
                if (dl[ax] == 0 && d <= pos[ax]) lv[ax] |= (uint32_t)(__ldg(a.valid + i - d * str[ax]) != 0) << j;
                if (dr[ax] == 0 && pos[ax] + d < dims[ax])
                    rv[ax] |= (uint32_t)(__ldg(a.valid + i + d * str[ax]) != 0) << j;
            }
        }
        bool stop = false;
        #pragma unroll
        for (int j = 0; j < R; ++j) {
            const int d = d0 + j;
            bool open = false;
            #pragma unroll
            for (int ax = 0; ax < DIM; ++ax) {
                if (dl[ax] == 0) {
                    if (lv[ax] >> j & 1) dl[ax] = d;
                    else if (pos[ax] == d) dl[ax] = -1;
                }
                if (dr[ax] == 0) {
                    if (rv[ax] >> j & 1) dr[ax] = d;
                    else if (pos[ax] + d == dims[ax] - 1) dr[ax] = -1;
                }
                if (dl[ax] > 0 && dr[ax] > 0) best = min(best, dl[ax] + dr[ax]);
                open |= dl[ax] == 0 || dr[ax] == 0;
            }
            if (!open || d >= best - 1) { stop = true; break; }
        }
        if (stop) break;
    }
    // Eq. 1 along every axis whose bracket is the shortest, averaged
    int nbest = 0;
    double acc[3] = {0.0, 0.0, 0.0};
    #pragma unroll
    for (int ax = 0; ax < DIM; ++ax) {
        if (dl[ax] <= 0 || dr[ax] <= 0 || dl[ax] + dr[ax] != best) continue;
        const double wr = __ddiv_rn((double)dl[ax], (double)best);
        const double wl = __dsub_rn(1.0, wr);
        const int64_t il = i - dl[ax] * str[ax], ir = i + dr[ax] * str[ax];
        #pragma unroll
        for (int c = 0; c < 3; ++c)
            if (c < k)
                acc[c] = __dadd_rn(acc[c], __dadd_rn(__dmul_rn(wl, __ldg(a.values + il * k + c)),
                                                     __dmul_rn(wr, __ldg(a.values + ir * k + c))));
        ++nbest;
    }
    #pragma unroll
    for (int c = 0; c < 3; ++c)
        if (c < k)
            a.out[i * k + c] = nbest ? __ddiv_rn(acc[c], (double)nbest)
                                     : __longlong_as_double(0x7ff8000000000000LL);
    a.filled[i] = nbest ? 1 : 0;
}

template <int DIM>
__global__ void __launch_bounds__(128) gridfill_hole_kernel(FillArgs a) {
    const unsigned long long nh = *a.n_holes;
    for (unsigned long long h = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; h < nh;
         h += (unsigned long long)gridDim.x * blockDim.x)
        fill_hole<DIM>(a, a.holes[h]);
}

// Grow-only per-device scratch (hole list + counter), reused across calls so a
// call costs no allocation; calls on one device are serialised by the mutex.
struct Scratch {
    void* ptr = nullptr;
    size_t bytes = 0;
};
std::mutex g_scratch_mu;
Scratch g_scratch[64];

}  // namespace

extern "C" lag_status lag_gridfill(int32_t dim, const int64_t* dims, int32_t k, const double* values,
                                   const uint8_t* valid, double* out, uint8_t* filled, void* stream) {
    lag_ctx_s* ctx = nullptr;
    if ((dim != 2 && dim != 3) || !dims || k < 1 || k > 3 || !values || !valid || !out || !filled) {
        lag_set_error(ctx, "lag_gridfill: bad arguments");
        return LAG_EINVAL;
    }
    FillArgs a{};
    a.values = values; a.valid = valid; a.out = out; a.filled = filled;
    a.dim = dim; a.k = k;
    a.n = 1;
    for (int ax = 0; ax < 3; ++ax) {
        a.dims[ax] = ax < dim ? dims[ax] : 1;
        if (a.dims[ax] < 1 || a.dims[ax] > INT_MAX / 2) {
            lag_set_error(ctx, "lag_gridfill: lattice extent must be in [1, 2^30]");
            return LAG_EINVAL;
        }
        a.n *= a.dims[ax];
    }
    cudaPointerAttributes at{};
    for (const void* p : {(const void*)values, (const void*)valid, (const void*)out, (const void*)filled}) {
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            lag_set_error(ctx, "lag_gridfill: arrays must be device memory");
            return LAG_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    Scratch& sc = g_scratch[dev & 63];
    const size_t need = 16 + (size_t)a.n * sizeof(int64_t);
    if (sc.bytes < need) {
        if (sc.ptr) cudaFree(sc.ptr);
        sc.ptr = nullptr;
        sc.bytes = 0;
        if (cudaMalloc(&sc.ptr, need) != cudaSuccess) {
            cudaGetLastError();
            lag_set_error(ctx, "lag_gridfill: scratch allocation of %zu bytes failed", need);
            return LAG_ENOMEM;
        }
        sc.bytes = need;
    }
    void* scratch = sc.ptr;
    cudaError_t e = cudaSuccess;
    a.n_holes = (unsigned long long*)scratch;
    a.holes = (int64_t*)((char*)scratch + 16);
    e = cudaMemsetAsync(a.n_holes, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
        gridfill_copy_kernel<<<(unsigned)((a.n + 255) / 256), 256, 0, s>>>(a);
        if (dim == 2) gridfill_hole_kernel<2><<<nsm * 16, 128, 0, s>>>(a);
        else gridfill_hole_kernel<3><<<nsm * 16, 128, 0, s>>>(a);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { lag_set_error(ctx, "lag_gridfill: %s", cudaGetErrorString(e)); return LAG_ECUDA; }
    return LAG_OK;
}
