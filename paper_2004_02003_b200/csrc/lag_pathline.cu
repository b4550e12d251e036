// lag_pathline.cu — pathline stitching from the basis flows of successive
// intervals (§3.2: "a trajectory can be stitched together by using
// basis flows of successive nonoverlapping intervals"; barycentric
// interpolation of end positions over a neighbourhood of basis flows,
// P:262-274).
//
// Reading R16: the seeds sit on a uniform lattice whose Delaunay
// triangulation is degenerate (cospherical cube corners); ties are broken by
// the fixed Kuhn (Freudenthal) template.  In the cube at index i with local
// coordinates f sorted descending f_(1) >= ... >= f_(d) (ties: lower axis
// first), the simplex vertices are v_0 = i, v_j = v_{j-1} + e_{pi_j} and the
// weights w_0 = 1 - f_(1), w_j = f_(j) - f_(j+1), w_d = f_(d).
//
// One thread per query pathline; per interval a handful of dependent 8-24 B
// gathers from that interval's end-position lattice (L2-resident for the
// lattice sizes of one block).  Latency-bound by design: K dependent steps.
#include "lag.h"
#include "lag_internal.h"

#include <cstdint>

namespace {

constexpr uint8_t ST_COMPLETE = 0, ST_OUT_OF_HULL = 1, ST_INVALID_FLOW = 2;

struct StitchArgs {
    const double* ends;     // [K][n][dim]
    const uint8_t* valid;   // [K][n] or null
    const double* starts;   // [m][dim]
    double* path;           // [m][K+1][dim]
    uint8_t* status;        // [m]
    int64_t dims[3];
    int64_t n, m;
    double origin[3], spacing[3];
    int K;
};

template <int D>
__global__ void __launch_bounds__(128) stitch_kernel(StitchArgs a) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.m) return;
    const double nan = __longlong_as_double(0x7ff8000000000000LL);
    double x[D];
    double* out = a.path + q * (int64_t)(a.K + 1) * D;
    #pragma unroll
    for (int c = 0; c < D; ++c) out[c] = x[c] = a.starts[q * D + c];
    const int64_t str[3] = {1, a.dims[0], a.dims[0] * a.dims[1]};
    uint8_t st = ST_COMPLETE;
    int k = 0;
    for (; k < a.K; ++k) {
        double u[D];
        bool outside = false;
        #pragma unroll
        for (int c = 0; c < D; ++c) {
            u[c] = __ddiv_rn(__dsub_rn(x[c], a.origin[c]), a.spacing[c]);
            outside |= !(u[c] >= 0.0 && u[c] <= (double)(a.dims[c] - 1));      // NaN -> outside
        }
        if (outside) { st = ST_OUT_OF_HULL; break; }
        int64_t base = 0;
        double f[D];
        int ax[D];
        #pragma unroll
        for (int c = 0; c < D; ++c) {
            int64_t i = (int64_t)floor(u[c]);
            i = i < a.dims[c] - 2 ? i : a.dims[c] - 2;
            f[c] = __dsub_rn(u[c], (double)i);
            base += i * str[c];
            ax[c] = c;
        }
        // stable descending sort of (f, axis): insertion sort on D <= 3 items
        #pragma unroll
        for (int s = 1; s < D; ++s)
            #pragma unroll
            for (int t = s; t > 0; --t)
                if (f[ax[t]] > f[ax[t - 1]]) { const int tmp = ax[t]; ax[t] = ax[t - 1]; ax[t - 1] = tmp; }
        double w[D + 1];
        int64_t v[D + 1];
        w[0] = __dsub_rn(1.0, f[ax[0]]);
        v[0] = base;
        #pragma unroll
        for (int j = 1; j <= D; ++j) {
            w[j] = j < D ? __dsub_rn(f[ax[j - 1]], f[ax[j]]) : f[ax[D - 1]];
            v[j] = v[j - 1] + str[ax[j - 1]];
        }
        const double* E = a.ends + (int64_t)k * a.n * D;
        if (a.valid) {
            const uint8_t* ok = a.valid + (int64_t)k * a.n;
            bool bad = false;
            #pragma unroll
            for (int j = 0; j <= D; ++j) bad |= w[j] > 0.0 && !ok[v[j]];
            if (bad) { st = ST_INVALID_FLOW; break; }
        }
        double xn[D];
        #pragma unroll
        for (int c = 0; c < D; ++c) {
            double s = 0.0;
            #pragma unroll
            for (int j = 0; j <= D; ++j) s = __dadd_rn(s, __dmul_rn(w[j], __ldg(E + v[j] * D + c)));
            xn[c] = s;
        }
        #pragma unroll
        for (int c = 0; c < D; ++c) out[(k + 1) * D + c] = x[c] = xn[c];
    }
    for (int r = k + 1; r <= a.K; ++r)
        #pragma unroll
        for (int c = 0; c < D; ++c) out[r * D + c] = nan;
    a.status[q] = st;
}

}  // namespace

extern "C" lag_status lag_stitch(int32_t dim, const int64_t* dims, const double* origin, const double* spacing,
                                 int32_t K, const double* ends, const uint8_t* valid, int64_t m,
                                 const double* starts, double* path, uint8_t* status, void* stream) {
    lag_ctx_s* ctx = nullptr;
    if ((dim != 2 && dim != 3) || !dims || !origin || !spacing || K < 0 || m < 0 ||
        (K > 0 && !ends) || (m > 0 && (!starts || !path || !status))) {
        lag_set_error(ctx, "lag_stitch: bad arguments");
        return LAG_EINVAL;
    }
    StitchArgs a{};
    a.ends = ends; a.valid = valid; a.starts = starts; a.path = path; a.status = status;
    a.K = K; a.m = m; a.n = 1;
    for (int ax = 0; ax < 3; ++ax) {
        a.dims[ax] = ax < dim ? dims[ax] : 1;
        a.origin[ax] = ax < dim ? origin[ax] : 0.0;
        a.spacing[ax] = ax < dim ? spacing[ax] : 1.0;
        if ((ax < dim && a.dims[ax] < 2) || !(a.spacing[ax] > 0.0) || !isfinite(a.spacing[ax]) ||
            !isfinite(a.origin[ax])) {
            lag_set_error(ctx, "lag_stitch: dims must be >= 2, spacing finite and > 0, origin finite");
            return LAG_EINVAL;
        }
        a.n *= a.dims[ax];
    }
    if (m == 0) return LAG_OK;
    cudaPointerAttributes at{};
    for (const void* p : {(const void*)ends, (const void*)valid, (const void*)starts, (const void*)path,
                          (const void*)status}) {
        if (!p) continue;
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            lag_set_error(ctx, "lag_stitch: arrays must be device memory");
            return LAG_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)((m + 127) / 128);
    if (dim == 2) stitch_kernel<2><<<blocks, 128, 0, s>>>(a);
    else stitch_kernel<3><<<blocks, 128, 0, s>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { lag_set_error(ctx, "lag_stitch: %s", cudaGetErrorString(e)); return LAG_ECUDA; }
    return LAG_OK;
}
