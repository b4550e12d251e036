// lag_ftle.cu — finite-time Lyapunov exponent of an extracted flow map.
//
// The paper's qualitative output is FTLE fields computed post hoc from the
// basis flows (§4.3); SPEC.md:460-468 states the operation: the
// flow-map gradient by central differences on the seed lattice (one-sided at
// the lattice faces), the right Cauchy-Green tensor C = J^T J, and
// FTLE = ln(sqrt(lambda_max(C))) / |T|, with lambda_max <= 0 giving 0 (counted).
//
// One thread per lattice node (x fastest; one CTA row per (y, z) line, no
// index division).  The 2*dim neighbour end positions are read through L1/L2
// (three consecutive planes stay resident in L2), so HBM sees each end
// position about once: the kernel is HBM-bound at 8*dim B read + 8 B written
// per node.  lambda_max: closed form in 2D; in 3D a cyclic Jacobi
// eigenvalue iteration in f64, accurate to rounding relative to ||C||
// (a trigonometric closed form loses ~sqrt(eps) near repeated eigenvalues).
#include "lag.h"
#include "lag_internal.h"

#include <cstdint>
#include <mutex>

namespace {

struct FtleArgs {
    const double* ends;     // [n][dim]
    double* out;            // [n]
    unsigned long long* n_degenerate;
    int64_t dims[3];
    double inv_sp[3], inv_sp2[3];   // 1 / seed spacing, 1 / (2 * spacing)
    double inv_absT;
};

// dF/dX_a at lattice index p along axis a (numpy.gradient, edge_order=1):
// interior (f[i+1] - f[i-1]) / (2 dx); faces (f[1] - f[0]) / dx, (f[n-1] - f[n-2]) / dx.
// (Multiplied by the reciprocal: within 1 ulp of the division.)
template <int DIM>
__device__ __forceinline__ void grad_axis(const FtleArgs& a, int64_t i, int64_t p, int64_t n, int64_t str,
                                          int ax, double J[DIM][DIM]) {
    if (n < 2) {
        #pragma unroll
        for (int c = 0; c < DIM; ++c) J[c][ax] = 0.0;
        return;
    }
    const int64_t lo = p > 0 ? i - str : i, hi = p < n - 1 ? i + str : i;
    const double inv = (p > 0 && p < n - 1) ? a.inv_sp2[ax] : a.inv_sp[ax];
    #pragma unroll
    for (int c = 0; c < DIM; ++c)
        J[c][ax] = (__ldg(a.ends + hi * DIM + c) - __ldg(a.ends + lo * DIM + c)) * inv;
}

__device__ __forceinline__ void jacobi_rotate(double A[3][3], int p, int q) {
    // rotation angle zeroing A[p][q]: with d = A[q][q] - A[p][p] the smaller
    // root of t^2 + (d / apq) t - 1 = 0 is t = 2 apq sgn(d) / (|d| + sqrt(d^2 + 4 apq^2))
    const double apq = A[p][q];
    if (apq == 0.0) return;
    const double d = A[q][q] - A[p][p];
    const double t = copysign(1.0, d) * (2.0 * apq) / (fabs(d) + sqrt(fma(d, d, 4.0 * apq * apq)));
    const double c = rsqrt(fma(t, t, 1.0)), s = t * c;
    A[p][p] -= t * apq;
    A[q][q] += t * apq;
    A[p][q] = A[q][p] = 0.0;
    const int r = 3 - p - q;
    const double arp = A[r][p], arq = A[r][q];
    A[r][p] = A[p][r] = c * arp - s * arq;
    A[r][q] = A[q][r] = s * arp + c * arq;
}

template <int DIM>
__global__ void __launch_bounds__(128) ftle_kernel(FtleArgs a) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= a.dims[0]) return;
    const int64_t pos[3] = {x, blockIdx.y, blockIdx.z};
    const int64_t str[3] = {1, a.dims[0], a.dims[0] * a.dims[1]};
    const int64_t i = x + pos[1] * str[1] + pos[2] * str[2];
    double J[DIM][DIM];
    #pragma unroll
    for (int ax = 0; ax < DIM; ++ax) grad_axis<DIM>(a, i, pos[ax], a.dims[ax], str[ax], ax, J);
    double C[3][3];
    bool finite = true;
    #pragma unroll
    for (int p = 0; p < DIM; ++p)
        #pragma unroll
        for (int q = 0; q < DIM; ++q) {
            double s = 0.0;
            #pragma unroll
            for (int c = 0; c < DIM; ++c) s = fma(J[c][p], J[c][q], s);
            C[p][q] = s;
            finite &= isfinite(s);
        }
    double lam;
    if (!finite) {
        a.out[i] = __longlong_as_double(0x7ff8000000000000LL);
        return;
    }
    if (DIM == 2) {
        const double h = 0.5 * (C[0][0] - C[1][1]);
        lam = 0.5 * (C[0][0] + C[1][1]) + hypot(h, C[0][1]);
    } else {
        #pragma unroll 1
        for (int sweep = 0; sweep < 8; ++sweep) {
            const double off = fabs(C[0][1]) + fabs(C[0][2]) + fabs(C[1][2]);
            const double diag = fabs(C[0][0]) + fabs(C[1][1]) + fabs(C[2][2]);
            if (off <= 1e-18 * diag || off == 0.0) break;
            jacobi_rotate(C, 0, 1);
            jacobi_rotate(C, 0, 2);
            jacobi_rotate(C, 1, 2);
        }
        lam = fmax(C[0][0], fmax(C[1][1], C[2][2]));
    }
    if (!(lam > 0.0)) {
        a.out[i] = 0.0;
        atomicAdd(a.n_degenerate, 1ull);
        return;
    }
    a.out[i] = 0.5 * log(lam) * a.inv_absT;
}

// per-device degenerate-tensor counter, allocated once (calls serialised)
std::mutex g_cnt_mu;
unsigned long long* g_cnt[64];

}  // namespace

extern "C" lag_status lag_ftle(int32_t dim, const int64_t* dims, const double* spacing, double T,
                               const double* ends, double* ftle, int64_t* n_degenerate, void* stream) {
    lag_ctx_s* ctx = nullptr;
    if ((dim != 2 && dim != 3) || !dims || !spacing || !ends || !ftle || !(T == T) || T == 0.0 ||
        !isfinite(T)) {
        lag_set_error(ctx, "lag_ftle: bad arguments");
        return LAG_EINVAL;
    }
    FtleArgs a{};
    a.ends = ends; a.out = ftle;
    a.inv_absT = 1.0 / fabs(T);
    for (int ax = 0; ax < 3; ++ax) {
        a.dims[ax] = ax < dim ? dims[ax] : 1;
        const double h = ax < dim ? spacing[ax] : 1.0;
        if (a.dims[ax] < 1 || !(h > 0.0) || !isfinite(h)) {
            lag_set_error(ctx, "lag_ftle: dims must be >= 1 and spacing finite and > 0");
            return LAG_EINVAL;
        }
        a.inv_sp[ax] = 1.0 / h;
        a.inv_sp2[ax] = 1.0 / (2.0 * h);
    }
    if (a.dims[1] > 65535 || a.dims[2] > 65535) {
        lag_set_error(ctx, "lag_ftle: lattice y/z extent above 65535");
        return LAG_EINVAL;
    }
    cudaPointerAttributes at{};
    for (const void* p : {(const void*)ends, (const void*)ftle}) {
        if (cudaPointerGetAttributes(&at, p) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
            cudaGetLastError();
            lag_set_error(ctx, "lag_ftle: arrays must be device memory");
            return LAG_EINVAL;
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_cnt_mu);
    unsigned long long*& cnt = g_cnt[dev & 63];
    if (!cnt && cudaMalloc((void**)&cnt, sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        cnt = nullptr;
        lag_set_error(ctx, "lag_ftle: counter allocation failed");
        return LAG_ENOMEM;
    }
    a.n_degenerate = cnt;
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), s);
    if (e == cudaSuccess) {
        const dim3 grid((unsigned)((a.dims[0] + 127) / 128), (unsigned)a.dims[1], (unsigned)a.dims[2]);
        if (dim == 2) ftle_kernel<2><<<grid, 128, 0, s>>>(a);
        else ftle_kernel<3><<<grid, 128, 0, s>>>(a);
        e = cudaGetLastError();
    }
    unsigned long long h_cnt = 0;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) { lag_set_error(ctx, "lag_ftle: %s", cudaGetErrorString(e)); return LAG_ECUDA; }
    if (n_degenerate) *n_degenerate = (int64_t)h_cnt;
    return LAG_OK;
}
