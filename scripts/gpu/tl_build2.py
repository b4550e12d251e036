"""Build liblag_TL2.so: %globaltimer stamps of the overlapped COMM cycle
(LAG_XCHG_PEER_OVERLAP), slot = cycle in the interval (0..63), per slot:
  0 pass-1 entry (CTA 0)      1 end of the exchange CTAs (max)
  2 end of pass-1 advect CTAs (max over warps)
  3 pass-2 start after its wait (CTA 0)  4 end of pass 2 (max over warps)
  5 first pass-1 advect CTA past its wait   6 pass-2 CTA 0 scheduled
read with lag_tl2_read (16 words per slot, 64 slots)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
TL = r'''namespace lag {
static __device__ unsigned long long g_tl2[64 * 16];
__device__ __forceinline__ unsigned long long tl_now() {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t;
}
__device__ __forceinline__ void tl2_set(int slot, int k) { g_tl2[(slot & 63) * 16 + k] = tl_now(); }
__device__ __forceinline__ void tl2_max(int slot, int k) { atomicMax(&g_tl2[(slot & 63) * 16 + k], tl_now()); }
'''
subs = [
    "namespace lag {\n\nconstexpr int kTile = 32;=>" + TL + "\nconstexpr int kTile = 32;",
    # pass 1
    """    griddep_launch();
    if ((int)blockIdx.x < xf.ncta) {
        xchg_pack_signal(xf.x, blockIdx.x, xf.ncta);
        xchg_wait_pull(xf.x, xf.ap, blockIdx.x, xf.ncta);
        return;
    }
    griddep_wait();
    advect_body<DIM, false, FROZEN, true>(a, blockIdx.x - xf.ncta, gridDim.x - xf.ncta);=>"""
    """    griddep_launch();
    if (blockIdx.x == 0 && threadIdx.x == 0) lag::tl2_set(a.cycle, 0);
    if ((int)blockIdx.x < xf.ncta) {
        xchg_pack_signal(xf.x, blockIdx.x, xf.ncta);
        xchg_wait_pull(xf.x, xf.ap, blockIdx.x, xf.ncta);
        if ((threadIdx.x & 31) == 0) lag::tl2_max(a.cycle, 1);
        return;
    }
    griddep_wait();
    if (blockIdx.x == xf.ncta && threadIdx.x == 0) lag::tl2_set(a.cycle, 5);
    advect_body<DIM, false, FROZEN, true>(a, blockIdx.x - xf.ncta, gridDim.x - xf.ncta);
    if ((threadIdx.x & 31) == 0) lag::tl2_max(a.cycle, 2);""",
    # pass 2 (PASSES advect_kernel)
    """    griddep_wait();
    griddep_launch();
    advect_body<DIM, BTO, FROZEN, PASSES>(a, blockIdx.x, gridDim.x);=>"""
    """    if (PASSES && blockIdx.x == 0 && threadIdx.x == 0) tl2_set(a.cycle, 6);
    griddep_wait();
    griddep_launch();
    if (PASSES && blockIdx.x == 0 && threadIdx.x == 0) tl2_set(a.cycle, 3);
    advect_body<DIM, BTO, FROZEN, PASSES>(a, blockIdx.x, gridDim.x);
    if (PASSES && (threadIdx.x & 31) == 0) tl2_max(a.cycle, 4);""",
    'extern "C" int32_t lag_abi_version(void) { return LAG_ABI_VERSION; }=>extern "C" int32_t lag_abi_version(void) { return LAG_ABI_VERSION; }\n'
    'extern "C" __attribute__((visibility("default"))) int lag_tl2_read(unsigned long long* h) { return (int)cudaMemcpyFromSymbol(h, lag::g_tl2, sizeof(lag::g_tl2)); }',
]
out = os.environ.get("TL_OUT", os.path.join(ROOT, "paper_2004_02003_b200", "liblag_TL2.so"))
extra = [e for e in os.environ.get("TL_EXTRA", "").split("@@") if e]
sys.exit(subprocess.call([sys.executable, os.path.join(ROOT, "scripts", "build_variant.py"), out] + subs + extra))
