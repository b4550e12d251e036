"""Build the %globaltimer-instrumented liblag_TL.so used by tl_peer.py (the
substitutions match the sources of commit a23c29d, where the timeline in
profiles/r2_comm_timeline_n2.txt was taken).  TL_OUT / TL_EXTRA: output and
extra substitutions ("old=>new", separated by @@)."""
import subprocess, sys, os
OUT = os.environ.get("TL_OUT", "paper_2004_02003_b200/liblag_TL.so")
EXTRA = [e for e in os.environ.get("TL_EXTRA", "").split("@@") if e]
TL = r'''namespace lag {
static __device__ unsigned long long g_tl[1024 * 16];
__device__ __forceinline__ void tl_max(unsigned long long seq, int k) {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(&g_tl[(seq & 1023) * 16 + k], t);
}
__device__ __forceinline__ void tl_stamp(unsigned long long seq, int k) {
    unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl[(seq & 1023) * 16 + k] = t;
}
'''
subs = [
 # infra (lag_kernels.cuh is included once per TU)
 "namespace lag {\n\nconstexpr int kTile = 32;=>" + TL + "\nconstexpr int kTile = 32;",
 # advect: entry of CTA 0 (k=5) and the last warp's signal (k=6)
 "    advect_body<DIM, BTO, FROZEN, PASSES>(a, blockIdx.x, gridDim.x);=>    const unsigned long long tseq = a.n_sig ? a.sig_value : 512ull + (unsigned long long)a.cycle;\n    if (blockIdx.x == 0 && threadIdx.x == 0) tl_stamp(tseq, 5);\n    advect_body<DIM, BTO, FROZEN, PASSES>(a, blockIdx.x, gridDim.x);\n    if ((threadIdx.x & 31) == 0) tl_max(tseq, 10);",
 "                        *reinterpret_cast<volatile unsigned long long*>(a.sig_flag[k]) = a.sig_value;\n                    __threadfence_system();=>                        *reinterpret_cast<volatile unsigned long long*>(a.sig_flag[k]) = a.sig_value;\n                    __threadfence_system();\n                    tl_stamp(a.sig_value, 6);",
 # exchange: entry (0), halo signalled (1), wait done (2), pulled (3), appended (4)
 "__device__ __forceinline__ void xchg_pack_signal(const XchgArgs& x, int cta, int ncta) {=>__device__ __forceinline__ void xchg_pack_signal(const XchgArgs& x, int cta, int ncta) {\n    if (cta == 0 && threadIdx.x == 0) tl_stamp(x.seq, 0);\n    if (threadIdx.x == 0) tl_max(x.seq, 11);",
 "    __syncthreads();                                  // the CTA's packs are visible to thread 0=>    __syncthreads();\n    if (threadIdx.x == 0) tl_max(x.seq, 8);",
 "        __threadfence();\n        if (atomicAdd(x.done_ctas, 1u) == (uint32_t)ncta - 1) {   // last CTA: halo(seq) ready=>        __threadfence();\n        tl_max(x.seq, 12);\n        if (atomicAdd(x.done_ctas, 1u) == (uint32_t)ncta - 1) {\n            tl_stamp(x.seq, 9);",
 "            for (int p = 0; p < x.npeers; ++p) *reinterpret_cast<volatile unsigned long long*>(x.halo_flag[p]) = x.seq;\n        }=>            for (int p = 0; p < x.npeers; ++p) *reinterpret_cast<volatile unsigned long long*>(x.halo_flag[p]) = x.seq;\n            tl_stamp(x.seq, 1);\n        }",
 "    __syncthreads();\n    // remote loads=>    __syncthreads();\n    if (cta == 0 && threadIdx.x == 0) tl_stamp(x.seq, 2);\n    if (threadIdx.x == 0) tl_max(x.seq, 13);\n    // remote loads",
 "    if (x.do_append) append_body(ap, cta, ncta);                         // hand-offs of cycle seq-1 (all CTAs)\n}=>    if (cta == 0 && threadIdx.x == 0) tl_stamp(x.seq, 3);\n    __syncthreads();\n    if (threadIdx.x == 0) tl_max(x.seq, 14);\n    if (x.do_append) append_body(ap, cta, ncta);\n    if (cta == 0 && threadIdx.x == 0) tl_stamp(x.seq, 4);\n    __syncthreads();\n    if (threadIdx.x == 0) { unsigned long long t; asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t)); atomicMax(&g_tl[(x.seq & 1023) * 16 + 7], t); }\n}",
 # readers
 'extern "C" int32_t lag_abi_version(void) { return LAG_ABI_VERSION; }=>extern "C" int32_t lag_abi_version(void) { return LAG_ABI_VERSION; }\nextern "C" __attribute__((visibility("default"))) int lag_tl_read_api(unsigned long long* h) { return (int)cudaMemcpyFromSymbol(h, lag::g_tl, sizeof(lag::g_tl)); }\n__global__ void tl_empty_kernel(int i) { if (threadIdx.x == 0 && blockIdx.x == 0) lag::tl_stamp(600 + i, 5); __syncthreads(); if (threadIdx.x == 0) lag::tl_max(600 + i, 10); }\nextern "C" __attribute__((visibility("default"))) int lag_tl_empty(int n, int blocks, void* stream) { for (int i = 0; i < n; ++i) tl_empty_kernel<<<blocks, 128, 0, (cudaStream_t)stream>>>(i); return (int)cudaGetLastError(); }',
 "unsigned long long& lag_peer_seq(PeerState* ps) { return ps->seq; }=>unsigned long long& lag_peer_seq(PeerState* ps) { return ps->seq; }\nextern \"C\" __attribute__((visibility(\"default\"))) int lag_tl_read_peer(unsigned long long* h) { return (int)cudaMemcpyFromSymbol(h, lag::g_tl, sizeof(lag::g_tl)); }",
]
sys.exit(subprocess.call([sys.executable, "scripts/build_variant.py", OUT] + subs + EXTRA))
