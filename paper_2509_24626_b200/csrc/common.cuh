// common.cuh -- small device helpers shared by the sm_100a kernels of
// libsparseserve.so.  No method arithmetic lives here.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>

#include <mutex>

#include "sparseserve.h"

namespace ss {

constexpr int kBlockTokens = 32;
constexpr int kHeadDim = 128;

// Multiprocessor count of the current device (148 on B200), queried once per
// device: grids of the persistent kernels are sized to it.
inline int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

// Development A/B knobs (environment variables such as SS_SEL_CHUNK) exist only
// in the debug build (-DSS_DEBUG_KNOBS, libsparseserve_debug.so, used by
// tools/ and a few subprocess tests).  The shipped library ignores the
// environment: every call does exactly what include/sparseserve.h states.
inline int knob(const char* name, int dflt) {
#ifdef SS_DEBUG_KNOBS
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

// 16-byte streaming load, no L1 allocation (read-once data).
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 16-byte store as a volatile asm: keeps program order with the volatile loads
// above, so a batch of loads is fully in flight before its stores are issued.
__device__ __forceinline__ void stg_v4(void* p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

// TMA bulk prefetch of [p, p+bytes) into L2 (no shared memory, no completion
// tracking): lets a warp run a whole tile / block ahead of its register or
// shared-memory pipeline.  bytes must be a multiple of 16.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---- mbarrier / TMA bulk copy / ldmatrix / mma.sync wrappers (PTX, one
// instruction each) shared by the attention and select kernels ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr)
                 : "memory");
}
// D[16x8] += A[16x16] B[16x8], bf16 in, f32 accumulate
__device__ __forceinline__ void hmma(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// Force-load a kernel under CUDA lazy module loading (cudaFuncGetAttributes
// loads the function).  A kernel first launched while a persistent kernel
// spins on work it produces can otherwise stall behind the load.
template <typename K>
inline bool preload_fn(K* k) {
    cudaFuncAttributes a;
    return cudaFuncGetAttributes(&a, (const void*)k) == cudaSuccess;
}

// One shared-memory / L1 carve-out for every kernel of a decode step (percent
// of the unified on-SM memory given to shared memory; < 0 leaves the driver's
// choice).  Kernels of different request groups co-run and alternate on each
// SM; a kernel whose preferred split differs from the SM's current one makes
// the SM reconfigure (drain) before its CTAs can land.
constexpr int kCarveoutDefault = -1;
template <typename K>
inline void set_carveout(K* k) {
    const int v = knob("SS_CARVEOUT", kCarveoutDefault);
    if (v >= 0) cudaFuncSetAttribute((const void*)k, cudaFuncAttributePreferredSharedMemoryCarveout, v);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Inclusive warp scan (int).
__device__ __forceinline__ int warp_incl_scan(int v) {
    int lane = lane_id();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Block-wide exclusive scan for NT threads (NT multiple of 32, <= 1024).
// `sw` must hold >= 33 ints of shared memory.  Returns exclusive prefix and
// writes the block total to `total`.  Contains __syncthreads().
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* sw, int& total) {
    constexpr int NWARP = NT / 32;
    int lane = lane_id(), w = warp_id();
    int incl = warp_incl_scan(v);
    if (lane == 31) sw[w] = incl;
    __syncthreads();
    if (w == 0) {
        int x = lane < NWARP ? sw[lane] : 0;
        int xi = warp_incl_scan(x);
        if (lane < NWARP) sw[lane] = xi - x;
        if (lane == NWARP - 1) sw[32] = xi;
    }
    __syncthreads();
    int res = sw[w] + incl - v;
    total = sw[32];
    __syncthreads();
    return res;
}

template <int NT>
__device__ __forceinline__ int block_sum(int v, int* sw) {
    int total;
    (void)block_excl_scan<NT>(v, sw, total);
    return total;
}

}  // namespace ss

#define SS_LAUNCH_CHECK()                                  \
    do {                                                   \
        if (cudaPeekAtLastError() != cudaSuccess) return SS_ERR_CUDA; \
    } while (0)
