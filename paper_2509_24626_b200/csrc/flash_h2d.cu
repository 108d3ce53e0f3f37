// flash_h2d.cu -- S4 FlashH2D GPU-direct loading (§3.2.1:
// "SparseServe launches a single GPU kernel that loads all selected KV blocks
// from DRAM in parallel ... by leveraging unified virtual addressing (UVA)").
//
// B200 design (differs from the paper's "one thread block per KV block", which
// needs the miss count on the host): a persistent grid reads the miss count
// from device memory (written by kv_cache_lookup_insert), so there is no host
// round trip.  One warp copies one block at a time; each lane keeps 16
// independent 16-byte zero-copy loads from host-mapped memory in flight
// (ld.global.nc.v4 over PCIe), then stores them to the HBM cache slot.  16 CTAs
// of 4 warps keep 512 KB of reads in flight -- above the bandwidth-delay
// product of a PCIe Gen5 x16 link (~55 GB/s x ~3-8 us under load) -- on only
// 16 of the 148 SMs.
//
// Roofline: host-link bound; algorithmic bytes = block_bytes per miss over
// PCIe (+ the same bytes written to HBM).
#include <stdlib.h>

#include "common.cuh"

namespace ss {

// Small per-SM footprint (4 warps, ~8K registers, no shared memory) so the
// gather can co-reside with the HBM-bound select / attention kernels of the
// other half-batch running on another stream; 148 x 4 warps x 4 KiB of loads
// in flight (2.4 MB) is still far above the PCIe bandwidth-delay product.
constexpr int kH2DThreadsMax = 512;
constexpr int kH2DCtas = 16;

template <int kH2DUnroll>
__global__ void __launch_bounds__(kH2DThreadsMax)
flash_h2d_kernel(const uint4* __restrict__ host, int64_t host_blocks,
                 const int64_t* __restrict__ miss_keys, const int32_t* __restrict__ miss_slots,
                 const int32_t* __restrict__ counts, int max_misses, uint4* __restrict__ pool,
                 int64_t vpb, uint32_t zero) {
    if (counts[3] != 0) return;
    const int n = min(counts[1], max_misses);
    const int lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // work unit = one batch of 32 x kH2DUnroll 16-byte loads (8 KiB with the
    // default 16) of one block; units are dealt round-robin to the warps, so the
    // warps of a call finish within one batch latency of each other (a whole-
    // block unit leaves a two-batch tail)
    constexpr int64_t kBatch = 32 * kH2DUnroll;
    const int64_t upb = (vpb + kBatch - 1) / kBatch;  // units per block
    const int64_t nu = (int64_t)n * upb;
    for (int64_t u = gw; u < nu; u += nw) {
        const int64_t i = u / upb, part = u - i * upb;
        const int64_t phys = miss_keys[i] % host_blocks;
        const uint4* src = host + phys * vpb;
        uint4* dst = pool + (int64_t)miss_slots[i] * vpb;
        const int64_t v0 = part * kBatch + lane;
        if (v0 + 32 * (kH2DUnroll - 1) < vpb) {
            uint4 r[kH2DUnroll];
#pragma unroll
            for (int k = 0; k < kH2DUnroll; ++k) r[k] = ldg_stream(src + v0 + 32 * k);
            // `zero` is 0 at run time but opaque to the compiler: every store
            // depends on ALL loads of the batch, so ptxas cannot interleave
            // stores with loads and all kH2DUnroll loads are in flight together
            uint32_t fold = 0;
#pragma unroll
            for (int k = 0; k < kH2DUnroll; ++k) fold ^= r[k].w;
            const uint32_t dep = fold & zero;
#pragma unroll
            for (int k = 0; k < kH2DUnroll; ++k) {
                uint4 x = r[k];
                x.x ^= dep;
                stg_v4(dst + v0 + 32 * k, x);
            }
        } else {
            for (int64_t v = v0; v < min(vpb, (part + 1) * kBatch); v += 32) stg_v4(dst + v, ldg_stream(src + v));
        }
    }
}

ss_status launch_flash_h2d(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
                           const int32_t* miss_slots, const int32_t* counts, int max_misses,
                           void* pool_kv, int64_t block_bytes, cudaStream_t stream) {
    if (max_misses <= 0) return SS_OK;
    // experiment knob: SS_H2D_SKIP=1 launches nothing (the step without PCIe time)
    static const bool skip = getenv("SS_H2D_SKIP") && atoi(getenv("SS_H2D_SKIP")) != 0;
    if (skip) return SS_OK;
    int64_t warps_needed = (int64_t)max_misses * 2;  // ~2 units per block (bf16)
    static const int threads = getenv("SS_H2D_THREADS") ? atoi(getenv("SS_H2D_THREADS")) : 128;
    int64_t grid = (warps_needed * 32 + threads - 1) / threads;
    // Few CTAs on purpose: zero-copy PCIe loads in flight on an SM slow down
    // the HBM-bound kernels co-running on that SM (measured: a select kernel
    // sharing the GPU with a 148-CTA gather ran 3.7x slower, with a 16-CTA one
    // 1.2x slower), while 16 CTAs x 4 warps x 32 lanes x 16 x 16 B = 512 KB in
    // flight cover the link's bandwidth-delay product.
    static const int max_ctas = getenv("SS_H2D_CTAS") ? atoi(getenv("SS_H2D_CTAS")) : kH2DCtas;
    if (grid > max_ctas) grid = max_ctas;
    // loads in flight per lane: 16 (default) keeps 512 KB in flight on 16 SMs
    static const int unroll = getenv("SS_H2D_UNROLL") ? atoi(getenv("SS_H2D_UNROLL")) : 16;
    auto kern = unroll >= 16 ? flash_h2d_kernel<16> : flash_h2d_kernel<8>;
    kern<<<(int)grid, threads, 0, stream>>>(
        (const uint4*)host_kv, host_blocks, miss_keys, miss_slots, counts, max_misses,
        (uint4*)pool_kv, block_bytes / 16, 0u);
    SS_LAUNCH_CHECK();
    return SS_OK;
}


// ---------------------------------------------------------------------------
// FlashH2D server (flash_h2d_serve): ONE persistent launch serves the ordered
// sequence of gathers ("jobs") of a whole decode step -- one job per (layer,
// request group) -- so the PCIe link does not drain and refill at every layer
// boundary.  Job j's inputs are valid once ready[j] != 0 (ss_flag_signal
// after its kv_cache_lookup_insert); its work units are handed out by an
// atomic cursor, and a warp always takes a unit of the lowest-numbered ready
// job with units left, so warps done with job j start the next job's loads
// while others still finish job j, and a late job never blocks ready ones.  The warp that completes
// job j's last unit publishes done[j] = 1 (release), which ss_flag_wait turns
// into a stream dependency for that job's attention.
//
// flags (device int32, zeroed by the caller before each launch):
//   [0, nj) ready   [nj, 2nj) done   [2nj, 3nj) unit cursor
//   [3nj, 4nj) finished units        [4nj] abort
// A job that is not ready within the timeout aborts the server: every job not
// yet done gets counts[3] = SS_ERR_CUDA (downstream attention becomes a no-op,
// the error is visible in the counts) and done = 1, so nothing waits forever.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t gtimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int ld_acquire_gpu(const int32_t* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int32_t* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int kU>
__global__ void __launch_bounds__(kH2DThreadsMax)
flash_h2d_server_kernel(const uint4* __restrict__ host, int64_t host_blocks,
                        const ss_h2d_job* __restrict__ jobs, int njobs, int64_t vpb,
                        int32_t* flags, uint32_t zero, uint64_t timeout_ns) {
    int32_t* ready = flags;
    int32_t* done = flags + njobs;
    int32_t* cursor = flags + 2 * njobs;
    int32_t* fin = flags + 3 * njobs;
    int32_t* abort_flag = flags + 4 * njobs;
    const int lane = lane_id();
    constexpr int64_t kBatch = 32 * kU;
    const int upb = (int)((vpb + kBatch - 1) / kBatch);  // units per block
    // Out-of-order service: lane 0 of a warp takes a unit of the LOWEST-numbered
    // ready job that still has units left (jobs below `lo` are fully handed
    // out), so a job whose producer is late never holds up later ready jobs --
    // nor, through their consumers, the hardware queues the late producer may be
    // waiting in.
    int lo = 0;
    bool aborted = false;
    uint64_t t_idle = gtimer_ns();
    const uint4* hsrc = host;
    while (true) {
        int pj = -1, pu = 0, pnu = 0;
        if (lane == 0) {
            for (int jj = lo; jj < njobs; ++jj) {
                if (ld_acquire_gpu(ready + jj) == 0) continue;
                const int32_t* cnt = jobs[jj].counts;
                const int err = __ldcg(cnt + 3);
                const int n = err ? 0 : min(__ldcg(cnt + 1), jobs[jj].max_misses);
                const int nu = n * upb;
                const int peek = *(volatile int32_t*)(cursor + jj);
                if (nu == 0) {  // nothing to load: the first warp here publishes done
                    if (peek == 0 && atomicAdd(cursor + jj, 1) == 0) st_release_gpu(done + jj, 1);
                    if (jj == lo) ++lo;
                    continue;
                }
                if (peek >= nu) {
                    if (jj == lo) ++lo;
                    continue;
                }
                const int u = atomicAdd(cursor + jj, 1);
                if (u >= nu) {
                    if (jj == lo) ++lo;
                    continue;
                }
                pj = jj;
                pu = u;
                pnu = nu;
                break;
            }
        }
        pj = __shfl_sync(0xffffffffu, pj, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        if (pj < 0) {
            if (lo >= njobs) break;  // every job handed out
            int stop = 0;
            if (lane == 0) {
                if (*(volatile int32_t*)abort_flag) {
                    stop = 1;
                } else if (gtimer_ns() - t_idle > timeout_ns) {
                    atomicExch(abort_flag, 1);
                    stop = 1;
                } else {
                    __nanosleep(64);
                }
            }
            if (__shfl_sync(0xffffffffu, stop, 0)) {
                aborted = true;
                break;
            }
            continue;
        }
        pu = __shfl_sync(0xffffffffu, pu, 0);
        pnu = __shfl_sync(0xffffffffu, pnu, 0);
        if (lane == 0) t_idle = gtimer_ns();
        const ss_h2d_job jb = jobs[pj];
        uint4* pool = (uint4*)jb.pool_kv;
        {
            const int i = pu / upb, part = pu - i * upb;
            const int64_t phys = __ldcg(jb.miss_keys + i) % host_blocks;
            const uint4* src = hsrc + phys * vpb;
            uint4* dst = pool + (int64_t)__ldcg(jb.miss_slots + i) * vpb;
            const int64_t v0 = (int64_t)part * kBatch + lane;
            if (v0 + 32 * (kU - 1) < vpb) {
                uint4 r[kU];
#pragma unroll
                for (int k = 0; k < kU; ++k) r[k] = ldg_stream(src + v0 + 32 * k);
                uint32_t fold = 0;
#pragma unroll
                for (int k = 0; k < kU; ++k) fold ^= r[k].w;
                const uint32_t dep = fold & zero;
#pragma unroll
                for (int k = 0; k < kU; ++k) {
                    uint4 x = r[k];
                    x.x ^= dep;
                    stg_v4(dst + v0 + 32 * k, x);
                }
            } else {
                for (int64_t v = v0; v < min(vpb, (int64_t)(part + 1) * kBatch); v += 32)
                    stg_v4(dst + v, ldg_stream(src + v));
            }
        }
        __threadfence();  // this lane's pool stores are visible GPU-wide ...
        __syncwarp();
        if (lane == 0) {  // ... before the unit is counted
            const int f = atomicAdd(fin + pj, 1);
            if (f == pnu - 1) {
                __threadfence();
                st_release_gpu(done + pj, 1);
            }
        }
    }
    if (aborted && lane == 0) {
        for (int jj = 0; jj < njobs; ++jj) {
            if (ld_acquire_gpu(done + jj) == 0) {
                atomicExch(jobs[jj].counts + 3, (int)SS_ERR_CUDA);
                __threadfence();
                st_release_gpu(done + jj, 1);
            }
        }
    }
}

__global__ void flag_wait_kernel(const int32_t* flag, uint64_t timeout_ns) {
    const uint64_t t0 = gtimer_ns();
    while (ld_acquire_gpu(flag) == 0) {
        if (gtimer_ns() - t0 > timeout_ns) break;
        __nanosleep(128);
    }
}

static uint64_t serve_timeout_ns() {
    static const uint64_t t = getenv("SS_SERVE_TIMEOUT_MS") ? (uint64_t)atoll(getenv("SS_SERVE_TIMEOUT_MS")) * 1000000ull
                                                            : 3000000000ull;  // 3 s
    return t;
}

ss_status launch_flash_h2d_serve(const void* host_kv, int64_t host_blocks, const ss_h2d_job* jobs,
                                 int njobs, int64_t block_bytes, int32_t* flags, cudaStream_t stream) {
    if (njobs <= 0) return SS_OK;
    static const int threads = getenv("SS_H2D_THREADS") ? atoi(getenv("SS_H2D_THREADS")) : 128;
    static const int ctas = getenv("SS_H2D_CTAS") ? atoi(getenv("SS_H2D_CTAS")) : kH2DCtas;
    flash_h2d_server_kernel<16><<<ctas, threads, 0, stream>>>(
        (const uint4*)host_kv, host_blocks, jobs, njobs, block_bytes / 16, flags, 0u, serve_timeout_ns());
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_flag_wait(const int32_t* flag, cudaStream_t stream) {
    flag_wait_kernel<<<1, 32, 0, stream>>>(flag, serve_timeout_ns());
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_h2d() {
    return preload_fn(flash_h2d_kernel<16>) && preload_fn(flash_h2d_kernel<8>) &&
           preload_fn(flash_h2d_server_kernel<16>) && preload_fn(flag_wait_kernel);
}

}  // namespace ss
