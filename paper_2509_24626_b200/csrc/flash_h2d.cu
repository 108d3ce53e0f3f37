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
constexpr int kServerSmemKB = 0;  // shared memory reserved per server CTA (dedicated SMs; 0: none)

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
    int64_t warps_needed = (int64_t)max_misses * 2;  // ~2 units per block (bf16)
    const int threads = knob("SS_H2D_THREADS", 128);
    int64_t grid = (warps_needed * 32 + threads - 1) / threads;
    // Few CTAs on purpose: zero-copy PCIe loads in flight on an SM slow down
    // the HBM-bound kernels co-running on that SM (measured: a select kernel
    // sharing the GPU with a 148-CTA gather ran 3.7x slower, with a 16-CTA one
    // 1.2x slower), while 16 CTAs x 4 warps x 32 lanes x 16 x 16 B = 512 KB in
    // flight cover the link's bandwidth-delay product.
    const int max_ctas = knob("SS_H2D_CTAS", kH2DCtas);
    if (grid > max_ctas) grid = max_ctas;
    // loads in flight per lane: 16 (default) keeps 512 KB in flight on 16 SMs
    auto kern = knob("SS_H2D_UNROLL", 16) >= 16 ? flash_h2d_kernel<16> : flash_h2d_kernel<8>;
    set_carveout(kern);
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
// while others still finish job j, and a late job never blocks ready ones.  The
// warp that completes job j's last unit publishes done[j] = 1 (release), which
// ss_flag_wait turns into a stream dependency for that job's attention.
//
// flags (device int32, zeroed by the caller before each launch):
//   [0, nj) ready   [nj, 2nj) done   [2nj, 3nj) unit cursor
//   [3nj, 4nj) finished units        [4nj] abort
// A server that sees no ready job for `timeout` aborts: every job not yet done
// gets done = 2 (SS_H2D_DONE_ABORTED).  The abort is sticky where it matters:
// the job's ss_flag_wait (stream-ordered after the job's producer, so after
// any counts[3] = 0 that producer writes) sees done == 2 and sets counts[3] =
// SS_ERR_CUDA, which turns the attention that follows into a no-op and makes
// the error visible in the step's counts.  A flag_wait that itself times out
// does the same.
//
// stats (optional, device uint64 [8], zeroed by the caller): [0] sum over the
// server's warps of the ns spent with no unit to serve (polling), [1] warps,
// [2] first unit start (globaltimer ns), [3] last unit end, [4] ns from the
// first unit start to the last unit end during which NO warp was copying
// (link idle, from a per-warp busy count), [5] 1 + the first job found not
// ready at an abort (0: no abort).
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

constexpr int kDoneServed = 1;
constexpr int kDoneAborted = 2;

// Link-idle accounting: `busy` counts the warps copying right now; the warp
// that takes it 1 -> 0 stamps the idle start, the warp that takes it 0 -> 1
// adds the elapsed idle time.  (Approximate at the ns level: the stamp and the
// count are two words; good enough for an idle fraction.)
struct ServeStats {
    unsigned long long* s;
    __device__ __forceinline__ void busy_begin(int32_t* busy, uint64_t* idle_t0) {
        if (s == nullptr) return;
        const uint64_t now = gtimer_ns();
        if (atomicAdd(busy, 1) == 0) {
            const uint64_t t0 = atomicExch((unsigned long long*)idle_t0, 0ull);
            if (t0 != 0 && now > t0) atomicAdd(s + 4, now - t0);
            atomicCAS(s + 2, 0ull, (unsigned long long)now);  // first unit start
        }
    }
    __device__ __forceinline__ void busy_end(int32_t* busy, uint64_t* idle_t0) {
        if (s == nullptr) return;
        const uint64_t now = gtimer_ns();
        atomicMax(s + 3, now);
        if (atomicSub(busy, 1) == 1) atomicExch((unsigned long long*)idle_t0, now);
    }
};

template <int kU>
__global__ void __launch_bounds__(kH2DThreadsMax)
flash_h2d_server_kernel(const uint4* __restrict__ host, int64_t host_blocks,
                        const ss_h2d_job* __restrict__ jobs, int njobs, int64_t vpb,
                        int32_t* flags, uint32_t zero, uint64_t timeout_ns,
                        unsigned long long* stats) {
    int32_t* ready = flags;
    int32_t* done = flags + njobs;
    int32_t* cursor = flags + 2 * njobs;
    int32_t* fin = flags + 3 * njobs;
    int32_t* abort_flag = flags + 4 * njobs;
    // link-idle bookkeeping lives in stats[6] (busy warps) and stats[7] (idle start)
    int32_t* busy = stats ? (int32_t*)(stats + 6) : nullptr;
    uint64_t* idle_t0 = stats ? (uint64_t*)(stats + 7) : nullptr;
    ServeStats st{stats};
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
    uint64_t t_idle = gtimer_ns();   // start of the current no-work stretch
    uint64_t idle_sum = 0;
    bool polling = false;
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
                    if (peek == 0 && atomicAdd(cursor + jj, 1) == 0) st_release_gpu(done + jj, kDoneServed);
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
                if (!polling) {
                    polling = true;
                    t_idle = gtimer_ns();
                }
                if (*(volatile int32_t*)abort_flag) {
                    stop = 1;
                } else if (gtimer_ns() - t_idle > timeout_ns) {
                    if (atomicExch(abort_flag, 1) == 0 && stats) {
                        int first = lo;
                        while (first < njobs && ld_acquire_gpu(ready + first) != 0) ++first;
                        stats[5] = (unsigned long long)(first + 1);
                    }
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
        if (lane == 0 && polling) idle_sum += gtimer_ns() - t_idle;
        polling = false;
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
                // (statistics atomics after the loads are issued: their round
                // trip overlaps the PCIe latency instead of delaying it)
                if (lane == 0) st.busy_begin(busy, idle_t0);
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
                if (lane == 0) st.busy_begin(busy, idle_t0);
                for (int64_t v = v0; v < min(vpb, (int64_t)(part + 1) * kBatch); v += 32)
                    stg_v4(dst + v, ldg_stream(src + v));
            }
        }
        __threadfence();  // this lane's pool stores are visible GPU-wide ...
        __syncwarp();
        if (lane == 0) {  // ... before the unit is counted
            st.busy_end(busy, idle_t0);
            const int f = atomicAdd(fin + pj, 1);
            if (f == pnu - 1) {
                __threadfence();
                st_release_gpu(done + pj, kDoneServed);
            }
        }
    }
    if (lane == 0 && stats) {
        if (polling) idle_sum += gtimer_ns() - t_idle;
        atomicAdd(stats + 0, idle_sum);
        atomicAdd(stats + 1, 1ull);
    }
    if (aborted && lane == 0) {
        for (int jj = 0; jj < njobs; ++jj) {
            if (ld_acquire_gpu(done + jj) == 0) {
                atomicExch(jobs[jj].counts + 3, (int)SS_ERR_CUDA);
                __threadfence();
                st_release_gpu(done + jj, kDoneAborted);
            }
        }
    }
}

// Pipelined server (default): each warp keeps TWO units in flight.  It claims
// and issues the loads of its next unit BEFORE it stores, fences and counts
// the current one, so the PCIe link always has this warp's next 8 KiB of
// reads outstanding while the current unit's HBM stores drain and its
// completion atomics round-trip (inside a decode step those take microseconds:
// HBM is saturated by the other request groups' select / attention).  Same job
// protocol, statistics and abort as flash_h2d_server_kernel.
struct SrvUnit {
    int pj, pu, pnu;  // job, unit, units of the job (pj < 0: none)
};

template <int kU>
__global__ void __launch_bounds__(256)
flash_h2d_server_pipe_kernel(const uint4* __restrict__ host, int64_t host_blocks,
                             const ss_h2d_job* __restrict__ jobs, int njobs, int64_t vpb,
                             int32_t* flags, uint32_t zero, uint64_t timeout_ns,
                             unsigned long long* stats) {
    int32_t* ready = flags;
    int32_t* done = flags + njobs;
    int32_t* cursor = flags + 2 * njobs;
    int32_t* fin = flags + 3 * njobs;
    int32_t* abort_flag = flags + 4 * njobs;
    int32_t* busy = stats ? (int32_t*)(stats + 6) : nullptr;
    uint64_t* idle_t0 = stats ? (uint64_t*)(stats + 7) : nullptr;
    ServeStats st{stats};
    const int lane = lane_id();
    constexpr int64_t kBatch = 32 * kU;
    const int upb = (int)((vpb + kBatch - 1) / kBatch);
    int lo = 0;
    bool aborted = false;
    uint64_t t_idle = gtimer_ns(), idle_sum = 0;
    bool polling = false;

    // one scan for a unit of the lowest ready job with units left (lane 0 scans,
    // the result is broadcast); pj < 0 if none right now
    auto try_claim = [&]() -> SrvUnit {
        int pj = -1, pu = 0, pnu = 0;
        if (lane == 0) {
            for (int jj = lo; jj < njobs; ++jj) {
                if (ld_acquire_gpu(ready + jj) == 0) continue;
                const int32_t* cnt = jobs[jj].counts;
                const int err = __ldcg(cnt + 3);
                const int n = err ? 0 : min(__ldcg(cnt + 1), jobs[jj].max_misses);
                const int nu = n * upb;
                const int peek = *(volatile int32_t*)(cursor + jj);
                if (nu == 0) {
                    if (peek == 0 && atomicAdd(cursor + jj, 1) == 0) st_release_gpu(done + jj, kDoneServed);
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
        SrvUnit r;
        r.pj = __shfl_sync(0xffffffffu, pj, 0);
        r.pu = __shfl_sync(0xffffffffu, pu, 0);
        r.pnu = __shfl_sync(0xffffffffu, pnu, 0);
        lo = __shfl_sync(0xffffffffu, lo, 0);
        return r;
    };
    // source / destination of a unit (lane's first vector)
    auto addr = [&](const SrvUnit& x, const uint4*& src, uint4*& dst, int64_t& v0) {
        const ss_h2d_job& jb = jobs[x.pj];
        const int i = x.pu / upb, part = x.pu - i * upb;
        src = host + (__ldcg(jb.miss_keys + i) % host_blocks) * vpb;
        dst = (uint4*)jb.pool_kv + (int64_t)__ldcg(jb.miss_slots + i) * vpb;
        v0 = (int64_t)part * kBatch + lane;
    };
    auto full_unit = [&](int64_t v0) { return v0 - lane + kBatch <= vpb; };
    // issue a unit's loads into r (full units only)
    auto issue = [&](const SrvUnit& x, uint4 (&r)[kU], const uint4*& src, uint4*& dst, int64_t& v0) {
        addr(x, src, dst, v0);
        if (full_unit(v0)) {
#pragma unroll
            for (int k = 0; k < kU; ++k) r[k] = ldg_stream(src + v0 + 32 * k);
        }
        if (lane == 0) st.busy_begin(busy, idle_t0);
    };
    // store a unit (every store depends on all loads through an opaque zero, so
    // ptxas keeps the loads together), fence, count; the last unit of a job
    // publishes done
    auto retire = [&](const SrvUnit& x, uint4 (&r)[kU], const uint4* src, uint4* dst, int64_t v0) {
        if (full_unit(v0)) {
            uint32_t fold = 0;
#pragma unroll
            for (int k = 0; k < kU; ++k) fold ^= r[k].w;
            const uint32_t dep = fold & zero;
#pragma unroll
            for (int k = 0; k < kU; ++k) {
                uint4 y = r[k];
                y.x ^= dep;
                stg_v4(dst + v0 + 32 * k, y);
            }
        } else {
            const int part = x.pu % upb;
            for (int64_t v = v0; v < min(vpb, (int64_t)(part + 1) * kBatch); v += 32) stg_v4(dst + v, ldg_stream(src + v));
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            st.busy_end(busy, idle_t0);
            const int f = atomicAdd(fin + x.pj, 1);
            if (f == x.pnu - 1) {
                __threadfence();
                st_release_gpu(done + x.pj, kDoneServed);
            }
        }
    };
    // blocking claim: polls until a unit is ready, every job is handed out
    // (pj < 0, done), or the timeout aborts (pj < 0, aborted)
    auto claim_wait = [&]() -> SrvUnit {
        while (true) {
            SrvUnit x = try_claim();
            if (x.pj >= 0) {
                if (lane == 0 && polling) idle_sum += gtimer_ns() - t_idle;
                polling = false;
                return x;
            }
            if (lo >= njobs) return x;
            int stop = 0;
            if (lane == 0) {
                if (!polling) {
                    polling = true;
                    t_idle = gtimer_ns();
                }
                if (*(volatile int32_t*)abort_flag) {
                    stop = 1;
                } else if (gtimer_ns() - t_idle > timeout_ns) {
                    if (atomicExch(abort_flag, 1) == 0 && stats) {
                        int first = lo;
                        while (first < njobs && ld_acquire_gpu(ready + first) != 0) ++first;
                        stats[5] = (unsigned long long)(first + 1);
                    }
                    stop = 1;
                } else {
                    __nanosleep(64);
                }
            }
            if (__shfl_sync(0xffffffffu, stop, 0)) {
                aborted = true;
                return x;
            }
        }
    };

    uint4 rA[kU], rB[kU];
    const uint4 *sA = nullptr, *sB = nullptr;
    uint4 *dA = nullptr, *dB = nullptr;
    int64_t vA = 0, vB = 0;
    SrvUnit cur = claim_wait();
    if (cur.pj >= 0) issue(cur, rA, sA, dA, vA);
    // two steps per iteration so the register buffers alternate statically
    while (cur.pj >= 0) {
        SrvUnit nxt = try_claim();
        if (nxt.pj >= 0) issue(nxt, rB, sB, dB, vB);
        retire(cur, rA, sA, dA, vA);
        if (nxt.pj < 0) {
            nxt = claim_wait();
            if (nxt.pj < 0) break;
            issue(nxt, rB, sB, dB, vB);
        }
        cur = try_claim();
        if (cur.pj >= 0) issue(cur, rA, sA, dA, vA);
        retire(nxt, rB, sB, dB, vB);
        if (cur.pj < 0) {
            cur = claim_wait();
            if (cur.pj < 0) break;
            issue(cur, rA, sA, dA, vA);
        }
    }
    if (lane == 0 && stats) {
        if (polling) idle_sum += gtimer_ns() - t_idle;
        atomicAdd(stats + 0, idle_sum);
        atomicAdd(stats + 1, 1ull);
    }
    if (aborted && lane == 0) {
        for (int jj = 0; jj < njobs; ++jj) {
            if (ld_acquire_gpu(done + jj) == 0) {
                atomicExch(jobs[jj].counts + 3, (int)SS_ERR_CUDA);
                __threadfence();
                st_release_gpu(done + jj, kDoneAborted);
            }
        }
    }
}

// Stream-ordered wait for a done flag.  flag == 2 (the server aborted this
// job) or a wait that times out marks the job failed in its counts word (this
// kernel runs after the job's producer, so the mark cannot be overwritten by
// it): the attention that follows is a no-op and the step reports the error.
__global__ void flag_wait_kernel(const int32_t* flag, int32_t* counts, uint64_t timeout_ns) {
    const uint64_t t0 = gtimer_ns();
    int v;
    while ((v = ld_acquire_gpu(flag)) == 0) {
        if (gtimer_ns() - t0 > timeout_ns) break;
        __nanosleep(128);
    }
    if (v != kDoneServed && counts != nullptr) {
        atomicExch(counts + 3, (int)SS_ERR_CUDA);
        __threadfence();
    }
}

static uint64_t timeout_ns_of(int64_t timeout_us) {
    return timeout_us > 0 ? (uint64_t)timeout_us * 1000ull : 3000000000ull;  // default 3 s
}

ss_status launch_flash_h2d_serve(const void* host_kv, int64_t host_blocks, const ss_h2d_job* jobs,
                                 int njobs, int64_t block_bytes, int32_t* flags, int64_t timeout_us,
                                 unsigned long long* stats, cudaStream_t stream) {
    if (njobs <= 0) return SS_OK;
    const int threads = knob("SS_H2D_THREADS", 128);
    const int ctas = knob("SS_H2D_CTAS", kH2DCtas);
    // pipelined form: measured equal in the C2 step (43.8 vs 44.6 GB/s, link idle
    // 0.8 vs 3 %: the in-step rate is capped elsewhere), so
    // the simpler, 94-register form stays the default
    const bool pipe = knob("SS_H2D_PIPE", 0) != 0;
    const bool u16 = knob("SS_H2D_UNROLL", 16) >= 16;
    auto kern = pipe ? (u16 ? flash_h2d_server_pipe_kernel<16> : flash_h2d_server_pipe_kernel<8>)
                     : (u16 ? flash_h2d_server_kernel<16> : flash_h2d_server_kernel<8>);
    set_carveout(kern);
    // Dedicated SMs: a server CTA that reserves (without using) most of an SM's
    // shared memory keeps the HBM-bound select / attention / cache CTAs off its
    // SM.  Measured (tools/kbench.py overlap): CTAs that share an SM with the
    // server's zero-copy loads run several times slower (their loads queue
    // behind the PCIe-latency ones), and the kernel waits for them.
    const int smem = knob("SS_H2D_SMEM_KB", kServerSmemKB) * 1024;
    if (smem > 0 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SS_ERR_CUDA;
    kern<<<ctas, threads, smem, stream>>>(
        (const uint4*)host_kv, host_blocks, jobs, njobs, block_bytes / 16, flags, 0u,
        timeout_ns_of(timeout_us), stats);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_flag_wait(const int32_t* flag, int32_t* counts, int64_t timeout_us, cudaStream_t stream) {
    set_carveout(flag_wait_kernel);
    flag_wait_kernel<<<1, 32, 0, stream>>>(flag, counts, timeout_ns_of(timeout_us));
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_h2d() {
    return preload_fn(flash_h2d_kernel<16>) && preload_fn(flash_h2d_kernel<8>) &&
           preload_fn(flash_h2d_server_kernel<16>) && preload_fn(flash_h2d_server_kernel<8>) &&
           preload_fn(flash_h2d_server_pipe_kernel<16>) && preload_fn(flash_h2d_server_pipe_kernel<8>) && preload_fn(flag_wait_kernel);
}

}  // namespace ss
