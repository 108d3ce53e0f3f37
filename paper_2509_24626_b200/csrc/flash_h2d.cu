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

}  // namespace ss
