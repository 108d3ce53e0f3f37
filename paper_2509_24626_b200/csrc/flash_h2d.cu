// flash_h2d.cu -- S4 FlashH2D GPU-direct loading (§3.2.1:
// "SparseServe launches a single GPU kernel that loads all selected KV blocks
// from DRAM in parallel ... by leveraging unified virtual addressing (UVA)").
//
// B200 design (differs from the paper's "one thread block per KV block", which
// needs the miss count on the host): a persistent grid reads the miss count
// from device memory (written by kv_cache_lookup_insert), so there is no host
// round trip.  One warp copies one block at a time; each lane keeps 8
// independent 16-byte zero-copy loads from host-mapped memory in flight
// (ld.global.nc.v4 over PCIe), then stores them to the HBM cache slot.  With
// up to 2 x 148 CTAs of 16 warps this keeps up to ~19 MB of reads in flight, far
// above the bandwidth-delay product of a PCIe Gen5 x16 link (~64 GB/s x ~2 us).
//
// Roofline: host-link bound; algorithmic bytes = block_bytes per miss over
// PCIe (+ the same bytes written to HBM).
#include "common.cuh"

namespace ss {

constexpr int kH2DThreads = 512;
constexpr int kH2DUnroll = 8;

__global__ void __launch_bounds__(kH2DThreads)
flash_h2d_kernel(const uint4* __restrict__ host, int64_t host_blocks,
                 const int64_t* __restrict__ miss_keys, const int32_t* __restrict__ miss_slots,
                 const int32_t* __restrict__ counts, int max_misses, uint4* __restrict__ pool,
                 int64_t vpb) {
    if (counts[3] != 0) return;
    const int n = min(counts[1], max_misses);
    const int lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * kH2DThreads + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * kH2DThreads) >> 5;
    for (int64_t i = gw; i < n; i += nw) {
        const int64_t phys = miss_keys[i] % host_blocks;
        const uint4* src = host + phys * vpb;
        uint4* dst = pool + (int64_t)miss_slots[i] * vpb;
        int64_t v = lane;
        for (; v + 32 * (kH2DUnroll - 1) < vpb; v += 32 * kH2DUnroll) {
            uint4 r[kH2DUnroll];
#pragma unroll
            for (int u = 0; u < kH2DUnroll; ++u) r[u] = ldg_stream(src + v + 32 * u);
#pragma unroll
            for (int u = 0; u < kH2DUnroll; ++u) dst[v + 32 * u] = r[u];
        }
        for (; v < vpb; v += 32) dst[v] = ldg_stream(src + v);
    }
}

ss_status launch_flash_h2d(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
                           const int32_t* miss_slots, const int32_t* counts, int max_misses,
                           void* pool_kv, int64_t block_bytes, cudaStream_t stream) {
    if (max_misses <= 0) return SS_OK;
    int64_t warps_needed = max_misses;
    int64_t grid = (warps_needed * 32 + kH2DThreads - 1) / kH2DThreads;
    if (grid > 2 * kNumSMs) grid = 2 * kNumSMs;
    flash_h2d_kernel<<<(int)grid, kH2DThreads, 0, stream>>>(
        (const uint4*)host_kv, host_blocks, miss_keys, miss_slots, counts, max_misses,
        (uint4*)pool_kv, block_bytes / 16);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

}  // namespace ss
