// meta_update.cu -- S0 block_meta_update ("Once a KV block
// reaches its capacity, its associated metadata is created"; per-channel
// bounding cuboid, reading R1).
//
// One CTA of 128 threads per block, thread c owns channel c and walks the 32
// tokens (each token row is read by the CTA as one coalesced 256 B / 512 B
// row).  Min/max use the total order of the bit patterns (-0 < +0), so the
// result is one of the input elements, bit-exact.  The result is scattered into
// the tiled metadata layout of include/sparseserve.h.
//
// Roofline: reads 32*d*es bytes, writes 2*d*es bytes per block (8.5 KiB bf16);
// amortised over 32 decode steps (one block fills every 32 tokens), so it is
// off the per-step critical path.
#include "common.cuh"

namespace ss {

// Order-preserving signed integer of a float bit pattern (-0 < +0).
__device__ __forceinline__ int32_t ord_bits16(uint16_t u) {
    int32_t s = (int32_t)(int16_t)u;
    return s < 0 ? (s ^ 0x7FFF) : s;
}
__device__ __forceinline__ int64_t ord_bits32(uint32_t u) {
    int64_t s = (int64_t)(int32_t)u;
    return s < 0 ? (s ^ 0x7FFFFFFFLL) : s;
}

template <typename E>
__global__ void __launch_bounds__(128) meta_update_kernel(const E* __restrict__ keys,
                                                          int64_t key_stride,
                                                          const int64_t* __restrict__ dst_idx,
                                                          int64_t n, E* __restrict__ meta) {
    constexpr int CPC = 16 / sizeof(E);
    const int c = threadIdx.x;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const E* kb = keys + i * key_stride;
        E vmin = kb[c], vmax = vmin;
        if constexpr (sizeof(E) == 2) {
            int32_t omin = ord_bits16(vmin), omax = omin;
#pragma unroll 8
            for (int t = 1; t < kBlockTokens; ++t) {
                E v = kb[t * kHeadDim + c];
                int32_t o = ord_bits16(v);
                if (o < omin) { omin = o; vmin = v; }
                if (o > omax) { omax = o; vmax = v; }
            }
        } else {
            int64_t omin = ord_bits32(vmin), omax = omin;
#pragma unroll 8
            for (int t = 1; t < kBlockTokens; ++t) {
                E v = kb[t * kHeadDim + c];
                int64_t o = ord_bits32(v);
                if (o < omin) { omin = o; vmin = v; }
                if (o > omax) { omax = o; vmax = v; }
            }
        }
        int64_t idx = dst_idx ? dst_idx[i] : i;
        if (idx < 0) continue;  // no destination row (kv_seal_blocks on a full block table)
        int64_t tile = idx >> 5;
        int r = (int)(idx & 31);
        E* mt = meta + tile * (int64_t)(64 * kHeadDim);
        int chunk = c / CPC, e = c % CPC;
        mt[((chunk * 2 + 0) * 32 + r) * CPC + e] = vmin;
        mt[((chunk * 2 + 1) * 32 + r) * CPC + e] = vmax;
    }
}

// NEXT-3 mean-of-keys metadata ("simply calculating the mean values
// of the token keys [45]"; reading R18): thread c sums channel c of the 32 keys
// in float64, t = 0..31 in order from +0.0 (bit-identical to the oracle's
// sequential sum), divides by 32 (exact) and rounds once to float32.  Tiled
// float32 layout (include/sparseserve.h): tile T = idx / 32 holds 32 blocks x
// d channels as [d/4 chunks][32 blocks][4 channels] (16 KiB), so lane r of a
// select warp reads block r's 16-byte chunks as contiguous 512-byte segments.
template <typename E>
__global__ void __launch_bounds__(128) meta_mean_kernel(const E* __restrict__ keys,
                                                        int64_t key_stride,
                                                        const int64_t* __restrict__ dst_idx,
                                                        int64_t n, float* __restrict__ meta) {
    const int c = threadIdx.x;
    for (int64_t i = blockIdx.x; i < n; i += gridDim.x) {
        const E* kb = keys + i * key_stride;
        double acc = 0.0;
#pragma unroll 8
        for (int t = 0; t < kBlockTokens; ++t) {
            const E v = kb[t * kHeadDim + c];
            const float f = sizeof(E) == 2 ? __uint_as_float((uint32_t)v << 16) : __uint_as_float((uint32_t)v);
            acc = __dadd_rn(acc, (double)f);
        }
        const float mu = __double2float_rn(acc * (1.0 / 32.0));
        const int64_t idx = dst_idx ? dst_idx[i] : i;
        if (idx < 0) continue;  // no destination row
        float* mt = meta + (idx >> 5) * (int64_t)(32 * kHeadDim);
        mt[((c >> 2) * 32 + (int)(idx & 31)) * 4 + (c & 3)] = mu;
    }
}

ss_status launch_meta_mean(const void* keys, int64_t key_stride, const int64_t* dst_idx, int64_t n,
                           float* meta, ss_dtype dt, cudaStream_t stream) {
    if (n == 0) return SS_OK;
    int grid = (int)(n < 65535 * 4 ? n : 65535 * 4);
    if (dt == SS_BF16)
        meta_mean_kernel<uint16_t><<<grid, 128, 0, stream>>>((const uint16_t*)keys, key_stride,
                                                               dst_idx, n, meta);
    else
        meta_mean_kernel<uint32_t><<<grid, 128, 0, stream>>>((const uint32_t*)keys, key_stride,
                                                               dst_idx, n, meta);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_meta_update(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                             int64_t n, void* meta, ss_dtype dt, cudaStream_t stream) {
    if (n == 0) return SS_OK;
    int grid = (int)(n < 65535 * 4 ? n : 65535 * 4);
    if (dt == SS_BF16)
        meta_update_kernel<uint16_t><<<grid, 128, 0, stream>>>(
            (const uint16_t*)keys, key_stride, dst_idx, n, (uint16_t*)meta);
    else
        meta_update_kernel<uint32_t><<<grid, 128, 0, stream>>>(
            (const uint32_t*)keys, key_stride, dst_idx, n, (uint32_t*)meta);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_meta() {
    return preload_fn(meta_update_kernel<uint16_t>) && preload_fn(meta_update_kernel<uint32_t>) &&
           preload_fn(meta_mean_kernel<uint16_t>) && preload_fn(meta_mean_kernel<uint32_t>);
}

}  // namespace ss
