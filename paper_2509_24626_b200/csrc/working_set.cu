// working_set.cu -- NEXT-2: decoding working-set estimation and working-set-aware
// admission (§3.3: "SparseServe tracks the KV blocks selected
// over the past w decoding steps (with w = 12 by default) and regards their
// union as the decoding working set"; Algorithm 1).
//
// ws_track keeps, per (request slot, KV head) of one layer, the step at which
// every block was last selected (last_sel) and a ring of the last w selections.
// At step t the union of the last w selections changes only by
//   - blocks selected at step t-w and not since (last_sel == t-w): leave
//   - blocks selected now that were outside the window (last_sel <= t-w): enter
// so the per-request block count ws_count[b] is maintained incrementally with
// 2k reads per (b, h) instead of re-unioning w sets.  One CTA per (b, h).
//
// ss_admit is Algorithm 1 lines 6-14 (host code, the scheduler's loop).
#include "common.cuh"

namespace ss {

constexpr int kWsThreads = 128;

__global__ void __launch_bounds__(kWsThreads)
ws_track_kernel(const int32_t* __restrict__ sel, int k, int Hkv, int max_blk, int64_t t, int w,
                int32_t* __restrict__ last_sel, int32_t* __restrict__ ring,
                int32_t* __restrict__ ws_count) {
    __shared__ int s_delta;
    const int pair = blockIdx.x;
    const int b = pair / Hkv;
    const int B = gridDim.x / Hkv;
    int32_t* ls = last_sel + (int64_t)pair * max_blk;
    int32_t* rg = ring + ((int64_t)(t % w) * B * Hkv + pair) * k;  // slot of step t-w (and t)
    const int32_t* sp = sel + (int64_t)pair * k;
    if (threadIdx.x == 0) s_delta = 0;
    __syncthreads();
    int delta = 0;
    // 1. leave: selected at step t-w and not selected since
    for (int r = threadIdx.x; r < k; r += kWsThreads) {
        const int32_t j = rg[r];
        if (j >= 0 && (int64_t)ls[j] == t - w) --delta;
    }
    __syncthreads();
    // 2. enter: selected now, outside the window until now; 3. stamp + ring
    for (int r = threadIdx.x; r < k; r += kWsThreads) {
        const int32_t j = sp[r];
        if (j >= 0) {
            if ((int64_t)ls[j] <= t - w) ++delta;
            ls[j] = (int32_t)t;
        }
        rg[r] = j;
    }
    if (delta) atomicAdd(&s_delta, delta);
    __syncthreads();
    if (threadIdx.x == 0 && s_delta) atomicAdd(&ws_count[b], s_delta);
}

ss_status launch_ws_track(const int32_t* sel, int k, const ss_dims& d, int max_blk, int64_t t,
                          int w, int32_t* last_sel, int32_t* ring, int32_t* ws_count,
                          cudaStream_t stream) {
    ws_track_kernel<<<d.batch * d.num_kv_heads, kWsThreads, 0, stream>>>(
        sel, k, d.num_kv_heads, max_blk, t, w, last_sel, ring, ws_count);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_ws() { return preload_fn(ws_track_kernel); }

}  // namespace ss
