// kv_cache.cu -- S3 kv_cache_lookup_insert: the HBM block cache of the KV cache
// manager ("sends the indices of the KV blocks required for the
// attention computation to the KV cache manager to trigger the KV cache
// loading"; "the remaining HBM is used to cache frequently
// accessed KV blocks and we employ the least recently used (LRU) cache
// eviction policy").  Batch-LRU semantics: readings R11/R12 in DESIGN.md;
// reference: oracle/oracle.c or_lru (must match bit-exactly, including the
// order array, which is always "slots sorted by (stamp, slot)").
//
// Device-only, no host synchronisation.  Data structures (caller-owned):
//   fwd[key] -> slot (dense direct-mapped table: a key is a dense index, so a
//   hash is unnecessary), slot_key[S], slot_stamp[S], order[S].
// Because `order` is kept sorted by (stamp, slot), the LRU victims of a call
// are simply the first M "eligible" entries of `order` (not hit, stamp < t),
// and the new order is [eligible entries not evicted, in old order] ++ [all
// slots with stamp == t, in slot order] -- two stable compactions.
//
// Kernels (stream-ordered, all grid-parallel except the tiny plan kernel):
//   A  lookup     : per selection entry: key, fwd probe, hit marks, per-CTA miss
//                   ranks (canonical order)
//   B1 elig_count : per 1024-entry chunk of `order`: # eligible
//   B2 plan       : 1 CTA: scans of per-CTA miss counts / eligible counts,
//                   capacity check, status + counts
//   B3 victims    : first M eligible -> victim list (evict old keys); the rest
//                   -> new order prefix
//   C  assign     : i-th miss -> i-th victim; fwd/slot_key/stamp; hit stamps
//   D1 teq_count  : per slot chunk: # slots with stamp == t
//   D2 teq_place  : stamp == t slots appended in slot order; new order copied
// On any status != 0 kernels B3..D2 are no-ops: the pool is untouched.
//
// Roofline: integer/latency bound; bytes ~ 12*E (+4 for fwd) + 26*S per call.
#include "common.cuh"

namespace ss {

constexpr int kCacheThreads = 256;
constexpr int kSlotChunk = 1024;  // slots per CTA in B1/B3/D1/D2 (4 per thread)
constexpr int kSlotPer = kSlotChunk / kCacheThreads;

struct CacheWs {
    uint8_t* touched;     // [S]
    int32_t* ctrl;        // [16]: 0 M, 1 hits, 2 status, 3 total_elig, 4 evictions, 5 kept, 6 invalid
    int32_t* miss_local;  // [E]
    int32_t* blk_miss;    // [nA]
    int32_t* blk_hit;     // [nA]
    int32_t* blk_off;     // [nA]
    int32_t* elig_cnt;    // [nS]
    int32_t* elig_off;    // [nS]
    int32_t* teq_cnt;     // [nS]
    int32_t* vict;        // [E]
    int32_t* new_order;   // [S]
};

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t carve(CacheWs* w, void* base, int64_t E, int S) {
    int64_t nA = (E + kCacheThreads - 1) / kCacheThreads;
    int64_t nS = (S + kSlotChunk - 1) / kSlotChunk;
    size_t off = 0;
    char* p = (char*)base;
    auto take = [&](size_t bytes) {
        char* r = p ? p + off : nullptr;
        off += align256(bytes);
        return r;
    };
    CacheWs t;
    t.ctrl = (int32_t*)take(16 * 4);
    t.touched = (uint8_t*)take((size_t)S);
    t.miss_local = (int32_t*)take((size_t)E * 4);
    t.blk_miss = (int32_t*)take((size_t)nA * 4);
    t.blk_hit = (int32_t*)take((size_t)nA * 4);
    t.blk_off = (int32_t*)take((size_t)nA * 4);
    t.elig_cnt = (int32_t*)take((size_t)nS * 4);
    t.elig_off = (int32_t*)take((size_t)nS * 4);
    t.teq_cnt = (int32_t*)take((size_t)nS * 4);
    t.vict = (int32_t*)take((size_t)E * 4);
    t.new_order = (int32_t*)take((size_t)S * 4);
    if (w) *w = t;
    return off;
}

size_t cache_ws_bytes(const ss_dims& d, int k, int S) {
    int64_t E = (int64_t)d.batch * d.num_kv_heads * k;
    return carve(nullptr, nullptr, E, S);
}

struct CacheArgs {
    ss_cache_pool pool;
    const int32_t* sel;
    const int32_t* req_ids;
    int32_t layer, num_layers, max_blk, k, Hkv;
    int64_t E;
    int64_t stamp;
    int32_t* slot_out;
    uint8_t* hit_out;
    int64_t* miss_keys;
    int32_t* miss_slots;
    int32_t* counts;
    CacheWs ws;
};

__device__ __forceinline__ int64_t cache_key(const CacheArgs& a, int64_t e, int32_t j) {
    int64_t b = e / ((int64_t)a.Hkv * a.k);
    int64_t h = (e / a.k) % a.Hkv;
    return (((int64_t)a.req_ids[b] * a.num_layers + a.layer) * a.Hkv + h) * a.max_blk + j;
}

// A: lookup
__global__ void __launch_bounds__(kCacheThreads) cache_lookup_kernel(CacheArgs a) {
    __shared__ int sw[64];
    const int64_t e = (int64_t)blockIdx.x * kCacheThreads + threadIdx.x;
    int is_miss = 0, is_hit = 0;
    if (e < a.E) {
        int32_t j = a.sel[e];
        int32_t so = -1;
        uint8_t ho = 0;
        if (j >= 0) {
            int64_t key = cache_key(a, e, j);
            if (key < 0 || key >= a.pool.fwd_len) {
                a.ws.ctrl[6] = 1;
            } else {
                int32_t f = a.pool.fwd[key];
                if (f >= 0) {
                    so = f;
                    ho = 1;
                    is_hit = 1;
                    a.ws.touched[f] = 1;
                } else {
                    is_miss = 1;
                }
            }
        }
        a.slot_out[e] = so;
        a.hit_out[e] = ho;
    }
    int tot;
    int rank = block_excl_scan<kCacheThreads>(is_miss, sw, tot);
    if (e < a.E) a.ws.miss_local[e] = is_miss ? rank : -1;
    int hits = block_sum<kCacheThreads>(is_hit, sw);
    if (threadIdx.x == 0) {
        a.ws.blk_miss[blockIdx.x] = tot;
        a.ws.blk_hit[blockIdx.x] = hits;
    }
}

__device__ __forceinline__ bool eligible(const CacheArgs& a, int32_t s) {
    return !a.ws.touched[s] && a.pool.slot_stamp[s] < a.stamp;
}

// B1: eligible count per chunk of `order`
__global__ void __launch_bounds__(kCacheThreads) cache_elig_count_kernel(CacheArgs a) {
    __shared__ int sw[64];
    const int S = a.pool.num_slots;
    const int p0 = blockIdx.x * kSlotChunk + threadIdx.x * kSlotPer;
    int c = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        int p = p0 + i;
        if (p < S) c += eligible(a, a.pool.order[p]);
    }
    int tot = block_sum<kCacheThreads>(c, sw);
    if (threadIdx.x == 0) a.ws.elig_cnt[blockIdx.x] = tot;
}

// B2: plan (single CTA of 1024 threads)
__global__ void __launch_bounds__(1024) cache_plan_kernel(CacheArgs a, int nA, int nS) {
    __shared__ int sw[64];
    int run = 0, hits = 0;
    for (int base = 0; base < nA; base += 1024) {
        int i = base + threadIdx.x;
        int v = i < nA ? a.ws.blk_miss[i] : 0;
        int tot;
        int ex = block_excl_scan<1024>(v, sw, tot);
        if (i < nA) a.ws.blk_off[i] = run + ex;
        run += tot;
        int hv = i < nA ? a.ws.blk_hit[i] : 0;
        hits += block_sum<1024>(hv, sw);
    }
    const int M = run;
    int erun = 0;
    for (int base = 0; base < nS; base += 1024) {
        int i = base + threadIdx.x;
        int v = i < nS ? a.ws.elig_cnt[i] : 0;
        int tot;
        int ex = block_excl_scan<1024>(v, sw, tot);
        if (i < nS) a.ws.elig_off[i] = erun + ex;
        erun += tot;
    }
    if (threadIdx.x == 0) {
        int status = a.ws.ctrl[6] ? 1 : (M > erun ? 3 : 0);
        a.ws.ctrl[0] = M;
        a.ws.ctrl[1] = hits;
        a.ws.ctrl[2] = status;
        a.ws.ctrl[3] = erun;
        a.ws.ctrl[5] = erun - M;
        a.counts[0] = status == 1 ? 0 : hits;
        a.counts[1] = status == 1 ? 0 : M;
        a.counts[2] = 0;
        a.counts[3] = status;
    }
}

// B3: victims + kept prefix of the new order
__global__ void __launch_bounds__(kCacheThreads) cache_victim_kernel(CacheArgs a) {
    __shared__ int sw[64];
    if (a.ws.ctrl[2] != 0) return;
    const int S = a.pool.num_slots;
    const int M = a.ws.ctrl[0];
    const int p0 = blockIdx.x * kSlotChunk + threadIdx.x * kSlotPer;
    int32_t sl[kSlotPer];
    bool el[kSlotPer];
    int c = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        int p = p0 + i;
        sl[i] = p < S ? a.pool.order[p] : -1;
        el[i] = p < S && eligible(a, sl[i]);
        c += el[i];
    }
    int tot;
    int rank = a.ws.elig_off[blockIdx.x] + block_excl_scan<kCacheThreads>(c, sw, tot);
    int ev = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        if (!el[i]) continue;
        if (rank < M) {
            a.ws.vict[rank] = sl[i];
            int64_t old = a.pool.slot_key[sl[i]];
            if (old != -1) {
                a.pool.fwd[old] = -1;
                ++ev;
            }
        } else {
            a.ws.new_order[rank - M] = sl[i];
        }
        ++rank;
    }
    int evs = block_sum<kCacheThreads>(ev, sw);
    if (threadIdx.x == 0 && evs) atomicAdd(&a.ws.ctrl[4], evs);
}

// C: assign misses to victims, stamp hits
__global__ void __launch_bounds__(kCacheThreads) cache_assign_kernel(CacheArgs a) {
    if (a.ws.ctrl[2] != 0) return;
    const int64_t e = (int64_t)blockIdx.x * kCacheThreads + threadIdx.x;
    if (e >= a.E) return;
    if (a.hit_out[e]) {
        a.pool.slot_stamp[a.slot_out[e]] = a.stamp;
        return;
    }
    int ml = a.ws.miss_local[e];
    if (ml < 0) return;
    int i = a.ws.blk_off[blockIdx.x] + ml;
    int32_t s = a.ws.vict[i];
    int64_t key = cache_key(a, e, a.sel[e]);
    a.slot_out[e] = s;
    a.miss_keys[i] = key;
    a.miss_slots[i] = s;
    a.pool.slot_key[s] = key;
    a.pool.fwd[key] = s;
    a.pool.slot_stamp[s] = a.stamp;
}

// D1: per slot chunk, # slots with stamp == t
__global__ void __launch_bounds__(kCacheThreads) cache_teq_count_kernel(CacheArgs a) {
    __shared__ int sw[64];
    if (a.ws.ctrl[2] != 0) return;
    const int S = a.pool.num_slots;
    const int s0 = blockIdx.x * kSlotChunk + threadIdx.x * kSlotPer;
    int c = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        int s = s0 + i;
        if (s < S) c += a.pool.slot_stamp[s] == a.stamp;
    }
    int tot = block_sum<kCacheThreads>(c, sw);
    if (threadIdx.x == 0) {
        a.ws.teq_cnt[blockIdx.x] = tot;
        if (blockIdx.x == 0) a.counts[2] = a.ws.ctrl[4];
    }
}

// D2: place stamp==t slots (slot order) after the kept prefix; copy the prefix
__global__ void __launch_bounds__(kCacheThreads) cache_teq_place_kernel(CacheArgs a) {
    __shared__ int sw[64];
    __shared__ int s_base;
    if (a.ws.ctrl[2] != 0) return;
    const int S = a.pool.num_slots;
    const int kept = a.ws.ctrl[5];
    if (threadIdx.x < 32) {
        int acc = 0;
        for (int c = threadIdx.x; c < (int)blockIdx.x; c += 32) acc += a.ws.teq_cnt[c];
        acc = warp_sum(acc);
        if (threadIdx.x == 0) s_base = kept + acc;
    }
    const int s0 = blockIdx.x * kSlotChunk + threadIdx.x * kSlotPer;
    bool f[kSlotPer];
    int c = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        int s = s0 + i;
        f[i] = s < S && a.pool.slot_stamp[s] == a.stamp;
        c += f[i];
        // copy the kept prefix of the new order (written by B3) into `order`
        if (s < kept) a.pool.order[s] = a.ws.new_order[s];
    }
    int tot;
    int ex = block_excl_scan<kCacheThreads>(c, sw, tot);  // syncs: s_base visible
    int pos = s_base + ex;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i)
        if (f[i]) a.pool.order[pos++] = s0 + i;
}

ss_status launch_cache(const ss_cache_pool& pool, const int32_t* sel, const int32_t* req_ids,
                       int layer, int num_layers, int max_blk, int k, const ss_dims& d,
                       int64_t stamp, int32_t* slot_out, uint8_t* hit_out, int64_t* miss_keys,
                       int32_t* miss_slots, int32_t* counts, void* ws, cudaStream_t stream) {
    CacheArgs a;
    a.pool = pool;
    a.sel = sel;
    a.req_ids = req_ids;
    a.layer = layer;
    a.num_layers = num_layers;
    a.max_blk = max_blk;
    a.k = k;
    a.Hkv = d.num_kv_heads;
    a.E = (int64_t)d.batch * d.num_kv_heads * k;
    a.stamp = stamp;
    a.slot_out = slot_out;
    a.hit_out = hit_out;
    a.miss_keys = miss_keys;
    a.miss_slots = miss_slots;
    a.counts = counts;
    const int S = pool.num_slots;
    carve(&a.ws, ws, a.E, S);
    const int nA = (int)((a.E + kCacheThreads - 1) / kCacheThreads);
    const int nS = (S + kSlotChunk - 1) / kSlotChunk;
    // ctrl and touched are adjacent at the start of the workspace
    size_t clear = (size_t)((char*)a.ws.touched - (char*)a.ws.ctrl) + (size_t)S;
    if (cudaMemsetAsync(a.ws.ctrl, 0, clear, stream) != cudaSuccess) return SS_ERR_CUDA;
    if (nA > 0) cache_lookup_kernel<<<nA, kCacheThreads, 0, stream>>>(a);
    cache_elig_count_kernel<<<nS, kCacheThreads, 0, stream>>>(a);
    cache_plan_kernel<<<1, 1024, 0, stream>>>(a, nA, nS);
    cache_victim_kernel<<<nS, kCacheThreads, 0, stream>>>(a);
    if (nA > 0) cache_assign_kernel<<<nA, kCacheThreads, 0, stream>>>(a);
    cache_teq_count_kernel<<<nS, kCacheThreads, 0, stream>>>(a);
    cache_teq_place_kernel<<<nS, kCacheThreads, 0, stream>>>(a);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

}  // namespace ss
