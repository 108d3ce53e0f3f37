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
//   hash is unnecessary), slot_key[S], slot_stamp[S], order[S] and its inverse
//   order_pos[S].
// Because `order` is kept sorted by (stamp, slot), the LRU victims of a call
// are simply the first M "eligible" entries of `order` (not hit, stamp < t),
// and the new order is [eligible entries not evicted, in old order] ++ [all
// slots with stamp == t, in slot order] -- two stable compactions.
//
// Three phases per call (chunk = 1024 order positions / slots), run as three
// stream-ordered kernels (default) or by ONE persistent kernel with grid
// barriers between them (cache_fused_kernel, SS_CACHE_FUSED=1; measured slower):
//   K1 lookup+count : entry CTAs probe fwd, mark hits, rank misses per CTA;
//                     chunk CTAs count stamp < t per order chunk and
//                     stamp == t per slot chunk; hits correct both counts
//                     through order_pos.  The LAST CTA (atomic ticket) scans
//                     the per-CTA counts, checks capacity, writes counts/status
//                     and publishes the stamp.
//   K2 victims      : first M eligible order entries -> victim list (evict old
//                     keys, mark victims); the rest -> new order prefix
//   K3 assign+place : entry CTAs assign the i-th miss the i-th victim
//                     (fwd / slot_key / stamp) and stamp hits; chunk CTAs append
//                     the stamp==t slots (hit | victim | already t) in slot order
//                     and copy the kept prefix into `order` / `order_pos`.
// On status != 0, K2 and K3 are no-ops: the pool is left byte-identical.
//
// Roofline: integer / latency bound; ~20 B per selection + ~30 B per slot.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"

namespace ss {

constexpr int kCacheThreads = 256;
constexpr int kSlotChunk = 1024;  // order positions / slots per chunk CTA (4 per thread)
constexpr int kSlotPer = kSlotChunk / kCacheThreads;

struct CacheWs {
    // ---- zero on entry to every call: zero-filled once by the caller, and
    // every call leaves them zero again (K2 / K3 clean up; no memset node) ----
    int32_t* ctrl;        // [16]: 0 M, 1 hits, 2 status, 3 total_elig, 4 evictions,
                          //       5 kept, 6 invalid, 7 K1 ticket; [8..9] = stamp (int64),
                          //       10 K3 ticket
    int64_t* ctrl64;      // = ctrl + 8
    uint8_t* touched;     // [S]  slot hit by this call
    uint8_t* victim;      // [S]  slot evicted/assigned by this call
    int32_t* elig_cnt;    // [nS] eligible entries per order chunk
    int32_t* teq_cnt;     // [nS] slots with stamp == t after the call, per slot chunk
    // ---- fully written before being read ----
    int32_t* miss_local;  // [E]
    int32_t* blk_miss;    // [nA]
    int32_t* blk_hit;     // [nA]
    int32_t* blk_off;     // [nA]
    int32_t* elig_off;    // [nS]
    int32_t* vict;        // [E]
    int32_t* new_order;   // [S]
    size_t zero_bytes;    // bytes from ctrl to the end of teq_cnt
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
    t.ctrl64 = t.ctrl ? (int64_t*)(t.ctrl + 8) : nullptr;
    t.touched = (uint8_t*)take((size_t)S);
    t.victim = (uint8_t*)take((size_t)S);
    t.elig_cnt = (int32_t*)take((size_t)nS * 4);
    t.teq_cnt = (int32_t*)take((size_t)nS * 4);
    t.zero_bytes = off;
    t.miss_local = (int32_t*)take((size_t)E * 4);
    t.blk_miss = (int32_t*)take((size_t)nA * 4);
    t.blk_hit = (int32_t*)take((size_t)nA * 4);
    t.blk_off = (int32_t*)take((size_t)nA * 4);
    t.elig_off = (int32_t*)take((size_t)nS * 4);
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
    int32_t nA, nS;
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

// The call's stamp: the host argument, or *clock (read on the device) when
// the pool has a device clock.  K1 reads it; its last CTA publishes it in
// ctrl64[0] for K2/K3.  The caller advances the clock between decode steps.
__device__ __forceinline__ int64_t stamp_pre_plan(const CacheArgs& a) {
    return a.pool.clock ? *a.pool.clock : a.stamp;
}
__device__ __forceinline__ int64_t stamp_post_plan(const CacheArgs& a) {
    return a.pool.clock ? a.ws.ctrl64[0] : a.stamp;
}

// ----------------------------------------------------------------------------
// K1: lookup + counts + (last CTA) plan
// ----------------------------------------------------------------------------
__device__ void cache_plan(const CacheArgs& a, int* sw) {
    // scans of per-CTA miss / hit counts and per-chunk eligible counts
    int run = 0, hits = 0;
    for (int base = 0; base < a.nA; base += kCacheThreads) {
        int i = base + threadIdx.x;
        int v = i < a.nA ? __ldcg(a.ws.blk_miss + i) : 0;
        int tot;
        int ex = block_excl_scan<kCacheThreads>(v, sw, tot);
        if (i < a.nA) a.ws.blk_off[i] = run + ex;
        run += tot;
        hits += block_sum<kCacheThreads>(i < a.nA ? __ldcg(a.ws.blk_hit + i) : 0, sw);
    }
    const int M = run;
    int erun = 0;
    for (int base = 0; base < a.nS; base += kCacheThreads) {
        int i = base + threadIdx.x;
        int v = i < a.nS ? __ldcg(a.ws.elig_cnt + i) : 0;
        int tot;
        int ex = block_excl_scan<kCacheThreads>(v, sw, tot);
        if (i < a.nS) a.ws.elig_off[i] = erun + ex;
        erun += tot;
    }
    if (threadIdx.x == 0) {
        int status = __ldcg(a.ws.ctrl + 6) ? 1 : (M > erun ? 3 : 0);
        a.ws.ctrl[0] = M;
        a.ws.ctrl[1] = hits;
        a.ws.ctrl[2] = status;
        a.ws.ctrl[3] = erun;
        a.ws.ctrl[5] = erun - M;
        a.counts[0] = status == 1 ? 0 : hits;
        a.counts[1] = status == 1 ? 0 : M;
        a.counts[2] = 0;
        a.counts[3] = status;
        a.ws.ctrl64[0] = stamp_pre_plan(a);
    }
}

// Phase 1 work item (entry item < nA, else order/slot chunk item - nA).
__device__ void p1_item(const CacheArgs& a, int item, int* sw, int64_t t) {
    if (item < a.nA) {
        // ---- entry CTA: probe fwd, mark hits, rank misses ----
        const int64_t e = (int64_t)item * kCacheThreads + threadIdx.x;
        int is_miss = 0, is_hit = 0;
        int ch_elig = -1, ch_teq = -1;  // chunks whose counters this hit moves
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
                        const int64_t st = a.pool.slot_stamp[f];
                        // a hit slot leaves the eligible set and joins stamp == t
                        if (st < t) {
                            ch_elig = a.pool.order_pos[f] / kSlotChunk;
                            ch_teq = f / kSlotChunk;
                        }
                    } else {
                        is_miss = 1;
                    }
                }
            }
            a.slot_out[e] = so;
            a.hit_out[e] = ho;
        }
        // warp-aggregated counter updates: recent (hit) slots crowd into the last
        // few order chunks, so per-hit atomics would serialise on a few words
        {
            const unsigned ge = __match_any_sync(0xffffffffu, ch_elig);
            if (ch_elig >= 0 && lane_id() == __ffs(ge) - 1) atomicSub(&a.ws.elig_cnt[ch_elig], __popc(ge));
            const unsigned gt = __match_any_sync(0xffffffffu, ch_teq);
            if (ch_teq >= 0 && lane_id() == __ffs(gt) - 1) atomicAdd(&a.ws.teq_cnt[ch_teq], __popc(gt));
        }
        int tot;
        int rank = block_excl_scan<kCacheThreads>(is_miss, sw, tot);
        if (e < a.E) a.ws.miss_local[e] = is_miss ? rank : -1;
        int hits = block_sum<kCacheThreads>(is_hit, sw);
        if (threadIdx.x == 0) {
            a.ws.blk_miss[item] = tot;
            a.ws.blk_hit[item] = hits;
        }
    } else {
        // ---- chunk CTA: stamp < t per order chunk, stamp == t per slot chunk ----
        const int S = a.pool.num_slots;
        const int c = item - a.nA;
        const int p0 = c * kSlotChunk + threadIdx.x * kSlotPer;
        int lt = 0, eq = 0;
#pragma unroll
        for (int i = 0; i < kSlotPer; ++i) {
            const int p = p0 + i;
            if (p < S) {
                lt += a.pool.slot_stamp[a.pool.order[p]] < t;
                eq += a.pool.slot_stamp[p] == t;
            }
        }
        lt = block_sum<kCacheThreads>(lt, sw);
        eq = block_sum<kCacheThreads>(eq, sw);
        if (threadIdx.x == 0) {
            if (lt) atomicAdd(&a.ws.elig_cnt[c], lt);
            if (eq) atomicAdd(&a.ws.teq_cnt[c], eq);
        }
    }
}

// Programmatic dependent launch (PDL, SS_CACHE_PDL=1) between the three kernels: K1 lets K2's
// CTAs launch at once (they take their SM slots while K1 runs and block in
// griddepcontrol.wait until K1 has completed and its writes are visible), and
// K2 does the same for K3 -- inside a decode step the next kernel no longer
// queues for slots behind other request groups' long select / attention CTAs.
__device__ __forceinline__ void pdl_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__global__ void __launch_bounds__(kCacheThreads) cache_lookup_count_kernel(CacheArgs a) {
    __shared__ int sw[64];
    pdl_launch_dependents();
    p1_item(a, blockIdx.x, sw, stamp_pre_plan(a));
    // ---- last CTA plans ----
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) sw[48] = atomicAdd(&a.ws.ctrl[7], 1);
    __syncthreads();
    if (sw[48] != (int)gridDim.x - 1) return;
    __threadfence();
    if (threadIdx.x == 0) a.ws.ctrl[7] = 0;  // K1 ticket back to zero
    cache_plan(a, sw);
}

// ----------------------------------------------------------------------------
// K2: victims + kept prefix of the new order
// ----------------------------------------------------------------------------
__device__ void p2_item(const CacheArgs& a, int item, int* sw, int M, int64_t t) {
    const int S = a.pool.num_slots;
    const int p0 = item * kSlotChunk + threadIdx.x * kSlotPer;
    int32_t sl[kSlotPer];
    bool el[kSlotPer];
    int c = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        int p = p0 + i;
        sl[i] = p < S ? a.pool.order[p] : -1;
        el[i] = p < S && !__ldcg(a.ws.touched + sl[i]) && a.pool.slot_stamp[sl[i]] < t;
        c += el[i];
    }
    int tot;
    int rank = __ldcg(a.ws.elig_off + item) + block_excl_scan<kCacheThreads>(c, sw, tot);
    int ev = 0;
#pragma unroll
    for (int i = 0; i < kSlotPer; ++i) {
        if (!el[i]) continue;
        const int32_t s = sl[i];
        if (rank < M) {
            a.ws.vict[rank] = s;
            a.ws.victim[s] = 1;
            atomicAdd(&a.ws.teq_cnt[s / kSlotChunk], 1);
            int64_t old = a.pool.slot_key[s];
            if (old != -1) {
                a.pool.fwd[old] = -1;
                ++ev;
            }
        } else {
            a.ws.new_order[rank - M] = s;
        }
        ++rank;
    }
    int evs = block_sum<kCacheThreads>(ev, sw);
    if (threadIdx.x == 0 && evs) atomicAdd(&a.ws.ctrl[4], evs);
}

__global__ void __launch_bounds__(kCacheThreads) cache_victim_kernel(CacheArgs a) {
    __shared__ int sw[64];
    pdl_wait();
    pdl_launch_dependents();
    if (a.ws.ctrl[2] != 0) return;
    p2_item(a, blockIdx.x, sw, a.ws.ctrl[0], stamp_post_plan(a));
}

// ----------------------------------------------------------------------------
// K3: assign misses / stamp hits (entry CTAs) || place stamp==t slots (chunk CTAs)
// ----------------------------------------------------------------------------
__device__ void p3_item(const CacheArgs& a, int item, int* sw, int* s_base_p, bool ok, int kept,
                        int evictions, int64_t t) {
    int& s_base = *s_base_p;
    const int S = a.pool.num_slots;
    if (item < a.nA) {
        const int64_t e = (int64_t)item * kCacheThreads + threadIdx.x;
        if (ok && e < a.E) {
            if (__ldcg(a.hit_out + e)) {
                a.pool.slot_stamp[__ldcg(a.slot_out + e)] = t;
            } else {
                const int ml = __ldcg(a.ws.miss_local + e);
                if (ml >= 0) {
                    const int i = __ldcg(a.ws.blk_off + item) + ml;
                    const int32_t s = __ldcg(a.ws.vict + i);
                    const int64_t key = cache_key(a, e, a.sel[e]);
                    a.slot_out[e] = s;
                    a.miss_keys[i] = key;
                    a.miss_slots[i] = s;
                    a.pool.slot_key[s] = key;
                    a.pool.fwd[key] = s;
                    a.pool.slot_stamp[s] = t;
                }
            }
        }
    } else {
        // chunk CTA c: slots [c*1024, (c+1)*1024) in slot order
        const int c = item - a.nA;
        if (ok && c == 0 && threadIdx.x == 0) a.counts[2] = evictions;
        if (threadIdx.x < 32) {
            int acc = 0;
            for (int cc = threadIdx.x; cc < c; cc += 32) acc += __ldcg(a.ws.teq_cnt + cc);
            acc = warp_sum(acc);
            if (threadIdx.x == 0) s_base = kept + acc;
        }
        const int s0 = c * kSlotChunk + threadIdx.x * kSlotPer;
        bool f[kSlotPer];
        int n = 0;
#pragma unroll
        for (int i = 0; i < kSlotPer; ++i) {
            const int s = s0 + i;
            // stamp == t after this call: hit, victim, or already stamped t (a
            // concurrent K3 entry CTA may be writing t into hit / victim slots;
            // their flags already decide those)
            f[i] = ok && s < S && (__ldcg(a.ws.touched + s) || __ldcg(a.ws.victim + s) || a.pool.slot_stamp[s] == t);
            n += f[i];
            // this chunk's per-call flags go back to zero (K1 set touched even
            // when the call fails)
            if (s < S) {
                a.ws.touched[s] = 0;
                a.ws.victim[s] = 0;
            }
            // copy the kept prefix of the new order (K2) into order / order_pos
            if (ok && s < kept) {
                const int32_t v = __ldcg(a.ws.new_order + s);
                a.pool.order[s] = v;
                a.pool.order_pos[v] = s;
            }
        }
        if (threadIdx.x == 0) a.ws.elig_cnt[c] = 0;
        int tot;
        int ex = block_excl_scan<kCacheThreads>(n, sw, tot);  // syncs: s_base visible
        int pos = s_base + ex;
#pragma unroll
        for (int i = 0; i < kSlotPer; ++i)
            if (f[i]) {
                a.pool.order[pos] = s0 + i;
                a.pool.order_pos[s0 + i] = pos;
                ++pos;
            }
        __syncthreads();  // s_base is reused by the CTA's next item
    }
}

// the last CTA of the final phase (every CTA has read ctrl / teq_cnt by now)
// zeroes the call-wide words, leaving the workspace ready for the next call
__device__ void cache_cleanup(const CacheArgs& a, int* sw, int ticket_idx, int nctas) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) sw[48] = atomicAdd(&a.ws.ctrl[ticket_idx], 1);
    __syncthreads();
    if (sw[48] != nctas - 1) return;
    __threadfence();
    for (int c = threadIdx.x; c < a.nS; c += kCacheThreads) a.ws.teq_cnt[c] = 0;
    __syncthreads();
    if (threadIdx.x < 16) a.ws.ctrl[threadIdx.x] = 0;
}

__global__ void __launch_bounds__(kCacheThreads) cache_assign_place_kernel(CacheArgs a) {
    __shared__ int sw[64];
    __shared__ int s_base;
    pdl_wait();
    p3_item(a, blockIdx.x, sw, &s_base, a.ws.ctrl[2] == 0, a.ws.ctrl[5], a.ws.ctrl[4], stamp_post_plan(a));
    cache_cleanup(a, sw, 10, gridDim.x);
}
// ----------------------------------------------------------------------------
// Fused form (SS_CACHE_FUSED=1): the three phases in ONE launch of a small persistent
// grid with two software grid barriers (plan by CTA 0 between them).  Inside a
// decode step the three separate kernels each queue for SM slots behind the
// other request groups' long select / attention CTAs; the fused call queues
// once.  Every cross-phase read goes through L2 (__ldcg).  The grid (<= 128
// CTAs of 256 threads, 8 K registers each) is far below what the 148 SMs hold,
// so every CTA becomes resident once co-running kernels release slots.
// ----------------------------------------------------------------------------
__device__ __forceinline__ void grid_barrier(int32_t* count, int32_t* gen, int n) {
    __syncthreads();
    if (threadIdx.x == 0) {
        int g;
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(g) : "l"(gen) : "memory");
        __threadfence();
        if (atomicAdd(count, 1) == n - 1) {
            atomicExch(count, 0);
            __threadfence();
            asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
        } else {
            int v = g;
            while (v == g) {
                __nanosleep(32);
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
            }
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kCacheThreads) cache_fused_kernel(CacheArgs a) {
    __shared__ int sw[64];
    __shared__ int s_base;
    // the clock advances only between decode steps: one read serves all phases
    const int64_t t = stamp_pre_plan(a);
    const int n1 = a.nA + a.nS;
    int32_t* bar_count = a.ws.ctrl + 11;
    int32_t* bar_gen = a.ws.ctrl + 12;
    for (int it = blockIdx.x; it < n1; it += gridDim.x) {
        p1_item(a, it, sw, t);
        __syncthreads();
    }
    grid_barrier(bar_count, bar_gen, gridDim.x);
    if (blockIdx.x == 0) cache_plan(a, sw);
    grid_barrier(bar_count, bar_gen, gridDim.x);
    const int status = __ldcg(a.ws.ctrl + 2);
    const int M = __ldcg(a.ws.ctrl + 0);
    const int kept = __ldcg(a.ws.ctrl + 5);
    if (status == 0)
        for (int it = blockIdx.x; it < a.nS; it += gridDim.x) {
            p2_item(a, it, sw, M, t);
            __syncthreads();
        }
    grid_barrier(bar_count, bar_gen, gridDim.x);
    const int evictions = __ldcg(a.ws.ctrl + 4);
    for (int it = blockIdx.x; it < n1; it += gridDim.x) {
        p3_item(a, it, sw, &s_base, status == 0, kept, evictions, t);
        __syncthreads();
    }
    cache_cleanup(a, sw, 10, gridDim.x);
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
    a.nA = (int)((a.E + kCacheThreads - 1) / kCacheThreads);
    a.nS = (S + kSlotChunk - 1) / kSlotChunk;
    // three kernels (default) or the fused form (SS_CACHE_FUSED=1; same results).
    // Measured in the C2 step: fused 54.8 us alone / 76 us in-step vs 38.7 / 56.6
    // for three kernels -- the 128-CTA grid serialises items per CTA and its
    // barriers cost more than two kernel boundaries (profiles/r01s3_cache_fused_ab.txt)
    const int fused = knob("SS_CACHE_FUSED", 0);
    const int fused_ctas = knob("SS_CACHE_CTAS", 128);
    if (fused) {
        const int grid = std::max(1, std::min(a.nA + a.nS, std::min(fused_ctas, num_sms())));
        cache_fused_kernel<<<grid, kCacheThreads, 0, stream>>>(a);
    } else {
        set_carveout(cache_lookup_count_kernel);
        set_carveout(cache_victim_kernel);
        set_carveout(cache_assign_place_kernel);
        cache_lookup_count_kernel<<<a.nA + a.nS, kCacheThreads, 0, stream>>>(a);
        // K2, K3: plain launches (default) or programmatic dependent launches
        // (SS_CACHE_PDL=1; griddepcontrol.wait is a no-op without).  Measured in
        // the C2 step: PDL makes the call faster (34 vs 39 us alone, 52 vs 57 in
        // the step) but the step slower (11.85 vs 11.0 ms median): the early-
        // resident K2/K3 CTAs take SM slots from the other groups' select.
        const int pdl = knob("SS_CACHE_PDL", 0);
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cudaLaunchConfig_t lc = {};
        lc.blockDim = dim3(kCacheThreads);
        lc.dynamicSmemBytes = 0;
        lc.stream = stream;
        lc.attrs = attr;
        lc.numAttrs = pdl ? 1 : 0;
        lc.gridDim = dim3(a.nS);
        if (cudaLaunchKernelEx(&lc, cache_victim_kernel, a) != cudaSuccess) return SS_ERR_CUDA;
        lc.gridDim = dim3(a.nA + a.nS);
        if (cudaLaunchKernelEx(&lc, cache_assign_place_kernel, a) != cudaSuccess) return SS_ERR_CUDA;
    }
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_cache() {
    return preload_fn(cache_lookup_count_kernel) && preload_fn(cache_victim_kernel) &&
           preload_fn(cache_assign_place_kernel) && preload_fn(cache_fused_kernel);
}

}  // namespace ss
