// sparse_attn.cu -- S5 sparse decode attention (§2.1:
// S = QK^T/sqrt(d), P = softmax(S), O = PV; PAPER.md:33 / :124: computed only
// over the KV blocks selected for the query token).  Readings R7 (tail block
// always attended), R9 (softmax renormalised over selected tokens + tail), R10
// (float32 output) in DESIGN.md; reference: oracle/oracle.c or_attention.
//
// B200 design: a persistent, stream-K split over "units".  A unit is one
// selected head-block (16 KiB K+V in bf16, contiguous in its HBM cache slot,
// PAPER.md:137 (H,N,D) layout) or the tail block of a (b, h) pair; a pair has
// Ku = k + 1 units (slot -1 / empty tail units are skipped).  The U = pairs*Ku
// units are cut into W equal contiguous ranges, one per warp (W = 148 SMs x NW
// warps), so every warp streams the same number of bytes whatever the per-pair
// split.  Each warp double-buffers whole blocks into its own shared memory with
// 1-D TMA bulk copies (cp.async.bulk + mbarrier complete_tx; SASS UBLKCP), so
// HBM reads are 16 KiB transactions issued by one lane while the warp computes
// on the previous block.  Pairs covered entirely by one warp are finalised in
// place; a pair cut by range boundaries leaves <= 1 partial (m, l, o) per
// contributing warp in the workspace and the last contributor (atomic ticket,
// self-resetting) merges them in warp order -- deterministic.
//
// Two compute paths share that schedule.  bf16 (default): sparse_attn_mma_kernel
// below -- tensor-core mma.sync over 2-D TMA, 128B-swizzled tiles.  f32 (and
// bf16 with SS_ATTN_MMA=0): sparse_attn_kernel -- per block, lane t computes
// token t's logits for the G query heads of the KV head (K row read with a
// lane-rotated chunk order: conflict-free 16-byte shared loads), an online
// softmax in exp2 domain, and lane l accumulates output dims 4l..4l+3 from the
// V rows in float32 (keeps the 1e-5 f32 tolerance).
//
// Roofline: HBM-bound; algorithmic bytes = block_bytes per attended unit
// (+ q, out: negligible).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <mutex>
#include <stdlib.h>

#include "common.cuh"

namespace ss {

constexpr int kAttnPartStride = 132;
// floats per (warp, seg, g) partial: m, l, pad, pad, o[128]
// at least this many units per warp: fewer, longer ranges when the problem is
// small.  Measured back to back with the bulk-load merge (profiles/r02_attn_min_units.txt):
// GQA (G = 4) two / one C3 request 17.3 / 16.5 us at 4 vs 18.6 / 18.5 at 8, but the
// full C3 batch (where 4 would already occupy every warp) 20.5 at 4 vs 20.0 at 8;
// MHA one C2 request group 25.7-25.9 us at 12 vs 26.7-26.8 at 8 alone, but the C2 step
// (request groups co-running) read 1476 tok/s with 12 against 1483-1511 over eight runs
// at 8 (r02bc), so MHA keeps 8
constexpr int kMinUnitsPerWarpGqaSmall = 4;
constexpr int kMinUnitsPerWarpGqa = 8;
constexpr int kMinUnitsPerWarpMha = 8;
constexpr int kTraceSlots = 12;       // debug timeline words per warp (AttnArgs::trace)

struct AttnArgs {
    const void* q;
    const void* pool;
    const int32_t* slot;
    const void* tail;
    const int32_t* tail_len;
    const int32_t* counts;
    float* out;
    float* part;
    int32_t* tickets;
    int k, B, Hq, Hkv;
    float scale_log2;
    // split form (sparse_decode_attn_part): mode 0 = every selected block + tail,
    // 1 = hit blocks (hit[] != 0) + tail, 2 = missed blocks only; lse (or null)
    // receives log2-domain log-sum-exp per (hq, b): m + log2(l), -inf if empty
    const uint8_t* hit;
    int mode;
    float* lse;
    int64_t U;  // pairs * (k + 1)
    int merge_bulk;  // 1: end-of-range merges through bulk loads (default); 0: registers (debug A/B)
    int W;      // total warps
    unsigned long long* trace;  // debug (SS_ATTN_TRACE=1): per warp globaltimer at entry / last unit / exit / merge start / merge end / partial flush / ticket / (m, l) loaded
};

__device__ __forceinline__ bool knob_attn_merge_bulk(const AttnArgs& a) { return a.merge_bulk != 0; }

template <bool BF16>
struct AttnTraits {
    static constexpr int ES = BF16 ? 2 : 4;
    static constexpr int BLOCK_ELEMS = 2 * kBlockTokens * kHeadDim;
    static constexpr int BLOCK_BYTES = BLOCK_ELEMS * ES;
    static constexpr int CPC = 16 / ES;             // elements per 16-byte chunk
    static constexpr int NCH = kHeadDim / CPC;      // chunks per K row
    static constexpr int NW = BF16 ? 6 : 3;         // warps per CTA (smem-limited)
};

template <bool BF16, int G>
struct WarpSmem {
    using T = AttnTraits<BF16>;
    alignas(128) unsigned char buf[2][T::BLOCK_BYTES];
    alignas(16) float4 q4[G][kHeadDim / 4];  // q (fp32) in 16-byte chunks, chunk order below
    alignas(16) float p[G][kBlockTokens];    // softmax numerators of the current block
    uint64_t bar[2][2];  // [stage][K half / V half]
};

__device__ __forceinline__ int64_t warp_of_unit(int64_t x, int64_t U, int W) {
    return ((x + 1) * (int64_t)W - 1) / U;
}

// q of the G heads of KV head (b, h): lane loads elements 4*lane .. 4*lane+3.
template <bool BF16, int G>
__device__ __forceinline__ void load_q(const AttnArgs& a, int b, int h, int lane, float4 (&r)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const int64_t qi = ((int64_t)b * a.Hq + (int64_t)h * G + g) * kHeadDim + 4 * lane;
        if (BF16) {
            uint2 raw = __ldg(reinterpret_cast<const uint2*>((const uint16_t*)a.q + qi));
            r[g] = make_float4(__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u),
                               __uint_as_float(raw.y << 16), __uint_as_float(raw.y & 0xFFFF0000u));
        } else {
            r[g] = __ldg(reinterpret_cast<const float4*>((const float*)a.q + qi));
        }
    }
}

// A warp whose range cut pair p has written its partial (m, l, o) of the G
// heads: take a ticket; true for the last contributor, which then merges all
// partials (merge_partials).
// The ticket is one acq_rel atomic: its release half (after the warp barrier,
// cumulative over every lane's partial stores) publishes this warp's partial,
// its acquire half makes the other contributors' partials visible to the last
// one -- no separate sequentially consistent fences (measured: each
// fence.sc.gpu cost ~0.8 us at the end of a launch, r02v).
__device__ __forceinline__ int atom_add_acq_rel_gpu(int32_t* p, int v) {
    int old;
    asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ bool partial_is_last(const AttnArgs& a, int64_t p) {
    const int lane = lane_id();
    const int Ku = a.k + 1;
    __syncwarp();
    int ticket = 0;
    if (lane == 0) ticket = atom_add_acq_rel_gpu(&a.tickets[p], 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    const int64_t wf = warp_of_unit(p * Ku, a.U, a.W);
    const int64_t wl = warp_of_unit((p + 1) * Ku - 1, a.U, a.W);
    return ticket == (int)(wl - wf);
}

// The last contributor merges all partials of pair p in warp order
// (deterministic) and writes the output, then resets the ticket.
template <int G, int UNR>
__device__ void merge_partials(const AttnArgs& a, int64_t p, int w) {
    const int lane = lane_id();
    const int Ku = a.k + 1;
    const int b = (int)(p / a.Hkv), h = (int)(p % a.Hkv);
    const int64_t wf = warp_of_unit(p * Ku, a.U, a.W);
    const int64_t wl = warp_of_unit((p + 1) * Ku - 1, a.U, a.W);
    auto trace = [&](int i) {
        if (a.trace != nullptr && lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[(int64_t)w * kTraceSlots + i] = t;
        }
    };
    trace(3);
    // merge the contributors' partials in warp order (deterministic).  Which of
    // its two partial slots contributor w2 used for p: slot 0 iff its range
    // starts inside p, i.e. floor(U*w2/W) >= p*Ku  <=>  U*w2 >= p*Ku*W (no
    // division: 64-bit integer division is a long software sequence).
    const int nc = (int)(wl - wf + 1);
    const int64_t pkw = p * Ku * (int64_t)a.W;
    auto base_of = [&](int i) -> int64_t {  // float offset of contributor i's head-0 partial
        const int64_t w2 = wf + i;
        return ((w2 * 2 + (a.U * w2 >= pkw ? 0 : 1)) * G) * kAttnPartStride;
    };
    // heads in chunks of GC (register pressure for G = 8)
    constexpr int GC = G < 4 ? G : 4;
#pragma unroll 1
    for (int g0 = 0; g0 < G; g0 += GC) {
        float mt[GC], lt[GC], oo[GC][4];
#pragma unroll
        for (int g = 0; g < GC; ++g) {
            mt[g] = -INFINITY;
            lt[g] = 0.f;
            oo[g][0] = oo[g][1] = oo[g][2] = oo[g][3] = 0.f;
        }
        // (m, l) of contributors lane, lane + 32, ...; the first 32 stay in
        // registers (nc <= 32 is the common case: one memory round trip)
        float m0[GC], l0[GC];
        int64_t b0 = 0;
#pragma unroll
        for (int g = 0; g < GC; ++g) m0[g] = -INFINITY, l0[g] = 0.f;
        for (int i = lane; i < nc; i += 32) {
            const int64_t bi = base_of(i) + g0 * kAttnPartStride;
#pragma unroll
            for (int g = 0; g < GC; ++g) {
                const float mv = __ldcg(a.part + bi + g * kAttnPartStride);
                mt[g] = fmaxf(mt[g], mv);
                if (i == lane) {
                    m0[g] = mv;
                    l0[g] = __ldcg(a.part + bi + g * kAttnPartStride + 1);
                }
            }
            if (i == lane) b0 = bi;
        }
#pragma unroll
        for (int g = 0; g < GC; ++g) mt[g] = warp_max(mt[g]);
        if (g0 == 0) trace(7);
        for (int i0 = 0; i0 < nc; i0 += 32) {
            // lane-parallel: contributor i0 + lane's partial offset and scale per head
            const int i = i0 + lane;
            int64_t base_i = b0;
            float sc_i[GC];
#pragma unroll
            for (int g = 0; g < GC; ++g) sc_i[g] = 0.f;
            if (i < nc) {
                if (i0 > 0) base_i = base_of(i) + g0 * kAttnPartStride;
#pragma unroll
                for (int g = 0; g < GC; ++g) {
                    const float* pp = a.part + base_i + g * kAttnPartStride;
                    const float mv = i0 == 0 ? m0[g] : __ldcg(pp);
                    const float lv = i0 == 0 ? l0[g] : __ldcg(pp + 1);
                    if (mt[g] != -INFINITY) {
                        sc_i[g] = exp2f(mv - mt[g]);
                        lt[g] += lv * sc_i[g];
                    }
                }
            }
            const int n = min(32, nc - i0);
#pragma unroll UNR
            for (int j = 0; j < n; ++j) {
                const int64_t bj = __shfl_sync(0xffffffffu, base_i, j);
#pragma unroll
                for (int g = 0; g < GC; ++g) {
                    const float sc = __shfl_sync(0xffffffffu, sc_i[g], j);
                    const float4 ov = __ldcg(reinterpret_cast<const float4*>(
                        a.part + bj + g * kAttnPartStride + 4 + 4 * lane));
                    oo[g][0] = fmaf(ov.x, sc, oo[g][0]);
                    oo[g][1] = fmaf(ov.y, sc, oo[g][1]);
                    oo[g][2] = fmaf(ov.z, sc, oo[g][2]);
                    oo[g][3] = fmaf(ov.w, sc, oo[g][3]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < GC; ++g) {
            const float lsum = warp_sum(lt[g]);
            const float inv = lsum > 0.f ? __frcp_rn(lsum) : 0.f;
            const int hq = h * G + g0 + g;
            if (a.lse != nullptr && lane == 0)
                a.lse[(int64_t)hq * a.B + b] = lsum > 0.f ? mt[g] + log2f(lsum) : -INFINITY;
            *reinterpret_cast<float4*>(a.out + ((int64_t)hq * a.B + b) * kHeadDim + 4 * lane) =
                make_float4(oo[g][0] * inv, oo[g][1] * inv, oo[g][2] * inv, oo[g][3] * inv);
        }
    }
    trace(4);
    if (lane == 0) a.tickets[p] = 0;
}

template <bool BF16, int G>
__global__ void __launch_bounds__(AttnTraits<BF16>::NW * 32, 1) sparse_attn_kernel(AttnArgs a) {
    using T = AttnTraits<BF16>;
    if (a.counts != nullptr && a.counts[3] != 0) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    WarpSmem<BF16, G>& sm = reinterpret_cast<WarpSmem<BF16, G>*>(smem_raw)[warp_id()];
    const int lane = lane_id();
    // warp w = warp_id * gridDim + CTA: with W < total warps the active warps
    // spread over all SMs (not packed into the first CTAs)
    const int w = warp_id() * gridDim.x + blockIdx.x;
    if (w >= a.W) return;  // W = min(total warps, U): every active warp owns >= 1 unit
    const int64_t u0 = a.U * w / a.W, u1 = a.U * (w + 1) / a.W;
    const int Ku = a.k + 1;

    if (lane == 0) {
        mbar_init(&sm.bar[0][0], 1);
        mbar_init(&sm.bar[0][1], 1);
        mbar_init(&sm.bar[1][0], 1);
        mbar_init(&sm.bar[1][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // ---- producer: next valid unit -> stage (lane 0 issues the bulk copy) ----
    // The unit descriptors of the warp's range are read 32 at a time into a
    // lane-distributed window (lane l: unit wbase + l), so finding the next
    // valid unit is a ballot, not a dependent global load per block.
    int64_t next_u = u0;
    int64_t bu0 = -1, bu1 = -1;  // unit held by stage 0 / 1 (-1: none)
    int64_t wbase = u0;
    int wkind = 0;               // 0 invalid, 1 pool slot, 2 tail block
    int64_t widx = 0;            // slot or pair index
    auto refill = [&]() {
        const int64_t u = wbase + lane;
        wkind = 0;
        if (u < u1) {
            const int64_t p = u / Ku;
            const int r = (int)(u % Ku);
            if (r < a.k) {
                int32_t sl = __ldg(a.slot + p * a.k + r);
                if (a.mode != 0 && ((__ldg(a.hit + p * a.k + r) != 0) != (a.mode == 1))) sl = -1;
                wkind = sl >= 0 ? 1 : 0;
                widx = sl;
            } else {
                wkind = (a.mode != 2 && __ldg(a.tail_len + p / a.Hkv) > 0) ? 2 : 0;
                widx = p;
            }
        }
    };
    refill();
    // Each stage holds one unit as two 8 KiB (bf16) halves with their own
    // mbarriers: the K half of the next unit is requested as soon as the
    // current unit's logits are done, half a block earlier than a whole-block
    // refill would allow (deeper pipeline at the same shared-memory budget).
    constexpr uint32_t HALF = T::BLOCK_BYTES / 2;
    const char* bsrc0 = nullptr;
    const char* bsrc1 = nullptr;  // source of the unit held by stage 0 / 1
    auto issue_half = [&](int stage, int half) {
        const char* src = stage ? bsrc1 : bsrc0;
        if (lane == 0 && src != nullptr) {
            // order this warp's earlier generic-proxy reads of the buffer
            // before the async-proxy (TMA) write that refills it
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.bar[stage][half], HALF);
            bulk_g2s(sm.buf[stage] + half * HALF, src + half * HALF, HALF, &sm.bar[stage][half]);
        }
    };
    // next valid unit -> stage: records it and requests its K half
    auto issue_k = [&](int stage) {
        while (true) {
            const unsigned m = __ballot_sync(0xffffffffu, wkind != 0 && wbase + lane >= next_u);
            if (m) {
                const int l = __ffs(m) - 1;
                next_u = wbase + l;
                const int kind = __shfl_sync(0xffffffffu, wkind, l);
                const int64_t idx = __shfl_sync(0xffffffffu, widx, l);
                const char* src = kind == 1 ? (const char*)a.pool + idx * T::BLOCK_BYTES
                                            : (const char*)a.tail + idx * T::BLOCK_BYTES;
                (stage ? bsrc1 : bsrc0) = src;
                (stage ? bu1 : bu0) = next_u++;
                issue_half(stage, 0);
                return;
            }
            if (wbase + 32 >= u1) {
                next_u = u1;
                (stage ? bu1 : bu0) = -1;
                (stage ? bsrc1 : bsrc0) = nullptr;
                return;
            }
            wbase += 32;
            refill();
        }
    };
    issue_k(0);
    issue_half(0, 1);
    issue_k(1);
    issue_half(1, 1);
    uint32_t phases = 0u;  // bit 2*stage + half = mbarrier phase
    int stage = 0;

    const int64_t p_first = u0 / Ku, p_last = (u1 - 1) / Ku;
    float4 qn[G];  // q of the next pair, prefetched in registers
    load_q<BF16, G>(a, (int)(p_first / a.Hkv), (int)(p_first % a.Hkv), lane, qn);
    for (int64_t p = p_first; p <= p_last; ++p) {
        const int b = (int)(p / a.Hkv), h = (int)(p % a.Hkv);
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) {
            // element c = 4*lane + i.  bf16: chunk c/8 = lane/2, half (c%8)/4 = lane&1
            if (BF16)
                sm.q4[g][(lane >> 1) + 16 * (lane & 1)] = qn[g];
            else
                sm.q4[g][lane] = qn[g];
        }
        if (p < p_last) load_q<BF16, G>(a, (int)((p + 1) / a.Hkv), (int)((p + 1) % a.Hkv), lane, qn);
        __syncwarp();
        float m[G], l[G], o[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            m[g] = -INFINITY;
            l[g] = 0.f;
            o[g][0] = o[g][1] = o[g][2] = o[g][3] = 0.f;
        }
        const int tl = __ldg(a.tail_len + b);

        while (true) {
            const int64_t cu = stage ? bu1 : bu0;
            if (cu < 0 || cu / Ku != p) break;
            const bool is_tail = (cu % Ku) == a.k;
            mbar_wait(&sm.bar[stage][0], (phases >> (2 * stage)) & 1u);
            phases ^= 1u << (2 * stage);
            const unsigned char* kb = sm.buf[stage];
            const unsigned char* vb = kb + kBlockTokens * kHeadDim * T::ES;
            // ---- logits: lane = token; 4 independent accumulators per head ----
            float sacc[G][4];
#pragma unroll
            for (int g = 0; g < G; ++g) sacc[g][0] = sacc[g][1] = sacc[g][2] = sacc[g][3] = 0.f;
            const unsigned char* krow = kb + lane * kHeadDim * T::ES;
#pragma unroll
            for (int c = 0; c < T::NCH; ++c) {
                const int cc = (c + lane) & (T::NCH - 1);
                const uint4 kv = *reinterpret_cast<const uint4*>(krow + cc * 16);
                const int a0 = (c & 1) * 2;
                if (BF16) {
                    const float k0 = __uint_as_float(kv.x << 16), k1 = __uint_as_float(kv.x & 0xFFFF0000u);
                    const float k2 = __uint_as_float(kv.y << 16), k3 = __uint_as_float(kv.y & 0xFFFF0000u);
                    const float k4 = __uint_as_float(kv.z << 16), k5 = __uint_as_float(kv.z & 0xFFFF0000u);
                    const float k6 = __uint_as_float(kv.w << 16), k7 = __uint_as_float(kv.w & 0xFFFF0000u);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float4 qa = sm.q4[g][cc], qb = sm.q4[g][cc + 16];
                        sacc[g][a0] = fmaf(qa.x, k0, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qa.y, k1, sacc[g][a0 + 1]);
                        sacc[g][a0] = fmaf(qa.z, k2, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qa.w, k3, sacc[g][a0 + 1]);
                        sacc[g][a0] = fmaf(qb.x, k4, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qb.y, k5, sacc[g][a0 + 1]);
                        sacc[g][a0] = fmaf(qb.z, k6, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qb.w, k7, sacc[g][a0 + 1]);
                    }
                } else {
                    const float k0 = __uint_as_float(kv.x), k1 = __uint_as_float(kv.y);
                    const float k2 = __uint_as_float(kv.z), k3 = __uint_as_float(kv.w);
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        const float4 qa = sm.q4[g][cc];
                        sacc[g][a0] = fmaf(qa.x, k0, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qa.y, k1, sacc[g][a0 + 1]);
                        sacc[g][a0] = fmaf(qa.z, k2, sacc[g][a0]);
                        sacc[g][a0 + 1] = fmaf(qa.w, k3, sacc[g][a0 + 1]);
                    }
                }
            }
            const bool valid = !is_tail || lane < tl;
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float s = (sacc[g][0] + sacc[g][1]) + (sacc[g][2] + sacc[g][3]);
                const float z = valid ? s * a.scale_log2 : -INFINITY;
                const float mnew = fmaxf(m[g], warp_max(z));
                const float corr = exp2f(m[g] - mnew);
                const float pp = exp2f(z - mnew);
                sm.p[g][lane] = pp;
                l[g] = l[g] * corr + warp_sum(pp);
                o[g][0] *= corr;
                o[g][1] *= corr;
                o[g][2] *= corr;
                o[g][3] *= corr;
                m[g] = mnew;
            }
            __syncwarp();
            // K half consumed: request the K half of this stage's next unit now
            issue_k(stage);
            mbar_wait(&sm.bar[stage][1], (phases >> (2 * stage + 1)) & 1u);
            phases ^= 1u << (2 * stage + 1);
            // ---- O += P V: lane owns dims 4*lane .. 4*lane+3 ----
            auto pv_token = [&](int t, const float (&pt)[G]) {
                float v0, v1, v2, v3;
                if (BF16) {
                    const uint2 vv = *reinterpret_cast<const uint2*>(vb + (t * kHeadDim + 4 * lane) * 2);
                    v0 = __uint_as_float(vv.x << 16);
                    v1 = __uint_as_float(vv.x & 0xFFFF0000u);
                    v2 = __uint_as_float(vv.y << 16);
                    v3 = __uint_as_float(vv.y & 0xFFFF0000u);
                } else {
                    const float4 vv = *reinterpret_cast<const float4*>(vb + (t * kHeadDim + 4 * lane) * 4);
                    v0 = vv.x;
                    v1 = vv.y;
                    v2 = vv.z;
                    v3 = vv.w;
                }
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    o[g][0] = fmaf(pt[g], v0, o[g][0]);
                    o[g][1] = fmaf(pt[g], v1, o[g][1]);
                    o[g][2] = fmaf(pt[g], v2, o[g][2]);
                    o[g][3] = fmaf(pt[g], v3, o[g][3]);
                }
            };
            if (!is_tail) {
#pragma unroll
                for (int t4 = 0; t4 < kBlockTokens; t4 += 4) {
                    float4 p4[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) p4[g] = *reinterpret_cast<const float4*>(&sm.p[g][t4]);
                    float pt[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) pt[g] = p4[g].x;
                    pv_token(t4 + 0, pt);
#pragma unroll
                    for (int g = 0; g < G; ++g) pt[g] = p4[g].y;
                    pv_token(t4 + 1, pt);
#pragma unroll
                    for (int g = 0; g < G; ++g) pt[g] = p4[g].z;
                    pv_token(t4 + 2, pt);
#pragma unroll
                    for (int g = 0; g < G; ++g) pt[g] = p4[g].w;
                    pv_token(t4 + 3, pt);
                }
            } else {
                // tail block: only the first tl rows hold data (the rest may be garbage)
                for (int t = 0; t < tl; ++t) {
                    float pt[G];
#pragma unroll
                    for (int g = 0; g < G; ++g) pt[g] = sm.p[g][t];
                    pv_token(t, pt);
                }
            }
            __syncwarp();
            issue_half(stage, 1);  // V half of this stage's next unit
            stage ^= 1;
        }

        // ---- flush pair p ----
        const bool full = (p * Ku >= u0) && ((p + 1) * Ku <= u1);
        if (full) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float inv = l[g] > 0.f ? __frcp_rn(l[g]) : 0.f;
                const int hq = h * G + g;
                *reinterpret_cast<float4*>(a.out + ((int64_t)hq * a.B + b) * kHeadDim + 4 * lane) =
                    make_float4(o[g][0] * inv, o[g][1] * inv, o[g][2] * inv, o[g][3] * inv);
                if (a.lse != nullptr && lane == 0)
                    a.lse[(int64_t)hq * a.B + b] = l[g] > 0.f ? m[g] + log2f(l[g]) : -INFINITY;
            }
            continue;
        }
        const int seg = (p == p_first) ? 0 : 1;
#pragma unroll
        for (int g = 0; g < G; ++g) {
            float* pp = a.part + (((int64_t)w * 2 + seg) * G + g) * kAttnPartStride;
            if (lane == 0) {
                pp[0] = m[g];
                pp[1] = l[g];
            }
            *reinterpret_cast<float4*>(pp + 4 + 4 * lane) =
                make_float4(o[g][0], o[g][1], o[g][2], o[g][3]);
        }
        if (partial_is_last(a, p)) merge_partials<G, 4>(a, p, w);
    }
}

// ============================================================================
// bf16 tensor-core variant (the north star's "tensor cores only for the
// batched-GQA QK^T/PV contractions").  Same unit schedule, pipeline and
// partial merge as above; per unit (one 32-token block of one (b, h) pair) one
// warp computes, transposed so that every MMA row is a real token / dim:
//   S^T[32 x 8]   = K[32 x 128] Q^T[128 x 8]     (columns 0..G-1 = the G heads)
//   O^T[128 x 8] += V^T[128 x 32] P^T[32 x 8]    (P split as bf16 hi + lo)
// with mma.sync m16n8k16 (bf16 in, f32 accumulate): 16 + 32 HMMA, 32 ldmatrix
// and 8 movmatrix (P^T from the S^T accumulator layout into the B-operand
// layout) per 16 KiB block, instead of ~2000 FMA/LDS instructions for G = 4.
// Why not tcgen05: a decode block contracts G <= 8 query heads with 32 tokens;
// tcgen05.mma wants >= 64-row tiles and a TMEM round trip per 32-token softmax
// step on the critical path of a kernel that is HBM/latency-bound at 1-4
// flop/byte, far below any tensor-core ridge.
//
// Staging: 2-D TMA (cp.async.bulk.tensor) with SWIZZLE_128B, so ldmatrix reads
// of 8 token rows (256 B apart in HBM) are bank-conflict-free.  A [2][32][128]
// block is four 32 x 64 boxes (K dims 0-63 | K 64-127 | V 0-63 | V 64-127),
// 4 KiB each; 16-byte chunk j of row r sits at chunk j ^ (r & 7).
//
// Precision: Q and K are exact in bf16 and the HMMA accumulates in f32, as the
// FMA path does; P is split p = hi + lo (both bf16, |p - hi - lo| <= 2^-17 p),
// so P V carries ~2^-17 relative error instead of bf16's 2^-9.
// ============================================================================
// Stages per warp (NS) and warps per CTA (NW) trade pipeline depth against the
// number of warps a pair is split across: NS x NW x 16 KiB stays ~192 KiB per
// CTA (one CTA per SM).  NS = 2, NW = 6 (round 1) splits a C3 pair over ~16
// warps; NS = 4, NW = 3 keeps the same bytes in flight per SM with half the
// warps, so half the partials to merge per pair.
template <int NS>
struct MmaCfg {
    static constexpr int NW = NS == 2 ? 6 : (NS == 3 ? 4 : 3);
};

template <int NS>
struct MmaWarpSmem {
    alignas(1024) unsigned char buf[NS][16384];  // [stage] K-lo | K-hi | V-lo | V-hi
    unsigned char merge_extra[4096];              // with buf: the merge's landing zone (C3, G = 4: 17 partials)
    uint64_t bar[NS][2];                          // [stage][K half / V half]
    uint64_t mbar;                                // end-of-range partial merge (bulk loads)
};

// End-of-range merge (the common case: the last contributor of a cut pair is
// usually the warp whose range ENDS in the pair, so it merges after its last
// unit, with its stage buffers idle).  The contributors' partials -- G heads x
// kAttnPartStride floats each, contiguous -- are pulled into those buffers by
// one bulk copy per contributor (lane i issues contributor i's), all on one
// mbarrier: one round trip per buffer-full of partials (C2: every partial at
// once; C3, G = 4: 15 of ~17), instead of one for (m, l) and one per 8
// contributors' o through registers (merge_partials; ~0.9 us per round trip at
// the end of a launch, r02v).  Rounds combine by the usual rescaling, in warp
// order (deterministic).
template <int G, int NS>
__device__ void merge_partials_bulk(const AttnArgs& a, int64_t p, int w, MmaWarpSmem<NS>& sm, uint32_t& phase) {
    constexpr int kBytes = G * kAttnPartStride * 4;
    constexpr int kCapBuf = (NS * 16384 + 4096) / kBytes;  // buf + merge_extra (contiguous)
    constexpr int kCap = kCapBuf < 32 ? kCapBuf : 32;  // contributors per round (lane-parallel)
    static_assert(kCap >= 1, "a partial must fit the stage buffers");
    const int lane = lane_id();
    const int Ku = a.k + 1;
    const int64_t wf = warp_of_unit(p * Ku, a.U, a.W);
    const int64_t wl = warp_of_unit((p + 1) * Ku - 1, a.U, a.W);
    const int nc = (int)(wl - wf + 1);
    auto trace = [&](int i) {
        if (a.trace != nullptr && lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[(int64_t)w * kTraceSlots + i] = t;
        }
    };
    trace(3);
    const int64_t pkw = p * Ku * (int64_t)a.W;
    unsigned char* dst = &sm.buf[0][0];
    float* P = reinterpret_cast<float*>(dst);
    float M[G], L[G], O[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        M[g] = -INFINITY;
        L[g] = 0.f;
        O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.f;
    }
    for (int r0 = 0; r0 < nc; r0 += kCap) {
        const int n = min(kCap, nc - r0);
        if (lane == 0) {
            // the previous round's shared-memory reads (generic proxy) before
            // this round's async-proxy writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.mbar, (uint32_t)(n * kBytes));
        }
        __syncwarp();
        if (lane < n) {
            const int64_t w2 = wf + r0 + lane;
            const int64_t off = ((w2 * 2 + (a.U * w2 >= pkw ? 0 : 1)) * G) * kAttnPartStride;
            // the partials were written through the generic proxy (acquired by
            // the ticket); order them before this async-proxy read
            asm volatile("fence.proxy.async.global;" ::: "memory");
            bulk_g2s(dst + lane * kBytes, a.part + off, kBytes, &sm.mbar);
        }
        mbar_wait(&sm.mbar, phase);
        phase ^= 1u;
        trace(r0 == 0 ? 7 : 9);
        // (1) lane-parallel over the round's n*G (contributor, head) items --
        // item i = j*G + g sits at P + i*kAttnPartStride, and lane t owns items
        // t, t+32, ..., all of head g = t % G: the head max, the scale factors
        // sc_i = 2^(m_i - M) (kept in the partial's pad word for step 2) and the
        // l sums reduce over the lanes of one head (xor strides >= G).
        // (2) every lane accumulates its 4 dims of o over the items (broadcast
        // loads of sc).  (Measured: one lane walking every item with dependent
        // loads / exp2 spent ~220 cycles per contributor at G = 4, r02ab +
        // tools/merge_probe.cu.)
        const int gl = lane % G;
        float mloc = -INFINITY;
        for (int i = lane; i < n * G; i += 32) mloc = fmaxf(mloc, P[i * kAttnPartStride]);
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) mloc = fmaxf(mloc, __shfl_xor_sync(0xffffffffu, mloc, o));
        float Mg = M[0];
#pragma unroll
        for (int g = 1; g < G; ++g)
            if (gl == g) Mg = M[g];
        const float mnew = fmaxf(Mg, mloc);
        const float corr_l = Mg == -INFINITY ? 0.f : exp2f(Mg - mnew);
        float lloc = 0.f;
        for (int i = lane; i < n * G; i += 32) {
            float* pi = P + i * kAttnPartStride;
            const float sc = mnew == -INFINITY ? 0.f : exp2f(pi[0] - mnew);
            lloc = fmaf(pi[1], sc, lloc);
            pi[2] = sc;
        }
#pragma unroll
        for (int o = 16; o >= G; o >>= 1) lloc += __shfl_xor_sync(0xffffffffu, lloc, o);
        __syncwarp();
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float cg = __shfl_sync(0xffffffffu, corr_l, g);
            L[g] = fmaf(L[g], cg, __shfl_sync(0xffffffffu, lloc, g));
            M[g] = __shfl_sync(0xffffffffu, mnew, g);
            O[g][0] *= cg, O[g][1] *= cg, O[g][2] *= cg, O[g][3] *= cg;
        }
#pragma unroll 4
        for (int j = 0; j < n; ++j) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float* pj = P + (j * G + g) * kAttnPartStride;
                const float sc = pj[2];
                const float4 ov = *reinterpret_cast<const float4*>(pj + 4 + 4 * lane);
                O[g][0] = fmaf(ov.x, sc, O[g][0]);
                O[g][1] = fmaf(ov.y, sc, O[g][1]);
                O[g][2] = fmaf(ov.z, sc, O[g][2]);
                O[g][3] = fmaf(ov.w, sc, O[g][3]);
            }
        }
        __syncwarp();
        trace(r0 == 0 ? 8 : 10);
    }
    const int b = (int)(p / a.Hkv), h = (int)(p % a.Hkv);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float inv = L[g] > 0.f ? __frcp_rn(L[g]) : 0.f;  // == 1.f / L (IEEE), no division subroutine
        const int hq = h * G + g;
        if (a.lse != nullptr && lane == 0)
            a.lse[(int64_t)hq * a.B + b] = L[g] > 0.f ? M[g] + log2f(L[g]) : -INFINITY;
        *reinterpret_cast<float4*>(a.out + ((int64_t)hq * a.B + b) * kHeadDim + 4 * lane) =
            make_float4(O[g][0] * inv, O[g][1] * inv, O[g][2] * inv, O[g][3] * inv);
    }
    trace(4);
    if (lane == 0) a.tickets[p] = 0;
}

// Per-stage unit descriptors kept in registers: a runtime stage index selects
// among statically indexed scalars (no local-memory array).
template <int NS>
struct StageRegs {
    int kind[NS], row[NS], pair[NS];
    __device__ __forceinline__ int get(const int (&a)[NS], int s) const {
        int v = a[0];
#pragma unroll
        for (int i = 1; i < NS; ++i)
            if (s == i) v = a[i];
        return v;
    }
    __device__ __forceinline__ void set(int (&a)[NS], int s, int v) {
#pragma unroll
        for (int i = 0; i < NS; ++i)
            if (s == i) a[i] = v;
    }
};

__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* tm, int x, int y,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// 8x8 b16 transpose across the warp (fragment layout in and out)
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
    uint32_t y;
    asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}
__device__ __forceinline__ uint32_t bf16x2_bits(__nv_bfloat162 v) {
    return *reinterpret_cast<uint32_t*>(&v);
}

template <int G, int NS>
__global__ void __launch_bounds__(MmaCfg<NS>::NW * 32, 1)
sparse_attn_mma_kernel(const AttnArgs a, const __grid_constant__ CUtensorMap tm_pool,
                       const __grid_constant__ CUtensorMap tm_tail) {
    if (a.counts != nullptr && a.counts[3] != 0) return;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    MmaWarpSmem<NS>& sm = reinterpret_cast<MmaWarpSmem<NS>*>(base)[warp_id()];
    const int lane = lane_id();
    const int w = warp_id() * gridDim.x + blockIdx.x;
    if (w >= a.W) return;
    const int64_t u0 = a.U * w / a.W, u1 = a.U * (w + 1) / a.W;
    const int Ku = a.k + 1;
    const int r = lane >> 2, c = lane & 3;  // fragment row group / column pair
    auto trace = [&](int i) {
        if (a.trace != nullptr && lane == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            a.trace[(int64_t)w * kTraceSlots + i] = t;
        }
    };
    trace(0);

    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < NS; ++st) {
            mbar_init(&sm.bar[st][0], 1);
            mbar_init(&sm.bar[st][1], 1);
        }
        mbar_init(&sm.mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_pool)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm_tail)) : "memory");
    }
    __syncwarp();

    // ---- producer: the warp's unit descriptors, 32 at a time, lane-parallel.
    // Lane l holds unit wbase + l: kind (0 skip, 1 pool slot, 2 tail), the
    // tensor-map row of its K, and its pair -- one division per lane per 32
    // units; the consumer never divides.
    int64_t wbase = u0;
    int wkind = 0, wrow = 0, wpair = 0;
    auto refill = [&]() {
        const int64_t u = wbase + lane;
        wkind = 0;
        if (u < u1) {
            const int64_t p = u / Ku;
            const int rr = (int)(u - p * Ku);
            wpair = (int)p;
            if (rr < a.k) {
                int32_t sl = __ldg(a.slot + p * a.k + rr);
                if (a.mode != 0 && ((__ldg(a.hit + p * a.k + rr) != 0) != (a.mode == 1))) sl = -1;
                wkind = sl >= 0 ? 1 : 0;
                wrow = sl * 64;
            } else {
                wkind = (a.mode != 2 && __ldg(a.tail_len + p / a.Hkv) > 0) ? 2 : 0;
                wrow = (int)p * 64;
            }
        }
    };
    refill();
    int next_l = 0;   // next lane of the window to consider
    int q_pref_pair = -1;  // pair whose q was last prefetched
    // unit held by each stage: kind (0 = none), K row in the tensor map, pair (-1 = none)
    StageRegs<NS> sr;
#pragma unroll
    for (int st = 0; st < NS; ++st) sr.kind[st] = 0, sr.row[st] = 0, sr.pair[st] = -1;
    auto issue_half = [&](int stage, int half) {
        const int kind = sr.get(sr.kind, stage);
        if (lane == 0 && kind != 0) {
            const CUtensorMap* tm = kind == 1 ? &tm_pool : &tm_tail;
            const int row = sr.get(sr.row, stage) + 32 * half;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&sm.bar[stage][half], 8192);
            const uint32_t dst = smem_u32(sm.buf[stage]) + half * 8192;
            tma_2d(dst, tm, 0, row, &sm.bar[stage][half]);
            tma_2d(dst + 4096, tm, 64, row, &sm.bar[stage][half]);
        }
    };
    auto issue_k = [&](int stage) {
        while (true) {
            const unsigned m = __ballot_sync(0xffffffffu, wkind != 0 && lane >= next_l);
            if (m) {
                const int l = __ffs(m) - 1;
                next_l = l + 1;
                sr.set(sr.kind, stage, __shfl_sync(0xffffffffu, wkind, l));
                sr.set(sr.row, stage, __shfl_sync(0xffffffffu, wrow, l));
                const int np = __shfl_sync(0xffffffffu, wpair, l);
                sr.set(sr.pair, stage, np);
                issue_half(stage, 0);
                if (np != q_pref_pair) {
                    // a new pair: its q (G x 256 B) into L1 now, so the q loads at
                    // its start hit instead of stalling the warp ~1 us
                    q_pref_pair = np;
                    if (lane < 2 * G)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)a.q +
                            ((int64_t)(np / a.Hkv) * a.Hq + (int64_t)(np % a.Hkv) * G) * kHeadDim * 2 + lane * 128));
                }
                return;
            }
            if (wbase + 32 >= u1) {
                next_l = 32;
                sr.set(sr.kind, stage, 0);
                sr.set(sr.pair, stage, -1);
                return;
            }
            wbase += 32;
            next_l = 0;
            refill();
        }
    };
#pragma unroll
    for (int st = 0; st < NS; ++st) {
        issue_k(st);
        issue_half(st, 1);
    }
    uint32_t phases = 0u;
    int stage = 0;

    // per-lane ldmatrix addressing: matrix mi = lane / 8, row rr = lane % 8
    const int mi = lane >> 3, rr = lane & 7;
    // QK, A = K[token][dim] (non-transposed): matrices {tok 0-7, 8-15, 0-7, 8-15}
    // x {dims lo 8, lo, hi 8, hi} of a 16-token x 16-dim tile
    const uint32_t k_off = (uint32_t)((8 * (mi & 1) + rr) * 128);
    const uint32_t k_hi = (uint32_t)(mi >> 1);
    // PV, A = V^T (transposed load of V[token][dim]): matrices {dims lo, hi, lo,
    // hi} x {tok 0-7, 0-7, 8-15, 8-15}
    const uint32_t v_off = (uint32_t)((8 * (mi >> 1) + rr) * 128);
    const uint32_t v_hi = (uint32_t)(mi & 1);

    const int64_t p_first = u0 / Ku, p_last = (u1 - 1) / Ku;
    for (int64_t p = p_first; p <= p_last; ++p) {
        const int b = (int)(p / a.Hkv), h = (int)(p % a.Hkv);
        // Q^T fragment (B operand): k-step s holds head r's dims 16s+2c, +1 (b0)
        // and 16s+8+2c, +1 (b1); heads r >= G are zero columns
        uint32_t qb[8][2];
        {
            const uint32_t* qp = reinterpret_cast<const uint32_t*>(
                (const uint16_t*)a.q + ((int64_t)b * a.Hq + (int64_t)h * G + (r < G ? r : 0)) * kHeadDim);
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                qb[s][0] = r < G ? __ldg(qp + 8 * s + c) : 0u;
                qb[s][1] = r < G ? __ldg(qp + 8 * s + 4 + c) : 0u;
            }
        }
        // running max / sum of heads 2c, 2c+1; O^T tile md: rows dims 16md + r
        // (+8), columns heads 2c, 2c+1
        float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
        float o[8][4];
#pragma unroll
        for (int md = 0; md < 8; ++md) o[md][0] = o[md][1] = o[md][2] = o[md][3] = 0.f;
        const int tl = __ldg(a.tail_len + b);

        while (sr.get(sr.pair, stage) == (int)p) {
            const bool is_tail = sr.get(sr.kind, stage) == 2;
            mbar_wait(&sm.bar[stage][0], (phases >> (2 * stage)) & 1u);
            phases ^= 1u << (2 * stage);
            const uint32_t kb = smem_u32(sm.buf[stage]);
            // ---- S^T = K Q^T: m-tile mt = tokens 16mt..16mt+15; two partial
            // accumulators per tile (dims 0-63 / 64-127) halve the HMMA chains ----
            float sa[2][2][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) sa[mt][hh][0] = sa[mt][hh][1] = sa[mt][hh][2] = sa[mt][hh][3] = 0.f;
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const uint32_t chunk = (uint32_t)(2 * (s & 3)) + k_hi;
                const uint32_t col = ((chunk ^ (uint32_t)rr) << 4) + (uint32_t)(s >> 2) * 4096u;
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) {
                    uint32_t ka[4];
                    ldsm_x4(kb + col + mt * 2048 + k_off, ka);
                    hmma(sa[mt][s >> 2], ka, qb[s][0], qb[s][1]);
                }
            }
            // lane holds S^T at tokens t(mt, e2) = 16mt + 8*e2 + r, heads 2c + e
            float z[2][2][2];  // [mt][e2][e]
            float rmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const bool valid = !is_tail || (16 * mt + 8 * e2 + r) < tl;
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const float sv = sa[mt][0][2 * e2 + e] + sa[mt][1][2 * e2 + e];
                        z[mt][e2][e] = valid ? sv * a.scale_log2 : -INFINITY;
                        rmax[e] = fmaxf(rmax[e], z[mt][e2][e]);
                    }
                }
            // reduce over the 8 row groups (lane bits 2..4)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                rmax[e] = fmaxf(rmax[e], __shfl_xor_sync(0xffffffffu, rmax[e], 4));
                rmax[e] = fmaxf(rmax[e], __shfl_xor_sync(0xffffffffu, rmax[e], 8));
                rmax[e] = fmaxf(rmax[e], __shfl_xor_sync(0xffffffffu, rmax[e], 16));
            }
            float corr[2], rsum[2] = {0.f, 0.f};
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const float mnew = fmaxf(m[e], rmax[e]);
                corr[e] = exp2f(m[e] - mnew);
                m[e] = mnew;
            }
            // P^T as the PV B operand: k-step ks = tokens 16ks..16ks+15; b0 =
            // tokens 16ks+2c, +1 of head r, b1 = tokens 16ks+8+2c, +1.  The
            // accumulator layout holds (token r-row, head pair) -> movmatrix.
            uint32_t pbh[2][2], pbl[2][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int e2 = 0; e2 < 2; ++e2) {
                    const float p0 = exp2f(z[mt][e2][0] - m[0]);
                    const float p1 = exp2f(z[mt][e2][1] - m[1]);
                    rsum[0] += p0;
                    rsum[1] += p1;
                    const __nv_bfloat162 hi = __floats2bfloat162_rn(p0, p1);
                    const float2 hf = __bfloat1622float2(hi);
                    const __nv_bfloat162 lo = __floats2bfloat162_rn(p0 - hf.x, p1 - hf.y);
                    pbh[mt][e2] = movm_t(bf16x2_bits(hi));
                    pbl[mt][e2] = movm_t(bf16x2_bits(lo));
                }
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                rsum[e] += __shfl_xor_sync(0xffffffffu, rsum[e], 4);
                rsum[e] += __shfl_xor_sync(0xffffffffu, rsum[e], 8);
                rsum[e] += __shfl_xor_sync(0xffffffffu, rsum[e], 16);
                l[e] = l[e] * corr[e] + rsum[e];
            }
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                o[md][0] *= corr[0];
                o[md][1] *= corr[1];
                o[md][2] *= corr[0];
                o[md][3] *= corr[1];
            }
            __syncwarp();
            issue_k(stage);  // K half consumed: next unit's K into this stage
            mbar_wait(&sm.bar[stage][1], (phases >> (2 * stage + 1)) & 1u);
            phases ^= 1u << (2 * stage + 1);
            const uint32_t vb = kb + 8192;
            if (is_tail && tl < kBlockTokens) {
                // rows >= tl of a tail may hold anything (0 * NaN = NaN): zero them
                unsigned char* vp = sm.buf[stage] + 8192;
                for (int i = lane; i < 2 * kBlockTokens * 8; i += 32) {
                    const int half = i / (kBlockTokens * 8), row = (i / 8) % kBlockTokens;
                    if (row >= tl)
                        *reinterpret_cast<uint4*>(vp + half * 4096 + row * 128 + (i % 8) * 16) =
                            make_uint4(0, 0, 0, 0);
                }
                __syncwarp();
            }
            // ---- O^T += V^T P^T: m-tile md = dims 16md..16md+15 ----
#pragma unroll
            for (int md = 0; md < 8; ++md) {
                const uint32_t chunk = (uint32_t)(2 * (md & 3)) + v_hi;
                const uint32_t col = ((chunk ^ (uint32_t)rr) << 4) + (uint32_t)(md >> 2) * 4096u;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    uint32_t va[4];
                    ldsm_x4_t(vb + col + ks * 2048 + v_off, va);
                    hmma(o[md], va, pbh[ks][0], pbh[ks][1]);
                    hmma(o[md], va, pbl[ks][0], pbl[ks][1]);
                }
            }
            __syncwarp();
            issue_half(stage, 1);  // V half of this stage's next unit
            stage = stage + 1 == NS ? 0 : stage + 1;
        }

        // ---- flush pair p: lane holds heads 2c + e, dims 16md + r (+8) ----
        if (p == p_last) trace(1);
        const bool full = (p * Ku >= u0) && ((p + 1) * Ku <= u1);
        if (full) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                if (2 * c + e < G) {
                    const float inv = l[e] > 0.f ? __frcp_rn(l[e]) : 0.f;
                    float* op = a.out + ((int64_t)(h * G + 2 * c + e) * a.B + b) * kHeadDim + r;
                    if (a.lse != nullptr && r == 0)
                        a.lse[(int64_t)(h * G + 2 * c + e) * a.B + b] = l[e] > 0.f ? m[e] + log2f(l[e]) : -INFINITY;
#pragma unroll
                    for (int md = 0; md < 8; ++md) {
                        op[16 * md] = o[md][e] * inv;
                        op[16 * md + 8] = o[md][2 + e] * inv;
                    }
                }
            }
            continue;
        }
        const int seg = (p == p_first) ? 0 : 1;
        unsigned long long t_flush = 0;
        if (a.trace != nullptr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_flush));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (2 * c + e < G) {
                float* pp = a.part + (((int64_t)w * 2 + seg) * G + 2 * c + e) * kAttnPartStride;
                if (r == 0) {
                    pp[0] = m[e];
                    pp[1] = l[e];
                }
#pragma unroll
                for (int md = 0; md < 8; ++md) {
                    pp[4 + 16 * md + r] = o[md][e];
                    pp[4 + 16 * md + 8 + r] = o[md][2 + e];
                }
            }
        }
        // the last contributor merges: mid-range through registers (units still
        // in flight in the stages), at the range end through bulk loads into the
        // idle stage buffers.  (Measured: deferring a mid-range cut pair's ticket
        // to the range end shortened the stragglers' streaming but made some
        // warps last for two pairs -- two serial merges in the tail, r02z.)
        if (partial_is_last(a, p)) {
            if (a.trace != nullptr && lane == 0) a.trace[(int64_t)w * kTraceSlots + 5] = t_flush;
            trace(6);
            uint32_t mphase = 0;
            if (p == p_last && knob_attn_merge_bulk(a))
                merge_partials_bulk<G, NS>(a, p, w, sm, mphase);
            else
                merge_partials<G, (G >= 8 ? 4 : 8)>(a, p, w);  // contributors' loads per batch (C3, G = 4: 8 measured better than 4)
        }
    }
    trace(2);
}

template <bool BF16, int G>
static size_t attn_smem_bytes() {
    return sizeof(WarpSmem<BF16, G>) * AttnTraits<BF16>::NW;
}

static int attn_total_warps(ss_dtype dt) {
    return num_sms() * (dt == SS_BF16 ? AttnTraits<true>::NW : AttnTraits<false>::NW);
}

static bool attn_trace_on() {
    return knob("SS_ATTN_TRACE", 0) != 0;
}

static size_t attn_ws_bytes_core(const ss_dims& d, ss_dtype dt) {
    int G = d.num_q_heads / d.num_kv_heads;
    size_t W = attn_total_warps(dt);
    size_t part = W * 2 * G * kAttnPartStride * 4;
    size_t pairs = (size_t)d.batch * d.num_kv_heads;
    return ((part + pairs * 4) + 255) & ~(size_t)255;
}

size_t attn_ws_bytes(const ss_dims& d, int k, ss_dtype dt) {
    // + debug timeline (kTraceSlots x u64 per warp) after the core workspace when traced
    return attn_ws_bytes_core(d, dt) + (attn_trace_on() ? (size_t)attn_total_warps(dt) * kTraceSlots * 8 : 0);
}

// [rows][128] bf16 view of a KV array (row = one token's K or V vector of a
// head-block; block b = rows 64b .. 64b+63), 32 x 64 boxes, 128-byte swizzle.
static bool encode_kv_map(CUtensorMap* m, const void* base, uint64_t rows) {
    auto enc = tensor_map_encoder();
    if (enc == nullptr) return false;
    const cuuint64_t gdim[2] = {(cuuint64_t)kHeadDim, (cuuint64_t)rows};
    const cuuint64_t gstride[1] = {(cuuint64_t)kHeadDim * 2};
    const cuuint32_t box[2] = {64, (cuuint32_t)kBlockTokens};
    const cuuint32_t estride[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box,
               estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int NS>
constexpr size_t mma_smem() {  // + base alignment slack
    return sizeof(MmaWarpSmem<NS>) * MmaCfg<NS>::NW + 1024;
}
// (+ 1 KiB static shared memory) within the 227 KiB a CTA may use on sm_100
static_assert(mma_smem<2>() + 1024 <= 232448 && mma_smem<3>() + 1024 <= 232448 && mma_smem<4>() + 1024 <= 232448,
              "attention CTA exceeds the shared-memory limit");
constexpr int kAttnStages = 2;  // default stages per warp (NS); SS_ATTN_STAGES=3|4 (debug A/B)

static int mma_stages() {
    const int ns = knob("SS_ATTN_STAGES", kAttnStages);
    return (ns == 3 || ns == 4) ? ns : 2;
}
static int mma_nw(int ns) { return ns == 2 ? MmaCfg<2>::NW : ns == 3 ? MmaCfg<3>::NW : MmaCfg<4>::NW; }

template <int G, int NS>
static ss_status launch_attn_mma_t(const AttnArgs& a, const void* pool, const void* tail,
                                   cudaStream_t stream) {
    CUtensorMap tm_pool, tm_tail;
    // the pool's slot count is not part of the call: its map spans the whole
    // int32 row range (TMA reads only the boxes requested = valid slots)
    if (!encode_kv_map(&tm_pool, pool, (uint64_t)INT32_MAX) ||
        !encode_kv_map(&tm_tail, tail, (uint64_t)a.B * a.Hkv * 2 * kBlockTokens))
        return SS_ERR_CUDA;
    auto kern = sparse_attn_mma_kernel<G, NS>;
    constexpr int NW = MmaCfg<NS>::NW;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mma_smem<NS>()) !=
        cudaSuccess)
        return SS_ERR_CUDA;
    // persistent NW-warp CTAs, one per SM (default).  SS_ATTN_CTA_WARPS=1
    // launches one-warp CTAs instead (each warp's stages its own CTA,
    // dispatched into whatever SM space co-running kernels leave); warps never
    // synchronise, so the kernel is the same (warp w = warp_id * gridDim + CTA).
    // Measured (NS = 2): 0.89 vs 0.85 of HBM peak alone at C2, no in-step difference.
    set_carveout(kern);
    const int cta_warps = knob("SS_ATTN_CTA_WARPS", NW);
    if (cta_warps == NW)
        kern<<<num_sms(), NW * 32, mma_smem<NS>(), stream>>>(a, tm_pool, tm_tail);
    else
        kern<<<a.W, 32, sizeof(MmaWarpSmem<NS>) + 1024, stream>>>(a, tm_pool, tm_tail);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

template <bool BF16, int G>
static ss_status launch_attn_t(AttnArgs a, cudaStream_t stream) {
    auto kern = sparse_attn_kernel<BF16, G>;
    size_t smem = attn_smem_bytes<BF16, G>();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return SS_ERR_CUDA;
    set_carveout(kern);
    kern<<<num_sms(), AttnTraits<BF16>::NW * 32, smem, stream>>>(a);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

// Split-form merge: out = (O_a 2^lse_a + O_b 2^lse_b) / (2^lse_a + 2^lse_b) per
// (hq, b) row (the standard log-sum-exp combination of two disjoint token sets'
// softmax-normalised outputs); both empty -> 0.  One warp per row.
__global__ void __launch_bounds__(256) attn_merge_kernel(const float* __restrict__ oa,
                                                         const float* __restrict__ la,
                                                         const float* __restrict__ ob,
                                                         const float* __restrict__ lb, int64_t rows,
                                                         const int32_t* counts, float* __restrict__ out) {
    if (counts != nullptr && counts[3] != 0) return;
    const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (row >= rows) return;
    const int lane = lane_id();
    const float xa = la[row], xb = lb[row];
    const float mx = fmaxf(xa, xb);
    float wa = 0.f, wb = 0.f;
    if (mx != -INFINITY) {
        wa = exp2f(xa - mx);
        wb = exp2f(xb - mx);
    }
    const float inv = (wa + wb) > 0.f ? 1.f / (wa + wb) : 0.f;
    const float4 va = reinterpret_cast<const float4*>(oa + row * kHeadDim)[lane];
    const float4 vb = reinterpret_cast<const float4*>(ob + row * kHeadDim)[lane];
    float4 r;
    r.x = (va.x * wa + vb.x * wb) * inv;
    r.y = (va.y * wa + vb.y * wb) * inv;
    r.z = (va.z * wa + vb.z * wb) * inv;
    r.w = (va.w * wa + vb.w * wb) * inv;
    reinterpret_cast<float4*>(out + row * kHeadDim)[lane] = r;
}

ss_status launch_attn_merge(const float* oa, const float* la, const float* ob, const float* lb,
                            int64_t rows, const int32_t* counts, float* out, cudaStream_t stream) {
    if (rows <= 0) return SS_OK;
    const int64_t threads = rows * 32;
    attn_merge_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(oa, la, ob, lb, rows, counts, out);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_sparse_attn(const void* q, const void* pool_kv, const int32_t* slot, int k,
                             const void* tail_kv, const int32_t* tail_len, const ss_dims& d,
                             ss_dtype dt, float scale, const int32_t* counts, float* out, void* ws,
                             cudaStream_t stream, const uint8_t* hit, int mode, float* lse) {
    AttnArgs a;
    a.hit = hit;
    a.mode = mode;
    a.lse = lse;
    a.q = q;
    a.pool = pool_kv;
    a.slot = slot;
    a.tail = tail_kv;
    a.tail_len = tail_len;
    a.counts = counts;
    a.out = out;
    a.k = k;
    a.B = d.batch;
    a.Hq = d.num_q_heads;
    a.Hkv = d.num_kv_heads;
    a.scale_log2 = scale * 1.4426950408889634f;
    const int G = d.num_q_heads / d.num_kv_heads;
    a.U = (int64_t)d.batch * d.num_kv_heads * (k + 1);
    a.merge_bulk = knob("SS_ATTN_MERGE_BULK", 1);
    // at least kMinUnitsPerWarpGqa / Mha units (16 KiB each in bf16) per warp: fewer, longer
    // ranges when the problem is small (C3: ~16 partials per pair to merge instead
    // of ~28); W <= U keeps every range non-empty
    const int min_units_dflt =
        G == 1 ? kMinUnitsPerWarpMha
               : (a.U >= (int64_t)num_sms() * 6 * kMinUnitsPerWarpGqaSmall ? kMinUnitsPerWarpGqa : kMinUnitsPerWarpGqaSmall);
    const int min_units = knob("SS_ATTN_MIN_UNITS", min_units_dflt);
    // bf16 tensor-core path (SS_ATTN_MMA=0 selects the CUDA-core FMA path)
    const int use_mma = knob("SS_ATTN_MMA", 1);
    const int ns = mma_stages();
    const int total_warps = (dt == SS_BF16 && use_mma) ? num_sms() * mma_nw(ns) : attn_total_warps(dt);
    a.W = (int)std::max<int64_t>(1, std::min<int64_t>(total_warps, a.U / std::max(1, min_units)));
    size_t part = (size_t)a.W * 2 * G * kAttnPartStride * 4;
    a.part = (float*)ws;
    a.tickets = (int32_t*)((char*)ws + part);
    a.trace = attn_trace_on() ? (unsigned long long*)((char*)ws + attn_ws_bytes_core(d, dt)) : nullptr;
#define SS_ATTN_CASE(GG)                                                                    \
    case GG:                                                                                \
        if (dt == SS_BF16 && use_mma)                                                      \
            return ns == 4 ? launch_attn_mma_t<GG, 4>(a, pool_kv, tail_kv, stream)        \
                 : ns == 3 ? launch_attn_mma_t<GG, 3>(a, pool_kv, tail_kv, stream)        \
                           : launch_attn_mma_t<GG, 2>(a, pool_kv, tail_kv, stream);       \
        return dt == SS_BF16 ? launch_attn_t<true, GG>(a, stream) : launch_attn_t<false, GG>(a, stream);
    switch (G) {
        SS_ATTN_CASE(1)
        SS_ATTN_CASE(2)
        SS_ATTN_CASE(4)
        SS_ATTN_CASE(8)
        default:
            return SS_ERR_UNSUPPORTED;
    }
#undef SS_ATTN_CASE
}

bool preload_attn() {
    bool ok = preload_fn(attn_merge_kernel);
#define SS_PL(GG)                                              \
    ok &= preload_fn(sparse_attn_mma_kernel<GG, 2>);          \
    ok &= preload_fn(sparse_attn_mma_kernel<GG, 3>);          \
    ok &= preload_fn(sparse_attn_mma_kernel<GG, 4>);          \
    ok &= preload_fn(sparse_attn_kernel<true, GG>);           \
    ok &= preload_fn(sparse_attn_kernel<false, GG>);
    SS_PL(1) SS_PL(2) SS_PL(4) SS_PL(8)
#undef SS_PL
    return ok;
}

}  // namespace ss
