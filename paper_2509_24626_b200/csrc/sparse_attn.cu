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
// Per block, lane t computes token t's logits for the G query heads of the KV
// head (K row read with a lane-rotated chunk order: conflict-free 16-byte
// shared loads), an online softmax in exp2 domain, and lane l accumulates
// output dims 4l..4l+3 from the V rows.  float32 CUDA-core math: at 1 (MHA) to
// 4 (GQA G=4) flop per HBM byte the kernel is far below the tensor-core ridge
// and fp32 keeps the 2e-3 / 1e-5 tolerances with margin.
//
// Roofline: HBM-bound; algorithmic bytes = block_bytes per attended unit
// (+ q, out: negligible).
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"

namespace ss {

constexpr int kAttnPartStride = 132;
constexpr int kMinUnitsPerWarp = 16;  // floats per (warp, seg, g) partial: m, l, pad, pad, o[128]

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
    int64_t U;  // pairs * (k + 1)
    int W;      // total warps
    int l2pf;   // L2 prefetch of the following unit
};

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
                const int32_t sl = __ldg(a.slot + p * a.k + r);
                wkind = sl >= 0 ? 1 : 0;
                widx = sl;
            } else {
                wkind = __ldg(a.tail_len + p / a.Hkv) > 0 ? 2 : 0;
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
                const float inv = l[g] > 0.f ? 1.f / l[g] : 0.f;
                const int hq = h * G + g;
                *reinterpret_cast<float4*>(a.out + ((int64_t)hq * a.B + b) * kHeadDim + 4 * lane) =
                    make_float4(o[g][0] * inv, o[g][1] * inv, o[g][2] * inv, o[g][3] * inv);
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
        __threadfence();
        __syncwarp();
        int ticket = 0;
        if (lane == 0) ticket = atomicAdd(&a.tickets[p], 1);
        ticket = __shfl_sync(0xffffffffu, ticket, 0);
        const int64_t wf = warp_of_unit(p * Ku, a.U, a.W);
        const int64_t wl = warp_of_unit((p + 1) * Ku - 1, a.U, a.W);
        if (ticket != (int)(wl - wf)) continue;
        __threadfence();
        // merge the contributors' partials in warp order (deterministic): the
        // (m, l) of all (contributor, head) pairs are read lane-parallel, then
        // every head's o with independent loads (all heads in one pass)
        const int nc = (int)(wl - wf + 1);
        float mt[G], lt[G], oo[G][4];
#pragma unroll
        for (int g = 0; g < G; ++g) {
            mt[g] = -INFINITY;
            lt[g] = 0.f;
            oo[g][0] = oo[g][1] = oo[g][2] = oo[g][3] = 0.f;
        }
        auto part_of = [&](int i, int g) -> const float* {
            const int64_t w2 = wf + i;
            const int s2 = ((a.U * w2 / a.W) / Ku == p) ? 0 : 1;
            return a.part + ((w2 * 2 + s2) * G + g) * kAttnPartStride;
        };
        for (int i = lane; i < nc; i += 32) {
#pragma unroll
            for (int g = 0; g < G; ++g) mt[g] = fmaxf(mt[g], __ldcg(part_of(i, g)));
        }
#pragma unroll
        for (int g = 0; g < G; ++g) mt[g] = warp_max(mt[g]);
        for (int i = lane; i < nc; i += 32) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float* pp = part_of(i, g);
                if (mt[g] != -INFINITY) lt[g] += __ldcg(pp + 1) * exp2f(__ldcg(pp) - mt[g]);
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) lt[g] = warp_sum(lt[g]);
#pragma unroll 2
        for (int i = 0; i < nc; ++i) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                if (mt[g] == -INFINITY) continue;
                const float* pp = part_of(i, g);
                const float sc = exp2f(__ldcg(pp) - mt[g]);
                const float4 ov = __ldcg(reinterpret_cast<const float4*>(pp + 4 + 4 * lane));
                oo[g][0] = fmaf(ov.x, sc, oo[g][0]);
                oo[g][1] = fmaf(ov.y, sc, oo[g][1]);
                oo[g][2] = fmaf(ov.z, sc, oo[g][2]);
                oo[g][3] = fmaf(ov.w, sc, oo[g][3]);
            }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
            const float inv = lt[g] > 0.f ? 1.f / lt[g] : 0.f;
            const int hq = h * G + g;
            *reinterpret_cast<float4*>(a.out + ((int64_t)hq * a.B + b) * kHeadDim + 4 * lane) =
                make_float4(oo[g][0] * inv, oo[g][1] * inv, oo[g][2] * inv, oo[g][3] * inv);
        }
        if (lane == 0) a.tickets[p] = 0;
    }
}

template <bool BF16, int G>
static size_t attn_smem_bytes() {
    return sizeof(WarpSmem<BF16, G>) * AttnTraits<BF16>::NW;
}

static int attn_total_warps(ss_dtype dt) {
    return kNumSMs * (dt == SS_BF16 ? AttnTraits<true>::NW : AttnTraits<false>::NW);
}

size_t attn_ws_bytes(const ss_dims& d, int k, ss_dtype dt) {
    int G = d.num_q_heads / d.num_kv_heads;
    size_t W = attn_total_warps(dt);
    size_t part = W * 2 * G * kAttnPartStride * 4;
    size_t pairs = (size_t)d.batch * d.num_kv_heads;
    return ((part + pairs * 4) + 255) & ~(size_t)255;
}

template <bool BF16, int G>
static ss_status launch_attn_t(AttnArgs a, cudaStream_t stream) {
    auto kern = sparse_attn_kernel<BF16, G>;
    size_t smem = attn_smem_bytes<BF16, G>();
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return SS_ERR_CUDA;
    kern<<<kNumSMs, AttnTraits<BF16>::NW * 32, smem, stream>>>(a);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_sparse_attn(const void* q, const void* pool_kv, const int32_t* slot, int k,
                             const void* tail_kv, const int32_t* tail_len, const ss_dims& d,
                             ss_dtype dt, float scale, const int32_t* counts, float* out, void* ws,
                             cudaStream_t stream) {
    AttnArgs a;
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
    static const int l2pf = getenv("SS_ATTN_L2PF") ? atoi(getenv("SS_ATTN_L2PF")) : 0;  // measured slower
    a.l2pf = l2pf;
    // at least kMinUnitsPerWarp units (256 KiB in bf16) per warp: fewer, longer
    // ranges when the problem is small (C3: ~8 partials per pair to merge instead
    // of ~28); W <= U keeps every range non-empty
    static const int min_units = getenv("SS_ATTN_MIN_UNITS") ? atoi(getenv("SS_ATTN_MIN_UNITS"))
                                                              : kMinUnitsPerWarp;
    a.W = (int)std::max<int64_t>(1, std::min<int64_t>(attn_total_warps(dt), a.U / std::max(1, min_units)));
    size_t part = (size_t)a.W * 2 * G * kAttnPartStride * 4;
    a.part = (float*)ws;
    a.tickets = (int32_t*)((char*)ws + part);
#define SS_ATTN_CASE(GG)                                                                    \
    case GG:                                                                                \
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

}  // namespace ss
