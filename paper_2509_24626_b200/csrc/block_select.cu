// block_select.cu -- S1 block scoring + S2 top-k ("DSAs compute
// dot products between the metadata vectors and the query token to obtain
// approximate attention scores for all KV blocks.  DSAs then select the top-k
// most critical KV blocks"; readings R2-R6 in DESIGN.md).
//
// Score (must be bit-identical to oracle/oracle.c or_block_score):
//   S(j) = max_g  sum_{c=0..127} max(q_{g,c} * M_{j,c}, q_{g,c} * m_{j,c})
// in float64, summed sequentially c = 0..127 from +0.0, then +0.0.
//
// Exactness argument.  A bf16 (or f32) metadata element X converts EXACTLY to
// float64 (F2F), q*X is exact in float64 (<= 48 significant bits), and one
// DFMA rounds (acc + q*X) once -- the same rounding as the oracle's
// `acc = acc + max(q*M, q*m)` with its exact product.  G == 1: the sign of q
// is warp-uniform per channel, so a per-channel LOP3 mask picks M (q >= 0) or
// m (q < 0) from the two bf16 words before the convert: one select, one F2F,
// one DFMA per channel.  G > 1: min and max are converted once per channel and
// each head adds q+ * M then q- * m (q+ = max(q,0), q- = min(q,0)); the extra
// term is an exact +-0 and leaves acc unchanged (acc is never -0).
//
// Work decomposition.  One CTA per (pair, chunk) work item; a CTA scores
// CH = 1024 blocks (SS_SEL_CHUNK) of one (b, h) pair.  Warp w owns metadata tiles w, w+8, ...; lane r of a warp owns
// block r of the tile, so every 16-byte chunk load of the warp is one
// contiguous 512-byte segment of the tiled layout (fully coalesced, streaming,
// no L1 allocation).  Scores become order-preserving 64-bit keys in shared
// memory; a CTA-wide radix select (8-bit digits, MSB first) finds the k-th
// largest key, ties broken by lower block index, and the chosen blocks are
// compacted in ascending order.  With more than one chunk per pair, chunk
// candidates go to the workspace and the LAST CTA of the pair (atomic ticket,
// self-resetting) merges them with the same select.  The global top-k is always
// inside the union of per-chunk top-k sets, so the result is exact.
//
// Roofline: HBM-bound on the metadata stream: 512 B per block per (b, h) in
// bf16 (1 KiB f32); fp64 work = 2*G*128 DFMA per block.
#include <stdlib.h>

#include <algorithm>

#include <cooperative_groups.h>

#include "common.cuh"

namespace ss {

constexpr int kSelThreads = 256;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kSelChunkMax = 4096;  // blocks per CTA (upper bound; smem sizing)
constexpr int kSelChunkGqa = 2048;  // measured best at C3 (tools/kbench.py)
constexpr int kSelChunkDefault = 1024;  // measured best at C2 (tools/kbench.py)
constexpr int kSelMaxMerge = 8192;

struct SelSmemLayout {
    // G > 1: qpn[c*G + g] = (q+, q-); G == 1: q (f64) [128] + masks [128]
    static size_t bytes(int G, int nkeys) {
        return (size_t)kHeadDim * G * 16 + (size_t)nkeys * 8 + (size_t)nkeys * 4 + 256 * 4 + 64 * 4;
    }
};

__device__ __forceinline__ uint64_t ord_key(double s) {
    uint64_t b = (uint64_t)__double_as_longlong(s);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Integer-built float64 operands (no F2F conversion).  A bf16 half-word h with
// its 15 magnitude bits shifted into the float64 exponent/fraction fields (the
// sign kept in bit 63) is the float64 whose value is EXACTLY h * 2^-896, for
// every finite h including +-0 and subnormals (the 8-bit exponent lands in the
// low bits of the 11-bit field; bf16 subnormals become float64 subnormals,
// which DFMA handles at full rate).  q is pre-scaled by 2^896 (exact; a finite
// bf16/f32 |q| < 2^128 stays below DBL_MAX), so fma(q*2^896, X', acc) rounds
// acc + q*X once, exactly as the oracle does.  2.5 integer ops per channel
// (arithmetic shift + LOP3 mask) replace a quarter-rate F2F.
constexpr double kQScale = 0x1p896;
__device__ __forceinline__ double bf16_lo_scaled(uint32_t w) {  // bits 15..0
    return __hiloint2double(((int32_t)(w << 16) >> 3) & (int32_t)0x8FFFFFFF, 0);
}
__device__ __forceinline__ double bf16_hi_scaled(uint32_t w) {  // bits 31..16
    return __hiloint2double(((int32_t)w >> 3) & (int32_t)0x8FFFE000, 0);
}
// the high words of bf16_lo_scaled / bf16_hi_scaled (the low word is 0)
__device__ __forceinline__ int32_t bf16_lo_hiword(uint32_t w) {
    return ((int32_t)(w << 16) >> 3) & (int32_t)0x8FFFFFFF;
}
__device__ __forceinline__ int32_t bf16_hi_hiword(uint32_t w) {
    return ((int32_t)w >> 3) & (int32_t)0x8FFFE000;
}
__device__ __forceinline__ double f32_scaled(uint32_t x) {
    return __hiloint2double(((int32_t)x >> 3) & (int32_t)0x8FFFFFFF, (int32_t)(x << 29));
}

// Ordered compaction: the positions p in [0, n) with pred(p), ascending, into
// out[]; returns their count.  Each warp owns a contiguous range and walks it
// 32 consecutive positions at a time (ballot + popc ranks): conflict-free
// shared-memory reads.  (The per-thread contiguous ranges it replaces read with
// a stride of n / NT words -- a 32-way bank conflict at 4096 positions: 8.9 us
// of the C3 select's epilogue, r02ah.)  Contains __syncthreads().
template <int NT, typename Pred>
__device__ int cta_compact(int n, int* sw, int32_t* out, Pred pred) {
    constexpr int NWARP = NT / 32;
    const int lane = lane_id(), w = warp_id();
    const int per_w = ((n + NWARP - 1) / NWARP + 31) / 32 * 32;
    const int a = min(n, w * per_w), b = min(n, a + per_w);
    int cnt = 0;
    for (int base = a; base < b; base += 32) {
        const int p = base + lane;
        cnt += __popc(__ballot_sync(0xffffffffu, p < b && pred(p)));
    }
    __syncthreads();  // sw may still be read by a previous scan
    if (lane == 0) sw[w] = cnt;
    __syncthreads();
    int off = 0, tot = 0;
#pragma unroll
    for (int i = 0; i < NWARP; ++i) {
        const int c = sw[i];
        off += i < w ? c : 0;
        tot += c;
    }
    for (int base = a; base < b; base += 32) {
        const int p = base + lane;
        const bool f = p < b && pred(p);
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) out[off + __popc(m & ((1u << lane) - 1u))] = p;
        off += __popc(m);
    }
    __syncthreads();
    return tot;
}

// ---------------------------------------------------------------------------
// CTA-wide top-k over keys[0..n): largest keys, ties -> lower position.
// Writes the selected positions, ascending, to out_pos (smem or global via
// functor).  k_sel = min(k, n) positions are produced.
// ---------------------------------------------------------------------------
// The bits above the highest bit in which the keys differ are common to all of
// them: the radix passes start at the digit holding that bit (one reduction
// instead of up to 7 passes whose histograms put every key into ONE bin -- the
// scores share sign, exponent and leading mantissa bits -- and serialise on its
// shared-memory atomic; measured, r02ac).  Returns the first shift and sets
// prefix / mask to the common bits.  Uses hist as scratch; contains __syncthreads().
template <int NT, typename K>
__device__ int radix_common_prefix(const K* keys, int n, int* hist, K& prefix, K& mask) {
    constexpr int NB = (int)sizeof(K) * 8;
    const int tid = threadIdx.x, lane = lane_id(), w = warp_id();
    K kmin = ~(K)0, kmax = 0;
    for (int i = tid; i < n; i += NT) {
        const K key = keys[i];
        kmin = key < kmin ? key : kmin;
        kmax = key > kmax ? key : kmax;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const K a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    K* red = reinterpret_cast<K*>(hist);  // [NT/32] min, [NT/32] max
    __syncthreads();  // hist may still be read by a previous select
    if (lane == 0) {
        red[w] = kmin;
        red[NT / 32 + w] = kmax;
    }
    __syncthreads();
    kmin = red[0];
    kmax = red[NT / 32];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) {
        kmin = red[i] < kmin ? red[i] : kmin;
        kmax = red[NT / 32 + i] > kmax ? red[NT / 32 + i] : kmax;
    }
    __syncthreads();
    const K diff = kmin ^ kmax;
    if (diff == 0) {  // every key equal: all bits common
        prefix = kmin;
        mask = ~(K)0;
        return -8;
    }
    const int hb = NB - 1 - (sizeof(K) == 8 ? __clzll((long long)diff) : __clz((int)diff));
    const int shift = hb / 8 * 8;
    mask = shift + 8 >= NB ? (K)0 : (~(K)0) << (shift + 8);
    prefix = kmin & mask;
    return shift;
}

// CP: start below the keys' common prefix (the tensor-core selects' merges of
// fp64 scores that share sign, exponent and leading mantissa bits); the MHA
// chunk top-k measured ~3 % slower with the extra reduction (r02ad), so off there.
template <int NT, bool AGG = true, bool CP = false, typename Emit>
__device__ void cta_topk_t(const uint64_t* keys, int n, int k_sel, int* hist, int* sw, Emit emit) {
    const int tid = threadIdx.x;
    uint64_t prefix = 0, mask = 0;
    int rem = k_sel;
    if (k_sel < n) {
        const int shift0 = CP ? radix_common_prefix<NT>(keys, n, hist, prefix, mask) : 56;
        for (int shift = shift0; shift >= 0; shift -= 8) {
            for (int i = tid; i < 256; i += NT) hist[i] = 0;
            __syncthreads();
            {  // (measured: warp-aggregated match_any voting was slower, r02o)
                for (int i = tid; i < n; i += NT) {
                    const uint64_t key = keys[i];
                    if ((key & mask) == prefix) atomicAdd(&hist[(int)((key >> shift) & 0xFF)], 1);
                }
            }
            __syncthreads();
            if (tid < 32) {
                // lane l owns digits 255-8l .. 248-8l (descending)
                int c[8], s = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    c[i] = hist[255 - (tid * 8 + i)];
                    s += c[i];
                }
                int incl = warp_incl_scan(s);
                int above = incl - s;
                if (above < rem && rem <= incl) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        if (above < rem && rem <= above + c[i]) {
                            sw[40] = 255 - (tid * 8 + i);
                            sw[41] = rem - above;
                            sw[42] = c[i];
                        }
                        above += c[i];
                    }
                }
            }
            __syncthreads();
            int digit = sw[40];
            rem = sw[41];
            int cnt = sw[42];
            __syncthreads();
            prefix |= (uint64_t)digit << shift;
            mask |= 0xFFull << shift;
            if (cnt == rem) break;  // every key with this prefix is taken
        }
    } else {
        mask = 0;
        prefix = 0;
        rem = n;  // all (every key matches the empty prefix)
    }
    // Compaction in position order: each warp owns a contiguous range, walked 32
    // consecutive positions at a time (ballots; conflict-free shared reads --
    // per-thread contiguous ranges read with a stride of n / NT, see cta_compact).
    // Keys equal to the k-th take the remaining rem places in position order.
    constexpr int NWARP = NT / 32;
    const int lane = lane_id(), w = warp_id();
    const int per_w = ((n + NWARP - 1) / NWARP + 31) / 32 * 32;
    const int a = min(n, w * per_w), b = min(n, a + per_w);
    const unsigned lt = (1u << lane) - 1u;
    int eq = 0;
    for (int base = a; base < b; base += 32) {
        const int p = base + lane;
        eq += __popc(__ballot_sync(0xffffffffu, p < b && (keys[p] & mask) == prefix));
    }
    __syncthreads();
    if (lane == 0) sw[w] = eq;
    __syncthreads();
    int er0 = 0;
#pragma unroll
    for (int i = 0; i < NWARP; ++i) er0 += i < w ? sw[i] : 0;
    __syncthreads();
    int nsel = 0;
    {
        int er = er0;
        for (int base = a; base < b; base += 32) {
            const int p = base + lane;
            const uint64_t km = p < b ? (keys[p] & mask) : 0;
            const unsigned me = __ballot_sync(0xffffffffu, p < b && km == prefix);
            const bool s = p < b && (km > prefix || (km == prefix && er + __popc(me & lt) < rem));
            nsel += __popc(__ballot_sync(0xffffffffu, s));
            er += __popc(me);
        }
    }
    if (lane == 0) sw[w] = nsel;
    __syncthreads();
    int o = 0;
#pragma unroll
    for (int i = 0; i < NWARP; ++i) o += i < w ? sw[i] : 0;
    {
        int er = er0;
        for (int base = a; base < b; base += 32) {
            const int p = base + lane;
            const uint64_t km = p < b ? (keys[p] & mask) : 0;
            const unsigned me = __ballot_sync(0xffffffffu, p < b && km == prefix);
            const bool s = p < b && (km > prefix || (km == prefix && er + __popc(me & lt) < rem));
            const unsigned ms = __ballot_sync(0xffffffffu, s);
            if (s) emit(o + __popc(ms & lt), p);
            o += __popc(ms);
            er += __popc(me);
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
template <bool AGG, typename Emit>
__device__ __forceinline__ void cta_topk(const uint64_t* keys, int n, int k_sel, int* hist, int* sw, Emit emit) {
    cta_topk_t<kSelThreads, AGG>(keys, n, k_sel, hist, sw, emit);
}

#ifdef SS_DEBUG_KNOBS
// debug timeline of the select kernels (SS_SEL_TRACE=1): per CTA, globaltimer
// at start / tile phase done / threshold / rescoring / chunk top-k / merge start /
// merge end, and the candidate count; read by ss_debug_sel_trace
__device__ unsigned long long g_sel_trace[16384 * 12];
#endif
__device__ __forceinline__ void sel_stamp(int on, int slot, unsigned long long v = 0) {
#ifdef SS_DEBUG_KNOBS
    if (on && threadIdx.x == 0) {
        if (slot != 7) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
        if (blockIdx.x < 16384) g_sel_trace[blockIdx.x * 12 + slot] = v;
    }
#else
    (void)on, (void)slot, (void)v;
#endif
}

namespace cg = cooperative_groups;

// Cluster epilogue of the MHA select (block_select_kernel<..., CLU = true>):
// the chunks of a pair are the CTAs of one thread-block cluster, every CTA
// holds the exact ordered keys of its chunk, and the pair's top-k is taken
// through distributed shared memory instead of per-chunk top-k sets merged by
// the last CTA through the global workspace (r02am: 5 us of chunk top-k + 3 us
// of merge + a ticket round trip after 31 us of scoring at one C2 request
// group).  As in block_select_tcc_kernel: a cluster-wide 256-bin histogram
// LINEAR in float(score) (monotone: fl32 of an fp64 score is non-decreasing),
// the bin b* holding the k-th largest, tau_f = a lower edge of b* one bin below
// it; every block of the top-k has float(score) >= float(k-th) >= tau_f.  The
// candidates (~k per PAIR) keep their EXACT keys; a CTA with more than k keeps
// its exact local top-k; the lists go to the leader CTA at their rank's offset
// (ascending j) and the leader takes the exact top-k (ties -> lower j).
template <int NT>
__device__ void mha_cluster_topk(cg::cluster_group& cluster, int CS, const uint64_t* keys, int n_loc, int j0,
                                 int k, int32_t* cpos, uint64_t* ckeys, int* hist, int* sw,
                                 unsigned long long* xch, uint64_t* gkey_local, int32_t* sel_pair, int tr) {
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    constexpr int NWARP = NT / 32;
    const int rank = (int)cluster.block_rank();
    auto fval = [](uint64_t key) {  // inverse of ord_key, rounded to float
        const uint64_t b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
        return (float)__longlong_as_double((long long)b);
    };
    for (int i = tid; i < 256; i += NT) hist[i] = 0;
    {   // (a) float min / max of the chunk's scores -> own xch[0..1]
        float mn = INFINITY, mx = -INFINITY;
        for (int i = tid; i < n_loc; i += NT) {
            const float v = fval(keys[i]);
            mn = fminf(mn, v);
            mx = fmaxf(mx, v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            sw[warp] = __float_as_int(mn);
            sw[16 + warp] = __float_as_int(mx);
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < NWARP; ++w) {
                mn = fminf(mn, __int_as_float(sw[w]));
                mx = fmaxf(mx, __int_as_float(sw[16 + w]));
            }
            xch[0] = (unsigned long long)(uint32_t)__float_as_int(mn);
            xch[1] = (unsigned long long)(uint32_t)__float_as_int(mx);
        }
    }
    cluster.sync();  // #1
    float Lmin = INFINITY, Lmax = -INFINITY;
    for (int rk = 0; rk < CS; ++rk) {
        const unsigned long long* rx = cluster.map_shared_rank(xch, rk);
        Lmin = fminf(Lmin, __int_as_float((int)(uint32_t)rx[0]));
        Lmax = fmaxf(Lmax, __int_as_float((int)(uint32_t)rx[1]));
    }
    // (b) linear histogram over [Lmin, Lmax], summed over the cluster
    const float scale = Lmax > Lmin ? 256.f / (Lmax - Lmin) : 0.f;
    auto bin_of = [&](float v) { return min(255, (int)((v - Lmin) * scale)); };
    for (int i = tid; i < n_loc; i += NT) atomicAdd(&hist[bin_of(fval(keys[i]))], 1);
    cluster.sync();  // #2
    int tot = 0;
    for (int rk = 0; rk < CS; ++rk) tot += cluster.map_shared_rank(hist, rk)[tid];  // NT == 256 bins
    cluster.sync();  // #3: remote reads done before hist is overwritten
    hist[tid] = tot;
    __syncthreads();
    if (tid < 32) {
        int cnt8[8], s8 = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            cnt8[i] = hist[255 - (tid * 8 + i)];
            s8 += cnt8[i];
        }
        const int incl = warp_incl_scan(s8);
        int above = incl - s8;
        if (above < k && k <= incl) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (above < k && k <= above + cnt8[i]) sw[40] = 255 - (tid * 8 + i);
                above += cnt8[i];
            }
        }
    }
    __syncthreads();
    const int bstar = sw[40];
    float tau = bstar >= 1 ? __fsub_rd(Lmin, 0.f) + __fdiv_rd((float)(bstar - 1), scale) : -INFINITY;
    if (!(tau <= Lmax)) tau = -INFINITY;
    sel_stamp(tr, 2);
    // (c) candidates: float(score) >= tau, positions ascending
    const int n_cand = cta_compact<NT>(n_loc, sw, cpos, [&](int p2) { return fval(keys[p2]) >= tau; });
    // (d) gather into the leader: [keys u64 x CS*k][j i32 x CS*k]
    const int n_out = min(n_cand, k);
    if (tid == 0) xch[4] = (unsigned long long)n_out;
    cluster.sync();  // #4
    int off = 0, n_all = 0;
    for (int rk = 0; rk < CS; ++rk) {
        const int cr = (int)cluster.map_shared_rank(xch, rk)[4];
        off += rk < rank ? cr : 0;
        n_all += cr;
    }
    uint64_t* gkey = cluster.map_shared_rank(gkey_local, 0);
    int32_t* gj = reinterpret_cast<int32_t*>(gkey + (size_t)CS * k);
    if (n_cand > k) {  // local exact top-k first (ties: lower position = lower j)
        for (int i = tid; i < n_cand; i += NT) ckeys[i] = keys[cpos[i]];
        __syncthreads();
        cta_topk_t<NT, true, false>(ckeys, n_cand, k, hist, sw, [&](int o, int pp) {
            gkey[off + o] = ckeys[pp];
            gj[off + o] = j0 + cpos[pp];
        });
    } else {
        for (int i = tid; i < n_cand; i += NT) {
            gkey[off + i] = keys[cpos[i]];
            gj[off + i] = j0 + cpos[i];
        }
    }
    sel_stamp(tr, 4);
    cluster.sync();  // #5: the gathered list complete in the leader; others exit after this
    if (rank != 0) return;
    sel_stamp(tr, 5);
    const int32_t* lj = reinterpret_cast<const int32_t*>(gkey_local + (size_t)CS * k);
    cta_topk_t<NT, true, false>(gkey_local, n_all, k, hist, sw, [&](int o, int pp) { sel_pair[o] = lj[pp]; });
    sel_stamp(tr, 6);
}

// G > 1 (min/max): the all-fp64 GQA kernel now serves calls that ask for every
// score (debug / tests) and f32 inputs; bf16 selections run on the tensor
// cores (block_select_tc_kernel).  One CTA per SM gives it the registers to
// keep its load ring and G x TT accumulators without spilling.
template <bool BF16, int G, bool ICV, bool MEAN, int TT, bool CLU = false>
__global__ void __launch_bounds__(kSelThreads, (G > 1 && !MEAN) ? 1 : 2)
block_select_kernel(const void* __restrict__ q, const void* __restrict__ meta,
                    const int32_t* __restrict__ n_blk_arr, int max_blk, int k, int Hq, int Hkv,
                    int nchunks, int CH, int npairs, int l2pf, int32_t* __restrict__ sel, double* __restrict__ scores,
                    uint64_t* __restrict__ cand_key, int32_t* __restrict__ cand_j,
                    int32_t* __restrict__ tickets) {
    constexpr int ES = BF16 ? 2 : 4;
    constexpr int CPC = 16 / ES;               // channels per 16-byte chunk
    constexpr int NCH = kHeadDim / CPC;        // chunks per row (16 bf16, 32 f32)
    constexpr int TILE_ELEMS = 64 * kHeadDim;  // 32 blocks * 2 * d
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* qpn = (double2*)smem_raw;                                  // [128*G]
    // GQA bf16 (SELQ): ONE DFMA per head and channel.  The sign of q_{g,c} is
    // the same for every lane, and the min / max operands are integer-built
    // float64s whose low words are 0, so the operand of head g is the high word
    // hN ^ (f_g & (hM ^ hN)) (one LOP3 on the integer pipe, f_g = all ones
    // when q_{g,c} >= 0, else 0) and
    // acc + q * (q >= 0 ? M : m) == acc + max(q M, q m), rounded once.
    constexpr bool SELQ = BF16 && ICV && G > 1 && !MEAN;
    double* qs = (double*)smem_raw;                                     // [128*G] (SELQ)
    int32_t* qf = (int32_t*)(smem_raw + kHeadDim * G * 8);              // [128*G] (SELQ)
    uint64_t* keys = (uint64_t*)(smem_raw + kHeadDim * G * 16);         // [nkeys]
    const int nkeys_cap = max(CH, min(nchunks * k, kSelMaxMerge));
    int32_t* jpos = (int32_t*)(keys + nkeys_cap);                       // [nkeys]
    int* hist = (int*)(jpos + nkeys_cap);                               // [256]
    int* sw = hist + 256;                                               // [64]

    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    // persistent: CTAs stride over (pair, chunk) work items, so the grid is fully
    // resident and a FlashH2D kernel of another request group can co-reside
    const int tr = (l2pf & 16) ? 1 : 0;  // debug timeline (SS_SEL_TRACE=1)
    sel_stamp(tr, 0);
    for (int item = blockIdx.x; item < nchunks * npairs; item += gridDim.x) {
    __syncthreads();  // previous item's shared-memory readers are done
    const int pair = item / nchunks;
    const int b = pair / Hkv, h = pair % Hkv;
    const int ci = item % nchunks;  // chunk index
    const int nb = n_blk_arr[b];
    const int nch_b = max(1, (nb + CH - 1) / CH);
    if constexpr (CLU) {
        // one cluster per pair (grid = pairs x nchunks, no persistence): a chunk
        // past n_blk still joins the cluster barriers with no block
        if (k >= nb) {  // every block selected (uniform over the cluster)
            if (ci == 0)
                for (int i = tid; i < k; i += kSelThreads) sel[(size_t)pair * k + i] = i < nb ? i : -1;
            return;
        }
    } else {
        if (ci >= nch_b) continue;
    }

    const int j0 = ci * CH;
    const int nb_chunk = max(0, min(CH, nb - j0));  // 0 if nb == 0 (or a CLU chunk past nb)
    const int ntiles = (nb_chunk + 31) / 32;
    constexpr size_t TILE_BYTES = MEAN ? (size_t)32 * kHeadDim * 4 : (size_t)TILE_ELEMS * ES;
    const char* meta_pair = (const char*)meta + ((size_t)pair * (max_blk / 32)) * TILE_BYTES;

    // G > 1 min/max: a warp pass scores TT tiles, tl and (TT = 2) tl + 8 (lane r:
    // block r of each); pass p has tl = warp + 8*TT*p.  The 16-byte chunk loads run GD steps
    // ahead in a register ring that carries across passes (the next pass's
    // first chunks load during this pass's last steps), and the first GD steps
    // are issued before the q setup below (they do not depend on q).
    constexpr int GD = 3, GR = GD + 1;
    static_assert(NCH % GR == 0, "ring slot of step s must be s % GR in every pass");
    uint4 rnA[GR], rxA[GR], rnB[GR], rxB[GR];
    const int npass = (G > 1 && !MEAN) ? (ntiles - warp + TT * kSelWarps - 1) / (TT * kSelWarps) : 0;
    auto pass_ptr = [&](int p, const char*& pa, const char*& pb) {
        const int tl = warp + p * TT * kSelWarps;
        pa = meta_pair + (size_t)(j0 / 32 + tl) * TILE_BYTES + lane * 16;
        pb = (TT == 2 && tl + kSelWarps < ntiles) ? pa + (size_t)kSelWarps * TILE_BYTES : pa;
    };
    auto ring_load = [&](const char* pa, const char* pb, int step, int slot) {
        rnA[slot] = ldg_stream(pa + (size_t)((step * 2 + 0) * 32) * 16);
        rxA[slot] = ldg_stream(pa + (size_t)((step * 2 + 1) * 32) * 16);
        if constexpr (TT == 2) {
            rnB[slot] = ldg_stream(pb + (size_t)((step * 2 + 0) * 32) * 16);
            rxB[slot] = ldg_stream(pb + (size_t)((step * 2 + 1) * 32) * 16);
        }
    };
    if constexpr (G > 1 && !MEAN) {
        if (npass > 0) {
            const char *pa, *pb;
            pass_ptr(0, pa, pb);
#pragma unroll
            for (int st = 0; st < GD; ++st) ring_load(pa, pb, st, st);
        }
    }

    // G == 1 (MHA): q as float64 plus per-channel select masks (q >= 0 -> max
    // row, else min row), so each channel costs one LOP3-select, one exact
    // f32->f64 convert and ONE DFMA: acc + q*(q>=0 ? M : m) == acc + max(qM, qm).
    double* qd1 = (double*)smem_raw;                        // [128]
    uint32_t* qmask1 = (uint32_t*)(smem_raw + kHeadDim * 8); // [128] (bf16 uses 64)
    if constexpr (G == 1 && !MEAN) {
        for (int c = tid; c < kHeadDim; c += kSelThreads) {
            size_t qi = ((size_t)b * Hq + h) * kHeadDim + c;
            double qv = BF16 ? (double)__uint_as_float(((uint32_t)((const uint16_t*)q)[qi]) << 16)
                             : (double)((const float*)q)[qi];
            qd1[c] = ICV ? qv * kQScale : qv;
        }
        __syncthreads();
        for (int i = tid; i < kHeadDim / (BF16 ? 2 : 1); i += kSelThreads) {
            uint32_t m;
            if (BF16)
                m = (qd1[2 * i] >= 0.0 ? 0x0000FFFFu : 0u) | (qd1[2 * i + 1] >= 0.0 ? 0xFFFF0000u : 0u);
            else
                m = qd1[i] >= 0.0 ? 0xFFFFFFFFu : 0u;
            qmask1[i] = m;
        }
    }
    // G > 1: q for the G query heads of this KV head, as (q+, q-) = (max(q,0), min(q,0)).
    // NEXT-3 mean metadata: q of the G heads as float64 (x 2^896 with ICV), [c][g]
    double* qm = (double*)smem_raw;
    if constexpr (MEAN)
    for (int i = tid; i < kHeadDim * G; i += kSelThreads) {
        const int g = i % G, c = i / G;
        const size_t qi = ((size_t)b * Hq + (size_t)h * G + g) * kHeadDim + c;
        const double qd = BF16 ? (double)__uint_as_float(((uint32_t)((const uint16_t*)q)[qi]) << 16)
                               : (double)((const float*)q)[qi];
        qm[i] = ICV ? qd * kQScale : qd;
    }
    if constexpr (G > 1 && !MEAN)
    for (int i = tid; i < kHeadDim * G; i += kSelThreads) {
        int g = i % G, c = i / G;
        size_t qi = ((size_t)b * Hq + (size_t)h * G + g) * kHeadDim + c;
        double qd;
        if (BF16)
            qd = (double)__uint_as_float(((uint32_t)((const uint16_t*)q)[qi]) << 16);
        else
            qd = (double)((const float*)q)[qi];
        if (ICV) qd *= kQScale;
        if constexpr (SELQ) {
            qs[i] = qd;                  // q * 2^896, signed
            qf[i] = qd >= 0.0 ? -1 : 0;  // all ones: the max row M, 0: the min row m
        } else {
            qpn[i] = make_double2(qd > 0.0 ? qd : 0.0, qd < 0.0 ? qd : 0.0);
        }
    }
    __syncthreads();


    // NEXT-3: S(j) = max_g sum_c q_{g,c} mu_{j,c}.  Tile [32 chunks][32 blocks][4 ch]
    // float32: lane r scores block r; chunk s (channels 4s..4s+3) of the warp's 32
    // blocks is one contiguous 512-byte segment.  One exact operand build per
    // channel, G DFMAs (the products q*mu are exact: <= 48 significant bits).
    if constexpr (MEAN)
    for (int tl = warp; tl < ntiles; tl += kSelWarps) {
        const char* tb = meta_pair + (size_t)(j0 / 32 + tl) * TILE_BYTES + lane * 16;
        constexpr int NCM = kHeadDim / 4, D = 8, R = D + 1;
        uint4 mv[R];
#pragma unroll
        for (int s = 0; s < D; ++s) mv[s] = ldg_stream(tb + (size_t)s * 512);
        double acc[G];
#pragma unroll
        for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll
        for (int s = 0; s < NCM; ++s) {
            if (s + D < NCM) mv[(s + D) % R] = ldg_stream(tb + (size_t)(s + D) * 512);
            const uint32_t w4[4] = {mv[s % R].x, mv[s % R].y, mv[s % R].z, mv[s % R].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int c = 4 * s + e;
                const double x = ICV ? f32_scaled(w4[e]) : (double)__uint_as_float(w4[e]);
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g] = __fma_rn(qm[c * G + g], x, acc[g]);
            }
        }
        double sc = acc[0];
#pragma unroll
        for (int g = 1; g < G; ++g) sc = acc[g] > sc ? acc[g] : sc;
        sc = sc + 0.0;
        const int pos = tl * 32 + lane;
        keys[pos] = ord_key(sc);
        if (scores != nullptr && j0 + pos < nb) scores[(size_t)pair * max_blk + j0 + pos] = sc;
    }

    if constexpr (G == 1 && !MEAN)
    for (int tl = warp; tl < ntiles; tl += kSelWarps) {
        const int tile = j0 / 32 + tl;
        const char* tb = meta_pair + (size_t)tile * TILE_ELEMS * ES + lane * 16;
        if ((l2pf & 1) && lane == 0 && tl + kSelWarps < ntiles)  // next tile of this warp -> L2
            prefetch_l2_bulk(meta_pair + (size_t)(tile + kSelWarps) * TILE_ELEMS * ES, TILE_ELEMS * ES);
        // fully unrolled over the NCH chunks, loads kept D chunks ahead
        constexpr int D = 6, R = D + 1;
        uint4 mn[R], mx[R];
        // (debug experiment SS_SEL_L2PF=2: read the min rows only -- wrong scores,
        // half the metadata bytes: the step-time effect of a half-size read)
        const bool half_exp = (l2pf & 2) != 0;
#pragma unroll
        for (int s = 0; s < D; ++s) {
            mn[s] = ldg_stream(tb + (size_t)((s * 2 + 0) * 32) * 16);
            mx[s] = half_exp ? mn[s] : ldg_stream(tb + (size_t)((s * 2 + 1) * 32) * 16);
        }
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < NCH; ++s) {
            if (s + D < NCH) {
                mn[(s + D) % R] = ldg_stream(tb + (size_t)(((s + D) * 2 + 0) * 32) * 16);
                mx[(s + D) % R] = half_exp ? mn[(s + D) % R]
                                           : ldg_stream(tb + (size_t)(((s + D) * 2 + 1) * 32) * 16);
            }
            const uint4 wn = mn[s % R], wx = mx[s % R];
            const uint4 mk = *reinterpret_cast<const uint4*>(qmask1 + s * (BF16 ? 4 : 4));
            const uint32_t an[4] = {wn.x, wn.y, wn.z, wn.w};
            const uint32_t ax[4] = {wx.x, wx.y, wx.z, wx.w};
            const uint32_t am[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const uint32_t y = (ax[i] & am[i]) | (an[i] & ~am[i]);
                if (BF16) {
                    const double2 qq = *reinterpret_cast<const double2*>(qd1 + s * 8 + 2 * i);
                    acc = __fma_rn(qq.x, ICV ? bf16_lo_scaled(y) : (double)__uint_as_float(y << 16), acc);
                    acc = __fma_rn(qq.y, ICV ? bf16_hi_scaled(y) : (double)__uint_as_float(y & 0xFFFF0000u), acc);
                } else {
                    acc = __fma_rn(qd1[s * 4 + i], ICV ? f32_scaled(y) : (double)__uint_as_float(y), acc);
                }
            }
        }
        const double s = acc + 0.0;
        const int pos = tl * 32 + lane;
        const int j = j0 + pos;
        keys[pos] = ord_key(s);
        if (scores != nullptr && j < nb) scores[(size_t)pair * max_blk + j] = s;
    }

    if constexpr (G > 1 && !MEAN)
    for (int p = 0; p < npass; ++p) {
        // two tiles per warp pass: each shared-memory (q+, q-) load serves two
        // blocks, and two independent DFMA chains / load streams per lane
        const int tl = warp + p * TT * kSelWarps;
        const bool two = TT == 2 && tl + kSelWarps < ntiles;
        const char *tbA, *tbB, *nxA, *nxB;
        pass_ptr(p, tbA, tbB);
        const bool has_next = p + 1 < npass;
        if (has_next) pass_ptr(p + 1, nxA, nxB);
        double accA[G], accB[G];
#pragma unroll
        for (int g = 0; g < G; ++g) accA[g] = accB[g] = 0.0;
        // fully unrolled over the NCH chunks; the min / max elements are built
        // once (exact) and shared by the G heads: acc_g += q+_g * M + q-_g * m
        // (one term is an exact 0)
        constexpr int R = GR;
        uint4 (&mnA)[GR] = rnA; uint4 (&mxA)[GR] = rxA;
        uint4 (&mnB)[GR] = rnB; uint4 (&mxB)[GR] = rxB;
#pragma unroll
        for (int s = 0; s < NCH; ++s) {
            if (s + GD < NCH)
                ring_load(tbA, tbB, s + GD, (s + GD) % GR);
            else if (has_next)
                ring_load(nxA, nxB, s + GD - NCH, (s + GD) % GR);
            const uint32_t wnA[4] = {mnA[s % R].x, mnA[s % R].y, mnA[s % R].z, mnA[s % R].w};
            const uint32_t wxA[4] = {mxA[s % R].x, mxA[s % R].y, mxA[s % R].z, mxA[s % R].w};
            const uint32_t wnB[4] = {mnB[s % R].x, mnB[s % R].y, mnB[s % R].z, mnB[s % R].w};
            const uint32_t wxB[4] = {mxB[s % R].x, mxB[s % R].y, mxB[s % R].z, mxB[s % R].w};
#pragma unroll
            for (int e = 0; e < CPC; ++e) {
                double dminA, dmaxA, dminB, dmaxB;
                if (BF16 && ICV) {
                    const int w = e >> 1;
                    dminA = (e & 1) ? bf16_hi_scaled(wnA[w]) : bf16_lo_scaled(wnA[w]);
                    dmaxA = (e & 1) ? bf16_hi_scaled(wxA[w]) : bf16_lo_scaled(wxA[w]);
                    dminB = (e & 1) ? bf16_hi_scaled(wnB[w]) : bf16_lo_scaled(wnB[w]);
                    dmaxB = (e & 1) ? bf16_hi_scaled(wxB[w]) : bf16_lo_scaled(wxB[w]);
                } else if (ICV) {
                    dminA = f32_scaled(wnA[e]);
                    dmaxA = f32_scaled(wxA[e]);
                    dminB = f32_scaled(wnB[e]);
                    dmaxB = f32_scaled(wxB[e]);
                } else if (BF16) {
                    const int w = e >> 1;
                    dminA = (double)__uint_as_float((e & 1) ? (wnA[w] & 0xFFFF0000u) : (wnA[w] << 16));
                    dmaxA = (double)__uint_as_float((e & 1) ? (wxA[w] & 0xFFFF0000u) : (wxA[w] << 16));
                    dminB = (double)__uint_as_float((e & 1) ? (wnB[w] & 0xFFFF0000u) : (wnB[w] << 16));
                    dmaxB = (double)__uint_as_float((e & 1) ? (wxB[w] & 0xFFFF0000u) : (wxB[w] << 16));
                } else {
                    dminA = (double)__uint_as_float(wnA[e]);
                    dmaxA = (double)__uint_as_float(wxA[e]);
                    dminB = (double)__uint_as_float(wnB[e]);
                    dmaxB = (double)__uint_as_float(wxB[e]);
                }
                const int c = s * CPC + e;
                if constexpr (SELQ) {
                    const int w = e >> 1;
                    const int32_t hNA = (e & 1) ? bf16_hi_hiword(wnA[w]) : bf16_lo_hiword(wnA[w]);
                    const int32_t hMA = (e & 1) ? bf16_hi_hiword(wxA[w]) : bf16_lo_hiword(wxA[w]);
                    const int32_t dA = hMA ^ hNA;   // hN ^ (d & mask) picks M or m: one LOP3
                    int32_t hNB = 0, dB = 0;
                    if constexpr (TT == 2) {
                        hNB = (e & 1) ? bf16_hi_hiword(wnB[w]) : bf16_lo_hiword(wnB[w]);
                        dB = ((e & 1) ? bf16_hi_hiword(wxB[w]) : bf16_lo_hiword(wxB[w])) ^ hNB;
                    }
                    double qv[G];
                    int32_t fv[G];
#pragma unroll
                    for (int g = 0; g < G; g += 2) {
                        const double2 t = *reinterpret_cast<const double2*>(qs + c * G + g);
                        qv[g] = t.x;
                        qv[g + 1] = t.y;
                    }
#pragma unroll
                    for (int g = 0; g < G; g += (G >= 4 ? 4 : 2)) {
                        if constexpr (G >= 4) {
                            const int4 t = *reinterpret_cast<const int4*>(qf + c * G + g);
                            fv[g] = t.x; fv[g + 1] = t.y; fv[g + 2] = t.z; fv[g + 3] = t.w;
                        } else {
                            const int2 t = *reinterpret_cast<const int2*>(qf + c * G + g);
                            fv[g] = t.x; fv[g + 1] = t.y;
                        }
                    }
#pragma unroll
                    for (int g = 0; g < G; ++g) {
                        accA[g] = __fma_rn(qv[g], __hiloint2double(hNA ^ (fv[g] & dA), 0), accA[g]);
                        if constexpr (TT == 2)
                            accB[g] = __fma_rn(qv[g], __hiloint2double(hNB ^ (fv[g] & dB), 0), accB[g]);
                    }
                } else {
#pragma unroll
                for (int g = 0; g < G; ++g) {
                    const double2 qq = qpn[c * G + g];
                    {
                        accA[g] = __fma_rn(qq.x, dmaxA, accA[g]);
                        accA[g] = __fma_rn(qq.y, dminA, accA[g]);
                        if constexpr (TT == 2) {
                            accB[g] = __fma_rn(qq.x, dmaxB, accB[g]);
                            accB[g] = __fma_rn(qq.y, dminB, accB[g]);
                        }
                    }
                }
                }
            }
        }
        double sA = accA[0], sB = accB[0];
#pragma unroll
        for (int g = 1; g < G; ++g) {
            sA = accA[g] > sA ? accA[g] : sA;
            sB = accB[g] > sB ? accB[g] : sB;
        }
        sA = sA + 0.0;
        sB = sB + 0.0;
        const int posA = tl * 32 + lane, posB = (tl + kSelWarps) * 32 + lane;
        keys[posA] = ord_key(sA);
        if (scores != nullptr && j0 + posA < nb) scores[(size_t)pair * max_blk + j0 + posA] = sA;
        if (two) {
            keys[posB] = ord_key(sB);
            if (scores != nullptr && j0 + posB < nb) scores[(size_t)pair * max_blk + j0 + posB] = sB;
        }
    }
    __syncthreads();
    sel_stamp(tr, 1);
    if constexpr (CLU) {
        cg::cluster_group cluster = cg::this_cluster();
        unsigned long long* xch = (unsigned long long*)(sw + 64);  // [32]
        uint64_t* ckeys = (uint64_t*)(xch + 32);                   // [CH]
        uint64_t* gkey = ckeys + CH;                                // leader: [nchunks * k] keys, then j
        mha_cluster_topk<kSelThreads>(cluster, nchunks, keys, nb_chunk, j0, k, jpos, ckeys, hist, sw, xch, gkey,
                                      sel + (size_t)pair * k, tr);
        return;
    }

    const int kc = min(k, nb_chunk);
    int32_t* sel_pair = sel + (size_t)pair * k;
    if (nch_b == 1) {
        cta_topk<G == 1>(keys, nb_chunk, kc, hist, sw, [&](int o, int p) { sel_pair[o] = j0 + p; });
        for (int r = kc + tid; r < k; r += kSelThreads) sel_pair[r] = -1;
        continue;
    }
    // Multi-chunk: emit candidates, then the last CTA of the pair merges.
    uint64_t* ck = cand_key + ((size_t)pair * nchunks + ci) * k;
    int32_t* cj = cand_j + ((size_t)pair * nchunks + ci) * k;
    cta_topk<G == 1>(keys, nb_chunk, kc, hist, sw, [&](int o, int p) {
        ck[o] = keys[p];
        cj[o] = j0 + p;
    });
    __threadfence();
    __syncthreads();
    sel_stamp(tr, 4);
    if (tid == 0) sw[48] = atomicAdd(&tickets[pair], 1);
    __syncthreads();
    if (sw[48] != nch_b - 1) continue;
    __threadfence();
    // Merge: candidates of chunk c are ascending in j and chunks are ordered,
    // so position order == j order and the tie rule carries over.
    int n = 0;
    for (int c = 0; c < nch_b; ++c) {
        int sz = min(CH, nb - c * CH);
        int kcc = min(k, sz);
        const uint64_t* sk = cand_key + ((size_t)pair * nchunks + c) * k;
        const int32_t* sj = cand_j + ((size_t)pair * nchunks + c) * k;
        for (int i = tid; i < kcc; i += kSelThreads) {
            keys[n + i] = __ldcg(sk + i);
            jpos[n + i] = __ldcg(sj + i);
        }
        n += kcc;
    }
    __syncthreads();
    const int kf = min(k, nb);
    sel_stamp(tr, 5);
    cta_topk<G == 1>(keys, n, kf, hist, sw, [&](int o, int p) { sel_pair[o] = jpos[p]; });
    for (int r = kf + tid; r < k; r += kSelThreads) sel_pair[r] = -1;
    if (tid == 0) tickets[pair] = 0;
    sel_stamp(tr, 6);
    }  // work items
}

// ---------------------------------------------------------------------------
// GQA select on the tensor cores, exact by filtering (bf16, G = 2, 4, 8).
//
// The score is a dense contraction: S_g(j) = sum_c max(q_gc M_jc, q_gc m_jc)
// = sum over the 256 "channels" [m_j0..m_j127, M_j0..M_j127] of
// [q-_g ; q+_g] (q+ = max(q, 0), q- = min(q, 0); one of the two products is an
// exact 0).  So a warp computes approximate scores of 16 blocks x 8 heads per
// mma.sync m16n8k16 (bf16 x bf16 products are exact in the f32 accumulator;
// the A operand is the metadata tile exactly as stored, ldmatrix'd from
// shared memory; the B operand is q), and a second mma over |A| x |B| gives
// sum_c |q_gc X_jc|, which bounds the f32 accumulation error:
//     |s~_j - S_j| <= eps_j = 2^-10 * max_g sum|t| + 2^-100
// (f32 accumulation of 256 exact products, even with truncating adds, errs
// by < 2^-13.9 sum|t|; the margin is 16x; the fp64 oracle's own rounding is
// < 2^-45 sum|t|).  With L_j = s~_j - eps_j, U_j = s~_j + eps_j and tau the
// k-th largest L_j of the chunk, every block of the exact top-k has U_j >= tau
// (k blocks have S >= L >= tau; a block with U < tau has S < tau).  Those
// candidates -- k plus the few within 2 eps of the threshold -- are rescored
// EXACTLY (the oracle's fp64 sequential sum, as block_select_kernel does) and
// the exact top-k with the same tie rule is taken among them: the selection is
// bit-identical to the oracle's.  Non-finite approximations make a block a
// candidate (L = -inf, U = +inf).  The fp64 work drops from every block to
// ~k per chunk, the integer operand building disappears, and the kernel is
// left with the metadata stream: 16 KiB tiles by 1-D TMA bulk copies, one
// stage per warp, 4 warps per CTA, 2 CTAs per SM.
// ---------------------------------------------------------------------------
constexpr int kTcWarps = 4;
constexpr int kTcThreads = kTcWarps * 32;
constexpr int kTileBytes = 64 * kHeadDim * 2;  // 32 blocks x [min|max] x 128 ch, bf16
constexpr int kSelTcStages = 1;  // tile stages per warp (SS_SEL_TC_STAGES, debug A/B)
constexpr int kSelTcRot = 0;     // start-tile rotation multiplier per CTA (SS_SEL_ROT, debug A/B)
constexpr int kSelTcPf = 0;      // L2 prefetch distance in tiles (SS_SEL_TC_PF, debug A/B)

__device__ __forceinline__ uint32_t ord32(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b >> 31) ? ~b : (b | 0x80000000u);
}

// k-th largest (1-based) 32-bit key of keys[0..n): CTA radix select, 8-bit
// digits MSB first.  Contains __syncthreads().
__device__ uint32_t cta_kth_u32(const uint32_t* keys, int n, int kk, int* hist, int* sw) {
    const int tid = threadIdx.x;
    uint32_t prefix = 0, mask = 0;
    int rem = kk;
    // the candidate filter only needs a LOWER bound of the k-th largest key (a
    // smaller tau admits more candidates, all rescored exactly): start below the
    // keys' common prefix and stop after two digits -- the lower edge of the
    // bin holding the k-th key, 16 bits below the keys' spread
    const int shift0 = radix_common_prefix<kTcThreads>(keys, n, hist, prefix, mask);
    const int shift_end = shift0 - 8;
    for (int shift = shift0; shift >= 0 && shift >= shift_end; shift -= 8) {
        for (int i = tid; i < 256; i += kTcThreads) hist[i] = 0;
        __syncthreads();
        for (int i = tid; i < n; i += kTcThreads) {
            const uint32_t key = keys[i];
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1);
        }
        __syncthreads();
        if (tid < 32) {
            int cnt[8], s = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt[i] = hist[255 - (tid * 8 + i)];
                s += cnt[i];
            }
            const int incl = warp_incl_scan(s);
            int above = incl - s;
            if (above < rem && rem <= incl) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (above < rem && rem <= above + cnt[i]) {
                        sw[40] = 255 - (tid * 8 + i);
                        sw[41] = rem - above;
                    }
                    above += cnt[i];
                }
            }
        }
        __syncthreads();
        const uint32_t digit = (uint32_t)sw[40];
        rem = sw[41];
        __syncthreads();
        prefix |= digit << shift;
        mask |= 0xFFu << shift;
    }
    return prefix;
}

template <int G, int NS>
__global__ void __launch_bounds__(kTcThreads, NS == 1 ? 2 : 1)
block_select_tc_kernel(const void* __restrict__ q, const void* __restrict__ meta,
                       const int32_t* __restrict__ n_blk_arr, int max_blk, int k, int Hq, int Hkv,
                       int nchunks, int CH, int region_bytes, int rot_mul, int pf_dist, int tr,
                       int32_t* __restrict__ sel,
                       uint64_t* __restrict__ cand_key, int32_t* __restrict__ cand_j,
                       int32_t* __restrict__ tickets) {
    extern __shared__ __align__(128) unsigned char tc_smem[];
    unsigned char* smem_raw = tc_smem;
    // [region: tile stages (tile phase) | keys u64 + jpos i32 (select phase)]
    // [lo f32 [CH]][hi f32 [CH]][qs f64 [128 G]][qf i32 [128 G]][hist 256][sw 64][bar]
    unsigned char* stage_base = smem_raw;
    uint64_t* keys = (uint64_t*)smem_raw;
    float* lo = (float*)(smem_raw + region_bytes);
    float* hi = lo + CH;
    double* qs = (double*)(hi + CH);
    int32_t* qf = (int32_t*)(qs + kHeadDim * G);
    int* hist = (int*)(qf + kHeadDim * G);
    int* sw = hist + 256;
    uint64_t* bars = (uint64_t*)(sw + 64);
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    sel_stamp(tr, 0);
    const int pair = blockIdx.x / nchunks, ci = blockIdx.x % nchunks;
    const int b = pair / Hkv, h = pair % Hkv;
    const int nb = n_blk_arr[b];
    const int nch_b = max(1, (nb + CH - 1) / CH);
    if (ci >= nch_b) return;
    const int j0 = ci * CH;
    const int nb_chunk = min(CH, nb - j0);
    const int ntiles = (nb_chunk + 31) / 32;
    const char* meta_pair = (const char*)meta + ((size_t)pair * (max_blk / 32)) * kTileBytes;
    const uint16_t* qb16 = (const uint16_t*)q + ((size_t)b * Hq + (size_t)h * G) * kHeadDim;

    // ---- exact-path q (x 2^896, signed) and max-row masks; mma B fragments ----
    for (int i = tid; i < kHeadDim * G; i += kTcThreads) {
        const int g = i % G, c = i / G;
        const double qd = (double)__uint_as_float(((uint32_t)qb16[(size_t)g * kHeadDim + c]) << 16) * kQScale;
        qs[i] = qd;
        qf[i] = qd >= 0.0 ? -1 : 0;
    }
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < NS; ++st) mbar_init(&bars[warp * NS + st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // B fragment of chunk s (k rows 0-7: the min channels 8s..8s+7 -> q-, rows
    // 8-15: the max channels -> q+; column n = head): lane holds rows 2c, 2c+1
    // (b0) and 2c+8, 2c+9 (b1) of column r
    const int r = lane >> 2, c = lane & 3;
    uint32_t qb[16][2], qa[16][2];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        uint32_t w = 0;
        if (r < G) w = __ldg(reinterpret_cast<const uint32_t*>(qb16 + (size_t)r * kHeadDim + 8 * s + 2 * c));
        const uint32_t neg = ((w & 0x8000u) ? 0x0000FFFFu : 0u) | ((w & 0x80000000u) ? 0xFFFF0000u : 0u);
        qb[s][0] = w & neg;   // q- (q < 0, incl. -0: an exact zero product either way)
        qb[s][1] = w & ~neg;  // q+
        qa[s][0] = qb[s][0] & 0x7FFF7FFFu;
        qa[s][1] = qb[s][1] & 0x7FFF7FFFu;
    }
    __syncthreads();

    // ---- tile phase: approximate scores + error bounds -> lo / hi ----
    // NS stages per warp; the warp's i-th tile is logical tile warp + i * kTcWarps,
    // read from physical tile (logical + rot) % ntiles: CTAs start at different
    // offsets of their chunks instead of all streaming the same address phase
    const int rot = ntiles > 0 ? (int)(((int64_t)blockIdx.x * rot_mul) % ntiles) : 0;
    const int my_tiles = ntiles > warp ? (ntiles - warp + kTcWarps - 1) / kTcWarps : 0;
    auto phys = [&](int i) { int t = warp + i * kTcWarps + rot; return t >= ntiles ? t - ntiles : t; };
    auto issue = [&](int i) {
        if (lane == 0 && i < my_tiles) {
            const int st = i % NS;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[warp * NS + st], kTileBytes);
            bulk_g2s(stage_base + (size_t)(warp * NS + st) * kTileBytes,
                     meta_pair + (size_t)(j0 / 32 + phys(i)) * kTileBytes, kTileBytes, &bars[warp * NS + st]);
        }
    };
    uint32_t phases = 0;
    const int mi = lane >> 3, rr = lane & 7;
    // ldmatrix row address of A (16 blocks x 16 k) for chunk s, m-tile mt:
    // matrices {min, blocks 0-7}, {min, 8-15}, {max, 0-7}, {max, 8-15}
    const uint32_t a_off = (uint32_t)((mi >> 1) * 512 + (8 * (mi & 1) + rr) * 16);
#pragma unroll
    for (int i = 0; i < NS; ++i) issue(i);
    // L2 prefetch of the warp's tiles pf_dist ahead (no shared memory: more
    // bytes in flight from DRAM than the stages alone hold)
    if (lane == 0)
        for (int i = NS; i < NS + pf_dist && i < my_tiles; ++i)
            prefetch_l2_bulk(meta_pair + (size_t)(j0 / 32 + phys(i)) * kTileBytes, kTileBytes);
    for (int i = 0; i < my_tiles; ++i) {
        const int st = i % NS, t = phys(i);
        if (lane == 0 && pf_dist > 0 && i + NS + pf_dist < my_tiles)
            prefetch_l2_bulk(meta_pair + (size_t)(j0 / 32 + phys(i + NS + pf_dist)) * kTileBytes, kTileBytes);
        mbar_wait(&bars[warp * NS + st], (phases >> st) & 1u);
        phases ^= 1u << st;
        unsigned char* stage = stage_base + (size_t)(warp * NS + st) * kTileBytes;
        const uint32_t sb = smem_u32(stage);
        float ds[2][4], da[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) ds[mt][e] = da[mt][e] = 0.f;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                uint32_t af[4];
                ldsm_x4(sb + s * 1024 + mt * 256 + a_off, af);
                hmma(ds[mt], af, qb[s][0], qb[s][1]);
                af[0] &= 0x7FFF7FFFu;
                af[1] &= 0x7FFF7FFFu;
                af[2] &= 0x7FFF7FFFu;
                af[3] &= 0x7FFF7FFFu;
                hmma(da[mt], af, qa[s][0], qa[s][1]);
            }
        }
        __syncwarp();
        issue(i + NS);  // the stage is consumed: the warp's tile i + NS into it
        // lane: rows r, r + 8 of each m-tile, heads 2c, 2c + 1
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                float sv = -INFINITY, av = 0.f;
                int bad = 0;  // a non-finite approximation makes the block a candidate
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (2 * c + e < G) {
                        const float dv = ds[mt][2 * half + e], dav = da[mt][2 * half + e];
                        bad |= !(fabsf(dv) <= 3.0e38f) || !(dav <= 3.0e38f);
                        sv = fmaxf(sv, dv);
                        av = fmaxf(av, dav);
                    }
                }
                // max over the quad's heads (the 4 lanes share rows r, r + 8)
                sv = fmaxf(sv, __shfl_xor_sync(0xffffffffu, sv, 1));
                sv = fmaxf(sv, __shfl_xor_sync(0xffffffffu, sv, 2));
                av = fmaxf(av, __shfl_xor_sync(0xffffffffu, av, 1));
                av = fmaxf(av, __shfl_xor_sync(0xffffffffu, av, 2));
                bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
                bad |= __shfl_xor_sync(0xffffffffu, bad, 2);
                const bool anybad = bad != 0;
                const int jj = t * 32 + 16 * mt + 8 * half + r;
                if (c == 0 && jj < nb_chunk) {
                    const float eps = __fmaf_ru(av, 0x1p-10f, 0x1p-100f);
                    if (anybad || !(eps <= 3.0e38f)) {
                        lo[jj] = -INFINITY;
                        hi[jj] = INFINITY;
                    } else {
                        lo[jj] = __fsub_rd(sv, eps);
                        hi[jj] = __fadd_ru(sv, eps);
                    }
                }
            }
    }
    __syncthreads();
    sel_stamp(tr, 1);

    // ---- threshold and candidates ----
    const int kk = min(k, nb_chunk);
    uint32_t* lkey = (uint32_t*)lo;   // in place: lo[] -> ord32(lo[])
    for (int i = tid; i < nb_chunk; i += kTcThreads) lkey[i] = ord32(lo[i]);
    __syncthreads();
    const uint32_t tau = kk < nb_chunk ? cta_kth_u32(lkey, nb_chunk, kk, hist, sw) : 0u;
    // per-chunk layout after the tile phase: candidate positions at the region
    // start, their exact keys after CH positions, the rescoring stage from there
    // to the end of hi[] (the region and lo / hi are dead by then)
    int32_t* jpos = (int32_t*)smem_raw;
    uint64_t* ckeys = (uint64_t*)(smem_raw + (size_t)CH * 4);
    const int n_cand = cta_compact<kTcThreads>(nb_chunk, sw, jpos, [&](int p) { return ord32(hi[p]) >= tau; });
    __syncthreads();
    sel_stamp(tr, 2);
    sel_stamp(tr, 7, (unsigned long long)n_cand);

    // ---- exact fp64 rescoring of the candidates (the oracle's arithmetic) ----
    // A candidate's 512 B of metadata are 32 scattered 16-byte pieces of its
    // tile; a batch of candidates is first staged into shared memory by the
    // whole CTA with cp.async (all pieces in flight at once), then each thread
    // rescores one candidate from shared memory.  (Loading them per thread
    // serialised ~8 global round trips per candidate.)
    {
        // one batch of (up to) kTcThreads candidates per round trip: ~k + a few
        // candidates fit at once (the former stage, behind the merge's key space,
        // held 32: five DRAM round trips with one warp rescoring, r02ac)
        unsigned char* cstage = smem_raw + (((size_t)CH * 4 + (size_t)n_cand * 8 + 127) & ~(size_t)127);
        const int stage_end = region_bytes + 8 * CH;  // end of hi[]
        const int batch = max(1, min(kTcThreads, (stage_end - (int)(cstage - smem_raw)) / 512));
        for (int base = 0; base < n_cand; base += batch) {
            const int nbt = min(batch, n_cand - base);
            for (int i = tid; i < nbt * 32; i += kTcThreads) {
                const int ci2 = i >> 5, pc = i & 31;       // candidate, piece (chunk s = pc / 2, min|max = pc % 2)
                const int p = jpos[base + ci2];
                const char* src = meta_pair + (size_t)(j0 / 32 + p / 32) * kTileBytes + (size_t)pc * 512 + (p % 32) * 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(cstage + ci2 * 512 + pc * 16)),
                             "l"(src)
                             : "memory");
            }
            asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
            __syncthreads();
            if (tid < nbt) {
                const uint4* cp = reinterpret_cast<const uint4*>(cstage + tid * 512);
                double acc[G];
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll 4
                for (int s = 0; s < 16; ++s) {
                    const uint4 wn4 = cp[2 * s], wx4 = cp[2 * s + 1];
                    const uint32_t wn[4] = {wn4.x, wn4.y, wn4.z, wn4.w};
                    const uint32_t wx[4] = {wx4.x, wx4.y, wx4.z, wx4.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int w = e >> 1, ch = 8 * s + e;
                        const int32_t hN = (e & 1) ? bf16_hi_hiword(wn[w]) : bf16_lo_hiword(wn[w]);
                        const int32_t hM = (e & 1) ? bf16_hi_hiword(wx[w]) : bf16_lo_hiword(wx[w]);
                        const int32_t dd = hM ^ hN;
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            acc[g] = __fma_rn(qs[ch * G + g], __hiloint2double(hN ^ (qf[ch * G + g] & dd), 0), acc[g]);
                    }
                }
                double sc = acc[0];
#pragma unroll
                for (int g = 1; g < G; ++g) sc = acc[g] > sc ? acc[g] : sc;
                ckeys[base + tid] = ord_key(sc + 0.0);
            }
            __syncthreads();
        }
    }

    sel_stamp(tr, 3);
    // ---- exact top-k among the candidates (positions ascending = j ascending) ----
    int32_t* sel_pair = sel + (size_t)pair * k;
    if (nch_b == 1) {
        cta_topk_t<kTcThreads, true, true>(ckeys, n_cand, kk, hist, sw, [&](int o, int pp) { sel_pair[o] = j0 + jpos[pp]; });
        for (int rr2 = kk + tid; rr2 < k; rr2 += kTcThreads) sel_pair[rr2] = -1;
        return;
    }
    uint64_t* ck = cand_key + ((size_t)pair * nchunks + ci) * k;
    int32_t* cj = cand_j + ((size_t)pair * nchunks + ci) * k;
    cta_topk_t<kTcThreads, true, true>(ckeys, n_cand, kk, hist, sw, [&](int o, int pp) {
        ck[o] = ckeys[pp];
        cj[o] = j0 + jpos[pp];
    });
    sel_stamp(tr, 4);
    __threadfence();
    __syncthreads();
    if (tid == 0) sw[48] = atomicAdd(&tickets[pair], 1);
    __syncthreads();
    if (sw[48] != nch_b - 1) return;
    __threadfence();
    sel_stamp(tr, 5);
    // merge layout: every chunk's candidates' keys, then their positions
    int32_t* mjpos = (int32_t*)(smem_raw + (size_t)max(CH, min(nchunks * k, kSelMaxMerge)) * 8);
    int n = 0;
    for (int cc = 0; cc < nch_b; ++cc) {
        const int sz = min(CH, nb - cc * CH);
        const int kcc = min(k, sz);
        const uint64_t* sk = cand_key + ((size_t)pair * nchunks + cc) * k;
        const int32_t* sj = cand_j + ((size_t)pair * nchunks + cc) * k;
        for (int i = tid; i < kcc; i += kTcThreads) {
            keys[n + i] = __ldcg(sk + i);
            mjpos[n + i] = __ldcg(sj + i);
        }
        n += kcc;
    }
    __syncthreads();
    const int kf = min(k, nb);
    cta_topk_t<kTcThreads, true, true>(keys, n, kf, hist, sw, [&](int o, int pp) { sel_pair[o] = mjpos[pp]; });
    for (int rr2 = kf + tid; rr2 < k; rr2 += kTcThreads) sel_pair[rr2] = -1;
    if (tid == 0) tickets[pair] = 0;
    sel_stamp(tr, 6);
}

// ---------------------------------------------------------------------------
// Cluster form of the tensor-core GQA select (the default for bf16 GQA).  The
// CS chunks of one (b, h) pair are the CS CTAs of one thread-block cluster, so
// the candidate threshold is taken over the WHOLE pair instead of per chunk:
//   1. tile phase as block_select_tc_kernel: approximate f32 scores with error
//      bounds, L_j <= S_j <= U_j, for the CTA's chunk;
//   2. tau' <= the k-th largest L_j of the pair, through distributed shared
//      memory: cluster min / max of the finite L, a 256-bin histogram LINEAR in
//      the value of L (monotone bins, few keys per bin -- the 8-bit radix digits
//      of the ordered keys put most keys into one or two bins whose shared
//      atomics serialise, r02ac), the bin b* holding the k-th largest, and tau'
//      = the smallest L in bin b* (<= the k-th largest);
//   3. candidates U_j >= tau' (and every block whose approximation is not
//      finite) are rescored EXACTLY (the oracle's fp64 sum): ~k per PAIR
//      instead of ~k per chunk, i.e. CS x fewer scattered 512-byte metadata
//      re-reads from DRAM -- those re-reads, issued by every CTA at once, were
//      the largest cost of the per-chunk form (r02ac/r02ad);
//   4. each CTA keeps its exact top-k (only when it has more than k
//      candidates) and writes (key, j) into the leader CTA's shared memory at
//      its rank's offset -- ascending j across the cluster -- and the leader
//      takes the exact top-k (ties -> lower j) and writes sel.
// Exactness: k blocks have S >= L >= (k-th largest L) >= tau', so a block with
// U < tau' has S < tau' and is beaten by k blocks; the union of the CTAs' exact
// local top-k sets contains the pair's exact top-k.  No global workspace, no
// tickets, no second launch-wide merge.
// ---------------------------------------------------------------------------
constexpr int kTccMaxCluster = 16;

template <int G, int NS>
__global__ void __launch_bounds__(kTcThreads, NS == 1 ? 2 : 1)
block_select_tcc_kernel(const void* __restrict__ q, const void* __restrict__ meta,
                        const int32_t* __restrict__ n_blk_arr, int max_blk, int k, int Hq, int Hkv,
                        int CS, int CH, int region_bytes, int tr, int32_t* __restrict__ sel,
                        const __grid_constant__ CUtensorMap tm_cand) {
    extern __shared__ __align__(128) unsigned char tc_smem[];
    unsigned char* smem_raw = tc_smem;
    // [region: tile stages | candidate positions, keys, rescoring stage | leader
    //  gather (key u64, j i32) at gather_off] [lo f32 [CH]][hi f32 [CH]]
    // [qs f64 [128 G]][qf i32 [128 G]][hist 256][sw 64][xch 32 x u64][bars]
    unsigned char* stage_base = smem_raw;
    float* lo = (float*)(smem_raw + region_bytes);
    float* hi = lo + CH;
    double* qs = (double*)(hi + CH);
    int32_t* qf = (int32_t*)(qs + kHeadDim * G);
    int* hist = (int*)(qf + kHeadDim * G);
    int* sw = hist + 256;
    unsigned long long* xch = (unsigned long long*)(sw + 64);  // cluster exchange slots
    uint64_t* bars = (uint64_t*)(xch + 32);
    cg::cluster_group cluster = cg::this_cluster();
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    sel_stamp(tr, 0);
    const int rank = (int)cluster.block_rank();
    const int pair = blockIdx.x / CS, ci = rank;
    const int b = pair / Hkv, h = pair % Hkv;
    const int nb = n_blk_arr[b];
    int32_t* sel_pair = sel + (size_t)pair * k;
    if (k >= nb) {  // every block is selected (uniform over the cluster: no barrier)
        if (rank == 0)
            for (int i = tid; i < k; i += kTcThreads) sel_pair[i] = i < nb ? i : -1;
        return;
    }
    const int j0 = ci * CH;
    const int nb_chunk = max(0, min(CH, nb - j0));
    const char* meta_pair = (const char*)meta + ((size_t)pair * (max_blk / 32)) * kTileBytes;
    const uint16_t* qb16 = (const uint16_t*)q + ((size_t)b * Hq + (size_t)h * G) * kHeadDim;

    for (int i = tid; i < kHeadDim * G; i += kTcThreads) {
        const int g = i % G, c = i / G;
        const double qd = (double)__uint_as_float(((uint32_t)qb16[(size_t)g * kHeadDim + c]) << 16) * kQScale;
        qs[i] = qd;
        qf[i] = qd >= 0.0 ? -1 : 0;
    }
    for (int i = tid; i < 256; i += kTcThreads) hist[i] = 0;
    if (lane == 0) {
#pragma unroll
        for (int st = 0; st < NS; ++st) mbar_init(&bars[warp * NS + st], 1);
        if (warp == 0) mbar_init(&bars[kTcWarps * NS], 1);  // candidate rescoring loads
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const int r = lane >> 2, c = lane & 3;
    uint32_t qb[16][2], qa[16][2];
#pragma unroll
    for (int s2 = 0; s2 < 16; ++s2) {
        uint32_t w = 0;
        if (r < G) w = __ldg(reinterpret_cast<const uint32_t*>(qb16 + (size_t)r * kHeadDim + 8 * s2 + 2 * c));
        const uint32_t neg = ((w & 0x8000u) ? 0x0000FFFFu : 0u) | ((w & 0x80000000u) ? 0xFFFF0000u : 0u);
        qb[s2][0] = w & neg;
        qb[s2][1] = w & ~neg;
        qa[s2][0] = qb[s2][0] & 0x7FFF7FFFu;
        qa[s2][1] = qb[s2][1] & 0x7FFF7FFFu;
    }
    __syncthreads();

    // ---- 1. tile phase, tiles of the PAIR handed out dynamically ----
    // (a static split left the cluster's CTAs 7.6 us apart at the end of the
    // phase -- CTAs sharing an SM stream slower -- and every cluster barrier
    // waits for the slowest, r02ad).  A warp takes tile t of the pair from a
    // counter in the leader's shared memory (DSMEM atomic, issued one tile
    // ahead), and writes its blocks' (L, U) into the OWNER CTA's lo / hi
    // (t*32 / CH), plus its own running min / max / count of the finite L.
    int* ctr_local = reinterpret_cast<int*>(&xch[31]);
    if (tid == 0) *ctr_local = 0;
    cluster.sync();  // #0: the leader's counter is zero; every CTA resident
    int* ctr = cluster.map_shared_rank(ctr_local, 0);
    const int ntiles_pair = (nb + 31) / 32;
    auto issue = [&](int st, int t) {
        if (lane == 0 && t < ntiles_pair) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            mbar_expect_tx(&bars[warp * NS + st], kTileBytes);
            bulk_g2s(stage_base + (size_t)(warp * NS + st) * kTileBytes, meta_pair + (size_t)t * kTileBytes,
                     kTileBytes, &bars[warp * NS + st]);
        }
    };
    int t_st0 = 0, t_st1 = 0;  // tile held by stage 0 / 1
    {
        int t0 = 0;
        if (lane == 0) t0 = atomicAdd(ctr, 1);
        t_st0 = __shfl_sync(0xffffffffu, t0, 0);
        issue(0, t_st0);
        if (NS == 2) {
            if (lane == 0) t0 = atomicAdd(ctr, 1);
            t_st1 = __shfl_sync(0xffffffffu, t0, 0);
            issue(1, t_st1);
        }
    }
    int pre_raw = 0;  // lane 0: the next tile index, requested one tile ahead
    if (lane == 0) pre_raw = atomicAdd(ctr, 1);
    float lmn = INFINITY, lmx = -INFINITY;
    int lcnt = 0;
    uint32_t phases = 0;
    const int mi = lane >> 3, rr = lane & 7;
    const uint32_t a_off = (uint32_t)((mi >> 1) * 512 + (8 * (mi & 1) + rr) * 16);
    for (int i = 0;; ++i) {
        const int st = NS == 2 ? (i & 1) : 0;
        const int t = st ? t_st1 : t_st0;
        if (t >= ntiles_pair) break;  // later grabs are larger: nothing left for this warp
        mbar_wait(&bars[warp * NS + st], (phases >> st) & 1u);
        phases ^= 1u << st;
        const uint32_t sb = smem_u32(stage_base + (size_t)(warp * NS + st) * kTileBytes);
        float ds[2][4], da[2][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 4; ++e) ds[mt][e] = da[mt][e] = 0.f;
#pragma unroll
        for (int s2 = 0; s2 < 16; ++s2) {
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                uint32_t af[4];
                ldsm_x4(sb + s2 * 1024 + mt * 256 + a_off, af);
                hmma(ds[mt], af, qb[s2][0], qb[s2][1]);
                af[0] &= 0x7FFF7FFFu;
                af[1] &= 0x7FFF7FFFu;
                af[2] &= 0x7FFF7FFFu;
                af[3] &= 0x7FFF7FFFu;
                hmma(da[mt], af, qa[s2][0], qa[s2][1]);
            }
        }
        __syncwarp();
        {   // the stage is consumed: the pre-requested tile into it, request the next
            const int tn = __shfl_sync(0xffffffffu, pre_raw, 0);
            if (st) t_st1 = tn; else t_st0 = tn;
            issue(st, tn);
            if (lane == 0 && tn < ntiles_pair) pre_raw = atomicAdd(ctr, 1);
        }
        const int owner = t * 32 / CH;
        float* lo_o = cluster.map_shared_rank(lo, owner);
        float* hi_o = cluster.map_shared_rank(hi, owner);
        const int jbase = t * 32 - owner * CH;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int half = 0; half < 2; ++half) {
                float sv = -INFINITY, av = 0.f;
                int bad = 0;
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    if (2 * c + e < G) {
                        const float dv = ds[mt][2 * half + e], dav = da[mt][2 * half + e];
                        bad |= !(fabsf(dv) <= 3.0e38f) || !(dav <= 3.0e38f);
                        sv = fmaxf(sv, dv);
                        av = fmaxf(av, dav);
                    }
                }
                sv = fmaxf(sv, __shfl_xor_sync(0xffffffffu, sv, 1));
                sv = fmaxf(sv, __shfl_xor_sync(0xffffffffu, sv, 2));
                av = fmaxf(av, __shfl_xor_sync(0xffffffffu, av, 1));
                av = fmaxf(av, __shfl_xor_sync(0xffffffffu, av, 2));
                bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
                bad |= __shfl_xor_sync(0xffffffffu, bad, 2);
                const int rel = 16 * mt + 8 * half + r;
                if (c == 0 && t * 32 + rel < nb) {
                    const float eps = __fmaf_ru(av, 0x1p-10f, 0x1p-100f);
                    if (bad != 0 || !(eps <= 3.0e38f)) {
                        lo_o[jbase + rel] = -INFINITY;
                        hi_o[jbase + rel] = INFINITY;
                    } else {
                        const float lv = __fsub_rd(sv, eps);
                        lo_o[jbase + rel] = lv;
                        hi_o[jbase + rel] = __fadd_ru(sv, eps);
                        lmn = fminf(lmn, lv);
                        lmx = fmaxf(lmx, lv);
                        ++lcnt;
                    }
                }
            }
    }
    sel_stamp(tr, 1);

    // ---- 2. tau' over the pair (distributed shared memory) ----
    const int kk = k;  // < nb here
    // (a) finite-L min / max / count of the L this CTA computed -> own xch[0..2]
    {
        float mn = lmn, mx = lmx;
        int cnt = lcnt;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        if (lane == 0) {
            sw[warp] = __float_as_int(mn);
            sw[8 + warp] = __float_as_int(mx);
            sw[16 + warp] = cnt;
        }
        __syncthreads();
        if (tid == 0) {  // (warp 0's values are this thread's)
            for (int wi = 1; wi < kTcWarps; ++wi) {
                mn = fminf(mn, __int_as_float(sw[wi]));
                mx = fmaxf(mx, __int_as_float(sw[8 + wi]));
                cnt += sw[16 + wi];
            }
            xch[0] = (unsigned long long)(uint32_t)__float_as_int(mn);
            xch[1] = (unsigned long long)(uint32_t)__float_as_int(mx);
            xch[2] = (unsigned long long)cnt;
        }
    }
    cluster.sync();  // #1: every lo / hi complete; every CTA's (min, max, count) visible
    float Lmin = INFINITY, Lmax = -INFINITY;
    int nfin = 0;
    for (int rk = 0; rk < CS; ++rk) {
        const unsigned long long* rx = cluster.map_shared_rank(xch, rk);
        Lmin = fminf(Lmin, __int_as_float((int)(uint32_t)rx[0]));
        Lmax = fmaxf(Lmax, __int_as_float((int)(uint32_t)rx[1]));
        nfin += (int)rx[2];
    }
    float tau = -INFINITY;  // every block a candidate unless k finite L exist
    if (nfin >= kk) {
        // (b) linear histogram of the finite L over [Lmin, Lmax]
        const float scale = Lmax > Lmin ? 256.f / (Lmax - Lmin) : 0.f;
        auto bin_of = [&](float v) { return min(255, (int)((v - Lmin) * scale)); };
        for (int i = tid; i < nb_chunk; i += kTcThreads) {
            const float v = lo[i];
            if (v != -INFINITY) atomicAdd(&hist[bin_of(v)], 1);
        }
        cluster.sync();  // #2
        // every CTA sums the cluster's histograms (bins tid, tid + 128) and finds b*
        int tot0 = 0, tot1 = 0;
        for (int rk = 0; rk < CS; ++rk) {
            const int* rh = cluster.map_shared_rank(hist, rk);
            tot0 += rh[tid];
            tot1 += rh[tid + 128];
        }
        cluster.sync();  // #3: remote reads of hist done before it is reused
        hist[tid] = tot0;
        hist[tid + 128] = tot1;
        __syncthreads();
        if (tid < 32) {
            int cnt8[8], s8 = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                cnt8[i] = hist[255 - (tid * 8 + i)];
                s8 += cnt8[i];
            }
            const int incl = warp_incl_scan(s8);
            int above = incl - s8;
            if (above < kk && kk <= incl) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (above < kk && kk <= above + cnt8[i]) sw[40] = 255 - (tid * 8 + i);
                    above += cnt8[i];
                }
            }
        }
        __syncthreads();
        const int bstar = sw[40];
        // (c) tau' = a lower edge of bin b*, one bin wide of margin: a key v in
        // bin b* has fl(fl(v - Lmin) * scale) >= b*, so v >= Lmin + (b* - 1) /
        // scale whatever the two roundings did (each is relative 2^-24; the
        // margin is a whole bin), and tau' <= the k-th largest L.  (Taking the
        // smallest L of bin b* instead cost one more pass and cluster barrier.)
        tau = bstar >= 1 ? __fsub_rd(Lmin, 0.f) + __fdiv_rd((float)(bstar - 1), scale) : -INFINITY;
        if (!(tau <= Lmax)) tau = -INFINITY;  // (scale overflowed / NaN: every block a candidate)
    }
    sel_stamp(tr, 2);

    // ---- 3. candidates of this chunk (U >= tau'), rescored exactly ----
    int32_t* jpos = (int32_t*)smem_raw;                    // [<= CH]
    uint64_t* ckeys = (uint64_t*)(smem_raw + (size_t)CH * 4);
    const int n_cand = cta_compact<kTcThreads>(nb_chunk, sw, jpos, [&](int p2) { return hi[p2] >= tau; });
    sel_stamp(tr, 7, (unsigned long long)n_cand);
    __syncthreads();
    sel_stamp(tr, 9);
    {
        uint32_t rphase = 0;
        unsigned char* cstage = smem_raw + (((size_t)CH * 4 + (size_t)n_cand * 8 + 127) & ~(size_t)127);
        const int stage_end = region_bytes + 8 * CH;
        const int batch = max(1, min(kTcThreads, (stage_end - (int)(cstage - smem_raw)) / 512));
        for (int base = 0; base < n_cand; base += batch) {
            const int nbt = min(batch, n_cand - base);
            // one 2-D TMA per candidate: its 32 16-byte pieces (one per (channel
            // chunk, min|max) row of its tile, 512 B apart) as ONE box of the
            // [rows][256] bf16 view of the metadata -- instead of 32 cp.async per
            // candidate (~600 outstanding 16-byte requests per CTA, r02ah)
            if (tid == 0) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_expect_tx(&bars[kTcWarps * NS], (uint32_t)(nbt * 512));
            }
            __syncthreads();
            if (tid < nbt) {
                const int p2 = jpos[base + tid];
                const int64_t blk = (int64_t)pair * max_blk + j0 + p2;  // the block's index in the whole array
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(cstage + tid * 512)),
                    "l"(reinterpret_cast<uint64_t>(&tm_cand)), "r"((int)(blk % 32) * 8), "r"((int)(blk / 32) * 32),
                    "r"(smem_u32(&bars[kTcWarps * NS]))
                    : "memory");
            }
            mbar_wait(&bars[kTcWarps * NS], rphase);
            rphase ^= 1u;
            if (base == 0) sel_stamp(tr, 8);
            if (tid < nbt) {
                const uint4* cp = reinterpret_cast<const uint4*>(cstage + tid * 512);
                double acc[G];
#pragma unroll
                for (int g = 0; g < G; ++g) acc[g] = 0.0;
#pragma unroll 4
                for (int s2 = 0; s2 < 16; ++s2) {
                    const uint4 wn4 = cp[2 * s2], wx4 = cp[2 * s2 + 1];
                    const uint32_t wn[4] = {wn4.x, wn4.y, wn4.z, wn4.w};
                    const uint32_t wx[4] = {wx4.x, wx4.y, wx4.z, wx4.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        const int w2 = e >> 1, ch = 8 * s2 + e;
                        const int32_t hN = (e & 1) ? bf16_hi_hiword(wn[w2]) : bf16_lo_hiword(wn[w2]);
                        const int32_t hM = (e & 1) ? bf16_hi_hiword(wx[w2]) : bf16_lo_hiword(wx[w2]);
                        const int32_t dd = hM ^ hN;
#pragma unroll
                        for (int g = 0; g < G; ++g)
                            acc[g] = __fma_rn(qs[ch * G + g], __hiloint2double(hN ^ (qf[ch * G + g] & dd), 0), acc[g]);
                    }
                }
                double sc = acc[0];
#pragma unroll
                for (int g = 1; g < G; ++g) sc = acc[g] > sc ? acc[g] : sc;
                ckeys[base + tid] = ord_key(sc + 0.0);
            }
            __syncthreads();
        }
    }
    sel_stamp(tr, 3);

    // ---- 4. (local exact top-k) -> the leader's gather area -> exact top-k ----
    const int n_out = min(n_cand, kk);
    if (tid == 0) xch[4] = (unsigned long long)n_out;
    cluster.sync();  // #5: counts visible; every CTA done with its own stage
    int off = 0, n_all = 0;  // this CTA's offset in the gathered list; its total (read before
    for (int rk = 0; rk < CS; ++rk) {  // the last barrier: the other CTAs exit after it)
        const int cr = (int)cluster.map_shared_rank(xch, rk)[4];
        off += rk < rank ? cr : 0;
        n_all += cr;
    }
    const int gather_off = CH * 12;  // leader region: [positions | keys] of its own candidates below
    unsigned char* lead = cluster.map_shared_rank(smem_raw, 0);
    uint64_t* gkey = reinterpret_cast<uint64_t*>(lead + gather_off);
    int32_t* gj = reinterpret_cast<int32_t*>(lead + gather_off + (size_t)CS * kk * 8);
    if (n_cand > kk) {
        cta_topk_t<kTcThreads, true, true>(ckeys, n_cand, kk, hist, sw, [&](int o, int pp) {
            gkey[off + o] = ckeys[pp];
            gj[off + o] = j0 + jpos[pp];
        });
    } else {
        for (int i = tid; i < n_cand; i += kTcThreads) {
            gkey[off + i] = ckeys[i];
            gj[off + i] = j0 + jpos[i];
        }
    }
    sel_stamp(tr, 4);
    cluster.sync();  // #6: the gathered list complete in the leader
    if (rank != 0) return;
    sel_stamp(tr, 5);
    const uint64_t* lkeys = reinterpret_cast<const uint64_t*>(smem_raw + gather_off);
    const int32_t* lj = reinterpret_cast<const int32_t*>(smem_raw + gather_off + (size_t)CS * kk * 8);
    cta_topk_t<kTcThreads, true, true>(lkeys, n_all, kk, hist, sw, [&](int o, int pp) { sel_pair[o] = lj[pp]; });
    sel_stamp(tr, 6);
}

// Blocks scored per CTA (the chunk): 1024 for MHA (G = 1), 2048 for GQA
// (G > 1: 4-8x the fp64 work per block, so longer CTAs amortise the q setup and
// the top-k).  Measured (tools/kbench.py, C2 / C3 full batch and one request
// group): a chooser that sized chunks to fill whole waves of resident CTAs lost
// to these fixed sizes everywhere (smaller chunks pay more top-k and merge work
// than the wave tail costs).  SS_SEL_CHUNK (multiple of 32, <= 4096) overrides.
static int sel_chunk_env() {
    int v = knob("SS_SEL_CHUNK", 0);  // debug build only
    if (v != 0 && (v < 32 || v > kSelChunkMax || (v % 32))) v = kSelChunkMax;
    return v;
}
constexpr int kSelChunkMin = 512;  // workspace sizing bound (SS_SEL_CHUNK may go lower)

// The chunk a call uses; doubled (up to kSelChunkMax) while the candidate merge
// of the pair's chunks would exceed kSelMaxMerge keys (its shared-memory bound).
// MHA (G = 1) chunk chooser: c chunks per pair of CH = ceil(max_blk / c)
// blocks (multiple of 32, >= kSelChunkMin); a CTA's time is ~proportional to
// its chunk, so a launch costs ~ceil(pairs * c / resident CTAs) waves x CH.
// Minimise that, ties -> fewer waves.  Full C2 batch (512 pairs): c = 4 (the
// round-1 1024); one request group (96 / 128 pairs): c = 3 / 2 -- one wave
// instead of 1.3 / 1.7 (measured alone, tools/kbench.py --batch 3 / 4: 0.73 /
// 0.78 of HBM vs 0.58 / 0.73 at 1024; profiles/r02_group_shape_sweep.txt).
// GQA (G > 1) keeps 2048: there the CTAs are issue-bound and more of them in
// flight beat whole waves (C3: 1.73 waves at 2048 157 us vs one wave at 4096
// 165 us, 1.19 waves at 3072 191 us).
static int sel_chunk_mha(int max_blk, int pairs) {
    const int resident = 2 * num_sms();  // __launch_bounds__(kSelThreads, 2)
    int best_ch = kSelChunkDefault;
    int64_t best_cost = INT64_MAX, best_waves = INT64_MAX;
    for (int c = 1; c <= 16; ++c) {
        const int ch = ((max_blk + c - 1) / c + 31) / 32 * 32;
        if (ch > kSelChunkMax) continue;
        if (ch < kSelChunkMin) break;
        const int chunks = (max_blk + ch - 1) / ch;
        const int64_t waves = ((int64_t)pairs * chunks + resident - 1) / resident;
        const int64_t cost = waves * ch;
        if (cost < best_cost || (cost == best_cost && waves < best_waves)) {
            best_cost = cost;
            best_waves = waves;
            best_ch = ch;
        }
    }
    return best_ch;
}

static int sel_chunk(int G, int max_blk, int k, int pairs) {
    int ch = sel_chunk_env() ? sel_chunk_env()
                             : (G > 1 ? kSelChunkGqa : sel_chunk_mha(max_blk, pairs));
    while ((size_t)((max_blk + ch - 1) / ch) * k > kSelMaxMerge && ch < kSelChunkMax) ch *= 2;
    return ch;
}

// Workspace: tickets [pairs] first (fixed place: they must stay zero between
// calls whatever chunk size a call picks), then the chunk candidates, sized for
// the smallest chunk.
size_t select_ws_bytes(const ss_dims& d, int max_blk, int k) {
    const int G = d.num_kv_heads > 0 ? d.num_q_heads / d.num_kv_heads : 1;
    const int ch = sel_chunk_env() ? sel_chunk_env() : kSelChunkMin;
    (void)G;
    int nchunks = (max_blk + ch - 1) / ch;
    size_t pairs = (size_t)d.batch * d.num_kv_heads;
    size_t nc = (size_t)pairs * nchunks * k;
    size_t bytes = ((pairs * 4 + 255) & ~(size_t)255) + nc * 8 + nc * 4;
    return (bytes + 255) & ~(size_t)255;
}

// MHA cluster form (block_select_kernel<..., CLU = true>): one cluster of
// nchunks CTAs per pair when no scores are requested and the pair has <= 8
// chunks; returns SS_ERR_UNSUPPORTED otherwise (the caller uses the workspace
// merge form).
template <bool BF16>
static ss_status launch_sel_mha_clu(const void* q, const void* meta, const int32_t* n_blk, int max_blk, int k,
                                    const ss_dims& d, int32_t* sel, cudaStream_t stream) {
    const size_t pairs = (size_t)d.batch * d.num_kv_heads;
    auto kern = block_select_kernel<BF16, 1, true, false, 2, true>;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kSelThreads);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // Only when every cluster is resident at once: a cluster's CTAs wait for
    // each other at five barriers, so in a multi-wave launch they hold SM slots
    // the next wave needs (measured: C2 full batch 213 vs 194 us; one C2 group
    // in clusters of 3, whose 96 clusters did not all fit, 62 vs 45 us; a group
    // in clusters of 2, all resident, 53 vs 56 us; r02an).  The chunk chooser's
    // chunk count is the cluster size; when its clusters do not all fit,
    // SS_ERR_UNSUPPORTED (the workspace form; measured: a smaller cluster of
    // longer chunks that fits was slower, one C2 group 46.8 vs 45.3 us, r02an).
    static int cached[9][2] = {};  // [cluster size] -> (smem, max active clusters)
    const int CH0 = sel_chunk(1, max_blk, k, (int)pairs);
    for (int cs = (max_blk + CH0 - 1) / CH0; cs >= 2 && cs == (max_blk + CH0 - 1) / CH0; --cs) {
        if (cs > 8) continue;
        const int CH = ((max_blk + cs - 1) / cs + 31) / 32 * 32;
        if (CH > kSelChunkMax) break;
        const int nchunks = (max_blk + CH - 1) / CH;
        if (nchunks != cs) continue;
        const int nkeys = max(CH, min(nchunks * k, kSelMaxMerge));
        const size_t smem = SelSmemLayout::bytes(1, nkeys) + 32 * 8 + (size_t)CH * 8 + (size_t)nchunks * k * 12;
        if (smem > 110 * 1024) continue;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
            return SS_ERR_CUDA;
        cfg.dynamicSmemBytes = smem;
        attr[0].val.clusterDim.x = (unsigned)nchunks;
        if (cached[cs][0] != (int)smem) {
            int nclu = 0;
            cfg.gridDim = dim3((unsigned)nchunks);
            if (cudaOccupancyMaxActiveClusters(&nclu, kern, &cfg) != cudaSuccess) nclu = 0;
            cached[cs][0] = (int)smem;
            cached[cs][1] = nclu;
        }
        if ((size_t)cached[cs][1] < pairs) continue;
        set_carveout(kern);
        cfg.gridDim = dim3((unsigned)(pairs * nchunks));
        const int l2pf = knob("SS_SEL_TRACE", 0) ? 16 : 0;
        if (cudaLaunchKernelEx(&cfg, kern, q, meta, n_blk, max_blk, k, (int)d.num_q_heads, (int)d.num_kv_heads,
                               nchunks, CH, (int)pairs, l2pf, sel, (double*)nullptr, (uint64_t*)nullptr,
                               (int32_t*)nullptr, (int32_t*)nullptr) != cudaSuccess)
            return SS_ERR_CUDA;
        return SS_OK;
    }
    return SS_ERR_UNSUPPORTED;
}

template <bool BF16, int G, bool ICV, bool MEAN, int TT = 2>
static ss_status launch_sel_t(const void* q, const void* meta, const int32_t* n_blk, int max_blk,
                              int k, const ss_dims& d, int32_t* sel, double* scores, void* ws,
                              cudaStream_t stream) {
    if constexpr (G == 1 && ICV && !MEAN) {
        if (scores == nullptr && knob("SS_SEL_MHA_CLU", 1) != 0) {
            const ss_status st = launch_sel_mha_clu<BF16>(q, meta, n_blk, max_blk, k, d, sel, stream);
            if (st != SS_ERR_UNSUPPORTED) return st;
        }
    }
    size_t pairs = (size_t)d.batch * d.num_kv_heads;
    const int CH = sel_chunk(G, max_blk, k, (int)pairs);
    int nchunks = (max_blk + CH - 1) / CH;
    size_t nc = pairs * nchunks * k;
    int32_t* tickets = (int32_t*)ws;
    uint64_t* cand_key = (uint64_t*)((char*)ws + ((pairs * 4 + 255) & ~(size_t)255));
    int32_t* cand_j = (int32_t*)((char*)cand_key + nc * 8);
    int nkeys = max(CH, min(nchunks * k, kSelMaxMerge));
    size_t smem = SelSmemLayout::bytes(G, nkeys);
    auto kern = block_select_kernel<BF16, G, ICV, MEAN, TT>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
        cudaSuccess)
        return SS_ERR_CUDA;
    const int items = nchunks * (int)pairs;
    // (measured: both the persistent grid and the L2 tile prefetch were slower
    // than a plain one-CTA-per-item grid; kept switchable for experiments)
    const int persist = knob("SS_SEL_PERSIST", 0);
    const int l2pf = knob("SS_SEL_L2PF", 0) | (knob("SS_SEL_TRACE", 0) ? 16 : 0);
    const int grid = (persist && items > 2 * num_sms()) ? 2 * num_sms() : items;
    set_carveout(kern);
    kern<<<grid, kSelThreads, smem, stream>>>(q, meta, n_blk, max_blk, k, d.num_q_heads,
                                              d.num_kv_heads, nchunks, CH, (int)pairs, l2pf, sel, scores, cand_key,
                                              cand_j, tickets);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

template <int G>
static ss_status launch_sel_tc(const void* q, const void* meta, const int32_t* n_blk, int max_blk, int k,
                               const ss_dims& d, int32_t* sel, void* ws, cudaStream_t stream) {
    const size_t pairs = (size_t)d.batch * d.num_kv_heads;
    // the largest chunk (<= 4096 blocks: fewer per-CTA threshold / rescoring /
    // top-k epilogues; C3 full batch: 138 us at 4096 vs 155 at 2048) that still
    // gives ~a wave of resident CTAs (2 per SM): one C3 request (8 pairs) gets
    // 1024-block chunks instead of 64 CTAs on 148 SMs
    int CH = kSelChunkMax;
    const int64_t target = (int64_t)2 * num_sms() * 4 / 5;
    while (CH > kSelChunkMin && (int64_t)pairs * ((max_blk + CH - 1) / CH) < target) CH /= 2;
    if (sel_chunk_env()) CH = sel_chunk_env();
    while ((size_t)((max_blk + CH - 1) / CH) * k > kSelMaxMerge && CH < kSelChunkMax) CH *= 2;
    const int nchunks = (max_blk + CH - 1) / CH;
    const size_t nc = pairs * nchunks * k;
    int32_t* tickets = (int32_t*)ws;
    uint64_t* cand_key = (uint64_t*)((char*)ws + ((pairs * 4 + 255) & ~(size_t)255));
    int32_t* cand_j = (int32_t*)((char*)cand_key + nc * 8);
    const int cap = std::max(CH, std::min(nchunks * k, kSelMaxMerge));
    const int ns = knob("SS_SEL_TC_STAGES", kSelTcStages) >= 2 ? 2 : 1;
    // region: the tile stages, later keys + positions + a candidate stage (>= 32 x 512 B)
    const int region = std::max(kTcWarps * ns * kTileBytes, ((cap * 12) + 127) / 128 * 128 + 32 * 512);
    const size_t smem = (size_t)region + (size_t)CH * 8 + (size_t)kHeadDim * G * 12 + 256 * 4 + 64 * 4 + 64;
    const int rot_mul = knob("SS_SEL_ROT", kSelTcRot);
    auto kern = ns == 2 ? block_select_tc_kernel<G, 2> : block_select_tc_kernel<G, 1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SS_ERR_CUDA;
    set_carveout(kern);
    kern<<<nchunks * (int)pairs, kTcThreads, smem, stream>>>(q, meta, n_blk, max_blk, k, d.num_q_heads,
                                                              d.num_kv_heads, nchunks, CH, region, rot_mul,
                                                              knob("SS_SEL_TC_PF", kSelTcPf), knob("SS_SEL_TRACE", 0), sel,
                                                              cand_key, cand_j, tickets);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

// Cluster form (block_select_tcc_kernel): CS CTAs per pair (power of two <= 16,
// chunks <= 4096 blocks), doubled while the launch has fewer than ~0.8 of a wave
// of CTAs; two tile stages per warp and one CTA per SM when the launch has at
// most one CTA per SM.  Returns SS_ERR_UNSUPPORTED when the shape does not fit
// (the caller falls back to the per-chunk form).
template <int G>
static ss_status launch_sel_tcc(const void* q, const void* meta, const int32_t* n_blk, int max_blk, int k,
                                const ss_dims& d, int32_t* sel, cudaStream_t stream) {
    const int64_t pairs = (int64_t)d.batch * d.num_kv_heads;
    int CS = 1;
    while (CS < kTccMaxCluster && (max_blk + CS - 1) / CS > kSelChunkMax) CS *= 2;
    if ((max_blk + CS - 1) / CS > kSelChunkMax) return SS_ERR_UNSUPPORTED;
    const int64_t target = (int64_t)2 * num_sms() * 4 / 5;
    while (CS < kTccMaxCluster && pairs * CS < target && (max_blk + 2 * CS - 1) / (2 * CS) >= 256) CS *= 2;
    if (CS == 16 && pairs * 12 >= target / 2) {
        // 16-CTA clusters (8 SMs each at two CTAs per SM) do not all fit in the
        // GPCs once there are more than ~8 of them; 12-CTA clusters (6 SMs) do
        // (measured: two C3 requests 95 us in 16-CTA clusters with a partial
        // second wave, 109 us in 8-CTA clusters at one CTA per SM, r02av)
        int nclu = 0;
        cudaLaunchConfig_t oc = {};
        cudaLaunchAttribute oa[1];
        oa[0].id = cudaLaunchAttributeClusterDimension;
        oa[0].val.clusterDim.x = 16;
        oa[0].val.clusterDim.y = 1;
        oa[0].val.clusterDim.z = 1;
        oc.attrs = oa;
        oc.numAttrs = 1;
        oc.gridDim = dim3(16);
        oc.blockDim = dim3(kTcThreads);
        // max active 16-CTA clusters of the 2-CTA-per-SM form, cached per shared-memory size
        static size_t fit_smem = 0;
        static int fit16 = 0;
        const int ch16 = ((max_blk + 15) / 16 + 31) / 32 * 32;
        oc.dynamicSmemBytes = (size_t)std::max(kTcWarps * kTileBytes, ch16 * 4 + 16 * k * 12) + (size_t)ch16 * 8 +
                              (size_t)kHeadDim * G * 12 + 256 * 4 + 64 * 4 + 32 * 8 + kTcWarps * 8 + 8;
        if (fit_smem != oc.dynamicSmemBytes) {
            auto k1 = block_select_tcc_kernel<G, 1>;
            cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)oc.dynamicSmemBytes);
            cudaFuncSetAttribute(k1, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            if (cudaOccupancyMaxActiveClusters(&nclu, k1, &oc) != cudaSuccess) nclu = 0;
            fit16 = nclu;
            fit_smem = oc.dynamicSmemBytes;
        }
        if (fit16 < pairs) CS = 12;
    }
    const int CH = ((max_blk + CS - 1) / CS + 31) / 32 * 32;
    // two stages per warp (one CTA per SM) when the launch has at most one CTA
    // per SM -- except for 16-CTA clusters, which need 16 SMs of one GPC at one
    // CTA per SM and did not all fit at once (C3 one request: a second wave of
    // clusters 32 us late, r02ad)
    const int ns = (pairs * CS <= num_sms() && CS <= 8) ? 2 : 1;
    // region: the tile stages; later the candidate positions / keys and the
    // rescoring stage; in the leader the gathered (key, j) list at CH * 12 --
    // which must end before hi[] does
    const int gather_end = CH * 12 + CS * k * 12;
    const int region = std::max(kTcWarps * ns * kTileBytes, ((gather_end - 8 * CH) + 127) / 128 * 128);
    const size_t smem = (size_t)region + (size_t)CH * 8 + (size_t)kHeadDim * G * 12 + 256 * 4 + 64 * 4 + 32 * 8 +
                        (size_t)kTcWarps * ns * 8 + 8;
    // candidate loads: the metadata as [B*Hkv*max_blk][256] bf16 rows of 512 B
    // (row 32T + 2s + mm of tile T = its channel chunk s, min|max), box 8 x 32
    CUtensorMap tm_cand;
    {
        auto enc = tensor_map_encoder();
        if (enc == nullptr) return SS_ERR_CUDA;
        const cuuint64_t gdim[2] = {256, (cuuint64_t)pairs * max_blk};
        const cuuint64_t gstride[1] = {512};
        const cuuint32_t box[2] = {8, 32};
        const cuuint32_t estride[2] = {1, 1};
        if (enc(&tm_cand, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(meta), gdim, gstride, box, estride,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return SS_ERR_CUDA;
    }
    if (smem > (size_t)(ns == 1 ? 113 * 1024 : 227 * 1024)) return SS_ERR_UNSUPPORTED;
    auto kern = ns == 2 ? block_select_tcc_kernel<G, 2> : block_select_tcc_kernel<G, 1>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SS_ERR_CUDA;
    if (CS > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return SS_ERR_CUDA;
    set_carveout(kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(pairs * CS));
    cfg.blockDim = dim3(kTcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int tr = knob("SS_SEL_TRACE", 0);
    if (cudaLaunchKernelEx(&cfg, kern, q, meta, n_blk, max_blk, k, (int)d.num_q_heads, (int)d.num_kv_heads, CS, CH,
                           region, tr, sel, tm_cand) != cudaSuccess)
        return SS_ERR_CUDA;
    return SS_OK;
}

ss_status launch_block_select(const void* q, const void* meta, const int32_t* n_blk, int max_blk,
                              int k, const ss_dims& d, ss_dtype dt, int32_t* sel, double* scores,
                              void* ws, cudaStream_t stream, bool mean) {
    int G = d.num_q_heads / d.num_kv_heads;
    {   // the largest chunk must keep the candidate merge within kSelMaxMerge keys
        const int ch = sel_chunk(G, max_blk, k, d.batch * d.num_kv_heads);  // the chunk the launch will use
        const int nchunks = (max_blk + ch - 1) / ch;
        if ((size_t)nchunks * k > kSelMaxMerge && nchunks > 1) return SS_ERR_UNSUPPORTED;
    }
    // integer-built float64 operands (default) or F2F conversions (SS_SEL_ICV=0,
    // A/B only: compiled into the debug build alone)
    const bool icv = knob("SS_SEL_ICV", 1) != 0;
    // GQA tiles per warp pass: 2 (default; G = 8 uses 1, which keeps its
    // accumulators and load ring in registers) or 1 (SS_SEL_TT=1, A/B)
    const bool tt1 = knob("SS_SEL_TT", 2) == 1;
#ifdef SS_DEBUG_KNOBS
#define SS_SEL_NOICV(BF, GG) return launch_sel_t<BF, GG, false, false>(SS_SEL_ARGS);
#else
#define SS_SEL_NOICV(BF, GG) (void)0;
#endif
#define SS_SEL_ARGS q, meta, n_blk, max_blk, k, d, sel, scores, ws, stream
    // GQA bf16 selections without a scores output: tensor-core scoring + exact
    // fp64 rescoring of the candidates (block_select_tc_kernel; SS_SEL_TC=0: the
    // all-fp64 kernel, which also serves calls that ask for every score)
    const bool tc = knob("SS_SEL_TC", 1) != 0 && !mean && dt == SS_BF16 && G > 1 && scores == nullptr;
    // cluster form of it (block_select_tcc_kernel); SS_SEL_TCC=0: the per-chunk form (debug A/B)
    const bool tcc = knob("SS_SEL_TCC", 1) != 0;
#define SS_SEL_CASE(GG)                                                                       \
    case GG:                                                                                  \
        if (GG > 1 && tc) {                                                                   \
            if (tcc) {                                                                        \
                const ss_status st_ = launch_sel_tcc<(GG > 1 ? GG : 2)>(q, meta, n_blk, max_blk, k, d, sel, stream); \
                if (st_ != SS_ERR_UNSUPPORTED) return st_;                                     \
            }                                                                                 \
            return launch_sel_tc<(GG > 1 ? GG : 2)>(q, meta, n_blk, max_blk, k, d, sel, ws, stream); \
        }                                                                                     \
        if (mean)                                                                             \
            return dt == SS_BF16 ? launch_sel_t<true, GG, true, true>(SS_SEL_ARGS)            \
                                 : launch_sel_t<false, GG, true, true>(SS_SEL_ARGS);          \
        if (!icv) {                                                                           \
            if (dt == SS_BF16) { SS_SEL_NOICV(true, GG) }                                     \
            else { SS_SEL_NOICV(false, GG) }                                                  \
        }                                                                                     \
        if (GG > 1 && (tt1 || GG == 8))                                                       \
            return dt == SS_BF16 ? launch_sel_t<true, GG, true, false, 1>(SS_SEL_ARGS)        \
                                 : launch_sel_t<false, GG, true, false, 1>(SS_SEL_ARGS);      \
        return dt == SS_BF16 ? launch_sel_t<true, GG, true, false>(SS_SEL_ARGS)               \
                             : launch_sel_t<false, GG, true, false>(SS_SEL_ARGS);
    switch (G) {
        SS_SEL_CASE(1)
        SS_SEL_CASE(2)
        SS_SEL_CASE(4)
        SS_SEL_CASE(8)
        default:
            return SS_ERR_UNSUPPORTED;
    }
#undef SS_SEL_CASE
#undef SS_SEL_ARGS
#undef SS_SEL_NOICV
}

bool preload_select() {
    bool ok = true;
#define SS_PL(GG)                                                                     \
    ok &= preload_fn(block_select_kernel<true, GG, true, true, 2>);                  \
    ok &= preload_fn(block_select_kernel<false, GG, true, true, 2>);                 \
    ok &= preload_fn(block_select_kernel<true, GG, true, false, 2>);                 \
    ok &= preload_fn(block_select_kernel<false, GG, true, false, 2>);                \
    ok &= preload_fn(block_select_kernel<true, GG, true, false, 1>);                 \
    ok &= preload_fn(block_select_kernel<false, GG, true, false, 1>);
    SS_PL(1) SS_PL(2) SS_PL(4) SS_PL(8)
#undef SS_PL
    ok &= preload_fn(block_select_tc_kernel<2, 1>) && preload_fn(block_select_tc_kernel<2, 2>);
    ok &= preload_fn(block_select_tc_kernel<4, 1>) && preload_fn(block_select_tc_kernel<4, 2>);
    ok &= preload_fn(block_select_tc_kernel<8, 1>) && preload_fn(block_select_tc_kernel<8, 2>);
    ok &= preload_fn(block_select_kernel<true, 1, true, false, 2, true>);
    ok &= preload_fn(block_select_kernel<false, 1, true, false, 2, true>);
    ok &= preload_fn(block_select_tcc_kernel<2, 1>) && preload_fn(block_select_tcc_kernel<2, 2>);
    ok &= preload_fn(block_select_tcc_kernel<4, 1>) && preload_fn(block_select_tcc_kernel<4, 2>);
    ok &= preload_fn(block_select_tcc_kernel<8, 1>) && preload_fn(block_select_tcc_kernel<8, 2>);
    return ok;
}

}  // namespace ss

#ifdef SS_DEBUG_KNOBS
// debug build only: copy the tensor-core select timeline (8 u64 per CTA, CTAs
// 0..n_ctas-1) to host memory
extern "C" int ss_debug_sel_trace(void* host, int n_ctas) {
    if (n_ctas > 16384) n_ctas = 16384;
    return cudaMemcpyFromSymbol(host, ss::g_sel_trace, (size_t)n_ctas * 12 * 8) == cudaSuccess ? 0 : 1;
}
#endif
