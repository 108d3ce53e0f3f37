/*
 * oracle.c -- plain, slow, obviously-correct CPU reference of the SparseServe
 * decode hot path (arXiv 2509.24626).  TEST INFRASTRUCTURE ONLY: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  It shares no code with the CUDA path (paper_2509_24626_b200/).
 *
 * Built with: gcc -O2 -fno-fast-math -ffp-contract=off -shared -fPIC
 * (no FMA contraction: every a*b+c below is a rounded product then a rounded
 * sum, exactly as written).
 *
 * Citations are to /root/reference/PAPER.md lines ("P:<line>") and to the
 * readings R1..R16 listed in DESIGN.md §3.
 *
 * Storage dtypes: dt == 0 -> bf16 (uint16 bit patterns), dt == 1 -> float32.
 * All arithmetic is done in float64 on the exactly-decoded values.
 *
 * Functions and their pins (tests/test_oracle_*.py):
 *   or_block_meta   S0  pinned: numpy min/max, hand-written signed-zero cases
 *   or_block_score  S1  pinned: exact rationals (fractions.Fraction), bound
 *                       soundness, M==m special case == exact dot product
 *   or_topk         S2  pinned: numpy.lexsort, order invariants, tie suites
 *   or_lru          S3  pinned: collections.OrderedDict LRU (one key per
 *                       call), hand-traced fixture tests/golden/lru_trace.json,
 *                       capacity error leaves state byte-identical
 *   or_gather       S4  pinned: numpy fancy-index byte comparison
 *   or_block_mean   NEXT-3 pinned: exact rational mean (fractions.Fraction),
 *                       numpy float64 mean, identical-token blocks (mean = key)
 *   or_block_score_mean NEXT-3 pinned: exact rationals; identical-token blocks
 *                       score exactly like the min/max bound (M = m = mu)
 *   or_attention    S5  pinned: torch scaled_dot_product_attention (fp64, CPU)
 *                       when k covers all blocks; masked-dense equivalence
 *   or_ws_estimate  NEXT-2 pinned: closed forms (constant selections -> k per
 *                       head, disjoint selections -> min(t+1, w) k, w = 1 ->
 *                       |sel|), monotone in w, brute-force Python set unions
 *   or_admit        NEXT-2 pinned: hand-traced Algorithm 1 cases (greedy in
 *                       order, later small requests still admitted, M_avl = 0)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_BLOCK_TOKENS 32

static double ld(const void* p, int dt, int64_t i) {
    if (dt == 0) {
        uint32_t u = ((uint32_t)((const uint16_t*)p)[i]) << 16;
        float f;
        memcpy(&f, &u, 4);
        return (double)f;
    }
    return (double)((const float*)p)[i];
}

static int64_t esize(int dt) { return dt == 0 ? 2 : 4; }

/* ------------------------------------------------------------------------
 * S0  block metadata ("Once a KV block reaches its capacity, its
 * associated metadata is created"; bounding cuboid = per-channel min and max
 * of the block's keys, P:94 and reading R1).
 * keys: block i's K half starts at element i*key_stride, laid out [32][d].
 * meta_out: [n][2][d], row 0 = per-channel min, row 1 = per-channel max,
 * stored as the raw element of the winning key (so the result is bit-exact).
 * Signed zero (reading R16): min prefers -0 over +0, max prefers +0 over -0.
 * ---------------------------------------------------------------------- */
void or_block_meta(const void* keys, int64_t key_stride, int64_t n, int dt, int d,
                   void* meta_out) {
    int64_t es = esize(dt);
    for (int64_t i = 0; i < n; ++i) {
        for (int c = 0; c < d; ++c) {
            int64_t imin = i * key_stride + c, imax = imin;
            double vmin = ld(keys, dt, imin), vmax = vmin;
            for (int t = 1; t < OR_BLOCK_TOKENS; ++t) {
                int64_t e = i * key_stride + (int64_t)t * d + c;
                double v = ld(keys, dt, e);
                if (v < vmin || (v == vmin && signbit(v) && !signbit(vmin))) { vmin = v; imin = e; }
                if (v > vmax || (v == vmax && !signbit(v) && signbit(vmax))) { vmax = v; imax = e; }
            }
            memcpy((char*)meta_out + ((i * 2 + 0) * d + c) * es, (const char*)keys + imin * es, es);
            memcpy((char*)meta_out + ((i * 2 + 1) * d + c) * es, (const char*)keys + imax * es, es);
        }
    }
}

/* ------------------------------------------------------------------------
 * S1  block criticality score ("compute dot products between the
 * metadata vectors and the query token to obtain approximate attention
 * scores"; reading R2: the Quest upper bound sum_c max(q_c*M_c, q_c*m_c);
 * R3: unscaled, float64, sequential sum c = 0..d-1 from +0.0; R4: GQA ->
 * max over the G query heads of a KV-head group).
 * q: [B][Hq][d]; meta: [B][Hkv][max_blk][2][d] (logical layout);
 * scores: [B][Hkv][max_blk], written for j < n_blk[b] only.
 * ---------------------------------------------------------------------- */
void or_block_score(const void* q, const void* meta, const int32_t* n_blk, int B, int Hq,
                    int Hkv, int d, int max_blk, int dt, double* scores) {
    int G = Hq / Hkv;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < Hkv; ++h)
            for (int j = 0; j < n_blk[b]; ++j) {
                int64_t mbase = (((int64_t)b * Hkv + h) * max_blk + j) * 2 * d;
                double best = 0.0;
                for (int g = 0; g < G; ++g) {
                    int64_t qbase = ((int64_t)b * Hq + (int64_t)h * G + g) * d;
                    double acc = 0.0;
                    for (int c = 0; c < d; ++c) {
                        double qc = ld(q, dt, qbase + c);
                        double lo = ld(meta, dt, mbase + c);      /* m_c (min) */
                        double hi = ld(meta, dt, mbase + d + c);  /* M_c (max) */
                        double a = qc * hi, bb = qc * lo;         /* exact products */
                        acc = acc + (a > bb ? a : bb);
                    }
                    if (g == 0 || acc > best) best = acc;
                }
                scores[((int64_t)b * Hkv + h) * max_blk + j] = best + 0.0; /* -0 -> +0 */
            }
}

/* ------------------------------------------------------------------------
 * NEXT-3  mean-of-keys metadata ("ranging from simply calculating the
 * mean values of the token keys [45] to finding the bounding cuboid of the
 * token keys [9]"; "other metadata construction methods [41, 45] can be
 * easily integrated").  Reading R18: one metadata vector per
 * block, mu_c = (sum_{t=0..31} K[t][c]) / 32 with the sum taken in float64
 * sequentially t = 0..31 from +0.0 (the division by 32 is exact), rounded
 * once to float32 (round-to-nearest-even) for storage.  meta_out: [n][d]
 * float32 whatever the key dtype.
 * ---------------------------------------------------------------------- */
void or_block_mean(const void* keys, int64_t key_stride, int64_t n, int dt, int d,
                   float* meta_out) {
    for (int64_t i = 0; i < n; ++i)
        for (int c = 0; c < d; ++c) {
            double acc = 0.0;
            for (int t = 0; t < OR_BLOCK_TOKENS; ++t)
                acc = acc + ld(keys, dt, i * key_stride + (int64_t)t * d + c);
            meta_out[i * d + c] = (float)(acc / 32.0);
        }
}

/* NEXT-3 score: S(j) = max_g sum_c q_{g,c} * mu_{j,c} -- the dot product of the
 * query with the block's metadata vector; float64, sequential in c from
 * +0.0, +0 canonical (R3, R4 as for the min/max score).  Every product is exact
 * in float64 (bf16 or f32 q times a float32 mu: <= 48 significant bits).
 * q: [B][Hq][d] dtype dt; meta: [B][Hkv][max_blk][d] float32. */
void or_block_score_mean(const void* q, const float* meta, const int32_t* n_blk, int B, int Hq,
                         int Hkv, int d, int max_blk, int dt, double* scores) {
    int G = Hq / Hkv;
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < Hkv; ++h)
            for (int j = 0; j < n_blk[b]; ++j) {
                const float* mu = meta + (((int64_t)b * Hkv + h) * max_blk + j) * d;
                double best = 0.0;
                for (int g = 0; g < G; ++g) {
                    int64_t qbase = ((int64_t)b * Hq + (int64_t)h * G + g) * d;
                    double acc = 0.0;
                    for (int c = 0; c < d; ++c) acc = acc + ld(q, dt, qbase + c) * (double)mu[c];
                    if (g == 0 || acc > best) best = acc;
                }
                scores[((int64_t)b * Hkv + h) * max_blk + j] = best + 0.0;
            }
}

/* ------------------------------------------------------------------------
 * S2  top-k ("select the top-k most critical KV blocks"; P:245 token
 * budget; reading R5: ties -> lowest block index; R6: k_eff = min(k, n_blk),
 * indices emitted ascending, -1 padded).
 * ---------------------------------------------------------------------- */
static const double* g_sort_scores;
static int cmp_desc_score_asc_idx(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    double sa = g_sort_scores[a], sb = g_sort_scores[b];
    if (sa > sb) return -1;
    if (sa < sb) return 1;
    return (a < b) ? -1 : (a > b);
}
static int cmp_i32(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    return (a < b) ? -1 : (a > b);
}

void or_topk(const double* scores, const int32_t* n_blk, int B, int Hkv, int max_blk, int k,
             int32_t* sel) {
    int32_t* idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(max_blk > 0 ? max_blk : 1));
    for (int b = 0; b < B; ++b)
        for (int h = 0; h < Hkv; ++h) {
            int n = n_blk[b];
            int keff = n < k ? n : k;
            for (int j = 0; j < n; ++j) idx[j] = j;
            g_sort_scores = scores + ((int64_t)b * Hkv + h) * max_blk;
            qsort(idx, (size_t)n, sizeof(int32_t), cmp_desc_score_asc_idx);
            qsort(idx, (size_t)keff, sizeof(int32_t), cmp_i32);
            int32_t* out = sel + ((int64_t)b * Hkv + h) * k;
            for (int r = 0; r < k; ++r) out[r] = r < keff ? idx[r] : -1;
        }
    free(idx);
}

/* ------------------------------------------------------------------------
 * S3  HBM block cache lookup / insert with LRU eviction ("sends the
 * indices of the KV blocks required ... to trigger the KV cache loading";
 * P:125 "least recently used (LRU) cache eviction policy"; reading R11/R12:
 * one pool per layer shared by all requests and heads, batch-LRU):
 *   1. keys in canonical order (b, h, r), key = ((req*L + layer)*Hkv + h)*max_blk + j
 *   2. hits: fwd[key] >= 0
 *   3. candidates: slots not hit in this call with stamp < t, ordered by
 *      (stamp asc, slot asc); never-used slots carry stamp -1
 *   4. more misses than candidates -> status 3 (capacity), no state change
 *   5. hit slots get stamp t; the i-th miss takes the i-th candidate
 *      (evicting its old key, if any) and gets stamp t
 * counts = {hits, misses, evictions, status}.  Returns status.
 * ---------------------------------------------------------------------- */
static const int64_t* g_sort_stamp;
static int cmp_stamp_slot(const void* pa, const void* pb) {
    int32_t a = *(const int32_t*)pa, b = *(const int32_t*)pb;
    int64_t sa = g_sort_stamp[a], sb = g_sort_stamp[b];
    if (sa < sb) return -1;
    if (sa > sb) return 1;
    return (a < b) ? -1 : (a > b);
}

int or_lru(int32_t* fwd, int64_t fwd_len, int64_t* slot_key, int64_t* slot_stamp, int32_t S,
           const int32_t* sel, const int32_t* req_ids, int layer, int L, int B, int Hkv,
           int max_blk, int k, int64_t t, int32_t* slot_out, uint8_t* hit_out,
           int64_t* miss_keys, int32_t* miss_slots, int32_t* counts) {
    int64_t E = (int64_t)B * Hkv * k;
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E > 0 ? E : 1));
    int64_t* miss_e = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E > 0 ? E : 1));
    uint8_t* hitmark = (uint8_t*)calloc((size_t)(S > 0 ? S : 1), 1);
    int32_t* cand = (int32_t*)malloc(sizeof(int32_t) * (size_t)(S > 0 ? S : 1));
    int32_t hits = 0, misses = 0, ncand = 0, evictions = 0, status = 0;

    for (int64_t e = 0; e < E; ++e) {
        int b = (int)(e / ((int64_t)Hkv * k));
        int h = (int)((e / k) % Hkv);
        int32_t j = sel[e];
        keys[e] = -1;
        slot_out[e] = -1;
        hit_out[e] = 0;
        if (j < 0) continue;
        int64_t key = (((int64_t)req_ids[b] * L + layer) * Hkv + h) * max_blk + j;
        if (key < 0 || key >= fwd_len) { status = 1; continue; }
        keys[e] = key;
        int32_t f = fwd[key];
        if (f >= 0) {
            hits++;
            hitmark[f] = 1;
            slot_out[e] = f;
            hit_out[e] = 1;
        } else {
            miss_e[misses++] = e;
        }
    }
    if (status == 0) {
        for (int32_t s = 0; s < S; ++s)
            if (!hitmark[s] && slot_stamp[s] < t) cand[ncand++] = s;
        g_sort_stamp = slot_stamp;
        qsort(cand, (size_t)ncand, sizeof(int32_t), cmp_stamp_slot);
        if (misses > ncand) status = 3;
    }
    if (status == 0) {
        for (int32_t s = 0; s < S; ++s)
            if (hitmark[s]) slot_stamp[s] = t;
        for (int32_t i = 0; i < misses; ++i) {
            int64_t e = miss_e[i];
            int32_t s = cand[i];
            if (slot_key[s] != -1) {
                fwd[slot_key[s]] = -1;
                evictions++;
            }
            slot_key[s] = keys[e];
            fwd[keys[e]] = s;
            slot_stamp[s] = t;
            slot_out[e] = s;
            miss_keys[i] = keys[e];
            miss_slots[i] = s;
        }
    }
    if (status == 1) hits = misses = evictions = 0; /* invalid key: nothing counted */
    counts[0] = hits;
    counts[1] = misses;
    counts[2] = evictions;
    counts[3] = status;
    free(keys);
    free(miss_e);
    free(hitmark);
    free(cand);
    return status;
}

/* ------------------------------------------------------------------------
 * S4  FlashH2D semantics (§3.2.1): every missed block is copied
 * byte-for-byte from its DRAM home into its HBM cache slot.  The physical host
 * block of a logical key is key % host_blocks (reading R15: aliasing for
 * benchmark host pools; host_blocks > every key means no aliasing).
 * ---------------------------------------------------------------------- */
void or_gather(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
               const int32_t* miss_slots, int32_t n_miss, void* pool_kv, int64_t block_bytes) {
    for (int32_t i = 0; i < n_miss; ++i) {
        int64_t phys = miss_keys[i] % host_blocks;
        memcpy((char*)pool_kv + (int64_t)miss_slots[i] * block_bytes,
               (const char*)host_kv + phys * block_bytes, (size_t)block_bytes);
    }
}

/* ------------------------------------------------------------------------
 * S5  sparse decode attention (§2.1: S = QK^T/sqrt(d), P = softmax(S),
 * O = PV; P:33 / P:124: restricted to the selected blocks; readings R7/R9:
 * the partial tail block (tail_len tokens) is always attended and softmax is
 * renormalised over selected tokens + tail; R10: float output; an empty
 * token set gives O = 0).
 * q: [B][Hq][d]; pool: [S][2][32][d]; slot: [B][Hkv][k] (-1 = none);
 * tail: [B][Hkv][2][32][d]; out: [Hq][B][d] (float64).
 * ---------------------------------------------------------------------- */
void or_attention(const void* q, const void* pool, const int32_t* slot, int k,
                  const void* tail, const int32_t* tail_len, int B, int Hq, int Hkv, int d,
                  int dt, double scale, double* out) {
    int G = Hq / Hkv;
    int64_t cap = (int64_t)k * OR_BLOCK_TOKENS + OR_BLOCK_TOKENS;
    double* z = (double*)malloc(sizeof(double) * (size_t)cap);
    const void** vsrc = (const void**)malloc(sizeof(void*) * (size_t)cap);
    int64_t* voff = (int64_t*)malloc(sizeof(int64_t) * (size_t)cap);
    for (int b = 0; b < B; ++b)
        for (int hq = 0; hq < Hq; ++hq) {
            int h = hq / G;
            int64_t qbase = ((int64_t)b * Hq + hq) * d;
            int64_t nt = 0;
            for (int r = 0; r < k; ++r) {
                int32_t s = slot[((int64_t)b * Hkv + h) * k + r];
                if (s < 0) continue;
                for (int t = 0; t < OR_BLOCK_TOKENS; ++t) {
                    int64_t kb = (((int64_t)s * 2 + 0) * OR_BLOCK_TOKENS + t) * d;
                    double dot = 0.0;
                    for (int c = 0; c < d; ++c) dot = dot + ld(q, dt, qbase + c) * ld(pool, dt, kb + c);
                    z[nt] = dot * scale;
                    vsrc[nt] = pool;
                    voff[nt] = (((int64_t)s * 2 + 1) * OR_BLOCK_TOKENS + t) * d;
                    nt++;
                }
            }
            for (int t = 0; t < tail_len[b]; ++t) {
                int64_t tb = ((((int64_t)b * Hkv + h) * 2 + 0) * OR_BLOCK_TOKENS + t) * d;
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot = dot + ld(q, dt, qbase + c) * ld(tail, dt, tb + c);
                z[nt] = dot * scale;
                vsrc[nt] = tail;
                voff[nt] = ((((int64_t)b * Hkv + h) * 2 + 1) * OR_BLOCK_TOKENS + t) * d;
                nt++;
            }
            double* o = out + ((int64_t)hq * B + b) * d;
            for (int c = 0; c < d; ++c) o[c] = 0.0;
            if (nt == 0) continue;
            double mx = z[0];
            for (int64_t i = 1; i < nt; ++i) if (z[i] > mx) mx = z[i];
            double den = 0.0;
            for (int64_t i = 0; i < nt; ++i) {
                double w = exp(z[i] - mx);
                den = den + w;
                for (int c = 0; c < d; ++c) o[c] = o[c] + w * ld(vsrc[i], dt, voff[i] + c);
            }
            for (int c = 0; c < d; ++c) o[c] = o[c] / den;
        }
    free(z);
    free(vsrc);
    free(voff);
}

/* ------------------------------------------------------------------------
 * NEXT-1  decode KV append and save path.
 * or_kv_append: "the resulting KV tensor is then saved into the
 * free slots in the corresponding KV blocks in HBM": if advance, tail_len[b]
 * += 1; then row tail_len[b]-1 of tail[b][h][0|1] <- new_kv[b][h][0|1].
 * new_kv: [B][Hkv][2][d]; tail: [B][Hkv][2][32][d] (storage dtype).
 * ---------------------------------------------------------------------- */
void or_kv_append(const void* new_kv, void* tail, int32_t* tail_len, int advance, int B, int Hkv,
                  int d, int dt) {
    int64_t es = esize(dt);
    for (int b = 0; b < B; ++b) {
        if (advance) tail_len[b] += 1;
        int row = tail_len[b] - 1;
        if (row < 0 || row >= OR_BLOCK_TOKENS) continue;
        for (int h = 0; h < Hkv; ++h)
            for (int half = 0; half < 2; ++half)
                memcpy((char*)tail + (((((int64_t)b * Hkv + h) * 2 + half) * OR_BLOCK_TOKENS + row) * d) * es,
                       (const char*)new_kv + ((((int64_t)b * Hkv + h) * 2 + half) * d) * es,
                       (size_t)(d * es));
    }
}

/* or_kv_seal: "Once a KV block reaches its capacity, its
 * associated metadata is created": for each listed request b (in list order)
 * and head h: staging[i][h] <- tail[b][h]; meta[b][h][n_blk[b]] <- per-channel
 * min/max of its 32 keys (or_block_meta); then (commit) n_blk[b] += 1,
 * tail_len[b] = 0.  meta: logical layout [B][Hkv][max_blk][2][d]. */
void or_kv_seal(const int32_t* fill_req, int n_fill, const void* tail, int32_t* tail_len,
                int32_t* n_blk, int max_blk, void* meta, void* staging, int Hkv, int d, int dt) {
    int64_t es = esize(dt);
    int64_t blk = (int64_t)2 * OR_BLOCK_TOKENS * d;  /* elements per [2][32][d] block */
    for (int i = 0; i < n_fill; ++i) {
        int b = fill_req[i];
        for (int h = 0; h < Hkv; ++h) {
            const char* src = (const char*)tail + ((int64_t)b * Hkv + h) * blk * es;
            memcpy((char*)staging + ((int64_t)i * Hkv + h) * blk * es, src, (size_t)(blk * es));
            void* m = (char*)meta + ((((int64_t)b * Hkv + h) * max_blk + n_blk[b]) * 2 * d) * es;
            or_block_meta(src, blk, 1, dt, d, m);
        }
    }
    for (int i = 0; i < n_fill; ++i) {
        n_blk[fill_req[i]] += 1;
        tail_len[fill_req[i]] = 0;
    }
}

/* or_d2h_scatter: "CPU threads redistribute the buffered data
 * into the corresponding DRAM KV blocks": block i -> host_kv[keys[i] % hb]. */
void or_d2h_scatter(const void* staging, int64_t n, const int64_t* keys, void* host_kv,
                    int64_t host_blocks, int64_t block_bytes) {
    for (int64_t i = 0; i < n; ++i)
        memcpy((char*)host_kv + (keys[i] % host_blocks) * block_bytes,
               (const char*)staging + i * block_bytes, (size_t)block_bytes);
}

/* ------------------------------------------------------------------------
 * NEXT-4  layer-segmented prefill, storage side (§3.4;
 * (N,H,D) -> (H,N,D) blocks): one layer of one request.
 *   k, v: [n_tok][Hkv][d] (N,H,D).  For head h and full block j < n_tok/32:
 *   block[h][j] = {K rows 32j..32j+31 of head h, V rows ...} ([2][32][d]);
 *   meta[b][h][j] = or_block_meta(block); host_kv[key % hb] = block with
 *   key = ((req*L + layer)*Hkv + h)*max_blk + j; the n_tok % 32 remaining rows
 *   go to tail[b][h][0|1][0..rem); n_blk[b] = n_tok/32, tail_len[b] = rem.
 *   meta: logical [B][Hkv][max_blk][2][d]; tail: [B][Hkv][2][32][d].
 * ---------------------------------------------------------------------- */
void or_prefill_save(const void* k, const void* v, int n_tok, int b, int req, int layer, int L,
                     int max_blk, int Hkv, int d, int dt, void* meta, void* tail, int32_t* n_blk,
                     int32_t* tail_len, void* host_kv, int64_t host_blocks) {
    int64_t es = esize(dt);
    int64_t row = (int64_t)d * es;
    int64_t bb = 2 * OR_BLOCK_TOKENS * row;
    int nb = n_tok / OR_BLOCK_TOKENS, rem = n_tok % OR_BLOCK_TOKENS;
    char* blk = (char*)malloc((size_t)bb);
    for (int h = 0; h < Hkv; ++h) {
        for (int j = 0; j < nb; ++j) {
            for (int t = 0; t < OR_BLOCK_TOKENS; ++t) {
                int64_t tok = (int64_t)j * OR_BLOCK_TOKENS + t;
                memcpy(blk + t * row, (const char*)k + (tok * Hkv + h) * row, (size_t)row);
                memcpy(blk + (OR_BLOCK_TOKENS + t) * row, (const char*)v + (tok * Hkv + h) * row, (size_t)row);
            }
            or_block_meta(blk, 2 * OR_BLOCK_TOKENS * d, 1, dt, d,
                          (char*)meta + ((((int64_t)b * Hkv + h) * max_blk + j) * 2 * d) * es);
            int64_t key = (((int64_t)req * L + layer) * Hkv + h) * max_blk + j;
            memcpy((char*)host_kv + (key % host_blocks) * bb, blk, (size_t)bb);
        }
        for (int t = 0; t < rem; ++t) {
            int64_t tok = (int64_t)nb * OR_BLOCK_TOKENS + t;
            char* tb = (char*)tail + ((int64_t)b * Hkv + h) * bb;
            memcpy(tb + t * row, (const char*)k + (tok * Hkv + h) * row, (size_t)row);
            memcpy(tb + (OR_BLOCK_TOKENS + t) * row, (const char*)v + (tok * Hkv + h) * row, (size_t)row);
        }
    }
    n_blk[b] = nb;
    tail_len[b] = rem;
    free(blk);
}

/* ------------------------------------------------------------------------
 * NEXT-2  decoding working set (§3.3: "tracks the KV blocks
 * selected over the past w decoding steps (with w = 12 by default) and regards
 * their union as the decoding working set"; per-head selection).
 *   hist: [T][L][B][Hkv][k] int32 selections of steps 0..T-1 (-1 = none).
 *   ws:   [T][B] out: ws[t][b] = sum over l, h of
 *         | union over s = max(0, t-w+1) .. t of hist[s][l][b][h][:] |  (blocks).
 * Written straight from the definition: a mark array per (t, b, l, h).
 * ---------------------------------------------------------------------- */
void or_ws_estimate(const int32_t* hist, int T, int L, int B, int Hkv, int k, int max_blk, int w,
                    int64_t* ws) {
    unsigned char* mark = (unsigned char*)malloc((size_t)(max_blk > 0 ? max_blk : 1));
    for (int t = 0; t < T; ++t)
        for (int b = 0; b < B; ++b) {
            int64_t tot = 0;
            for (int l = 0; l < L; ++l)
                for (int h = 0; h < Hkv; ++h) {
                    memset(mark, 0, (size_t)(max_blk > 0 ? max_blk : 1));
                    int s0 = t - w + 1 < 0 ? 0 : t - w + 1;
                    for (int s = s0; s <= t; ++s)
                        for (int i = 0; i < k; ++i) {
                            int32_t j = hist[((((int64_t)s * L + l) * B + b) * Hkv + h) * k + i];
                            if (j >= 0 && j < max_blk && !mark[j]) { mark[j] = 1; ++tot; }
                        }
                }
            ws[(int64_t)t * B + b] = tot;
        }
    free(mark);
}

/* ------------------------------------------------------------------------
 * NEXT-2  Algorithm 1 lines 6-14: B_res <- {}, M_used <- 0;
 * for req in B_init (in order): M_req <- estimateWS(req); if M_used + M_req <=
 * M_avl then B_res.add(req), M_used += M_req else S.reset(req).
 *   m_req [n] (estimateWS results), admit [n] out (1 added / 0 reset).
 *   Returns |B_res|.
 * ---------------------------------------------------------------------- */
int or_admit(const int64_t* m_req, int n, int64_t m_avl, uint8_t* admit) {
    int64_t m_used = 0;
    int cnt = 0;
    for (int i = 0; i < n; ++i) {
        if (m_used + m_req[i] <= m_avl) {
            admit[i] = 1;
            m_used += m_req[i];
            ++cnt;
        } else {
            admit[i] = 0;
        }
    }
    return cnt;
}
