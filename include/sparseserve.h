/*
 * sparseserve.h -- C ABI of the B200-native SparseServe decode hot path
 * (arXiv 2509.24626, "SparseServe"), libsparseserve.so.
 *
 * One decode step, per layer, runs the calls below in this order (PAPER.md:124
 * §3.1 "Model Executor": sparse attention for decoding requests; the indices of
 * the required KV blocks are sent to the KV cache manager to trigger loading):
 *
 *   ss_block_select        S1+S2  score every full 32-token block from its
 *                                 metadata, keep the top-k per (request, KV head)
 *   kv_cache_lookup_insert S3     HBM block cache: hits, LRU victims, miss list
 *   flash_h2d_gather       S4     FlashH2D: zero-copy gather of missed blocks
 *                                 from pinned host DRAM into HBM cache slots
 *   sparse_decode_attn     S5     attention over the selected blocks + tail
 *
 * and block_meta_update (S0) runs when a block fills.
 * Around them: flash_h2d_serve (S4 for a whole step in one persistent launch,
 * with ss_flag_signal / ss_flag_wait), ss_host_alloc (the NUMA-placed pinned
 * host KV pool), ss_decode_step_host (one captured step from host buffers),
 * and the NEXT-row calls (KV append / seal / FlashD2H save, working set,
 * admission, prefill layer save, mean-of-keys metadata).
 *
 * Conventions (all calls):
 *  - Every pointer is caller-owned.  "device" = cudaMalloc'd (or torch) memory
 *    on the current device; "host-mapped" = pinned host memory whose DEVICE
 *    address is passed (cudaHostAlloc / cudaHostRegister(...Mapped...) +
 *    cudaHostGetDevicePointer; under UVA that equals the host address).  The
 *    library never allocates, frees or keeps global state (exceptions, both
 *    explicit: the FlashD2H thread pool ss_d2h_create owns threads, and
 *    ss_host_alloc allocates the host pool the caller frees); calls are
 *    reentrant.
 *  - `stream` is a cudaStream_t passed as void*.  Every call is asynchronous on
 *    it and never synchronises with the host.
 *  - Host-side argument errors return SS_ERR_INVALID_ARG / SS_ERR_UNSUPPORTED
 *    before anything is launched.  A failed launch returns SS_ERR_CUDA and
 *    leaves cudaGetLastError() set.
 *  - Device-side errors (invalid cache key, cache capacity) are reported in the
 *    `counts` word written by kv_cache_lookup_insert; flash_h2d_gather and
 *    sparse_decode_attn given that `counts` become no-ops when counts[3] != 0.
 *  - Fixed geometry: head_dim = 128, block_tokens = 32 (§1:
 *    32-token blocks, 16 KB per LWM-7B head-block).  Layouts are dense and
 *    C-contiguous; all base pointers 16-byte aligned.
 *  - dtype: SS_BF16 (storage bf16, the paper's 2-byte KV) or
 *    SS_F32.  Scores are float64, attention accumulates and outputs float32.
 *
 * Semantics are defined by the CPU oracle (oracle/oracle.c) and DESIGN.md §3
 * readings R1..R20; the CUDA path must match it bit-exactly for indices,
 * masks, cache state and gathered bytes, and within 2e-3 (bf16) / 1e-5 (f32)
 * max-abs for attention outputs.
 */
#ifndef SPARSESERVE_H_
#define SPARSESERVE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SS_OK = 0,
    SS_ERR_INVALID_ARG = 1,
    SS_ERR_UNSUPPORTED = 2,
    SS_ERR_CAPACITY = 3,
    SS_ERR_CUDA = 4
} ss_status;

typedef enum { SS_BF16 = 0, SS_F32 = 1 } ss_dtype;

typedef struct {
    int32_t batch;        /* B: requests in the decode batch                       */
    int32_t num_q_heads;  /* Hq                                                    */
    int32_t num_kv_heads; /* Hkv; Hq % Hkv == 0, G = Hq/Hkv in {1,2,4,8}           */
    int32_t head_dim;     /* d: must be 128                                         */
    int32_t block_tokens; /* must be 32                                             */
} ss_dims;

/* ---------------------------------------------------------------------------
 * Metadata layout (HBM), shared by block_meta_update and ss_block_select.
 *
 * Logical index of a block: idx = (b * Hkv + h) * max_blk + j, max_blk % 32 == 0.
 * Logical content: {min[d], max[d]} per channel over the block's 32 keys
 * (PAPER.md:94 bounding cuboid; Quest min/max, reading R1).
 * Physical layout ("tiled", chosen so a warp reading 32 consecutive blocks
 * issues fully coalesced 512-byte loads): blocks are grouped in tiles of 32,
 * tile T = idx / 32, row r = idx % 32.  With CPC = 16 / sizeof(elem) channels
 * per 16-byte chunk (8 for bf16, 4 for f32), element (channel c, mm = 0 for
 * min / 1 for max) lives at element offset
 *     T * (64 * d)  +  (((c / CPC) * 2 + mm) * 32 + r) * CPC  +  c % CPC.
 * A tile is 32 * 2 * d elements (16 KiB in bf16).  This is a pure permutation
 * of the logical [..][max_blk][2][d] array (tests/layout.py).
 * ------------------------------------------------------------------------- */

/* S0  block_meta_update -- PAPER.md:125 "Once a KV block reaches its
 * capacity, its associated metadata is created."
 *   keys      device, dtype dt: block i's 32 keys at keys + i*key_stride
 *             (elements), laid out [32][d].  key_stride = 32*d for packed keys,
 *             2*32*d to read the K half of [2][32][d] KV blocks in place.
 *   dst_idx   device int64 [n]: logical meta index per block (< 0: block i is
 *             skipped), or NULL = 0..n-1.
 *   n         number of blocks (0 is a no-op).
 *   meta      device, tiled layout above; per-channel min/max under the total
 *             order of the bit patterns (-0 < +0; finite inputs only). */
ss_status block_meta_update(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                            int64_t n, void* meta, ss_dtype dt, int32_t head_dim,
                            void* stream);

/* S1+S2  ss_block_select -- PAPER.md:94 "compute dot products between the
 * metadata vectors and the query token to obtain approximate attention scores
 * for all KV blocks ... select the top-k most critical KV blocks".
 *   q        device [B][Hq][d] dtype dt.
 *   meta     device, tiled layout, max_blk blocks per (b, h).
 *   n_blk    device int32 [B]: full blocks of request b (0 <= n_blk <= max_blk).
 *   k        >= 1 blocks per (b, h).
 *   sel      device int32 [B][Hkv][k] out: the min(k, n_blk[b]) blocks with the
 *            largest score S(j) = max_{g<G} sum_{c=0..d-1} max(q_c M_c, q_c m_c)
 *            (float64, sequential in c, +0 canonical), ties -> lower j,
 *            written in ascending j, -1 padded.
 *   scores   device float64 [B][Hkv][max_blk] out (j < n_blk only), or NULL.
 *   ws       device workspace of ss_workspace_size(SS_WS_SELECT, ...) bytes,
 *            ZERO-FILLED ONCE before first use; every call leaves it zeroed.
 * Returns SS_ERR_UNSUPPORTED (nothing launched) when ceil(max_blk / 4096) * k >
 * 8192: the per-pair candidate merge would exceed its shared-memory bound. */
ss_status ss_block_select(const void* q, const void* meta, const int32_t* n_blk,
                          int32_t max_blk, int32_t k, ss_dims dims, ss_dtype dt, int32_t* sel,
                          double* scores, void* ws, size_t ws_bytes, void* stream);

/* NEXT-3  mean-of-keys metadata -- PAPER.md:94 "Different DSAs propose various
 * metadata construction methods, ranging from simply calculating the mean
 * values of the token keys [45] to finding the bounding cuboid of the token keys
 * [9]"; "other metadata construction methods [41, 45] can be
 * easily integrated into SparseServe".  An alternative to the min/max pair
 * above (reading R18 in DESIGN.md).
 *
 * Mean metadata layout (HBM): ONE float32 vector per block, whatever the KV
 * dtype: mu[c] = (sum_{t=0..31} K[t][c]) / 32, the sum in float64 sequentially
 * t = 0..31 from +0.0, rounded once to float32 (round-to-nearest-even).  Tiled
 * like the min/max layout: tile T = idx / 32, row r = idx % 32, channel c at
 * float offset  T * (32 * d)  +  ((c / 4) * 32 + r) * 4  +  c % 4  (a tile is
 * 16 KiB: the same bytes per block as bf16 min/max).
 *
 * block_meta_update_mean: arguments as block_meta_update; meta is the float32
 *   mean layout above (device).
 * ss_block_select_mean: arguments as ss_block_select, with meta the float32
 *   mean layout; the score is S(j) = max_{g<G} sum_{c=0..d-1} q_c * mu_c
 *   (float64, sequential in c, every product exact, +0 canonical); same top-k,
 *   tie rule, output order, padding, workspace (SS_WS_SELECT) and errors. */
ss_status block_meta_update_mean(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                                 int64_t n, float* meta, ss_dtype dt, int32_t head_dim,
                                 void* stream);
ss_status ss_block_select_mean(const void* q, const float* meta, const int32_t* n_blk,
                               int32_t max_blk, int32_t k, ss_dims dims, ss_dtype dt, int32_t* sel,
                               double* scores, void* ws, size_t ws_bytes, void* stream);

/* S3  kv_cache_lookup_insert -- PAPER.md:124-125: the executor sends the
 * indices of the required blocks to the KV cache manager; hot blocks are cached
 * in the remaining HBM with LRU eviction; DRAM is the authoritative home (no
 * write-back).  One pool per (GPU, layer), shared by all requests and heads
 * (reading R11).  All pool arrays are device memory owned by the caller:
 *   fwd        int32 [fwd_len]: key -> slot, -1 if not cached.  Initially -1.
 *   slot_key   int64 [S]: slot -> key, -1 if empty.          Initially -1.
 *   slot_stamp int64 [S]: stamp of last use, -1 if never used. Initially -1.
 *   order      int32 [S]: slots sorted by (slot_stamp, slot).  Initially 0..S-1.
 *   order_pos  int32 [S]: position of each slot in `order`.    Initially 0..S-1.
 * Batch-LRU (reading R12): key = ((req_ids[b]*L + layer)*Hkv + h)*max_blk + j
 * for every sel[b][h][r] >= 0, in canonical (b, h, r) order.  Hits keep their
 * slot and get slot_stamp = stamp.  The i-th miss takes the i-th slot, in
 * (stamp, slot) order, among slots not hit by this call with slot_stamp < stamp;
 * a previous key of that slot is evicted (fwd = -1).
 *   slot_out   int32 [B][Hkv][k]: cache slot per selection (-1 for padding).
 *   hit_out    uint8 [B][Hkv][k]: 1 = hit.
 *   miss_keys  int64 [B*Hkv*k], miss_slots int32 [B*Hkv*k]: the first counts[1]
 *              entries list the misses in canonical order.
 *   counts     int32 [4] = {hits, misses, evictions, status}; status 0 = OK,
 *              1 = a key >= fwd_len (nothing counted), 3 = more misses than
 *              evictable slots.  On status != 0 the pool is left byte-identical
 *              and the other outputs are unspecified.
 * Preconditions: req_ids unique; stamp >= every stamp previously used on the
 * pool.  ws: ss_workspace_size(SS_WS_CACHE, ...) bytes, ZERO-FILLED ONCE
 * before first use; every call (including a failing one) leaves it zeroed.
 * One workspace serves one call at a time (calls sharing it must be ordered). */
typedef struct {
    int32_t* fwd;
    int64_t fwd_len;
    int64_t* slot_key;
    int64_t* slot_stamp;
    int32_t* order;
    int32_t* order_pos;  /* inverse permutation of order.      Initially 0..S-1. */
    int32_t num_slots;
    /* Optional device int64 "clock" (NULL = use the `stamp` argument).  When
     * set, the call's stamp is *clock, read on the device (the `stamp`
     * argument is ignored); the caller advances it once per decode step (all
     * calls of one step share it), so a captured CUDA graph can replay decode
     * steps without host-side scalars. */
    int64_t* clock;
} ss_cache_pool;

ss_status kv_cache_lookup_insert(ss_cache_pool pool, const int32_t* sel, const int32_t* req_ids,
                                 int32_t layer, int32_t num_layers, int32_t max_blk, int32_t k,
                                 ss_dims dims, int64_t stamp, int32_t* slot_out,
                                 uint8_t* hit_out, int64_t* miss_keys, int32_t* miss_slots,
                                 int32_t* counts, void* ws, size_t ws_bytes, void* stream);

/* S4  flash_h2d_gather -- PAPER.md:143-149 §3.2.1 FlashH2D: one kernel loads
 * all selected, missing blocks from DRAM over UVA (GPU-direct, zero-copy).
 *   host_kv     host-mapped pinned memory, host_blocks blocks of block_bytes;
 *               logical key -> physical host block key % host_blocks
 *               (reading R15; host_blocks > every key = no aliasing).
 *   miss_keys / miss_slots / counts: as written by kv_cache_lookup_insert
 *               (device); the miss count counts[1] is read ON DEVICE, capped
 *               at max_misses; no-op if counts[3] != 0.
 *   pool_kv     device [S][block_bytes]; slot s <- host block, byte-exact.
 *   block_bytes multiple of 16 (16384 for a bf16 [2][32][128] block). */
ss_status flash_h2d_gather(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
                           const int32_t* miss_slots, const int32_t* counts, int32_t max_misses,
                           void* pool_kv, int64_t block_bytes, void* stream);

/* S4, pipelined form -- the same FlashH2D copy (§3.2.1) for
 * every gather of a decode step, served by ONE persistent launch so the host
 * link does not drain at each layer boundary.  Each job is one
 * flash_h2d_gather's arguments; a warp always serves the lowest-numbered
 * ready job with blocks left.
 *   jobs      device array of njobs ss_h2d_job (read-only except counts[3],
 *             see abort below).  pool_kv / max_misses / block_bytes as above.
 *   flags     device int32 [SS_H2D_FLAGS(njobs)], ZEROED by the caller before
 *             the launch: [0,nj) ready, [nj,2nj) done, [2nj,4nj) server
 *             scratch, [4nj] abort.  Job j starts once ready[j] != 0 (set it
 *             with ss_flag_signal, stream-ordered after the job's
 *             kv_cache_lookup_insert); done[j] becomes SS_H2D_DONE_SERVED
 *             (release, GPU scope) after all of job j's blocks are in HBM --
 *             wait for it with ss_flag_wait before reading the pool.
 *   timeout_us  abort after this long with no ready job (<= 0: 3 s).
 *   stats_or_null  device uint64 [SS_H2D_STATS], zeroed by the caller, or
 *             NULL: [0] sum over the server's warps of ns with nothing to
 *             serve, [1] warps, [2] first unit start / [3] last unit end
 *             (globaltimer ns), [4] ns between them with NO warp copying
 *             (link idle), [5] 1 + the job found not ready at an abort (0:
 *             none); [6..7] scratch.
 *   Errors: on abort every job not yet done gets done = SS_H2D_DONE_ABORTED
 *   (and counts[3] = SS_ERR_CUDA); its ss_flag_wait, which runs after the
 *   job's producer, then sets counts[3] = SS_ERR_CUDA again so a producer
 *   that ran late cannot clear it: the attention becomes a no-op and the
 *   error stays visible.  The launch never completes before every ready job
 *   is served, so a job whose producer runs only after the server (e.g. a
 *   profiler serialising kernels) aborts: use flash_h2d_gather there. */
#define SS_H2D_FLAGS(njobs) (4 * (njobs) + 1)
#define SS_H2D_STATS 8
#define SS_H2D_DONE_SERVED 1
#define SS_H2D_DONE_ABORTED 2
typedef struct {
    const int64_t* miss_keys;
    const int32_t* miss_slots;
    int32_t* counts;
    void* pool_kv;
    int32_t max_misses;
    int32_t reserved;
} ss_h2d_job;

ss_status flash_h2d_serve(const void* host_kv, int64_t host_blocks, const ss_h2d_job* jobs,
                          int32_t njobs, int64_t block_bytes, int32_t* flags, int64_t timeout_us,
                          uint64_t* stats_or_null, void* stream);

/* Stream-ordered flag signal / wait for flash_h2d_serve.
 *   ss_flag_signal: *flag = 1 (device int32 that was 0), after all prior work
 *                   on `stream` (a 1-byte memset: no kernel).
 *   ss_flag_wait:   later work on `stream` starts only after *flag != 0
 *                   (acquire, GPU scope), observed by a one-thread kernel.
 *                   If the flag reads SS_H2D_DONE_ABORTED, or nothing is
 *                   signalled within timeout_us (<= 0: 3 s), it sets
 *                   counts_or_null[3] = SS_ERR_CUDA (when given) so the job's
 *                   downstream calls become no-ops and the failure is
 *                   reported, never silent. */
ss_status ss_flag_signal(int32_t* flag, void* stream);
ss_status ss_flag_wait(const int32_t* flag, int32_t* counts_or_null, int64_t timeout_us, void* stream);

/* Load every kernel of the library now (CUDA lazy module loading would load
 * each one at its first launch; a first launch that has to wait behind a
 * spinning flash_h2d_serve can stall it).  flash_h2d_serve calls it itself on
 * its first call outside stream capture.  Idempotent; SS_ERR_CUDA on failure. */
ss_status ss_preload_kernels(void);

/* S5  sparse_decode_attn -- PAPER.md:71-72 §2.1 (S = QK^T/sqrt(d), P =
 * softmax(S), O = PV) restricted to the selected blocks.
 *   q         device [B][Hq][d] dtype dt.
 *   pool_kv   device [S][2][32][d] dtype dt (K then V of one head-block,
 *             PAPER.md:137 (H,N,D) layout).
 *   slot      device int32 [B][Hkv][k] (slot_out of S3; -1 entries skipped).
 *   tail_kv   device [B][Hkv][2][32][d]: the partial block of each (b, h);
 *             its first tail_len[b] tokens are always attended (reading R7).
 *   tail_len  device int32 [B], 0..31.
 *   softmax_scale  normally 1/sqrt(d).
 *   counts    device int32[4] from S3 or NULL; no-op if counts[3] != 0.
 *   out       device float32 [Hq][B][d] (head-major).  Softmax runs over the
 *             selected tokens + tail only (reading R9); empty set -> 0.
 *   ws        ss_workspace_size(SS_WS_ATTN, ...) bytes, ZERO-FILLED ONCE
 *             before first use; every call leaves it zeroed. */
ss_status sparse_decode_attn(const void* q, const void* pool_kv, const int32_t* slot, int32_t k,
                             const void* tail_kv, const int32_t* tail_len, ss_dims dims,
                             ss_dtype dt, float softmax_scale, const int32_t* counts,
                             float* out, void* ws, size_t ws_bytes, void* stream);

/* S5, split form -- the same attention over a SUBSET of the token set, plus
 * its log-sum-exp, so the part over the cache hits can run while FlashH2D
 * still loads the misses.  Softmax over disjoint token sets
 * combines exactly by log-sum-exp (PAPER.md:71-72 restated per subset):
 *   O = (O_a 2^lse_a + O_b 2^lse_b) / (2^lse_a + 2^lse_b).
 *   hit    device uint8 [B][Hkv][k] (hit_out of S3); required for mode 1/2.
 *   mode   0: every selected block + tail (= sparse_decode_attn)
 *          1: blocks with hit != 0 + tail    2: blocks with hit == 0 only.
 *   out    device float32 [Hq][B][d]: the subset's normalised output (0 if
 *          the subset is empty).
 *   lse    device float32 [Hq][B]: log2-domain log-sum-exp of the subset's
 *          scaled logits (z * log2(e) with z = q.k * softmax_scale): m + log2(l);
 *          -inf for an empty subset.
 *   Other arguments as sparse_decode_attn (same workspace size). */
ss_status sparse_decode_attn_part(const void* q, const void* pool_kv, const int32_t* slot,
                                  const uint8_t* hit, int32_t mode, int32_t k, const void* tail_kv,
                                  const int32_t* tail_len, ss_dims dims, ss_dtype dt,
                                  float softmax_scale, const int32_t* counts, float* out, float* lse,
                                  void* ws, size_t ws_bytes, void* stream);

/* Merge two split-form results over disjoint token sets (rows = Hq * B rows of
 * d = 128 floats): out = (out_a 2^lse_a + out_b 2^lse_b) / (2^lse_a + 2^lse_b),
 * 0 when both are empty.  out may alias out_a or out_b.  No-op if counts is
 * non-null and counts[3] != 0 (as the attention calls). */
ss_status sparse_attn_merge(const float* out_a, const float* lse_a, const float* out_b,
                            const float* lse_b, int64_t rows, const int32_t* counts, float* out,
                            void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-1: decode KV append + save path (PAPER.md:151-153 §3.2.2, :125).
 * Per decode step: kv_append for every layer (advance = 1 on the first layer
 * only, so every layer writes the same row and attends the new token), then
 * for the requests whose tail just filled: kv_seal_blocks per layer (metadata
 * of the new block + a contiguous device staging copy), flash_d2h_save per
 * layer (FlashD2H), and kv_commit once.
 * ------------------------------------------------------------------------- */

/* kv_append -- "the resulting KV tensor is then saved into the free slots in
 * the corresponding KV blocks in HBM".
 *   new_kv    device [B][Hkv][2][d] dtype dt: this step's K and V rows.
 *   tail_kv   device [B][Hkv][2][32][d]: row tail_len[b] - 1 of each (b, h)
 *             tail receives the new K / V row.
 *   tail_len  device int32 [B]; if advance != 0 it is first incremented (the
 *             new token is counted), then used.  Precondition: the resulting
 *             tail_len is in 1..32 (rows outside are not written). */
ss_status kv_append(const void* new_kv, void* tail_kv, int32_t* tail_len, int32_t advance,
                    ss_dims dims, ss_dtype dt, void* stream);

/* kv_seal_blocks -- "Once a KV block reaches its capacity, its associated
 * metadata is created".  For the n_fill requests fill_req
 * (device int32, unique, each with a full 32-token tail): the tail of every KV
 * head is copied to staging[i][h] (device [n_fill][Hkv][2][32][d], list order)
 * and its per-channel min/max is written to meta (tiled layout) as block
 * n_blk[b] of (b, h).  Counters are not changed (see kv_commit).
 * Precondition: n_blk[b] < max_blk (a row is free); a request whose block
 * table is full gets its staging copy but no metadata row (nothing out of
 * bounds is written).
 *   ws   device, ss_workspace_size(SS_WS_SEAL, ...) bytes, no initialisation. */
ss_status kv_seal_blocks(const int32_t* fill_req, int32_t n_fill, const void* tail_kv,
                         const int32_t* n_blk, int32_t max_blk, void* meta, void* staging,
                         void* ws, size_t ws_bytes, ss_dims dims, ss_dtype dt, void* stream);

/* kv_commit -- n_blk[b] += 1 and tail_len[b] = 0 for b in fill_req (device). */
ss_status kv_commit(const int32_t* fill_req, int32_t n_fill, int32_t* n_blk, int32_t* tail_len,
                    void* stream);

/* FlashD2H ("(1) the contiguous KV tensor is first copied
 * into a DRAM buffer with a single memcpy, and (2) once the transfer
 * completes, CPU threads redistribute the buffered data into the corresponding
 * DRAM KV blocks").  An engine owns a pool of CPU threads (created/destroyed
 * explicitly by the caller; the only library object with state).
 * flash_d2h_save enqueues on `stream`: one cudaMemcpyAsync of n_blocks x
 * block_bytes from device `staging` into pinned `host_buf`, then a host
 * function that scatters block i to host_kv + (keys[i] % host_blocks) *
 * block_bytes on the engine's threads and returns when all are written, so
 * later work on `stream` (or waiting on an event after it) sees them.
 *   keys      HOST int64 [n_blocks], copied at call time.
 *   host_buf  pinned, >= n_blocks * block_bytes, untouched until the stream
 *             passes the call.  host_kv: host memory (pinned for FlashH2D). */
typedef struct ss_d2h_engine ss_d2h_engine;
ss_status ss_d2h_create(int32_t num_threads, ss_d2h_engine** out);
ss_status ss_d2h_destroy(ss_d2h_engine* engine);
ss_status flash_d2h_save(ss_d2h_engine* engine, const void* staging, void* host_buf,
                         int64_t n_blocks, const int64_t* keys, void* host_kv, int64_t host_blocks,
                         int64_t block_bytes, void* stream);

/* ---------------------------------------------------------------------------
 * NEXT-2: decoding working set + working-set-aware admission (PAPER.md:199-207
 * §3.3, Algorithm 1).
 * ------------------------------------------------------------------------- */

/* ws_track -- "tracks the KV blocks selected over the past w decoding steps
 * (with w = 12 by default) and regards their union as the decoding working
 * set".  Call once per layer per step with that layer's state,
 * after ss_block_select.  For every (b, h): ws_count[b] += |U_t| - |U_{t-1}|
 * where U_t = union of sel over steps t-w+1..t, so after all layers of step t
 * ws_count[b] = sum over layers and heads of |U_t| (blocks; x block bytes =
 * the request's working set).
 *   sel       device int32 [B][Hkv][k] (-1 = none), this layer, step t.
 *   last_sel  device int32 [B][Hkv][max_blk], this layer: step a block was last
 *             selected; initialise to <= -w (e.g. INT32_MIN / 2).
 *   ring      device int32 [w][B][Hkv][k], this layer: initialise to -1.
 *   ws_count  device int32 [B], shared by the layers; initialise to 0.
 *   t         step index, strictly increasing by 1 per step, 0 <= t < 2^31.  */
ss_status ws_track(const int32_t* sel, int32_t k, ss_dims dims, int32_t max_blk, int64_t t,
                   int32_t w, int32_t* last_sel, int32_t* ring, int32_t* ws_count, void* stream);

/* ss_admit -- Algorithm 1 lines 6-14: for the candidate batch in order, admit a
 * request if M_used + M_req <= M_avl (M_used += M_req), else mark it for reset.
 * Host arrays: ws_bytes [n] (M_req), admit_out [n] (1 admitted / 0 reset).
 * Returns the number admitted (or -1 on invalid arguments). */
int32_t ss_admit(const int64_t* ws_bytes, int32_t n, int64_t m_avl, uint8_t* admit_out);

/* ---------------------------------------------------------------------------
 * NEXT-4: layer-segmented prefill, storage side (§3.4: "The KV
 * blocks of all finished layers can be immediately evicted after being saved
 * to DRAM"; (N,H,D) -> (H,N,D) blocks).
 * prefill_layer_save -- one prefill layer of one request (batch slot b, request
 * id req): k_nhd / v_nhd device [n_tok][Hkv][d] ((N,H,D) projection output).
 * Full blocks j < n_tok/32 of every head are re-laid out into staging (device
 * [Hkv][n_tok/32][2][32][d]), their metadata written (tiled meta, index
 * (b*Hkv+h)*max_blk + j) and saved to their DRAM home host_kv + (key %
 * host_blocks) * block_bytes, key = ((req*L + layer)*Hkv + h)*max_blk + j, with
 * one DMA copy per head (requires host_blocks % max_blk == 0: a head's blocks are
 * contiguous there); the remaining n_tok % 32 tokens become the tail (rows of
 * tail_kv[b][h]); n_blk[b] = n_tok/32, tail_len[b] = n_tok % 32.
 *   ws  device, ss_workspace_size(SS_WS_PREFILL, dims, max_blk, ...) bytes.
 * host_kv: pinned host memory (HOST address). n_tok <= 32 * max_blk. */
ss_status prefill_layer_save(const void* k_nhd, const void* v_nhd, int32_t n_tok, int32_t b,
                             int32_t req, int32_t layer, int32_t num_layers, int32_t max_blk,
                             ss_dims dims, ss_dtype dt, void* staging, void* meta, void* tail_kv,
                             int32_t* n_blk, int32_t* tail_len, void* host_kv, int64_t host_blocks,
                             void* ws, size_t ws_bytes, void* stream);

#define SS_WS_SELECT 0
#define SS_WS_CACHE 1
#define SS_WS_ATTN 2
#define SS_WS_SEAL 3
#define SS_WS_PREFILL 4

/* Workspace bytes for call `which` (SS_WS_*); num_slots is used by SS_WS_CACHE. */
size_t ss_workspace_size(int32_t which, ss_dims dims, int32_t max_blk, int32_t k,
                         int32_t num_slots);

/* Device address of pinned host memory (cudaHostGetDevicePointer). */
ss_status ss_host_device_pointer(void* host, void** dev);

/* Host KV pool memory (§3.1: DRAM holds every KV block;
 * PAPER.md:143-149 §3.2.1: FlashH2D reads it zero-copy over UVA; SURVEY.md
 * §8(e): each rank's partition on its GPU's NUMA node).
 *   ss_device_numa_node: NUMA node of CUDA device `device`'s PCIe root from
 *     sysfs, or -1 when unknown (single-node or virtualised hosts).
 *   ss_host_alloc: `bytes` of page-locked, device-mapped host memory; when
 *     numa_node >= 0 its pages are bound to that node before first touch
 *     (mbind), *bound_out (may be NULL) = 1 if that binding took effect.
 *     *host_out = host address (caller owns it: free with ss_host_free with
 *     the same bytes), *dev_out = its device address (for flash_h2d_*).
 *     SS_ERR_CAPACITY if the mapping fails, SS_ERR_CUDA if registration does
 *     (nothing is left allocated on error).  Contents are zero.
 *   ss_host_free: unregisters and unmaps; NULL is a no-op. */
int32_t ss_device_numa_node(int32_t device);
ss_status ss_host_alloc(size_t bytes, int32_t numa_node, void** host_out, void** dev_out,
                        int32_t* bound_out);
ss_status ss_host_free(void* host, size_t bytes);

const char* ss_status_string(ss_status s);
const char* ss_version(void);

/* One decode step from HOST buffers (the e2e path of the benchmark): copies
 * this step's queries host -> device, launches the step's instantiated CUDA
 * graph (every layer's S1..S5 (+S6) calls of this library, captured by the
 * caller), and copies the step's outputs device -> host, all enqueued on
 * `stream` in that order; nothing synchronises.
 *   graph_exec  cudaGraphExec_t of the captured step.
 *   q_host      pinned host [q_bytes] -> q_dev (the graph's query buffer).
 *   out_dev[i]  device outputs -> out_host[i] (pinned) [out_bytes[i]], i < n_out.
 * Errors: SS_ERR_INVALID_ARG (null pointers), SS_ERR_CUDA (enqueue failed). */
ss_status ss_decode_step_host(void* graph_exec, const void* q_host, void* q_dev, size_t q_bytes,
                              int32_t n_out, const void* const* out_dev, void* const* out_host,
                              const size_t* out_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSESERVE_H_ */
