// abi.cu -- the extern "C" boundary of libsparseserve.so (include/sparseserve.h):
// host-side argument validation, then one launch sequence per call.  No state,
// no allocation, no host synchronisation.
#include <cuda_runtime.h>

#include "common.cuh"

namespace ss {
ss_status launch_meta_update(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                             int64_t n, void* meta, ss_dtype dt, cudaStream_t stream);
ss_status launch_block_select(const void* q, const void* meta, const int32_t* n_blk, int max_blk,
                              int k, const ss_dims& d, ss_dtype dt, int32_t* sel, double* scores,
                              void* ws, cudaStream_t stream, bool mean);
ss_status launch_meta_mean(const void* keys, int64_t key_stride, const int64_t* dst_idx, int64_t n,
                           float* meta, ss_dtype dt, cudaStream_t stream);
size_t select_ws_bytes(const ss_dims& d, int max_blk, int k);
ss_status launch_cache(const ss_cache_pool& pool, const int32_t* sel, const int32_t* req_ids,
                       int layer, int num_layers, int max_blk, int k, const ss_dims& d,
                       int64_t stamp, int32_t* slot_out, uint8_t* hit_out, int64_t* miss_keys,
                       int32_t* miss_slots, int32_t* counts, void* ws, cudaStream_t stream);
size_t cache_ws_bytes(const ss_dims& d, int k, int S);
ss_status launch_flash_h2d(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
                           const int32_t* miss_slots, const int32_t* counts, int max_misses,
                           void* pool_kv, int64_t block_bytes, cudaStream_t stream);
ss_status launch_flash_h2d_serve(const void* host_kv, int64_t host_blocks, const ss_h2d_job* jobs,
                                 int njobs, int64_t block_bytes, int32_t* flags, int64_t timeout_us,
                                 unsigned long long* stats, cudaStream_t stream);
ss_status launch_flag_wait(const int32_t* flag, int32_t* counts, int64_t timeout_us, cudaStream_t stream);
ss_status launch_sparse_attn(const void* q, const void* pool_kv, const int32_t* slot, int k,
                             const void* tail_kv, const int32_t* tail_len, const ss_dims& d,
                             ss_dtype dt, float scale, const int32_t* counts, float* out, void* ws,
                             cudaStream_t stream, const uint8_t* hit = nullptr, int mode = 0,
                             float* lse = nullptr);
ss_status launch_attn_merge(const float* oa, const float* la, const float* ob, const float* lb,
                            int64_t rows, const int32_t* counts, float* out, cudaStream_t stream);
size_t attn_ws_bytes(const ss_dims& d, int k, ss_dtype dt);
ss_status launch_kv_append(const void* new_kv, void* tail_kv, int32_t* tail_len, int advance,
                           const ss_dims& d, ss_dtype dt, cudaStream_t stream);
ss_status launch_kv_seal(const int32_t* fill_req, int n_fill, const void* tail_kv,
                         const int32_t* n_blk, int max_blk, void* meta, void* staging, void* ws,
                         const ss_dims& d, ss_dtype dt, cudaStream_t stream);
ss_status launch_kv_commit(const int32_t* fill_req, int n_fill, int32_t* n_blk, int32_t* tail_len,
                           cudaStream_t stream);
ss_status launch_prefill_layer_save(const void* k_nhd, const void* v_nhd, int n_tok, int b, int req,
                                    int layer, int num_layers, int max_blk, const ss_dims& d,
                                    ss_dtype dt, void* staging, void* meta, void* tail_kv,
                                    int32_t* n_blk, int32_t* tail_len, void* host_kv,
                                    int64_t host_blocks, void* ws, cudaStream_t stream);
ss_status launch_ws_track(const int32_t* sel, int k, const ss_dims& d, int max_blk, int64_t t,
                          int w, int32_t* last_sel, int32_t* ring, int32_t* ws_count,
                          cudaStream_t stream);
bool preload_select();
bool preload_attn();
bool preload_cache();
bool preload_save();
bool preload_ws();
bool preload_meta();
bool preload_h2d();
}  // namespace ss

namespace {
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
bool dt_ok(ss_dtype dt) { return dt == SS_BF16 || dt == SS_F32; }
bool dims_ok(const ss_dims& d) {
    if (d.batch < 1 || d.num_q_heads < 1 || d.num_kv_heads < 1) return false;
    if (d.num_q_heads % d.num_kv_heads) return false;
    return true;
}
ss_status dims_supported(const ss_dims& d) {
    if (d.head_dim != ss::kHeadDim || d.block_tokens != ss::kBlockTokens) return SS_ERR_UNSUPPORTED;
    int G = d.num_q_heads / d.num_kv_heads;
    if (G != 1 && G != 2 && G != 4 && G != 8) return SS_ERR_UNSUPPORTED;
    return SS_OK;
}
}  // namespace

extern "C" {

ss_status block_meta_update(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                            int64_t n, void* meta, ss_dtype dt, int32_t head_dim, void* stream) {
    if (n < 0 || !dt_ok(dt)) return SS_ERR_INVALID_ARG;
    if (n == 0) return SS_OK;
    if (!keys || !meta || key_stride < 32 * head_dim) return SS_ERR_INVALID_ARG;
    if (head_dim != ss::kHeadDim) return SS_ERR_UNSUPPORTED;
    return ss::launch_meta_update(keys, key_stride, dst_idx, n, meta, dt, (cudaStream_t)stream);
}

ss_status ss_block_select(const void* q, const void* meta, const int32_t* n_blk, int32_t max_blk,
                          int32_t k, ss_dims dims, ss_dtype dt, int32_t* sel, double* scores,
                          void* ws, size_t ws_bytes, void* stream) {
    if (!q || !meta || !n_blk || !sel || !dt_ok(dt) || !dims_ok(dims)) return SS_ERR_INVALID_ARG;
    if (k < 1 || max_blk < 0 || (max_blk % 32) != 0) return SS_ERR_INVALID_ARG;
    if (!aligned16(q) || !aligned16(meta)) return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    size_t need = ss::select_ws_bytes(dims, max_blk, k);
    if (ws_bytes < need || (need && !ws)) return SS_ERR_INVALID_ARG;
    return ss::launch_block_select(q, meta, n_blk, max_blk, k, dims, dt, sel, scores, ws,
                                   (cudaStream_t)stream, false);
}

ss_status block_meta_update_mean(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                                 int64_t n, float* meta, ss_dtype dt, int32_t head_dim, void* stream) {
    if (n < 0 || !dt_ok(dt)) return SS_ERR_INVALID_ARG;
    if (n == 0) return SS_OK;
    if (!keys || !meta || key_stride < 32 * head_dim) return SS_ERR_INVALID_ARG;
    if (head_dim != ss::kHeadDim) return SS_ERR_UNSUPPORTED;
    return ss::launch_meta_mean(keys, key_stride, dst_idx, n, meta, dt, (cudaStream_t)stream);
}

ss_status ss_block_select_mean(const void* q, const float* meta, const int32_t* n_blk,
                               int32_t max_blk, int32_t k, ss_dims dims, ss_dtype dt, int32_t* sel,
                               double* scores, void* ws, size_t ws_bytes, void* stream) {
    if (!q || !meta || !n_blk || !sel || !dt_ok(dt) || !dims_ok(dims)) return SS_ERR_INVALID_ARG;
    if (k < 1 || max_blk < 0 || (max_blk % 32) != 0) return SS_ERR_INVALID_ARG;
    if (!aligned16(q) || !aligned16(meta)) return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    size_t need = ss::select_ws_bytes(dims, max_blk, k);
    if (ws_bytes < need || (need && !ws)) return SS_ERR_INVALID_ARG;
    return ss::launch_block_select(q, meta, n_blk, max_blk, k, dims, dt, sel, scores, ws,
                                   (cudaStream_t)stream, true);
}

ss_status kv_cache_lookup_insert(ss_cache_pool pool, const int32_t* sel, const int32_t* req_ids,
                                 int32_t layer, int32_t num_layers, int32_t max_blk, int32_t k,
                                 ss_dims dims, int64_t stamp, int32_t* slot_out,
                                 uint8_t* hit_out, int64_t* miss_keys, int32_t* miss_slots,
                                 int32_t* counts, void* ws, size_t ws_bytes, void* stream) {
    if (!pool.fwd || !pool.slot_key || !pool.slot_stamp || !pool.order || !pool.order_pos ||
        pool.num_slots < 1 ||
        pool.fwd_len < 1)
        return SS_ERR_INVALID_ARG;
    if (!sel || !req_ids || !slot_out || !hit_out || !miss_keys || !miss_slots || !counts)
        return SS_ERR_INVALID_ARG;
    if (!dims_ok(dims) || k < 1 || max_blk < 1 || num_layers < 1 || layer < 0 ||
        layer >= num_layers)
        return SS_ERR_INVALID_ARG;
    if ((int64_t)dims.batch * dims.num_kv_heads * k > (int64_t)1 << 30) return SS_ERR_UNSUPPORTED;
    size_t need = ss::cache_ws_bytes(dims, k, pool.num_slots);
    if (!ws || ws_bytes < need) return SS_ERR_INVALID_ARG;
    return ss::launch_cache(pool, sel, req_ids, layer, num_layers, max_blk, k, dims, stamp,
                            slot_out, hit_out, miss_keys, miss_slots, counts, ws,
                            (cudaStream_t)stream);
}

ss_status flash_h2d_gather(const void* host_kv, int64_t host_blocks, const int64_t* miss_keys,
                           const int32_t* miss_slots, const int32_t* counts, int32_t max_misses,
                           void* pool_kv, int64_t block_bytes, void* stream) {
    if (!host_kv || !miss_keys || !miss_slots || !counts || !pool_kv) return SS_ERR_INVALID_ARG;
    if (host_blocks < 1 || max_misses < 0 || block_bytes < 16 || (block_bytes % 16) != 0)
        return SS_ERR_INVALID_ARG;
    if (!aligned16(host_kv) || !aligned16(pool_kv)) return SS_ERR_INVALID_ARG;
    return ss::launch_flash_h2d(host_kv, host_blocks, miss_keys, miss_slots, counts, max_misses,
                                pool_kv, block_bytes, (cudaStream_t)stream);
}

ss_status ss_preload_kernels(void) {
    static const bool ok = ss::preload_select() & ss::preload_attn() & ss::preload_cache() &
                           ss::preload_save() & ss::preload_ws() & ss::preload_meta() & ss::preload_h2d();
    return ok ? SS_OK : SS_ERR_CUDA;
}

ss_status flash_h2d_serve(const void* host_kv, int64_t host_blocks, const ss_h2d_job* jobs,
                          int32_t njobs, int64_t block_bytes, int32_t* flags, int64_t timeout_us,
                          uint64_t* stats_or_null, void* stream) {
    if (njobs < 0) return SS_ERR_INVALID_ARG;
    if (njobs == 0) return SS_OK;
    if (!host_kv || !jobs || !flags || host_blocks < 1) return SS_ERR_INVALID_ARG;
    if (block_bytes < 16 || (block_bytes % 16) != 0 || !aligned16(host_kv)) return SS_ERR_INVALID_ARG;
    // every kernel of the library must be loaded before a server spins (lazy
    // module loading could otherwise stall a producer kernel's first launch
    // behind the spinning server); outside stream capture only
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing((cudaStream_t)stream, &cap) == cudaSuccess && cap == cudaStreamCaptureStatusNone) {
        if (ss_preload_kernels() != SS_OK) return SS_ERR_CUDA;
    }
    if (stats_or_null && (reinterpret_cast<uintptr_t>(stats_or_null) & 7)) return SS_ERR_INVALID_ARG;
    return ss::launch_flash_h2d_serve(host_kv, host_blocks, jobs, njobs, block_bytes, flags, timeout_us,
                                      reinterpret_cast<unsigned long long*>(stats_or_null),
                                      (cudaStream_t)stream);
}

ss_status ss_flag_signal(int32_t* flag, void* stream) {
    if (!flag) return SS_ERR_INVALID_ARG;
    // little-endian: byte 0 = 1 makes the (zeroed) int32 equal to 1
    if (cudaMemsetAsync(flag, 1, 1, (cudaStream_t)stream) != cudaSuccess) return SS_ERR_CUDA;
    return SS_OK;
}

ss_status ss_flag_wait(const int32_t* flag, int32_t* counts_or_null, int64_t timeout_us, void* stream) {
    if (!flag) return SS_ERR_INVALID_ARG;
    return ss::launch_flag_wait(flag, counts_or_null, timeout_us, (cudaStream_t)stream);
}

ss_status sparse_decode_attn(const void* q, const void* pool_kv, const int32_t* slot, int32_t k,
                             const void* tail_kv, const int32_t* tail_len, ss_dims dims,
                             ss_dtype dt, float softmax_scale, const int32_t* counts, float* out,
                             void* ws, size_t ws_bytes, void* stream) {
    if (!q || !pool_kv || !slot || !tail_kv || !tail_len || !out || !dt_ok(dt) || !dims_ok(dims))
        return SS_ERR_INVALID_ARG;
    if (k < 1) return SS_ERR_INVALID_ARG;
    if (!aligned16(q) || !aligned16(pool_kv) || !aligned16(tail_kv) || !aligned16(out))
        return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    size_t need = ss::attn_ws_bytes(dims, k, dt);
    if (!ws || ws_bytes < need) return SS_ERR_INVALID_ARG;
    return ss::launch_sparse_attn(q, pool_kv, slot, k, tail_kv, tail_len, dims, dt, softmax_scale,
                                  counts, out, ws, (cudaStream_t)stream);
}

ss_status sparse_decode_attn_part(const void* q, const void* pool_kv, const int32_t* slot,
                                  const uint8_t* hit, int32_t mode, int32_t k, const void* tail_kv,
                                  const int32_t* tail_len, ss_dims dims, ss_dtype dt,
                                  float softmax_scale, const int32_t* counts, float* out, float* lse,
                                  void* ws, size_t ws_bytes, void* stream) {
    if (!q || !pool_kv || !slot || !tail_kv || !tail_len || !out || !lse || !dt_ok(dt) || !dims_ok(dims))
        return SS_ERR_INVALID_ARG;
    if (mode < 0 || mode > 2 || (mode != 0 && !hit) || k < 1) return SS_ERR_INVALID_ARG;
    if (!aligned16(q) || !aligned16(pool_kv) || !aligned16(tail_kv) || !aligned16(out))
        return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    size_t need = ss::attn_ws_bytes(dims, k, dt);
    if (!ws || ws_bytes < need) return SS_ERR_INVALID_ARG;
    return ss::launch_sparse_attn(q, pool_kv, slot, k, tail_kv, tail_len, dims, dt, softmax_scale,
                                  counts, out, ws, (cudaStream_t)stream, hit, mode, lse);
}

ss_status sparse_attn_merge(const float* out_a, const float* lse_a, const float* out_b,
                            const float* lse_b, int64_t rows, const int32_t* counts, float* out,
                            void* stream) {
    if (rows < 0) return SS_ERR_INVALID_ARG;
    if (rows == 0) return SS_OK;
    if (!out_a || !lse_a || !out_b || !lse_b || !out) return SS_ERR_INVALID_ARG;
    if (!aligned16(out_a) || !aligned16(out_b) || !aligned16(out)) return SS_ERR_INVALID_ARG;
    return ss::launch_attn_merge(out_a, lse_a, out_b, lse_b, rows, counts, out, (cudaStream_t)stream);
}

ss_status kv_append(const void* new_kv, void* tail_kv, int32_t* tail_len, int32_t advance,
                    ss_dims dims, ss_dtype dt, void* stream) {
    if (!new_kv || !tail_kv || !tail_len || !dt_ok(dt) || !dims_ok(dims)) return SS_ERR_INVALID_ARG;
    if (!aligned16(new_kv) || !aligned16(tail_kv)) return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    return ss::launch_kv_append(new_kv, tail_kv, tail_len, advance, dims, dt, (cudaStream_t)stream);
}

ss_status kv_seal_blocks(const int32_t* fill_req, int32_t n_fill, const void* tail_kv,
                         const int32_t* n_blk, int32_t max_blk, void* meta, void* staging,
                         void* ws, size_t ws_bytes, ss_dims dims, ss_dtype dt, void* stream) {
    if (n_fill < 0 || !dt_ok(dt) || !dims_ok(dims)) return SS_ERR_INVALID_ARG;
    if (n_fill == 0) return SS_OK;
    if (!fill_req || !tail_kv || !n_blk || !meta || !staging || !ws) return SS_ERR_INVALID_ARG;
    if (max_blk < 32 || (max_blk % 32) || n_fill > dims.batch) return SS_ERR_INVALID_ARG;
    if (!aligned16(tail_kv) || !aligned16(staging)) return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    if (ws_bytes < (size_t)n_fill * dims.num_kv_heads * 8) return SS_ERR_INVALID_ARG;
    return ss::launch_kv_seal(fill_req, n_fill, tail_kv, n_blk, max_blk, meta, staging, ws, dims,
                              dt, (cudaStream_t)stream);
}

ss_status kv_commit(const int32_t* fill_req, int32_t n_fill, int32_t* n_blk, int32_t* tail_len,
                    void* stream) {
    if (n_fill < 0) return SS_ERR_INVALID_ARG;
    if (n_fill == 0) return SS_OK;
    if (!fill_req || !n_blk || !tail_len) return SS_ERR_INVALID_ARG;
    return ss::launch_kv_commit(fill_req, n_fill, n_blk, tail_len, (cudaStream_t)stream);
}

ss_status ws_track(const int32_t* sel, int32_t k, ss_dims dims, int32_t max_blk, int64_t t,
                   int32_t w, int32_t* last_sel, int32_t* ring, int32_t* ws_count, void* stream) {
    if (!sel || !last_sel || !ring || !ws_count || !dims_ok(dims)) return SS_ERR_INVALID_ARG;
    if (k < 1 || w < 1 || max_blk < 1 || t < 0 || t >= ((int64_t)1 << 31)) return SS_ERR_INVALID_ARG;
    return ss::launch_ws_track(sel, k, dims, max_blk, t, w, last_sel, ring, ws_count,
                               (cudaStream_t)stream);
}

ss_status prefill_layer_save(const void* k_nhd, const void* v_nhd, int32_t n_tok, int32_t b,
                             int32_t req, int32_t layer, int32_t num_layers, int32_t max_blk,
                             ss_dims dims, ss_dtype dt, void* staging, void* meta, void* tail_kv,
                             int32_t* n_blk, int32_t* tail_len, void* host_kv, int64_t host_blocks,
                             void* ws, size_t ws_bytes, void* stream) {
    if (!k_nhd || !v_nhd || !staging || !meta || !tail_kv || !n_blk || !tail_len || !host_kv || !ws)
        return SS_ERR_INVALID_ARG;
    if (!dt_ok(dt) || !dims_ok(dims) || n_tok < 0 || b < 0 || b >= dims.batch || req < 0)
        return SS_ERR_INVALID_ARG;
    if (max_blk < 32 || (max_blk % 32) || (int64_t)n_tok > 32LL * max_blk) return SS_ERR_INVALID_ARG;
    if (layer < 0 || layer >= num_layers || host_blocks < max_blk || (host_blocks % max_blk))
        return SS_ERR_INVALID_ARG;
    if (!aligned16(k_nhd) || !aligned16(v_nhd) || !aligned16(staging) || !aligned16(tail_kv))
        return SS_ERR_INVALID_ARG;
    ss_status st = dims_supported(dims);
    if (st != SS_OK) return st;
    if (ws_bytes < (size_t)dims.num_kv_heads * max_blk * 8) return SS_ERR_INVALID_ARG;
    return ss::launch_prefill_layer_save(k_nhd, v_nhd, n_tok, b, req, layer, num_layers, max_blk, dims,
                                         dt, staging, meta, tail_kv, n_blk, tail_len, host_kv,
                                         host_blocks, ws, (cudaStream_t)stream);
}

int32_t ss_admit(const int64_t* ws_bytes, int32_t n, int64_t m_avl, uint8_t* admit_out) {
    if (n < 0 || (n > 0 && (!ws_bytes || !admit_out))) return -1;
    int64_t used = 0;
    int32_t admitted = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (used + ws_bytes[i] <= m_avl) {
            admit_out[i] = 1;
            used += ws_bytes[i];
            ++admitted;
        } else {
            admit_out[i] = 0;
        }
    }
    return admitted;
}

size_t ss_workspace_size(int32_t which, ss_dims dims, int32_t max_blk, int32_t k,
                         int32_t num_slots) {
    if (!dims_ok(dims) || k < 1) return 0;
    switch (which) {
        case SS_WS_SELECT:
            return ss::select_ws_bytes(dims, max_blk, k);
        case SS_WS_CACHE:
            return ss::cache_ws_bytes(dims, k, num_slots);
        case SS_WS_SEAL:
            return ((size_t)dims.batch * dims.num_kv_heads * 8 + 255) & ~(size_t)255;
        case SS_WS_PREFILL:
            return ((size_t)dims.num_kv_heads * max_blk * 8 + 255) & ~(size_t)255;
        case SS_WS_ATTN:
            // sized for the larger (bf16 / f32 use different warp counts)
            {
                size_t a = ss::attn_ws_bytes(dims, k, SS_BF16), b = ss::attn_ws_bytes(dims, k, SS_F32);
                return a > b ? a : b;
            }
        default:
            return 0;
    }
}

ss_status ss_decode_step_host(void* graph_exec, const void* q_host, void* q_dev, size_t q_bytes,
                              int32_t n_out, const void* const* out_dev, void* const* out_host,
                              const size_t* out_bytes, void* stream) {
    if (!graph_exec || n_out < 0 || (q_bytes && (!q_host || !q_dev))) return SS_ERR_INVALID_ARG;
    if (n_out > 0 && (!out_dev || !out_host || !out_bytes)) return SS_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (q_bytes && cudaMemcpyAsync(q_dev, q_host, q_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        return SS_ERR_CUDA;
    if (cudaGraphLaunch((cudaGraphExec_t)graph_exec, s) != cudaSuccess) return SS_ERR_CUDA;
    for (int i = 0; i < n_out; ++i) {
        if (!out_dev[i] || !out_host[i]) return SS_ERR_INVALID_ARG;
        if (cudaMemcpyAsync(out_host[i], out_dev[i], out_bytes[i], cudaMemcpyDeviceToHost, s) != cudaSuccess)
            return SS_ERR_CUDA;
    }
    return SS_OK;
}

ss_status ss_host_device_pointer(void* host, void** dev) {
    if (!host || !dev) return SS_ERR_INVALID_ARG;
    return cudaHostGetDevicePointer(dev, host, 0) == cudaSuccess ? SS_OK : SS_ERR_CUDA;
}

const char* ss_status_string(ss_status s) {
    switch (s) {
        case SS_OK: return "SS_OK";
        case SS_ERR_INVALID_ARG: return "SS_ERR_INVALID_ARG";
        case SS_ERR_UNSUPPORTED: return "SS_ERR_UNSUPPORTED";
        case SS_ERR_CAPACITY: return "SS_ERR_CAPACITY";
        case SS_ERR_CUDA: return "SS_ERR_CUDA";
        default: return "SS_ERR_UNKNOWN";
    }
}

const char* ss_version(void) { return "sparseserve-b200 0.1 (sm_100a)"; }

}  // extern "C"
