// kv_save.cu -- NEXT-1: the decode-step KV append and the save path
// (§3.2.2: "the hidden states ... are projected into a KV tensor
// of shape (B, H, D) ... saved into the free slots in the corresponding KV
// blocks in HBM.  Once a KV block is full, it is asynchronously flushed into
// DRAM using a separate CUDA stream"; "Once a KV block reaches
// its capacity, its associated metadata is created"; PAPER.md:151-153 FlashD2H:
// "(1) the contiguous KV tensor is first copied into a DRAM buffer with a
// single memcpy, and (2) once the transfer completes, CPU threads redistribute
// the buffered data into the corresponding DRAM KV blocks").
//
//   kv_append      one CTA per request: (optionally) counts the new token in
//                  tail_len, writes its K and V rows of every KV head into the
//                  HBM tail block at row tail_len - 1
//   kv_seal_blocks for the requests whose tail just filled: copy the full tails
//                  into a contiguous staging buffer (list order) and build their
//                  metadata (meta_update kernel) as block n_blk[b]
//   kv_commit      n_blk[b] += 1, tail_len[b] = 0 for the sealed requests
//   flash_d2h_save one cudaMemcpyAsync of the staging blocks into pinned DRAM,
//                  then a host function hands the scatter to the engine's CPU
//                  threads (std::thread pool) and returns when every block is
//                  in its DRAM home host_kv[key % host_blocks] -- so work
//                  enqueued after it on the same stream sees the saved blocks.
//
// Roofline: append/seal move 2*d*es bytes per (request, head) per step and
// 16 KiB per sealed block (HBM, negligible); FlashD2H is host-link + host-DRAM
// bound (one bulk D2H copy instead of one cudaMemcpy per 16 KiB block).
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "common.cuh"

namespace ss {

ss_status launch_meta_update(const void* keys, int64_t key_stride, const int64_t* dst_idx,
                             int64_t n, void* meta, ss_dtype dt, cudaStream_t stream);

constexpr int kSaveThreads = 256;

// ---- kv_append ----------------------------------------------------------------
__global__ void __launch_bounds__(kSaveThreads)
kv_append_kernel(const uint4* __restrict__ new_kv, uint4* __restrict__ tail, int32_t* tail_len,
                 int advance, int Hkv, int row_vecs /* 16-byte vectors per token row */) {
    __shared__ int s_row;
    const int b = blockIdx.x;
    if (threadIdx.x == 0) {
        int t = tail_len[b];
        if (advance) {
            t += 1;
            tail_len[b] = t;
        }
        s_row = t - 1;
    }
    __syncthreads();
    const int row = s_row;
    if (row < 0 || row >= kBlockTokens) return;  // precondition violated: nothing written
    const int per_head = 2 * row_vecs;           // K row + V row
    for (int i = threadIdx.x; i < Hkv * per_head; i += kSaveThreads) {
        const int h = i / per_head, r = i % per_head;
        const int half = r / row_vecs, v = r % row_vecs;
        const int64_t src = (((int64_t)b * Hkv + h) * 2 + half) * row_vecs + v;
        const int64_t dst = ((((int64_t)b * Hkv + h) * 2 + half) * kBlockTokens + row) * row_vecs + v;
        tail[dst] = new_kv[src];
    }
}

// ---- kv_seal_blocks ------------------------------------------------------------
__global__ void __launch_bounds__(kSaveThreads)
kv_seal_copy_kernel(const int32_t* __restrict__ fill_req, const uint4* __restrict__ tail,
                    const int32_t* __restrict__ n_blk, int Hkv, int max_blk, int block_vecs,
                    uint4* __restrict__ staging, int64_t* __restrict__ dst_idx) {
    const int i = blockIdx.x, h = blockIdx.y;
    const int b = fill_req[i];
    const uint4* src = tail + ((int64_t)b * Hkv + h) * block_vecs;
    uint4* dst = staging + ((int64_t)i * Hkv + h) * block_vecs;
    for (int v = threadIdx.x; v < block_vecs; v += kSaveThreads) dst[v] = src[v];
    // a full block table (n_blk == max_blk) has no row for the new block: no
    // metadata is written (precondition of the call; the engine checks it)
    if (threadIdx.x == 0)
        dst_idx[(int64_t)i * Hkv + h] = n_blk[b] < max_blk ? ((int64_t)b * Hkv + h) * max_blk + n_blk[b] : -1;
}

__global__ void kv_commit_kernel(const int32_t* __restrict__ fill_req, int n_fill, int32_t* n_blk,
                                 int32_t* tail_len) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_fill; i += gridDim.x * blockDim.x) {
        const int b = fill_req[i];
        n_blk[b] += 1;
        tail_len[b] = 0;
    }
}

ss_status launch_kv_append(const void* new_kv, void* tail_kv, int32_t* tail_len, int advance,
                           const ss_dims& d, ss_dtype dt, cudaStream_t stream) {
    const int es = dt == SS_BF16 ? 2 : 4;
    kv_append_kernel<<<d.batch, kSaveThreads, 0, stream>>>((const uint4*)new_kv, (uint4*)tail_kv,
                                                           tail_len, advance, d.num_kv_heads,
                                                           kHeadDim * es / 16);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

ss_status launch_kv_seal(const int32_t* fill_req, int n_fill, const void* tail_kv,
                         const int32_t* n_blk, int max_blk, void* meta, void* staging, void* ws,
                         const ss_dims& d, ss_dtype dt, cudaStream_t stream) {
    if (n_fill == 0) return SS_OK;
    const int es = dt == SS_BF16 ? 2 : 4;
    const int block_vecs = 2 * kBlockTokens * kHeadDim * es / 16;
    int64_t* dst_idx = (int64_t*)ws;
    kv_seal_copy_kernel<<<dim3(n_fill, d.num_kv_heads), kSaveThreads, 0, stream>>>(
        fill_req, (const uint4*)tail_kv, n_blk, d.num_kv_heads, max_blk, block_vecs,
        (uint4*)staging, dst_idx);
    SS_LAUNCH_CHECK();
    // metadata of the staged blocks (their K halves, stride = one [2][32][d] block)
    return launch_meta_update(staging, 2 * kBlockTokens * kHeadDim, dst_idx,
                              (int64_t)n_fill * d.num_kv_heads, meta, dt, stream);
}

ss_status launch_kv_commit(const int32_t* fill_req, int n_fill, int32_t* n_blk, int32_t* tail_len,
                           cudaStream_t stream) {
    if (n_fill == 0) return SS_OK;
    kv_commit_kernel<<<(n_fill + 255) / 256, 256, 0, stream>>>(fill_req, n_fill, n_blk, tail_len);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

}  // namespace ss

// ---- FlashD2H: CPU-assisted saving (host side) --------------------------------
struct ss_d2h_engine {
    std::vector<std::thread> workers;
    std::mutex m;
    std::condition_variable cv;
    std::deque<std::function<void()>> q;
    bool stop = false;

    explicit ss_d2h_engine(int n) {
        for (int i = 0; i < n; ++i)
            workers.emplace_back([this] {
                for (;;) {
                    std::function<void()> task;
                    {
                        std::unique_lock<std::mutex> lk(m);
                        cv.wait(lk, [this] { return stop || !q.empty(); });
                        if (stop && q.empty()) return;
                        task = std::move(q.front());
                        q.pop_front();
                    }
                    task();
                }
            });
    }
    ~ss_d2h_engine() {
        {
            std::lock_guard<std::mutex> lk(m);
            stop = true;
        }
        cv.notify_all();
        for (auto& t : workers) t.join();
    }
};

namespace {
// One scatter of a batch of blocks, split into chunks so the D2H copy of chunk
// c+1 overlaps the CPU scatter of chunk c: stream order is
//   memcpy(c0), hostfn(c0 -> enqueue), memcpy(c1), hostfn(c1 -> enqueue), ...,
//   hostfn(wait): the last host function blocks the stream until every block
// is in DRAM, so work after it on the stream sees the saved blocks.
struct ScatterJob {
    ss_d2h_engine* eng;
    const char* src;  // pinned DRAM landing buffer, blocks back to back
    char* host_kv;
    std::vector<int64_t> keys;
    int64_t host_blocks, block_bytes;
    std::mutex dm;
    std::condition_variable dcv;
    int64_t pending = 0;  // enqueued, unfinished tasks
};

struct ChunkArg {
    ScatterJob* job;
    int64_t i0, i1;
};

void copy_blocks(ScatterJob* job, int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i)
        memcpy(job->host_kv + (job->keys[i] % job->host_blocks) * job->block_bytes,
               job->src + i * job->block_bytes, (size_t)job->block_bytes);
}

void CUDART_CB chunk_host_fn(void* p) {
    ChunkArg* c = (ChunkArg*)p;
    ScatterJob* job = c->job;
    const int nt = (int)job->eng->workers.size();
    if (nt == 0) {
        copy_blocks(job, c->i0, c->i1);
    } else {
        const int64_t n = c->i1 - c->i0;
        const int parts = (int)std::min<int64_t>(n, nt);
        {
            std::lock_guard<std::mutex> g(job->dm);
            job->pending += parts;
        }
        {
            std::lock_guard<std::mutex> lk(job->eng->m);
            for (int t = 0; t < parts; ++t) {
                const int64_t a = c->i0 + n * t / parts, b = c->i0 + n * (t + 1) / parts;
                job->eng->q.emplace_back([job, a, b] {
                    copy_blocks(job, a, b);
                    std::lock_guard<std::mutex> g(job->dm);
                    if (--job->pending == 0) job->dcv.notify_all();
                });
            }
        }
        job->eng->cv.notify_all();
    }
    delete c;
}

void CUDART_CB wait_host_fn(void* p) {
    ScatterJob* job = (ScatterJob*)p;
    {
        std::unique_lock<std::mutex> lk(job->dm);
        job->dcv.wait(lk, [job] { return job->pending == 0; });
    }
    delete job;
}

constexpr int64_t kD2HChunkBytes = 4 << 20;  // overlap granularity
}  // namespace

extern "C" {

ss_status ss_d2h_create(int32_t num_threads, ss_d2h_engine** out) {
    if (!out || num_threads < 0 || num_threads > 256) return SS_ERR_INVALID_ARG;
    *out = new ss_d2h_engine(num_threads);
    return SS_OK;
}

ss_status ss_d2h_destroy(ss_d2h_engine* eng) {
    delete eng;
    return SS_OK;
}

ss_status flash_d2h_save(ss_d2h_engine* eng, const void* staging, void* host_buf, int64_t n_blocks,
                         const int64_t* keys, void* host_kv, int64_t host_blocks,
                         int64_t block_bytes, void* stream) {
    if (!eng || n_blocks < 0) return SS_ERR_INVALID_ARG;
    if (n_blocks == 0) return SS_OK;
    if (!staging || !host_buf || !keys || !host_kv || host_blocks < 1 || block_bytes < 16)
        return SS_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    ScatterJob* job = new ScatterJob();
    job->eng = eng;
    job->src = (const char*)host_buf;
    job->host_kv = (char*)host_kv;
    job->keys.assign(keys, keys + n_blocks);
    job->host_blocks = host_blocks;
    job->block_bytes = block_bytes;
    const int64_t per = std::max<int64_t>(1, kD2HChunkBytes / block_bytes);
    for (int64_t i0 = 0; i0 < n_blocks; i0 += per) {
        const int64_t i1 = std::min(n_blocks, i0 + per);
        if (cudaMemcpyAsync((char*)host_buf + i0 * block_bytes, (const char*)staging + i0 * block_bytes,
                            (size_t)((i1 - i0) * block_bytes), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaLaunchHostFunc(s, chunk_host_fn, new ChunkArg{job, i0, i1}) != cudaSuccess)
            return SS_ERR_CUDA;  // (job leaks on this error path; the stream is broken anyway)
    }
    if (cudaLaunchHostFunc(s, wait_host_fn, job) != cudaSuccess) return SS_ERR_CUDA;
    return SS_OK;
}

}  // extern "C"

// ---- NEXT-4: layer-segmented prefill, storage side ------------------------------
// (§3.4: "The KV blocks of all finished layers can be
// immediately evicted after being saved to DRAM"; P:129/137 (N,H,D) -> (H,N,D)).
// One prefill layer of one request: the projection output K, V [n][Hkv][d]
// ((N,H,D) layout) is re-laid out on the GPU into per-head 32-token blocks
// [Hkv][nb][2][32][d] (staging) + the partial tail, the metadata of every full
// block is built, and since the blocks of one (request, layer, head) are
// contiguous in their DRAM home (keys j = 0..nb-1 are consecutive), the save is
// Hkv large DMA copies (cudaMemcpyAsync) -- no SM or CPU work for the bytes.
namespace ss {

__global__ void __launch_bounds__(kSaveThreads)
prefill_relayout_kernel(const uint4* __restrict__ k_nhd, const uint4* __restrict__ v_nhd, int n_tok,
                        int nb, int Hkv, int row_vecs, int b, int max_blk, uint4* __restrict__ staging,
                        uint4* __restrict__ tail, int64_t* __restrict__ dst_idx) {
    const int j = blockIdx.x, h = blockIdx.y;
    const int block_vecs = 2 * kBlockTokens * row_vecs;
    uint4* dst = j < nb ? staging + ((int64_t)h * nb + j) * block_vecs
                        : tail + ((int64_t)b * Hkv + h) * block_vecs;
    for (int i = threadIdx.x; i < block_vecs; i += kSaveThreads) {
        const int half = i / (kBlockTokens * row_vecs);
        const int t = (i / row_vecs) % kBlockTokens;
        const int v = i % row_vecs;
        const int64_t tok = (int64_t)j * kBlockTokens + t;
        if (tok < n_tok) {
            const uint4* src = half ? v_nhd : k_nhd;
            dst[i] = src[(tok * Hkv + h) * row_vecs + v];
        } else if (j < nb) {
            // (cannot happen: full blocks only)
        }
    }
    if (threadIdx.x == 0 && j < nb) dst_idx[(int64_t)h * nb + j] = ((int64_t)b * Hkv + h) * max_blk + j;
}

__global__ void prefill_counters_kernel(int32_t* n_blk, int32_t* tail_len, int b, int nb, int rem) {
    n_blk[b] = nb;
    tail_len[b] = rem;
}

ss_status launch_prefill_layer_save(const void* k_nhd, const void* v_nhd, int n_tok, int b, int req,
                                    int layer, int num_layers, int max_blk, const ss_dims& d,
                                    ss_dtype dt, void* staging, void* meta, void* tail_kv,
                                    int32_t* n_blk, int32_t* tail_len, void* host_kv,
                                    int64_t host_blocks, void* ws, cudaStream_t stream) {
    const int es = dt == SS_BF16 ? 2 : 4;
    const int row_vecs = kHeadDim * es / 16;
    const int nb = n_tok / kBlockTokens, rem = n_tok % kBlockTokens;
    const int Hkv = d.num_kv_heads;
    const int64_t bb = 2LL * kBlockTokens * kHeadDim * es;
    int64_t* dst_idx = (int64_t*)ws;
    const int grid_x = nb + (rem ? 1 : 0);
    if (grid_x > 0) {
        prefill_relayout_kernel<<<dim3(grid_x, Hkv), kSaveThreads, 0, stream>>>(
            (const uint4*)k_nhd, (const uint4*)v_nhd, n_tok, nb, Hkv, row_vecs, b, max_blk,
            (uint4*)staging, (uint4*)tail_kv, dst_idx);
        SS_LAUNCH_CHECK();
    }
    if (nb > 0) {
        ss_status st = launch_meta_update(staging, 2 * kBlockTokens * kHeadDim, dst_idx,
                                          (int64_t)nb * Hkv, meta, dt, stream);
        if (st != SS_OK) return st;
        for (int h = 0; h < Hkv; ++h) {
            const int64_t key0 = (((int64_t)req * num_layers + layer) * Hkv + h) * max_blk;
            const int64_t phys0 = key0 % host_blocks;
            if (cudaMemcpyAsync((char*)host_kv + phys0 * bb, (const char*)staging + (int64_t)h * nb * bb,
                                (size_t)(nb * bb), cudaMemcpyDeviceToHost, stream) != cudaSuccess)
                return SS_ERR_CUDA;
        }
    }
    prefill_counters_kernel<<<1, 1, 0, stream>>>(n_blk, tail_len, b, nb, rem);
    SS_LAUNCH_CHECK();
    return SS_OK;
}

bool preload_save() {
    return preload_fn(kv_append_kernel) && preload_fn(kv_seal_copy_kernel) && preload_fn(kv_commit_kernel) &&
           preload_fn(prefill_relayout_kernel) && preload_fn(prefill_counters_kernel);
}

}  // namespace ss
