// Probe: what a persistent one-CTA-per-SM launch costs on its own (the fixed
// part of a small sparse_decode_attn launch).  Three kernels back to back on
// one stream: stamp_a (1 thread, globaltimer at its end), body (148 CTAs x 192
// threads, S bytes of dynamic shared memory, globaltimer at every CTA's entry
// and exit, optionally one 16 KiB bulk copy per warp), stamp_c (1 thread,
// globaltimer at its start).  Prints the gaps previous-kernel-end -> first CTA
// entry, last CTA exit -> next kernel start, the body's entry/exit spread, and
// the CUDA-event time of the body alone (after a device spin, so host launch
// overhead is hidden).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void spin(long long ns) {
    unsigned long long t0 = gtime();
    while ((long long)(gtime() - t0) < ns) {}
}
__global__ void stamp(unsigned long long* out) { *out = gtime(); }

__global__ void body(unsigned long long* entry, unsigned long long* exit_, const char* src, int copy) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[8];
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) entry[blockIdx.x] = gtime();
    if (copy && lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[w])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[w])), "r"(16384));
        const char* g = src + ((size_t)(blockIdx.x * 6 + w) * 7919 % 65536) * 16384;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         s32(sm + w * 16384)),
                     "l"(g), "r"(16384), "r"(s32(&bar[w]))
                     : "memory");
        asm volatile(
            "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W;\n}" ::"r"(
                s32(&bar[w]))
            : "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) exit_[blockIdx.x] = gtime();
}

int main() {
    const int nsm = 148;
    unsigned long long *d_t, *h_t;
    cudaMalloc(&d_t, (2 + 2 * nsm) * 8);
    cudaMallocHost(&h_t, (2 + 2 * nsm) * 8);
    char* src;
    cudaMalloc(&src, (size_t)65536 * 16384);  // 1 GiB
    cudaMemset(src, 1, (size_t)65536 * 16384);
    cudaFuncSetAttribute(body, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int smems[3] = {0, 100 * 1024, 197 * 1024};
    for (int copy = 0; copy < 2; ++copy)
        for (int si = 0; si < 3; ++si) {
            const int S = copy ? (smems[si] < 6 * 16384 ? 6 * 16384 : smems[si]) : smems[si];
            double gap_in = 0, gap_out = 0, spread_in = 0, span = 0, ev = 0, ev_b2b = 0;
            const int reps = 20;
            for (int r = 0; r < reps + 2; ++r) {
                spin<<<1, 1>>>(200000);
                stamp<<<1, 1>>>(d_t);
                body<<<nsm, 192, S>>>(d_t + 2, d_t + 2 + nsm, src, copy);
                stamp<<<1, 1>>>(d_t + 1);
                cudaMemcpy(h_t, d_t, (2 + 2 * nsm) * 8, cudaMemcpyDeviceToHost);
                unsigned long long mn = ~0ull, mx = 0, emx = 0;
                for (int i = 0; i < nsm; ++i) {
                    mn = h_t[2 + i] < mn ? h_t[2 + i] : mn;
                    emx = h_t[2 + i] > emx ? h_t[2 + i] : emx;
                    mx = h_t[2 + nsm + i] > mx ? h_t[2 + nsm + i] : mx;
                }
                if (r < 2) continue;
                gap_in += (double)(mn - h_t[0]);
                gap_out += (double)(h_t[1] - mx);
                spread_in += (double)(emx - mn);
                span += (double)(mx - mn);
                spin<<<1, 1>>>(200000);
                cudaEventRecord(e0);
                body<<<nsm, 192, S>>>(d_t + 2, d_t + 2 + nsm, src, copy);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                ev += ms * 1e3;
                spin<<<1, 1>>>(2000000);
                cudaEventRecord(e0);
                for (int k = 0; k < 20; ++k) body<<<nsm, 192, S>>>(d_t + 2, d_t + 2 + nsm, src, copy);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
                ev_b2b += ms * 1e3 / 20;
            }
            printf("{\"copy16k_per_warp\": %d, \"smem_kib\": %d, \"gap_prev_end_to_first_entry_us\": %.2f, "
                   "\"entry_spread_us\": %.2f, \"entry_to_last_exit_us\": %.2f, \"gap_last_exit_to_next_start_us\": %.2f, "
                   "\"event_us_single\": %.2f, \"event_us_back_to_back\": %.2f}\n",
                   copy, S / 1024, gap_in / reps / 1e3, spread_in / reps / 1e3, span / reps / 1e3, gap_out / reps / 1e3,
                   ev / reps, ev_b2b / reps);
        }
    cudaError_t err = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(err));
    return 0;
}
