// Probe: can a 1-D TMA bulk copy (cp.async.bulk global->shared) source pinned,
// host-mapped memory, and at what bandwidth vs. 16-byte zero-copy loads?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_host_probe tools/tma_host_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int BB = 16384;

__global__ void tma_gather(const char* host, const int64_t* idx, int n, char* dst) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar[2];
    int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    char* buf = sm + w * 2 * BB;  // 4 warps per CTA
    uint64_t* b = (uint64_t*)(sm + 4 * 2 * BB) + w * 2;
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&b[0])));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&b[1])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    int gw = blockIdx.x * 4 + w, nw = gridDim.x * 4;
    uint32_t ph[2] = {0, 0};
    int st = 0;
    for (int i = gw; i < n; i += nw) {
        if (lane == 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&b[st])), "r"(BB));
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(s32(buf + st * BB)), "l"(host + idx[i] * BB), "r"(BB), "r"(s32(&b[st])) : "memory");
        }
        uint32_t done = 0;
        while (!done)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(done) : "r"(s32(&b[st])), "r"(ph[st]) : "memory");
        ph[st] ^= 1;
        // write back to HBM with a bulk store
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         ::"l"(dst + (int64_t)i * BB), "r"(s32(buf + st * BB)), "r"(BB) : "memory");
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
        st ^= 1;
    }
}

__global__ void ldg_gather(const uint4* host, const int64_t* idx, int n, uint4* dst) {
    int lane = threadIdx.x % 32;
    int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32, nw = gridDim.x * (int64_t)blockDim.x / 32;
    for (int64_t i = gw; i < n; i += nw) {
        const uint4* s = host + idx[i] * (BB / 16);
        uint4* d = dst + i * (BB / 16);
        for (int v = lane; v < BB / 16; v += 256) {
            uint4 r[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) r[u] = __ldg(s + v + 32 * u);
#pragma unroll
            for (int u = 0; u < 8; ++u) d[v + 32 * u] = r[u];
        }
    }
}

int main() {
    const int64_t HB = 1 << 16;  // 1 GiB host
    char* h;
    cudaHostAlloc(&h, HB * BB, cudaHostAllocMapped);
    for (int64_t i = 0; i < HB * BB; i += 4096) h[i] = (char)(i / 4096);
    const int n = 8192;
    int64_t* idx_h = new int64_t[n];
    for (int i = 0; i < n; ++i) idx_h[i] = (int64_t)((i * 2654435761ull) % HB);
    int64_t* idx;
    cudaMalloc(&idx, n * 8);
    cudaMemcpy(idx, idx_h, n * 8, cudaMemcpyHostToDevice);
    char *dst, *dst2;
    cudaMalloc(&dst, (int64_t)n * BB);
    cudaMalloc(&dst2, (int64_t)n * BB);
    char* hd;
    cudaHostGetDevicePointer((void**)&hd, h, 0);
    int smem = 4 * 2 * BB + 1024;
    cudaFuncSetAttribute(tma_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int grid : {148, 296}) {
        tma_gather<<<grid, 128, smem>>>(hd, idx, n, dst);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("tma_gather error: %s\n", cudaGetErrorString(e)); return 1; }
        cudaEventRecord(a);
        for (int r = 0; r < 3; ++r) tma_gather<<<grid, 128, smem>>>(hd, idx, n, dst);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("TMA bulk from host  ctas=%d: %.1f GB/s\n", grid, 3.0 * n * BB / ms / 1e6);
    }
    ldg_gather<<<296, 512>>>((const uint4*)hd, idx, n, (uint4*)dst2);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 3; ++r) ldg_gather<<<296, 512>>>((const uint4*)hd, idx, n, (uint4*)dst2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("LDG zero-copy       : %.1f GB/s\n", 3.0 * n * BB / ms / 1e6);
    // verify
    char* chk = new char[(int64_t)n * BB];
    cudaMemcpy(chk, dst, (int64_t)n * BB, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < n; ++i)
        if (memcmp(chk + (int64_t)i * BB, h + idx_h[i] * BB, BB)) ++bad;
    printf("TMA result mismatching blocks: %d / %d\n", bad, n);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
