// Probe: cycles one warp spends merging nc partials of G heads from shared
// memory (the sparse_decode_attn end-of-range merge's compute), in isolation.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/merge_probe tools/merge_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kStride = 132;

template <int G, int VAR>
__global__ void merge_probe(const float* src, float* out, long long* cyc, int nc) {
    extern __shared__ float P[];
    const int lane = threadIdx.x;
    for (int i = lane; i < nc * G * kStride; i += 32) P[i] = src[i];
    __syncwarp();
    float M[G], L[G], O[G][4];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        M[g] = -INFINITY;
        L[g] = 0.f;
        O[g][0] = O[g][1] = O[g][2] = O[g][3] = 0.f;
    }
    long long t0 = clock64();
    const int n = nc;
    float mnew[G], corr[G];
#pragma unroll
    for (int g = 0; g < G; ++g) mnew[g] = M[g];
#pragma unroll 1
    for (int j = 0; j < n; ++j)
#pragma unroll
        for (int g = 0; g < G; ++g) mnew[g] = fmaxf(mnew[g], P[(j * G + g) * kStride]);
#pragma unroll
    for (int g = 0; g < G; ++g) {
        corr[g] = M[g] == -INFINITY ? 0.f : exp2f(M[g] - mnew[g]);
        L[g] *= corr[g];
        O[g][0] *= corr[g], O[g][1] *= corr[g], O[g][2] *= corr[g], O[g][3] *= corr[g];
        M[g] = mnew[g];
    }
    long long t1 = clock64();
    if (VAR == 0) {
#pragma unroll 1
        for (int j = 0; j < n; ++j) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float* pj = P + (j * G + g) * kStride;
                const float2 ml = *reinterpret_cast<const float2*>(pj);
                const float sc = M[g] == -INFINITY ? 0.f : exp2f(ml.x - M[g]);
                L[g] = fmaf(ml.y, sc, L[g]);
                const float4 ov = *reinterpret_cast<const float4*>(pj + 4 + 4 * lane);
                O[g][0] = fmaf(ov.x, sc, O[g][0]);
                O[g][1] = fmaf(ov.y, sc, O[g][1]);
                O[g][2] = fmaf(ov.z, sc, O[g][2]);
                O[g][3] = fmaf(ov.w, sc, O[g][3]);
            }
        }
    } else {
#pragma unroll 4
        for (int j = 0; j < n; ++j) {
#pragma unroll
            for (int g = 0; g < G; ++g) {
                const float* pj = P + (j * G + g) * kStride;
                const float2 ml = *reinterpret_cast<const float2*>(pj);
                const float sc = exp2f(ml.x - M[g]);
                L[g] = fmaf(ml.y, sc, L[g]);
                const float4 ov = *reinterpret_cast<const float4*>(pj + 4 + 4 * lane);
                O[g][0] = fmaf(ov.x, sc, O[g][0]);
                O[g][1] = fmaf(ov.y, sc, O[g][1]);
                O[g][2] = fmaf(ov.z, sc, O[g][2]);
                O[g][3] = fmaf(ov.w, sc, O[g][3]);
            }
        }
    }
    long long t2 = clock64();
#pragma unroll
    for (int g = 0; g < G; ++g) {
        const float inv = L[g] > 0.f ? 1.f / L[g] : 0.f;
        *reinterpret_cast<float4*>(out + (g * 32 + lane) * 4) =
            make_float4(O[g][0] * inv, O[g][1] * inv, O[g][2] * inv, O[g][3] * inv);
    }
    long long t3 = clock64();
    if (lane == 0) {
        cyc[0] = t1 - t0;
        cyc[1] = t2 - t1;
        cyc[2] = t3 - t2;
    }
}

template <int G, int VAR>
void run(const float* src, float* out, long long* cyc, int nc) {
    long long h[3];
    for (int rep = 0; rep < 3; ++rep) {
        merge_probe<G, VAR><<<1, 32, nc * G * kStride * 4>>>(src, out, cyc, nc);
        cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    }
    printf("{\"G\": %d, \"variant\": %d, \"nc\": %d, \"max_pass_cyc\": %lld, \"sum_pass_cyc\": %lld, \"store_cyc\": %lld}\n", G,
           VAR, nc, h[0], h[1], h[2]);
}

int main() {
    float *src, *out;
    long long* cyc;
    cudaMalloc(&src, 32 * 8 * kStride * 4);
    cudaMalloc(&out, 8 * 128 * 4);
    cudaMalloc(&cyc, 64);
    cudaMemset(src, 0, 32 * 8 * kStride * 4);
    for (int nc : {8, 15}) {
        run<1, 0>(src, out, cyc, nc);
        run<4, 0>(src, out, cyc, nc);
        run<4, 1>(src, out, cyc, nc);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
