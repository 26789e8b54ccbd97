// Throughput of the legacy warp-level tensor-core path (mma.sync, HMMA SASS) on
// this B200: m16n8k8 TF32 and m16n8k16 BF16 with FP32 accumulators, and FFMA2 for
// comparison.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_mma tools/micro_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void tf32_kernel(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile(
                "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void bf16_kernel(float* out, int iters) {
    unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
    float c[8][4] = {};
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};"
                : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    float s = 0;
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma2_kernel(float* out, int iters) {
    float2 c[16];
    const float2 a = make_float2(threadIdx.x * 1e-3f, 1.0001f), b = make_float2(0.999f, 1e-4f);
    for (int t = 0; t < 16; ++t) c[t] = make_float2(t, t);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int t = 0; t < 16; ++t) c[t] = __ffma2_rn(a, c[t], b);
    }
    float s = 0;
    for (int t = 0; t < 16; ++t) s += c[t].x + c[t].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        const int blocks = sms * 2, threads = 32 * warps;
        float ms;
        tf32_kernel<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        tf32_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        double flop = 2.0 * 16 * 8 * 8 * 8.0 * iters * blocks * warps;
        printf("warps/block %2d  tf32 m16n8k8  %.1f TFLOP/s\n", warps, flop / ms / 1e9);
        bf16_kernel<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        bf16_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flop = 2.0 * 16 * 8 * 16 * 8.0 * iters * blocks * warps;
        printf("warps/block %2d  bf16 m16n8k16 %.1f TFLOP/s\n", warps, flop / ms / 1e9);
        ffma2_kernel<<<blocks, threads>>>(out, 16);
        cudaEventRecord(e0);
        ffma2_kernel<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flop = 2.0 * 2 * 16.0 * iters * blocks * threads;
        printf("warps/block %2d  ffma2         %.1f TFLOP/s\n", warps, flop / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
