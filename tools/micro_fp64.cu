#include <cstdio>
__global__ void fma_tp(double* out, long long* t, int n) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void ffma_tp(float* out, long long* t, int n) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
    const float b = 1.0000001f, c = 1e-9f;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void ddiv_lat(double* out, long long* t, int n) {
    double a = 1.0 + threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) a = 1.0 / (a + 1.0);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
    double* o; float* of; long long* t; long long h;
    cudaMalloc(&o, 8192); cudaMalloc(&of, 8192); cudaMalloc(&t, 8);
    const int n = 4096;
    for (int threads : {32, 256, 1024}) {
        fma_tp<<<1, threads>>>(o, t, n); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("DFMA threads=%4d: %.2f DFMA/clk/SM\n", threads, 8.0 * n * threads / h);
        ffma_tp<<<1, threads>>>(of, t, n); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("FFMA threads=%4d: %.2f FFMA/clk/SM\n", threads, 8.0 * n * threads / h);
    }
    ddiv_lat<<<1, 32>>>(o, t, 1000); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("DDIV+DADD dependent latency: %.1f cycles\n", h / 1000.0);
    int v; cudaDeviceGetAttribute(&v, cudaDevAttrSingleToDoublePrecisionPerfRatio, 0);
    printf("single/double perf ratio attribute: %d\n", v);
}
// dependent DFMA chain latency + block barrier cost
__global__ void dfma_lat(double* out, long long* t, int n) {
    double a = 1.0 + threadIdx.x;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) a = fma(a, 1.0000001, 1e-9);
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void bar_cost(long long* t, int n) {
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
__global__ void lds_lat(double* out, long long* t, int n) {
    __shared__ double s[64];
    if (threadIdx.x < 64) s[threadIdx.x] = 0.0;
    __syncthreads();
    int i = 0;
    double acc = 0;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) { double v = s[i]; acc += v; i = (int)v; }
    long long t1 = clock64();
    out[threadIdx.x] = acc;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
struct Extra { Extra() {
    double* o; long long* t; long long h;
    cudaMalloc(&o, 8192); cudaMalloc(&t, 8);
    dfma_lat<<<1, 32>>>(o, t, 1000); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.1f cycles\n", h / 1000.0);
    for (int th : {32, 256, 1024}) { bar_cost<<<1, th>>>(t, 1000); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads x%d threads: %.1f cycles\n", th, h / 1000.0); }
    lds_lat<<<1, 32>>>(o, t, 1000); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
    printf("LDS.64 + DADD dependent: %.1f cycles\n", h / 1000.0);
} } g_extra;
