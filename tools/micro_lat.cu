#include <cstdio>
__global__ void lat(double* out, long long* t, int n) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999, c = 1e-12;
    float fa = 1.0f + threadIdx.x, fb = 0.9999f, fc = 1e-6f;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) fa = fmaf(fa, fb, fc);
    long long t2 = clock64();
    double s = a;
    for (int i = 0; i < n; ++i) s = __shfl_sync(0xffffffffu, s, (threadIdx.x + 1) & 31);
    long long t3 = clock64();
    __shared__ double sm[64];
    sm[threadIdx.x] = s;
    __syncwarp();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) { idx = (int)sm[idx & 31] & 31; }
    long long t4 = clock64();
    out[threadIdx.x] = a + fa + s + idx;
    if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; }
}
int main() {
    double* o; long long* t; long long h[4];
    cudaMalloc(&o, 4096); cudaMalloc(&t, 64);
    lat<<<1, 32>>>(o, t, 1000);
    cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
    printf("DFMA dep latency %.1f, FFMA %.1f, SHFL(double) %.1f, LDS.64+cvt %.1f cycles\n", h[0]/1000.0, h[1]/1000.0, h[2]/1000.0, h[3]/1000.0);
}
