#include <cstdio>
__global__ void k(double a, double b, double* out, long long* t, int mode) {
    double x = a;
    float y = (float)a;
    __shared__ double s[64];
    s[threadIdx.x] = a;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) for (int i = 0; i < 1000; ++i) x = fma(x, b, 1e-9);
    if (mode == 1) for (int i = 0; i < 1000; ++i) y = fmaf(y, (float)b, 1e-9f);
    if (mode == 2) for (int i = 0; i < 1000; ++i) x = s[((int)x) & 31] + 1.0;
    if (mode == 3) for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffff, x, (i + 1) & 31);
    if (mode == 4) for (int i = 0; i < 1000; ++i) x = x * b;
    long long t1 = clock64();
    out[threadIdx.x] = x + y;
    if (threadIdx.x == 0) t[0] = t1 - t0;
}
int main() {
    double* o; long long* t; cudaMalloc(&o, 512); cudaMalloc(&t, 8);
    const char* names[] = {"dfma chain", "ffma chain", "lds+dadd chain", "shfl f64 chain", "dmul chain"};
    for (int m = 0; m < 5; ++m) {
        long long h;
        for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(1.0, 0.999999, o, t, m); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); }
        printf("%s: %.1f cycles/op\n", names[m], h / 1000.0);
    }
}
