#include <cstdio>
// per-step cost pieces of the LDL^T factorization loop
template <int MODE, int OWN>
__global__ void steps(double* out, long long* t, int np) {
    __shared__ double cb[2][128];
    const int tid = threadIdx.x;
    double av[OWN];
    int ai[OWN], aj[OWN];
    for (int r = 0; r < OWN; ++r) { int q = tid + 256 * r; ai[r] = q % 60; aj[r] = (q * 7) % 60; av[r] = 1.0 + q; }
    if (tid < 128) { cb[0][tid] = 2.0 + tid; cb[1][tid] = 3.0 + tid; }
    __syncthreads();
    long long t0 = clock64();
    double acc = 0;
    for (int k = 0; k < np; ++k) {
        double* c = cb[k & 1];
        if (MODE >= 1) {
#pragma unroll
            for (int r = 0; r < OWN; ++r) if (aj[r] == k && ai[r] >= k) c[ai[r]] = av[r];
        }
        __syncthreads();
        if (MODE >= 2) {
            const double dk = c[k];
            const double inv = dk != 0 ? 1.0 / dk : 0.0;
            if (MODE >= 3) {
                double ci[OWN], cj[OWN];
#pragma unroll
                for (int r = 0; r < OWN; ++r) { ci[r] = c[ai[r]]; cj[r] = c[aj[r]]; }
#pragma unroll
                for (int r = 0; r < OWN; ++r) av[r] = (aj[r] > k) ? av[r] - ci[r] * (cj[r] * inv) : av[r] * inv;
            } else acc += inv;
        }
    }
    long long t1 = clock64();
    double s = acc;
    for (int r = 0; r < OWN; ++r) s += av[r];
    out[tid] = s;
    if (tid == 0) t[0] = t1 - t0;
}
int main() {
    double* o; long long* t; long long h;
    cudaMalloc(&o, 8192); cudaMalloc(&t, 8);
    steps<0, 8><<<1, 256>>>(o, t, 60); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("bar only: %lld cyc/step\n", h / 60);
    steps<1, 8><<<1, 256>>>(o, t, 60); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("+publish: %lld cyc/step\n", h / 60);
    steps<2, 8><<<1, 256>>>(o, t, 60); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("+rcp: %lld cyc/step\n", h / 60);
    steps<3, 8><<<1, 256>>>(o, t, 60); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("+update: %lld cyc/step\n", h / 60);
    steps<3, 8><<<1, 128>>>(o, t, 60); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("+update 128 thr: %lld cyc/step\n", h / 60);
}
