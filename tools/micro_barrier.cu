// Cycles per barrier-separated step on one CTA of 256 threads (clock64):
//   0: __syncthreads only            1: LDS + DFMA + STS + __syncthreads
//   2: LDS + STS + __syncthreads     3: LDS + FFMA + STS + __syncthreads
//   4: LDS.64 + DADD(const) + STS    5: mode 1, shared reads of a warp-private slot
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro_barrier tools/micro_barrier.cu
#include <cstdio>
__global__ void k(int mode, int steps, double* out, long long* t) {
    __shared__ double buf[2][256];
    __shared__ float fbuf[2][256];
    const int tid = threadIdx.x;
    buf[0][tid] = 1.0 + tid * 1e-3;
    buf[1][tid] = 0.0;
    fbuf[0][tid] = 1.0f;
    fbuf[1][tid] = 0.0f;
    double acc = tid;
    float facc = tid;
    __syncthreads();
    const long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
        const int src = mode == 5 ? tid : (tid * 7 + s) & 255;
        if (mode == 1 || mode == 5) {
            acc = fma(acc, buf[s & 1][src], 1e-9);
            buf[(s + 1) & 1][tid] = acc;
        } else if (mode == 2) {
            buf[(s + 1) & 1][tid] = buf[s & 1][src];
        } else if (mode == 3) {
            facc = fmaf(facc, fbuf[s & 1][src], 1e-9f);
            fbuf[(s + 1) & 1][tid] = facc;
        } else if (mode == 4) {
            buf[(s + 1) & 1][tid] = buf[s & 1][src] + 1.0;
        }
        __syncthreads();
    }
    const long long t1 = clock64();
    out[tid] = acc + facc;
    if (tid == 0) t[0] = t1 - t0;
}
int main() {
    double* out;
    long long* t;
    cudaMalloc(&out, 256 * 8);
    cudaMalloc(&t, 8);
    for (int mode = 0; mode < 6; ++mode) {
        long long h = 0;
        for (int r = 0; r < 3; ++r) {
            k<<<1, 256>>>(mode, 600, out, t);
            cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        }
        printf("mode %d: %.1f cycles / step\n", mode, h / 600.0);
    }
    return 0;
}
