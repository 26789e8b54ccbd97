// Micro-benchmark of the in-CTA pose solve (ldlt_solve_cta) on one CTA, clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DPVO_LDLT_BLOCK=8 \
//      -o tools/micro_solve tools/micro_solve.cu
__device__ long long g_ph[8];
#define SOLVE_PROBE_BEGIN long long _pt = clock64(); if (threadIdx.x == 0) for (int _i = 0; _i < 8; ++_i) g_ph[_i] = 0;
#define SOLVE_PROBE(i) if (threadIdx.x == 0) { const long long _t = clock64(); g_ph[i] += _t - _pt; _pt = _t; }
__device__ long long g_loop[128];
#define SOLVE_LOOP_PROBE(i) if (threadIdx.x == 0 && (i) < 128) g_loop[i] = clock64();
#include "../paper_2208_04726_b200/csrc/ba.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
namespace pvo_dev {
namespace {
__global__ void micro(const double* sys, int np, double* x, long long* t) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Layout L = make_layout(np, 0);
    __syncthreads();
    const long long t0 = clock64();
    const bool ok = ldlt_solve_cta(sys, np, smem, L, x);
    const long long t1 = clock64();
    if (threadIdx.x == 0) {
        t[0] = t1 - t0;
        t[1] = ok;
        printf("  load %lld factor %lld store %lld backsub %lld | loop deltas", g_ph[0], g_ph[1], g_ph[2], g_ph[3]);
        for (int i = np - 1; i > np - 12 && i > 0; --i) printf(" %lld", g_loop[i - 1] - g_loop[i]);
        printf("\n");
    }
}
// the same solve repeated (enough warp-state samples for an ncu source view)
__global__ void micro_loop(const double* sys, int np, double* x, int reps) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Layout L = make_layout(np, 0);
    for (int r = 0; r < reps; ++r) ldlt_solve_cta(sys, np, smem, L, x);
}
}  // namespace
}  // namespace pvo_dev
int main(int argc, char** argv) {
    const int loop_np = argc > 1 ? atoi(argv[1]) : 0;  // profiling mode: micro_solve <np> <reps>
    for (int np : {42, 60, 96}) {
        if (loop_np && np != loop_np) continue;
        const int nent = np * (np + 1) / 2;
        std::vector<double> h(nent + np), A((size_t)np * np), b(np);
        int e = 0;
        for (int i = 0; i < np; ++i)
            for (int j = i; j < np; ++j) {
                const double v = (i == j) ? np + 1.0 + i : 0.5 / (1 + i + j);
                h[e++] = v;
                A[i * np + j] = A[j * np + i] = v;
            }
        for (int i = 0; i < np; ++i) h[nent + i] = b[i] = 1.0 + i;
        double *dsys, *dx;
        long long* dt;
        cudaMalloc(&dsys, sizeof(double) * h.size());
        cudaMalloc(&dx, sizeof(double) * np);
        cudaMalloc(&dt, 2 * sizeof(long long));
        cudaMemcpy(dsys, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
        const pvo_dev::Layout L = pvo_dev::make_layout(np, 0);
        cudaFuncSetAttribute(pvo_dev::micro, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
        long long t[2];
        if (loop_np) {
            cudaFuncSetAttribute(pvo_dev::micro_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
            pvo_dev::micro_loop<<<1, 256, L.total>>>(dsys, np, dx, argc > 2 ? atoi(argv[2]) : 200);
            cudaDeviceSynchronize();
        }
        {  // steady-state time per solve: 200 back-to-back solves in one launch (CUDA events)
            cudaFuncSetAttribute(pvo_dev::micro_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            pvo_dev::micro_loop<<<1, 256, L.total>>>(dsys, np, dx, 20);
            cudaEventRecord(e0);
            pvo_dev::micro_loop<<<1, 256, L.total>>>(dsys, np, dx, 200);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("np=%d loop: %.2f us per solve\n", np, ms * 1e3 / 200);
        }
        for (int rep = 0; rep < 3; ++rep) {
            pvo_dev::micro<<<1, 256, L.total>>>(dsys, np, dx, dt);
            cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
        }
        std::vector<double> x(np);
        cudaMemcpy(x.data(), dx, sizeof(double) * np, cudaMemcpyDeviceToHost);
        double res = 0;  // residual |A x - b|
        for (int i = 0; i < np; ++i) {
            double s = -b[i];
            for (int j = 0; j < np; ++j) s += A[i * np + j] * x[j];
            res = fmax(res, fabs(s));
        }
        printf("np=%d cycles=%lld ok=%lld residual=%.2e (%s)\n", np, t[0], t[1], res,
               cudaGetErrorString(cudaGetLastError()));
    }
}
