// Micro-benchmark of the BA pose solve (tools only): times the phases of
// ldlt_solve_cta with clock64 on one CTA.
#include "../paper_2208_04726_b200/csrc/ba.cu"

#include <cstdio>
#include <vector>

namespace pvo_dev {
namespace {
__global__ void micro(const double* sys, int np, double* x, long long* t) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Layout L = make_layout(np, 0);
    long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep) ldlt_solve_cta(sys, np, smem, L, x);
    long long t1 = clock64();
    if (threadIdx.x == 0) t[0] = (t1 - t0) / 10;
}
}  // namespace
}  // namespace pvo_dev

int main() {
    for (int np : {6, 30, 60, 96}) {
        const int nent = np * (np + 1) / 2;
        std::vector<double> h(nent + np);
        // SPD: diagonally dominant
        int e = 0;
        for (int i = 0; i < np; ++i)
            for (int j = i; j < np; ++j) h[e++] = (i == j) ? np + 1.0 + i : 0.5 / (1 + i + j);
        for (int i = 0; i < np; ++i) h[nent + i] = 1.0 + i;
        double *dsys, *dx;
        long long* dt;
        cudaMalloc(&dsys, sizeof(double) * h.size());
        cudaMalloc(&dx, sizeof(double) * np);
        cudaMalloc(&dt, sizeof(long long));
        cudaMemcpy(dsys, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
        const pvo_dev::Layout L = pvo_dev::make_layout(np, 0);
        cudaFuncSetAttribute(pvo_dev::micro, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
        pvo_dev::micro<<<1, 256, L.total>>>(dsys, np, dx, dt);
        long long t = 0;
        cudaMemcpy(&t, dt, sizeof(t), cudaMemcpyDeviceToHost);
        printf("np=%d  cycles/solve=%lld  err=%s\n", np, t, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
