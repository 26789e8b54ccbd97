#include "/tmp/ba_prof.cu"
#include <cstdio>
#include <vector>
namespace pvo_dev {
namespace {
__global__ void micro(const double* sys, int np, double* x, long long* t) {
    extern __shared__ __align__(16) unsigned char smem[];
    const Layout L = make_layout(np, 0);
    long long t0 = clock64();
    ldlt_solve_cta(sys, np, smem, L, x);
    if (threadIdx.x == 0) { t[0] = t0; for (int i = 0; i < 4; ++i) t[1 + i] = g_prof[i]; }
}
}
}
int main() {
    for (int np : {6, 42, 60, 96}) {
        const int nent = np * (np + 1) / 2;
        std::vector<double> h(nent + np);
        int e = 0;
        for (int i = 0; i < np; ++i) for (int j = i; j < np; ++j) h[e++] = (i == j) ? np + 1.0 + i : 0.5 / (1 + i + j);
        for (int i = 0; i < np; ++i) h[nent + i] = 1.0 + i;
        double *dsys, *dx; long long* dt;
        cudaMalloc(&dsys, sizeof(double) * h.size()); cudaMalloc(&dx, sizeof(double) * np); cudaMalloc(&dt, 8 * sizeof(long long));
        cudaMemcpy(dsys, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
        const pvo_dev::Layout L = pvo_dev::make_layout(np, 0);
        cudaFuncSetAttribute(pvo_dev::micro, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total);
        for (int rep = 0; rep < 3; ++rep) {
            pvo_dev::micro<<<1, 256, L.total>>>(dsys, np, dx, dt);
            long long t[5];
            cudaMemcpy(t, dt, sizeof(t), cudaMemcpyDeviceToHost);
            printf("np=%d rank %lld load %lld factor %lld subst %lld\n", np, t[1]-t[0], t[2]-t[1], t[3]-t[2], t[4]-t[3]);
        }
    }
}
