// Probe which TMA descriptor shapes the corr kernel uses are accepted on this
// GPU: one tensor copy per launch, variant chosen by argv[1].
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/micro_tma tools/micro_tma.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int rank, int c0, int c1, int c2, int c3, int bytes,
                      float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(bytes)
                     : "memory");
        if (rank == 4) {
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3, %4, %5}], [%6];" ::"r"(su32(sm)),
                "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(su32(&bar))
                : "memory");
        } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
                "%3}], [%4];" ::"r"(su32(sm)),
                "l"((uint64_t)&map), "r"(c0), "r"(c1), "r"(su32(&bar))
                : "memory");
        }
        asm volatile(
            "{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(
                su32(&bar))
            : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main(int argc, char** argv) {
    const int v = argc > 1 ? atoi(argv[1]) : 0;
    void* fnp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
    const int W = argc > 2 ? atoi(argv[2]) : 40, H = argc > 3 ? atoi(argv[3]) : 30, NF = 4;
    const int cx = argc > 4 ? atoi(argv[4]) : 0, cy = argc > 5 ? atoi(argv[5]) : 0;
    float* g;
    cudaMalloc(&g, sizeof(float) * W * H * 128 * NF);
    std::vector<float> h(W * H * 128 * NF);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    cudaMemcpy(g, h.data(), sizeof(float) * h.size(), cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 1 << 20);
    CUtensorMap map;
    int rank = 4, bytes = 0;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], es[4] = {1, 1, 1, 1};
    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE;
    if (v == 0 || v == 1 || v == 4) {  // planar gram {W, H, 8, NF}, box {12|16, 9, 5, 1}
        dims[0] = W; dims[1] = H; dims[2] = 8; dims[3] = NF;
        box[0] = v == 1 ? 16 : 12; box[1] = 9; box[2] = 5; box[3] = 1;
        bytes = box[0] * 9 * 5 * 4;
    } else if (v == 2) {  // feat {128, W, H, NF}, box {16, 9, 9, 1}, 64B swizzle
        dims[0] = 128; dims[1] = W; dims[2] = H; dims[3] = NF;
        box[0] = 16; box[1] = 9; box[2] = 9; box[3] = 1;
        sw = CU_TENSOR_MAP_SWIZZLE_64B;
        bytes = 16 * 81 * 4;
    } else if (v == 3) {  // patch 2-D {128, rows}, box {16, 9}
        rank = 2;
        dims[0] = 128; dims[1] = 64;
        box[0] = 16; box[1] = 9;
        bytes = 16 * 9 * 4;
    }
    cuuint64_t s = 4;
    for (int i = 0; i < rank; ++i) {
        if (i) strides[i - 1] = s;
        s *= dims[i];
    }
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, g, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                     v == 4 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d encode %d\n", v, (int)r);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    if (rank == 4 && v != 2) probe<<<1, 128, 65536>>>(map, rank, cx, cy, 0, 1, bytes, out);
    else if (rank == 4) probe<<<1, 128, 65536>>>(map, rank, 0, cx, cy, 1, bytes, out);
    else probe<<<1, 128, 65536>>>(map, rank, 0, 0, 0, 1, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %s\n", v, cudaGetErrorString(e));
    return 0;
}
