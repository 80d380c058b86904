// Standalone TMA probe: 3-D / 2-D boxes over a complex CANON array viewed as fp32.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include "../../paper_2202_14005_b200/csrc/sm100.cuh"
using namespace mdnn::sm100;

__global__ void k(const __grid_constant__ CUtensorMap tm, float* out, int rank, int c0, int c1, int c2, int bytes)
{
    __shared__ __align__(1024) float buf[8192];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar, bytes);
        if (rank == 3)
            tma_load_3d(buf, &tm, &bar, c0, c1, c2);
        else
            tma_load_2d(buf, &tm, &bar, c0, c1);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x)
        out[i] = buf[i];
}

int main(int argc, char** argv)
{
    int X = 36, Y = 20, P = 2;
    int bx = argc > 1 ? atoi(argv[1]) : 192, c0 = argc > 2 ? atoi(argv[2]) : -10, rank = argc > 3 ? atoi(argv[3]) : 3;
    float* d;
    cudaMalloc(&d, sizeof(float) * 2 * X * Y * P);
    float* o;
    cudaMalloc(&o, 1 << 20);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(2 * X), cuuint64_t(Y), cuuint64_t(P)};
    cuuint64_t strides[2] = {cuuint64_t(2 * X) * 4, cuuint64_t(2 * X) * Y * 4};
    cuuint32_t box[3] = {cuuint32_t(bx), 1, cuuint32_t(rank == 3 ? P : 1)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rank %d box %d c0 %d -> %d\n", rank, bx, c0, int(r));
    int bytes = bx * 4 * (rank == 3 ? P : 1);
    k<<<1, 128>>>(m, o, rank, c0, 3, 0, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    return 0;
}
