// Minimal TMA tensor store check (param-space tensor map, 3-D box).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
struct Pack { CUtensorMap m[2]; };
__global__ void k(const __grid_constant__ Pack p, int mode, int x, int y) {
    extern __shared__ __align__(128) float buf[];
    for (int i = threadIdx.x; i < 128 * 30; i += blockDim.x) buf[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned s = (unsigned)__cvta_generic_to_shared(buf);
        const void* tm = &p.m[mode];
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];"
                     :: "l"(tm), "r"(s), "r"(x), "r"(y), "r"(0) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
int main(int argc, char** argv) {
    int mode = atoi(argv[1]), X = atoi(argv[2]), Y = atoi(argv[3]);
    void* fnp; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
    auto fn = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
    float* d; cudaMalloc(&d, 256 * 64 * 4 * 4);
    Pack p;
    cuuint64_t gdim[3] = {256, 64, 4}, gstr[2] = {256 * 4, 256 * 64 * 4};
    cuuint32_t box[3] = {128, 30, 1}, es[3] = {1, 1, 1};
    CUresult r0 = fn(&p.m[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    // unaligned-window map: base + 4 floats (16 B), extent 251
    cuuint64_t gdim2[3] = {3, 3, 4};
    CUresult r1 = fn(&p.m[1], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d + 256 + 4, gdim2, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", (int)r0, (int)r1);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    k<<<1, 128, 100000>>>(p, mode, X, Y);
    printf("mode %d x %d y %d: %s\n", mode, X, Y, cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
