// rwmix.cu — achievable HBM bandwidth on this B200 for read:write stream mixes
// (1R1W copy, 3R1W, 1R3W, 2R1W) with a plain float4 grid-stride kernel; the
// ceiling each stencil's traffic mix can expect.  nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o rwmix tools/rwmix.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int NR, int NW>
__global__ void mix(const float4* __restrict__ a, const float4* __restrict__ b, const float4* __restrict__ c,
                    float4* __restrict__ x, float4* __restrict__ y, float4* __restrict__ z, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        float4 v = a[i];
        if (NR > 1) { float4 t = b[i]; v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w; }
        if (NR > 2) { float4 t = c[i]; v.x += t.x; v.y += t.y; v.z += t.z; v.w += t.w; }
        x[i] = v;
        if (NW > 1) y[i] = v;
        if (NW > 2) z[i] = v;
    }
}
static int g_blocks_per_sm = 8;
template <int NR, int NW>
void run(float4** p, size_t n, const char* name) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int i = 0; i < 3; ++i) mix<NR, NW><<<nsm * g_blocks_per_sm, 512>>>(p[0], p[1], p[2], p[3], p[4], p[5], n);
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) mix<NR, NW><<<nsm * g_blocks_per_sm, 512>>>(p[0], p[1], p[2], p[3], p[4], p[5], n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("\"%s\": %.1f, ", name, (double)(NR + NW) * n * 16 * it / (ms / 1e3) / 1e9);
}
int main(int argc, char** argv) {
    if (argc > 1) g_blocks_per_sm = atoi(argv[1]);   // 1 = 16 warps per SM (the k3d occupancy)
    const size_t n = (512ull << 20) / 16;      // 512 MiB per array
    float4* p[6];
    for (int i = 0; i < 6; ++i) { cudaMalloc(&p[i], n * 16); cudaMemset(p[i], 0, n * 16); }
    printf("{\"blocks_per_sm\": %d, \"GBps_512MiB_arrays\": {", g_blocks_per_sm);
    run<1, 1>(p, n, "1R1W");
    run<2, 1>(p, n, "2R1W");
    run<3, 1>(p, n, "3R1W");
    run<1, 3>(p, n, "1R3W");
    run<1, 2>(p, n, "1R2W");
    printf("\"end\": 0}}\n");
    return 0;
}
