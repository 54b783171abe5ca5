// microbench.cu — B200 (sm_100a) analogue of the paper's Table 2 (PAPER.md:
// 291-315: latency of shfl.up / shared-memory read / L1 hit, cycles) plus the
// issue-rate facts the kernel design depends on (FFMA register-bank form vs
// constant operand vs FFMA2).  Standalone: nvcc -gencode
// arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
//
// Latency: one warp, a dependent chain of N operations timed with clock64();
// cycles/op = elapsed / N.  Throughput: all SMs, many warps, independent
// chains; ops/clk/SM = total ops / (elapsed SM clocks * nSM).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int N = 4096;

// ---------------------------------------------------------------- latency
__global__ void lat_shfl_up(int* out, long long* cyc, int seed) {
    int v = threadIdx.x + seed;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __shfl_up_sync(0xffffffffu, v, 1) + 1;
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void lat_lds(int* out, long long* cyc, int seed) {
    __shared__ int s[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) s[i] = (i + 1) & 1023;
    __syncwarp();
    int v = (threadIdx.x + seed) & 1023;
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = s[v];
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// pointer chase in a 4 KiB array (L1-resident after the first pass)
__global__ void lat_ldg_l1(const int* __restrict__ a, int* out, long long* cyc, int seed) {
    int v = (threadIdx.x + seed) & 1023;
    for (int i = 0; i < 2048; ++i) v = __ldg(a + v);      // warm L1
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < N; ++i) v = __ldg(a + v);
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}

// pointer chase through L2: stride 8 KiB in a 64 MiB array, loads bypass L1
__global__ void lat_ldg_l2(const int* __restrict__ a, int* out, long long* cyc, int seed) {
    int v = seed;
    for (int i = 0; i < 256; ++i) v = __ldcg(a + v);
    long long t0 = clock64();
    for (int i = 0; i < 1024; ++i) v = __ldcg(a + v);
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) *cyc = (t1 - t0) * (N / 1024);
}

// ------------------------------------------------------------- throughput
template <int MODE>
__global__ void tput_fma(float* out, long long* cyc, float b, int iters) {
    float acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = threadIdx.x * 0.001f + k;
    float a = out[0] + 1.0f;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (MODE == 0) acc[k] = fmaf(acc[k], a, acc[(k + 1) & 7]);     // 3 registers
            if (MODE == 1) acc[k] = fmaf(acc[k], b, acc[k]);              // constant-bank operand
            if (MODE == 2) acc[k] = fmaf(acc[k], 1.0001f, acc[k]);        // immediate
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void tput_ffma2(float* out, long long* cyc, float b, int iters) {
    float2 acc[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = make_float2(threadIdx.x * 0.001f + k, k);
    const float2 a = make_float2(out[0] + 1.0f, out[1] + 1.0f);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[k] = __ffma2_rn(acc[k], a, acc[(k + 1) & 7]);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += acc[k].x + acc[k].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void tput_shfl(int* out, long long* cyc, int iters) {
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __shfl_up_sync(0xffffffffu, v[k], 1);
    }
    long long t1 = clock64();
    int s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void tput_lds128(int* out, long long* cyc, int iters) {
    __shared__ int4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    int4 acc = make_int4(0, 0, 0, 0);
    int idx = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int4 t = s[(idx + 32 * k + i) & 2047];
            acc.x ^= t.x; acc.y ^= t.y; acc.z ^= t.z; acc.w ^= t.w;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// SHFL and LDS.128 interleaved (independent chains): do they share one
// issue path (MIO)?  ops = 8 SHFL + 8 LDS.128 per thread-iteration; compare
// the time per iteration with tput_shfl + tput_lds128 (shared) vs their max.
__global__ void tput_mix(int* out, long long* cyc, int iters) {
    __shared__ int4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_int4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    int4 acc = make_int4(0, 0, 0, 0);
    int v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x + k;
    int idx = threadIdx.x & 31;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = __shfl_up_sync(0xffffffffu, v[k], 1);
            int4 t = s[(idx + 32 * k + i) & 2047];
            acc.x ^= t.x; acc.y ^= t.y; acc.z ^= t.z; acc.w ^= t.w;
        }
    }
    long long t1 = clock64();
    int r = acc.x + acc.y + acc.z + acc.w;
#pragma unroll
    for (int k = 0; k < 8; ++k) r += v[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

static int nsm() {
    int n;
    CK(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0));
    return n;
}

template <class F>
static double per_sm_rate(F launch, int blocks, int threads, int iters, double ops_per_thread_iter) {
    long long* dcyc;
    CK(cudaMalloc(&dcyc, blocks * sizeof(long long)));
    launch(dcyc);                       // warm-up
    CK(cudaDeviceSynchronize());
    launch(dcyc);
    CK(cudaDeviceSynchronize());
    long long* h = (long long*)malloc(blocks * sizeof(long long));
    CK(cudaMemcpy(h, dcyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost));
    long long mx = 0;
    for (int b = 0; b < blocks; ++b) mx = h[b] > mx ? h[b] : mx;
    free(h);
    CK(cudaFree(dcyc));
    const int n = nsm();
    // all blocks resident at once: ops per SM per clock
    return (double)blocks * threads * iters * ops_per_thread_iter / n / (double)mx;
}

int main() {
    int *dout, *a;
    long long* dc;
    CK(cudaMalloc(&dout, 1 << 24));
    CK(cudaMalloc(&dc, 64));
    CK(cudaMalloc(&a, 64 << 20));
    // L1 chase table: a[i] = (i + 33) % 1024 ; L2 chase: stride 2048 ints (8 KiB)
    int* h = (int*)malloc(64 << 20);
    const int n2 = (64 << 20) / 4;
    for (int i = 0; i < n2; ++i) h[i] = i < 1024 ? (i + 33) % 1024 : (i + 2048 * 7) % n2;
    CK(cudaMemcpy(a, h, 64 << 20, cudaMemcpyHostToDevice));
    free(h);
    long long cyc;
    printf("{\"table2_b200_cycles\": {");
    lat_shfl_up<<<1, 32>>>(dout, dc, 0);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("\"shfl_up_plus_iadd\": %.1f, ", (double)cyc / N);
    lat_lds<<<1, 32>>>(dout, dc, 0);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("\"lds_chase\": %.1f, ", (double)cyc / N);
    lat_ldg_l1<<<1, 32>>>(a, dout, dc, 0);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("\"ldg_l1_hit_chase\": %.1f, ", (double)cyc / N);
    lat_ldg_l2<<<1, 32>>>(a + 1024, dout, dc, 0);
    CK(cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost));
    printf("\"ldg_l2_hit_chase\": %.1f}, ", (double)cyc / N);
    const int nb = nsm() * 8, nt = 256, it = 2048;
    printf("\"per_sm_per_clk\": {");
    printf("\"ffma_3reg\": %.1f, ", per_sm_rate([&](long long* c) { tput_fma<0><<<nb, nt>>>((float*)dout, c, 1.0001f, it); }, nb, nt, it, 8));
    printf("\"ffma_const\": %.1f, ", per_sm_rate([&](long long* c) { tput_fma<1><<<nb, nt>>>((float*)dout, c, 1.0001f, it); }, nb, nt, it, 8));
    printf("\"ffma_imm\": %.1f, ", per_sm_rate([&](long long* c) { tput_fma<2><<<nb, nt>>>((float*)dout, c, 1.0001f, it); }, nb, nt, it, 8));
    printf("\"ffma2_fma_lanes\": %.1f, ", per_sm_rate([&](long long* c) { tput_ffma2<<<nb, nt>>>((float*)dout, c, 1.0001f, it); }, nb, nt, it, 16));
    printf("\"shfl_lanes\": %.1f, ", per_sm_rate([&](long long* c) { tput_shfl<<<nb, nt>>>(dout, c, it); }, nb, nt, it, 8));
    printf("\"lds128_lanes\": %.1f, ", per_sm_rate([&](long long* c) { tput_lds128<<<nb, nt>>>(dout, c, it); }, nb, nt, it, 8));
    // iterations of (1 SHFL + 1 LDS.128) per SM per clock, in lanes
    printf("\"shfl_plus_lds128_pair_lanes\": %.1f}}\n", per_sm_rate([&](long long* c) { tput_mix<<<nb, nt>>>(dout, c, it); }, nb, nt, it, 8));
    return 0;
}
