// fp64lat.cu -- dependent-issue latency and per-SM throughput of DFMA / DADD,
// 64-bit shuffles and shared loads on sm_100a (calibrates the latency model of
// the persistent PDHG kernels).  nvcc -arch=sm_100a -o fp64lat fp64lat.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k_dfma(double* out, long long* cyc, int n, double a, double b) {
    double x[CH];
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x + c;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) s += x[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl(double* out, long long* cyc, int n) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_lds(double* out, long long* cyc, int n) {
    __shared__ int nxt[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) nxt[i] = (i * 17 + 1) & 1023;
    __syncthreads();
    int p = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = nxt[p];
    long long t1 = clock64();
    out[threadIdx.x] = p;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_bar(double* out, long long* cyc, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = 0;
}
__global__ void k_div(double* out, long long* cyc, int n, double a) {
    double x = threadIdx.x + 2.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = a / x + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
    const int n = 4096;
#define RUN(name, call, per) call; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-40s %8.2f cyc per %s\n", name, (double)h / n, per);
    RUN("dfma 1 chain, 1 warp", (k_dfma<1><<<1, 32>>>(out, cyc, n, 1.0000001, 1e-9)), "dep step");
    RUN("dfma 2 chains, 1 warp", (k_dfma<2><<<1, 32>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 2");
    RUN("dfma 4 chains, 1 warp", (k_dfma<4><<<1, 32>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 4");
    RUN("dfma 8 chains, 1 warp", (k_dfma<8><<<1, 32>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 8");
    RUN("dfma 8 chains, 4 warps", (k_dfma<8><<<1, 128>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 8");
    RUN("dfma 8 chains, 16 warps", (k_dfma<8><<<1, 512>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 8");
    RUN("dfma 8 chains, 16 warps x 148 CTAs", (k_dfma<8><<<148, 512>>>(out, cyc, n, 1.0000001, 1e-9)), "step of 8");
    RUN("shfl.64 + dadd dependent", (k_shfl<<<1, 32>>>(out, cyc, n)), "step");
    RUN("lds dependent (pointer chase)", (k_lds<<<1, 32>>>(out, cyc, n)), "load");
    RUN("__syncthreads, 512 threads", (k_bar<<<1, 512>>>(out, cyc, n)), "barrier");
    RUN("ddiv + dadd dependent", (k_div<<<1, 32>>>(out, cyc, n, 3.0)), "step");
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
