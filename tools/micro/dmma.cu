// dmma.cu -- latency / throughput of mma.sync.m8n8k4.f64 on sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
    double d[CH][2];
    for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* out; long long* cyc; long long h;
    cudaMalloc(&out, 1 << 22); cudaMalloc(&cyc, 8);
    const int n = 4096;
#define RUN(name, call) call; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("%-44s %8.2f cyc per step\n", name, (double)h / n);
    RUN("dmma 1 chain 1 warp", (k<1><<<1, 32>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 2 chains 1 warp", (k<2><<<1, 32>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 4 chains 1 warp", (k<4><<<1, 32>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 4 chains 4 warps", (k<4><<<1, 128>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 1 chain 16 warps", (k<1><<<1, 512>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 2 chains 16 warps", (k<2><<<1, 512>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 4 chains 16 warps", (k<4><<<1, 512>>>(out, cyc, n, 1e-3, 1e-3)));
    RUN("dmma 4 chains 16 warps x 148", (k<4><<<148, 512>>>(out, cyc, n, 1e-3, 1e-3)));
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
