// Inter-SM signalling latency on B200: two CTAs ping-pong a step counter
// through L2 (relaxed polls; variants of the producer-side fence).
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void pingpong(unsigned* flags, double* data, long long* out, int iters) {
    const int b = blockIdx.x;
    if (threadIdx.x != 0 || b > 1) return;
    unsigned* mine = flags + b * 32;
    unsigned* other = flags + (1 - b) * 32;
    const long long t0 = clock64();
    double acc = 0;
    for (int i = 0; i < iters; ++i) {
        if (b == (i & 1)) {
            // producer: payload then flag
            data[b * 16] = (double)i;
            if (MODE == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i + 1) : "memory");
            if (MODE == 1) { __threadfence(); asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i + 1) : "memory"); }
            if (MODE == 2) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i + 1) : "memory");
        } else {
            unsigned v;
            do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(other) : "memory"); } while (v < (unsigned)(i + 1));
            if (MODE == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            acc += __ldcg(data + (1 - b) * 16);
            // mirror the counter so both sides advance
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"(i + 1) : "memory");
        }
        // wait until the other side has also reached i+1
        unsigned v;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(other) : "memory"); } while (v < (unsigned)(i + 1));
    }
    out[b] = clock64() - t0;
    out[2 + b] = (long long)acc;
}

__global__ void l2lat(const double* p, long long* out, int n) {
    // dependent chain of L2 loads (cg), stride 4 KB
    const long long t0 = clock64();
    long idx = 0;
    double s = 0;
    for (int i = 0; i < n; ++i) {
        double v = __ldcg(p + idx);
        s += v;
        idx = ((long)v + i * 512) & ((1 << 22) - 1);
    }
    out[0] = (clock64() - t0) / n;
    out[1] = (long long)s;
}

int main() {
    unsigned* f; double* d; long long* o;
    cudaMalloc(&f, 4096); cudaMalloc(&d, 64 << 20); cudaMalloc(&o, 64);
    cudaMemset(d, 0, 64 << 20);
    long long h[4];
    const int it = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int grid : {2, 148}) {
            cudaMemset(f, 0, 4096);
            if (mode == 0) pingpong<0><<<grid, 32>>>(f, d, o, it);
            if (mode == 1) pingpong<1><<<grid, 32>>>(f, d, o, it);
            if (mode == 2) pingpong<2><<<grid, 32>>>(f, d, o, it);
            cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
            printf("mode %d grid %d: %lld cycles per half round trip\n", mode, grid, h[0] / it);
        }
    }
    l2lat<<<1, 1>>>(d, o, 10000);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    printf("dependent L2 load latency: %lld cycles\n", h[0]);
    printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
