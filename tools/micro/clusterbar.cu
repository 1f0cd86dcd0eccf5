// clusterbar.cu -- cost of cluster-wide synchronisation variants on sm_100a
// (one DSMEM store per thread before each barrier; cycles per round, CTA 0).
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
template <int MODE>
__global__ void k(long long* cyc, double* out, int n) {
    __shared__ double buf[2][256];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank(), C = cl.num_blocks();
    double* peer = cl.map_shared_rank(&buf[0][0], (r + 1) % C);
    cl.sync();
    double acc = 0.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        peer[(i & 1) * 256 + threadIdx.x] = acc + i;  // DSMEM store into the neighbour
        if (MODE == 0) {
            cl.sync();
        } else if (MODE == 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else if (MODE == 2) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
        } else if (MODE == 3) {
            asm volatile("fence.acq_rel.cluster;\nbarrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
        } else if (MODE == 4) {
            __syncthreads();  // reference: CTA barrier only (no cluster ordering)
        }
        acc += buf[i & 1][threadIdx.x];
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(const char* name, int C, int threads, long long* cyc, double* out) {
    const int n = 2000;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(C);
    cfg.blockDim = dim3(threads);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k<MODE>, cyc, out, n);
    long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-52s C=%d T=%d %8.1f cyc per round (%s)\n", name, C, threads, (double)h / n, cudaGetErrorString(cudaGetLastError()));
}
int main() {
    long long* cyc; double* out;
    cudaMalloc(&cyc, 8); cudaMalloc(&out, 1 << 20);
    for (int C : {2, 8}) for (int T : {256, 512}) {
        if (T > 256) continue;
        run<0>("cg cluster.sync()", C, T, cyc, out);
        run<1>("arrive.release + wait.acquire", C, T, cyc, out);
        run<2>("arrive.relaxed + wait (no ordering)", C, T, cyc, out);
        run<3>("fence.acq_rel.cluster + arrive.relaxed + wait", C, T, cyc, out);
        run<4>("__syncthreads only (reference)", C, T, cyc, out);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
