// Standalone check of the strided 3-D tensor-map box used by the tensor-map
// sweep engine: loads one box per variant and prints what landed in smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tmap_test tmap_test.cu
// Measured on B200: boxes at plane stride 2 and negative / out-of-range
// origins work (zero fill); a box whose first column is not 16-B aligned
// (odd column for doubles) faults with "illegal instruction", so the sweep
// aligns its box origin down to an even column.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

struct Pad {
    char b[168];
};

template <int MODE>
__device__ __forceinline__ void body(const void* tmp, int x, int y, int z, int bytes, double* out,
                                     double* buf, uint64_t* barp) {
    uint64_t& bar = *barp;
    const void* tmv = tmp;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4 * 36; ++i) buf[i] = -1.0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(su32(buf)),
            "l"(tmv), "r"(x), "r"(y), "r"(z), "r"(su32(&bar))
            : "memory");
        asm volatile(
            "{\n\t.reg .pred P1;\nW:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
            "@!P1 bra W;\n}" ::"r"(su32(&bar))
            : "memory");
        for (int i = 0; i < 4 * 36; ++i) out[i] = buf[i];
    }
}

__global__ void k(const __grid_constant__ CUtensorMap tm, int x, int y, int z, int bytes,
                  double* out) {
    __shared__ __align__(128) double buf[4 * 36];
    __shared__ __align__(8) uint64_t bar;
    body<0>(&tm, x, y, z, bytes, out, buf, &bar);
}

// same parameter layout as cp_sweep2_tmap_kernel: 168-byte struct, int, map
__global__ void k2(const Pad pad, const int par, const __grid_constant__ CUtensorMap tm, int x,
                   int y, int z, int bytes, double* out) {
    __shared__ __align__(128) double buf[4 * 36];
    __shared__ __align__(8) uint64_t bar;
    body<1>(&tm, x, y, z, bytes, out, buf, &bar);
}

// dynamic shared memory after some static shared memory
__global__ void k3(const __grid_constant__ CUtensorMap tm, int x, int y, int z, int bytes,
                   double* out) {
    extern __shared__ __align__(128) unsigned char dyn[];
    __shared__ double red[8][6];
    __shared__ bool flag;
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { red[0][0] = 1.0; flag = true; }
    body<2>(&tm, x, y, z, bytes, out, reinterpret_cast<double*>(dyn) + 4 * 36 * 3, &bar);
    if (threadIdx.x == 0 && flag) out[0] += 0.0 * red[0][0];
}

int main() {
    const int pitch = 64, rows = 33, planes = 16;
    const long plane = 32 + 34L * pitch + 64;
    std::vector<double> h(planes * plane);
    for (int p = 0; p < planes; ++p)
        for (int j = 0; j < rows; ++j)
            for (int i = 0; i < pitch; ++i) h[p * plane + 32 + j * pitch + i] = p * 10000 + j * 100 + i;
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* o;
    cudaMalloc(&o, 4 * 36 * 8);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
    struct V {
        const char* name;
        unsigned bz, sz;
        int x;
        int bytes;
    } vs[] = {{"box{36,1,4} stride1 x=0", 4, 1, 0, 1152},
              {"box{36,1,4} stride1 x=-2", 4, 1, -2, 1152},
              {"box{36,1,8} stride2 x=0", 8, 2, 0, 1152},
              {"box{36,1,8} stride2 x=-2", 8, 2, -2, 1152}};
    for (auto& v : vs) {
        alignas(64) CUtensorMap tm;
        cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, (cuuint64_t)planes};
        cuuint64_t str[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)plane * 8};
        cuuint32_t box[3] = {36, 1, v.bz};
        cuuint32_t es[3] = {1, 1, v.sz};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d + 32, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int mode = 0; mode < 3; ++mode) {
        if (mode == 0) k<<<1, 32>>>(tm, v.x, 33, 1, v.bytes, o);
        if (mode == 1) k2<<<1, 32>>>(Pad{}, 0, tm, 60, 5, 1, v.bytes, o);
        if (mode == 2) k3<<<1, 32, 37120>>>(tm, v.x, 5, 1, v.bytes, o);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> ho(4 * 36);
        cudaMemcpy(ho.data(), o, ho.size() * 8, cudaMemcpyDeviceToHost);
        printf("mode %d %s: encode=%d kernel=%s  [0]=%g [1]=%g [2]=%g [36]=%g [72]=%g [108]=%g [143]=%g\n",
               mode, v.name, (int)r, cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[36], ho[72], ho[108],
               ho[143]);
        if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
