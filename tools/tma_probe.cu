// Standalone TMA probe: 4-D box loads (x, y, z, field) of a padded fp64 array with given box
// dims and start coordinates; prints OK / mismatch / the CUDA error per case.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void k(const __grid_constant__ CUtensorMap m, double* out, int n, int c0, int c1, int c2) {
    extern __shared__ __align__(128) unsigned char raw[];
    double* s = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
    uint64_t* bar = reinterpret_cast<uint64_t*>(s + n);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(n * 8) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5}], [%6];" ::"r"(su32(s)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(c2), "r"(0), "r"(su32(bar))
            : "memory");
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra W_%=;\n}" ::"r"(
                         su32(bar))
                     : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    int ci = -1;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncFn enc = reinterpret_cast<EncFn>(p);
    const int px = 40, py = 18, pz = 18, nf = 4;
    const size_t fsz = (size_t)px * py * pz;
    std::vector<double> h(fsz * nf);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
    double* d;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* out;
    cudaMalloc(&out, 1 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Case { int bx, by, bz, c0, c1, c2; } cases[] = {
        {20, 11, 11, 2, 0, 0}, {18, 10, 10, 3, 0, 0}, {18, 10, 10, 4, 0, 0}, {18, 10, 10, 2, 0, 0},
        {16, 8, 8, 4, 1, 1}, {20, 10, 10, 3, 0, 0}, {18, 11, 11, 3, 0, 0}, {18, 10, 10, 3, 1, 1},
        {20, 11, 11, 3, 0, 0}, {18, 11, 11, 2, 0, 0}, {18, 10, 11, 2, 0, 0}, {18, 11, 10, 2, 0, 0}, {20, 10, 10, 2, 0, 0},
        {16, 10, 10, 2, 0, 0}, {16, 11, 11, 2, 0, 0}, {24, 10, 10, 2, 0, 0}};
    for (auto c : cases) {
        if (only >= 0 && ++ci != only) continue;
        CUtensorMap m;
        const cuuint64_t dims[4] = {(cuuint64_t)px, (cuuint64_t)py, (cuuint64_t)pz, (cuuint64_t)nf};
        const cuuint64_t str[3] = {(cuuint64_t)px * 8, (cuuint64_t)px * py * 8, (cuuint64_t)fsz * 8};
        const cuuint32_t box[4] = {(cuuint32_t)c.bx, (cuuint32_t)c.by, (cuuint32_t)c.bz, (cuuint32_t)nf};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int n = c.bx * c.by * c.bz * nf;
        if (r != CUDA_SUCCESS) { printf("box %d %d %d c0 %d: encode error %d\n", c.bx, c.by, c.bz, c.c0, (int)r); continue; }
        k<<<1, 256, n * 8 + 256>>>(m, out, n, c.c0, c.c1, c.c2);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("box %d %d %d c0 %d c1 %d: %s\n", c.bx, c.by, c.bz, c.c0, c.c1, cudaGetErrorString(e)); return 1; }
        std::vector<double> o(n);
        cudaMemcpy(o.data(), out, n * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int f = 0; f < nf; ++f) for (int z = 0; z < c.bz; ++z) for (int y = 0; y < c.by; ++y) for (int x = 0; x < c.bx; ++x) {
            int gx = c.c0 + x, gy = c.c1 + y, gz = c.c2 + z;
            double want = (gx < px && gy < py && gz < pz) ? h[f * fsz + ((size_t)gz * py + gy) * px + gx] : 0.0;
            if (o[((f * c.bz + z) * c.by + y) * c.bx + x] != want) ++bad;
        }
        printf("box %d %d %d c0 %d c1 %d: %s (%d bad)\n", c.bx, c.by, c.bz, c.c0, c.c1, bad ? "MISMATCH" : "OK", bad);
    }
    return 0;
}
