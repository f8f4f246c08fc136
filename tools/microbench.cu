// Microbenchmark of phase-step costs on B200: N phases separated by a grid-wide
// cooperative barrier or a cluster barrier, with (a) no work, (b) one dependent
// global read-modify-write per thread, (c) a 7-point stencil read per thread.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE, int WORK>
__global__ void phases(double* a, int n, int nph) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
    for (int p = 0; p < nph; ++p) {
        if (WORK == 1)
            for (int i = tid; i < n; i += nth) a[i] = a[i] * 0.5 + 1.0;
        if (WORK == 2)
            for (int i = tid + 4096; i < n - 4096; i += nth)
                a[i] = a[i] + 1e-3 * (a[i - 1] + a[i + 1] + a[i - 64] + a[i + 64] + a[i - 4096] + a[i + 4096]);
        if (MODE == 0) cg::this_grid().sync();
        else if (MODE == 1) cg::this_cluster().sync();
        else __syncthreads();
    }
}

template <int MODE, int WORK>
float run(int blocks, int threads, int n, int nph, double* a) {
    void* fn = (void*)phases<MODE, WORK>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (MODE == 0) { attr[0].id = cudaLaunchAttributeCooperative; attr[0].val.cooperative = 1; }
    else if (MODE == 1) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = blocks; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    } else cfg.numAttrs = 0;
    void* args[] = {&a, &n, &nph};
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelExC(&cfg, fn, args);
    cudaEventRecord(e0);
    cudaLaunchKernelExC(&cfg, fn, args);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("err %s\n", cudaGetErrorString(err));
    return ms * 1000.f / nph;  // us per phase
}

int main() {
    double* a;
    const int n = 1 << 22;
    cudaMalloc(&a, n * sizeof(double) + (1 << 20));
    cudaMemset(a, 0, n * sizeof(double));
    const int nph = 2000;
    printf("us per phase (barrier + work)\n");
    for (int blocks : {1, 16, 148, 296, 592}) {
        printf("grid  blocks=%4d thr=256: empty %.3f  rmw(64K) %.3f  stencil(64K) %.3f  rmw(4M) %.3f\n", blocks,
               run<0, 0>(blocks, 256, 65536, nph, a), run<0, 1>(blocks, 256, 65536, nph, a),
               run<0, 2>(blocks, 256, 65536, nph, a), run<0, 1>(blocks, 256, n, 200, a));
    }
    for (int blocks : {1, 2, 8, 16}) {
        printf("clust blocks=%4d thr=512: empty %.3f  rmw(64K) %.3f  stencil(64K) %.3f\n", blocks,
               run<1, 0>(blocks, 512, 65536, nph, a), run<1, 1>(blocks, 512, 65536, nph, a),
               run<1, 2>(blocks, 512, 65536, nph, a));
    }
    printf("block blocks=1 thr=1024: empty %.3f  rmw(64K) %.3f  stencil(64K) %.3f\n", run<2, 0>(1, 1024, 65536, nph, a),
           run<2, 1>(1, 1024, 65536, nph, a), run<2, 2>(1, 1024, 65536, nph, a));
    // kernel-boundary cost: back-to-back tiny kernels in a graph
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    for (int k = 0; k < 500; ++k) phases<2, 1><<<1, 256, 0, st>>>(a, 256, 1);
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, st);
    cudaGraphLaunch(ge, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("graph of 500 tiny kernels: %.3f us per kernel\n", ms * 1000 / 500);
    return 0;
}
