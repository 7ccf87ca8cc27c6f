// Microbenchmark of per-sweep synchronisation floors on B200 (design input
// for the domino sweep; results in profiles/).  Build + run:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/probe tools/launch_probe.cu && /tmp/probe
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void empty_kernel(int *p) {
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
__global__ void pdl_kernel(int *p) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (p && threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}
__global__ void gridsync_kernel(int iters, int *p) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) {
        if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
        g.sync();
    }
}
// hand-rolled barrier: one atomic counter, sense by iteration
__global__ void flagsync_kernel(int iters, unsigned *ctr) {
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            const unsigned target = (unsigned)(i + 1) * gridDim.x;
            while (true) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (v >= target) break;
            }
        }
        __syncthreads();
    }
}

int main() {
    int *d;
    unsigned *ctr;
    cudaMalloc(&d, 4);
    cudaMalloc(&ctr, 4);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int N = 32, REP = 200;
    for (int blocks : {1, 148, 600, 1700}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
            for (int i = 0; i < N; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(512);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                cudaLaunchKernelEx(&cfg, pdl ? pdl_kernel : empty_kernel, d);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int w = 0; w < 10; ++w) cudaGraphLaunch(ge, s);
            cudaEventRecord(a, s);
            for (int r = 0; r < REP; ++r) cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("graph kernels blocks=%d x512 pdl=%d: %.3f us/kernel\n", blocks, pdl, 1e3 * ms / (REP * N));
        }
    }
    for (int per : {1, 2, 4}) {
        int blocks = nsm * per;
        int iters = 2000;
        void *args[] = {&iters, &d};
        cudaLaunchCooperativeKernel((void *)gridsync_kernel, blocks, 512, args, 0, s);
        cudaEventRecord(a, s);
        cudaLaunchCooperativeKernel((void *)gridsync_kernel, blocks, 512, args, 0, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("cg grid.sync blocks=%d x512: %.3f us/iter (%s)\n", blocks, 1e3 * ms / iters,
               cudaGetErrorString(cudaGetLastError()));
        cudaMemset(ctr, 0, 4);
        void *args2[] = {&iters, &ctr};
        cudaLaunchCooperativeKernel((void *)flagsync_kernel, blocks, 512, args2, 0, s);
        cudaMemsetAsync(ctr, 0, 4, s);
        cudaEventRecord(a, s);
        cudaLaunchCooperativeKernel((void *)flagsync_kernel, blocks, 512, args2, 0, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("atomic barrier blocks=%d x512: %.3f us/iter (%s)\n", blocks, 1e3 * ms / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
