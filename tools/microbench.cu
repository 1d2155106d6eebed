// Fixed-cost calibration on B200: launch floors, cluster barriers, DSMEM.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_empty(int* p) { if (threadIdx.x == 1000) p[0] = 1; }
__global__ void __cluster_dims__(8, 1, 1) k_empty_cl(int* p) { if (threadIdx.x == 1000) p[0] = 1; }
__global__ void __cluster_dims__(8, 1, 1) k_cl_sync(int* p) {
    cg::this_cluster().sync();
    if (threadIdx.x == 1000) p[0] = 1;
}
__global__ void __cluster_dims__(8, 1, 1) k_cl_dsmem(unsigned long long* p) {
    __shared__ unsigned long long tile[1024];
    auto cl = cg::this_cluster();
    cl.sync();
    int c = cl.block_rank();
    for (int r = 0; r < 8; r++) cl.map_shared_rank(tile, r)[c * 128 + threadIdx.x] = threadIdx.x + r;
    cl.sync();
    if (tile[threadIdx.x] == 12345) p[0] = 1;
}
__global__ void k_ldchain(const unsigned long long* a, unsigned long long* p, int n) {
    unsigned long long i = threadIdx.x;
    for (int k = 0; k < n; k++) i = a[i];
    if (i == 12345) p[0] = i;
}

template <class F>
float timeit(F f, int iters = 200) {
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; i++) f();
    cudaEventRecord(a);
    for (int i = 0; i < iters; i++) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1000 / iters;
}

int main() {
    int* d; cudaMalloc(&d, 4);
    unsigned long long* a; cudaMalloc(&a, 1 << 20);
    cudaMemset(a, 0, 1 << 20);
    cudaFuncSetAttribute(k_empty_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    cudaFuncSetAttribute(k_cl_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    printf("empty <<<16,128>>>            %6.2f us\n", timeit([&] { k_empty<<<16, 128>>>(d); }));
    printf("empty <<<16,512>>> 64KiB smem  %6.2f us\n", timeit([&] { k_empty<<<16, 512, 0>>>(d); }));
    printf("empty cluster8 <<<16,128>>>    %6.2f us\n", timeit([&] { k_empty_cl<<<16, 128>>>(d); }));
    printf("empty cluster8 120KiB smem     %6.2f us\n", timeit([&] { k_empty_cl<<<16, 128, 120 * 1024>>>(d); }));
    printf("cluster8 sync                  %6.2f us\n", timeit([&] { k_cl_sync<<<16, 128>>>(d); }));
    printf("cluster8 dsmem all-to-all      %6.2f us\n", timeit([&] { k_cl_dsmem<<<16, 128>>>(a); }));
    printf("cluster8 dsmem spread          %6.2f us\n", timeit([&] { k_cl_dsmem<<<16, 128, 120 * 1024>>>(a); }));
    for (int n : {1, 4, 16})
        printf("dependent global loads x%-2d     %6.2f us\n", n, timeit([&] { k_ldchain<<<1, 32>>>(a, (unsigned long long*)d, n); }));
    // graph-captured chains of 20 kernels: per-node cost
    cudaStream_t st; cudaStreamCreate(&st);
    auto graph_time = [&](auto launch, const char* name) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        for (int i = 0; i < 20; i++) launch(st);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int i = 0; i < 5; i++) cudaGraphLaunch(ge, st);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, st);
        for (int i = 0; i < 50; i++) cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("graph node %-28s %6.2f us\n", name, ms * 1000 / 50 / 20);
    };
    graph_time([&](cudaStream_t s) { k_empty<<<16, 128, 0, s>>>(d); }, "empty 16x128");
    graph_time([&](cudaStream_t s) { k_empty<<<148, 512, 0, s>>>(d); }, "empty 148x512");
    graph_time([&](cudaStream_t s) { k_empty_cl<<<16, 128, 0, s>>>(d); }, "empty cluster8 16x128");
    graph_time([&](cudaStream_t s) { k_empty_cl<<<128, 128, 120 * 1024, s>>>(d); }, "empty cluster8 128 spread");
    graph_time([&](cudaStream_t s) { k_cl_dsmem<<<16, 128, 0, s>>>(a); }, "cluster8 dsmem 16");
    graph_time([&](cudaStream_t s) { k_cl_dsmem<<<16, 128, 120 * 1024, s>>>(a); }, "cluster8 dsmem 16 spread");
    graph_time([&](cudaStream_t s) { k_ldchain<<<1, 32, 0, s>>>(a, (unsigned long long*)d, 4); }, "4 dependent loads");
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
}
