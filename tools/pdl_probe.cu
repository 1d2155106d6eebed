#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t[64][2];
__global__ void k(int id, int wait_ns, int trig_early) {
    unsigned long long t0; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    if (threadIdx.x == 0 && blockIdx.x == 0) g_t[id][0] = t0;
    if (trig_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    unsigned long long t; do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)wait_ns);
    if (!trig_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); g_t[id][1] = t; }
}
static void run(cudaStream_t s, int pdl, int n, int trig) {
    for (int i = 0; i < n; i++) {
        cudaLaunchConfig_t cfg{}; cfg.gridDim = 32; cfg.blockDim = 128; cfg.stream = s;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = at; cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, k, i, 3000, trig);
    }
}
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int graph = 0; graph < 2; graph++)
    for (int pdl = 0; pdl < 2; pdl++) for (int trig = 0; trig < 2; trig++) {
        const int n = 20;
        cudaGraphExec_t ge = nullptr;
        if (graph) {
            cudaGraph_t g; cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal); run(s, pdl, n, trig);
            cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
            size_t ne = 0; cudaGraphGetEdges(g, nullptr, nullptr, &ne);
            printf("edges %zu ", ne);
        }
        for (int it = 0; it < 3; it++) {
            cudaEventRecord(a, s);
            if (graph) cudaGraphLaunch(ge, s); else run(s, pdl, n, trig);
            cudaEventRecord(b, s); cudaStreamSynchronize(s);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        unsigned long long t[64][2]; cudaMemcpyFromSymbol(t, g_t, sizeof t);
        double gap = 0; for (int i = 1; i < n; i++) gap += (double)((long long)t[i][0] - (long long)t[i-1][1]);
        printf("graph %d pdl %d trig_early %d: total %.2f us (20 x 3 us), mean start-after-prev-end %.2f us  err=%s\n", graph, pdl, trig, ms * 1e3, gap / (n - 1) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
}
