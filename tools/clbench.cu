// Phase timing of the cluster transform (HC_TRACE build); standalone.
#define HC_TRACE 1
#include <cstdio>
#include <vector>
#include "../paper_2408_17063_b200/csrc/kernels.cuh"
#include "../paper_2408_17063_b200/csrc/host_tables.hpp"
using namespace hc;
int main() {
    const uint64_t primes[4] = {18014333006036993ull, 18014336227311617ull, 18014343743619073ull, 18014384546430977ull};
    DevCtx D;
    std::vector<Tw> twf, twi;
    std::vector<uint16_t> slot;
    int digits[4];
    build_host_ctx(D, twf, twi, slot, NPOLY, 3, primes, 65537, digits);
    Tw *dtf, *dti;
    cudaMalloc(&dtf, twf.size() * sizeof(Tw));
    cudaMalloc(&dti, twi.size() * sizeof(Tw));
    cudaMemcpy(dtf, twf.data(), twf.size() * sizeof(Tw), cudaMemcpyHostToDevice);
    cudaMemcpy(dti, twi.data(), twi.size() * sizeof(Tw), cudaMemcpyHostToDevice);
    D.twf = dtf; D.twi = dti;
    u64* buf; cudaMalloc(&buf, 16 * NPOLY * 8); cudaMemset(buf, 0, 16 * NPOLY * 8);
    cudaFuncSetAttribute(k_xform_cl<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    for (int nj : {1, 2, 14}) {
        ClJobs cj; memset(&cj, 0, sizeof cj);
        for (int i = 0; i < nj; i++) {
            cj.j[i].dir = 0; cj.j[i].k = i % 4; cj.j[i].ld = LD_U64; cj.j[i].ep = EP_STORE;
            cj.j[i].a = buf + (size_t)i * NPOLY; cj.j[i].out = buf + (size_t)i * NPOLY;
        }
        for (int it = 0; it < 5; it++) k_xform_cl<0><<<nj * CL, CNT, 120 * 1024>>>(D, cj);
        cudaDeviceSynchronize();
        static unsigned long long tr[4096][8];
        cudaMemcpyFromSymbol(tr, g_trace, sizeof tr);
        unsigned long long t0 = ~0ull, tend = 0;
        for (int b = 0; b < nj * CL; b++) { if (tr[b][0] < t0) t0 = tr[b][0]; if (tr[b][5] > tend) tend = tr[b][5]; }
        printf("jobs %d: span %.2f us\n", nj, (tend - t0) / 1e3);
        for (int b = 0; b < std::min(nj * CL, 16); b++)
            printf("  blk %2d start %6.2f  loads+A %6.2f  wait-start %6.2f  exchange %6.2f  passes %6.2f  store %6.2f\n", b,
                   (tr[b][0] - t0) / 1e3, (tr[b][1] - tr[b][0]) / 1e3, (tr[b][2] - tr[b][1]) / 1e3,
                   (tr[b][3] - tr[b][2]) / 1e3, (tr[b][4] - tr[b][3]) / 1e3, (tr[b][5] - tr[b][4]) / 1e3);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
