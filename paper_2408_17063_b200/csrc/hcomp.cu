// libhcomp: host orchestration + C ABI (include/hcomp.h) for the B200 Comp path.
//
// The Comp schedule (compress.py:273-367 with the reference's per-operation
// BGV semantics, bgv.py:579-770) is compiled once per (N, s) plan into job
// lists for the kernels in kernels.cuh and captured into one CUDA graph.
// DESIGN.md section 3 walks through the steps S1..S10 / T1..T4 / F1..F4 /
// D1..D2 named in the comments below.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../../include/hcomp.h"
#include "kernels.cuh"
#include "foldchain.cuh"
#include "ksfused.cuh"
#include "pyrng.hpp"
#include "host_tables.hpp"

using namespace hc;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            return fail(HC_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
        }                                                                             \
    } while (0)

extern "C" const char* hc_last_error(void) { return g_err.c_str(); }

extern "C" int hc_plain_row(void) { return PIDX; }
extern "C" uint64_t hc_prim_root_2n(uint64_t q, int n) { return prim_root_2n_host(q, n); }

extern "C" int hc_galois_tables(int n, uint32_t t, uint16_t* coef, uint16_t* perm) {
    if (galois_tables_host(n, t, coef, perm)) return fail(HC_ERR_ARG, "galois: n must be 8192 and t odd");
    return HC_OK;
}

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------
struct DevKey {
    u64* key = nullptr;        // [D_L][2][L+1][n] Montgomery form
    uint16_t* gal = nullptr;   // coefficient gather
    uint16_t* perm = nullptr;  // NTT-domain permutation
    uint16_t* igal = nullptr;  // inverse coefficient gather: source i -> (j | neg << 15) with gal[j] = i | neg << 15
    int tinv = 1;              // t^-1 mod 2n: gal[j] encodes (j * tinv) mod 2n (k_ksfused's closed-form gather)
};

// transform launches with at most this many jobs use the cluster kernel
static int CL_MAX_JOBS = 48;  // transform batches up to this size use clusters
static int g_cl_chunk = 15;  // co-resident 8-CTA clusters (cudaOccupancyMaxActiveClusters)
static int g_lane_max_blocks = 4;  // chunks up to this many blocks run the baby segment as lanes
static int g_vt2_jobs = 200;       // single-CTA launches of >= this many jobs: three 256-thread transforms per SM
static const int CL_SPREAD_SMEM = 120 * 1024;  // k_cl_intt2 (static smem beside it)
// schedule kernels launch with programmatic stream serialization (PDL): each
// starts while its predecessor drains and blocks in pdl_wait() (kernels.cuh)
// before touching the predecessor's data.  HC_PDL=0 disables it (A/B timing).
static int g_pdl = -1;
static bool pdl_on() {
    if (g_pdl < 0) {
        const char* e = getenv("HC_PDL");
        g_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    return g_pdl == 1;
}
// PDL only on the main chain: inside parallel branches (lanes) an early-launched
// kernel would hold SMs idle that the other branches need
static thread_local bool g_step_pdl = true;
static thread_local bool g_pdl_suspended = false;  // hc_comp_profile: launches timed one by one
template <typename... KArgs, typename... Args>
static cudaError_t launch_cl(void (*k)(KArgs...), int cluster, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args);
template <typename... KArgs, typename... Args>
static cudaError_t launch(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    int na = 0;
    if (pdl_on() && g_step_pdl && !g_pdl_suspended) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, args...);
}
// runtime cluster dimension (non-portable sizes), PDL as launch()
template <typename... KArgs, typename... Args>
static cudaError_t launch_cl(void (*k)(KArgs...), int cluster, dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    na++;
    if (pdl_on() && g_step_pdl && !g_pdl_suspended) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        na++;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

enum StepKind { ST_XF, ST_CO, ST_MA, ST_DX, ST_MEMSET = 5, ST_I2 = 6, ST_MB = 7, ST_ADD = 8, ST_FOLD = 9, ST_KF = 10 };  // values: bench.py per_kind_ms keys
struct Step {
    int kind = 0;
    int njobs = 0;
    int gy = 1;
    void* djobs = nullptr;
    // ST_MEMSET
    u64* out = nullptr;
    int rows = 0;  // ST_ADD: rows per job (gy: primes)
    size_t bytes = 0;
    std::vector<XJob> hjobs;  // ST_XF: host copy (cluster launches pass jobs by value)
    std::vector<Intt2Job> i2jobs;  // ST_I2
    std::vector<XJob> side;        // ST_XF cluster launch: ClJobs.side (res_f.c0 finish of a fold)
    int group = 0;            // consecutive steps with the same nonzero group run concurrently
    int cl = 0;               // ST_XF: launch as 8-CTA clusters (<= CL_MAX jobs)
    int jpc = 1;              // ST_XF cluster launch: transforms per cluster
    int lane = -1;            // in a group: steps of one lane run in order on one branch
    FcArgs fc{};              // ST_FOLD: the persistent fold chain (k_foldchain)
};

struct Schedule {
    std::vector<Step> steps;
    std::vector<void*> allocs;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    int cur_group = 0, next_group = 1, cur_lane = -1;
    bool cl_in_lane = false;  // allow cluster launches inside a lane
    // steps added between par_begin() and par_end() are independent: they are
    // captured on forked streams (parallel graph branches)
    void par_begin() { cur_group = next_group++; }
    void par_end() { cur_group = 0; }
    ~Schedule() {
        if (exec) cudaGraphExecDestroy(exec);
        for (void* p : allocs) cudaFree(p);
    }
};

struct Plan;

struct hc_ctx {
    int dev = 0, L = 3, n = NPOLY;
    u64 p = 0;
    DevCtx hctx{};             // host copy (device pointers inside)
    KFront kfront{};           // k_ksfused's front-stage constants (by value at its launches)
    DevCtx* d_ctx = nullptr;
    Tw* d_twf = nullptr;
    Tw* d_twi = nullptr;
    uint16_t* d_slot_of = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t side[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev_fork = nullptr, ev_join[4] = {nullptr, nullptr, nullptr, nullptr};
    // second copy engine for the inputs' H2D (cd on the caller's stream, cv here)
    cudaStream_t copy_s = nullptr;
    cudaEvent_t ev_copy0 = nullptr, ev_copy1 = nullptr;
    std::map<uint32_t, DevKey> keys;
    std::unique_ptr<Plan> plan;
    int digits[MAXL + 1] = {};
};

static void release_key(DevKey& k) {
    cudaFree(k.key);
    cudaFree(k.gal);
    cudaFree(k.perm);
    cudaFree(k.igal);
}

// (direction, loader, epilogue) combinations the schedules use; each gets a
// single-CTA (k_xf) and an 8-CTA cluster (k_xf_cl) instantiation.
#define XF_COMBOS(X)                  \
    X(0, LD_U64, EP_STORE)            \
    X(1, LD_U64, EP_STORE)            \
    X(0, LD_RED, EP_STORE)            \
    X(1, LD_RED, EP_STORE)            \
    X(1, LD_MONT, EP_RS)              \
    X(1, LD_MONT, EP_RESCALE_RD)      \
    X(1, LD_MONT, EP_RESCALE4)        \
    X(0, LD_U64, EP_ADDMONT)          \
    X(0, LD_DIG, EP_STORE_LAZY)       \
    X(0, LD_DIGGAL, EP_STORE_LAZY)    \
    X(0, LD_RED, EP_ADDRED)           \
    X(0, LD_DIGGAL, EP_KSACC)         \
    X(1, LD_KSFIN, EP_RESCALE)

static int kernels_configured = 0;
// co-resident 16-CTA clusters for k_foldchain (it needs D_1 = 7; 0: the fold
// chain runs as two launches per fold).  HC_FOLDCHAIN=0 disables it.
static int g_fc_clusters = 0;
static int g_i2_16 = 0;  // co-resident 16-CTA clusters (0: two-prime INTTs on 8-CTA clusters)
// co-resident 8-CTA transform clusters (one CTA per SM) on the current device
static int max_active_clusters(int* clusters) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(CL * 16);
    cfg.blockDim = dim3(CNT);
    cfg.dynamicSmemBytes = CL_SMEM;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CU(cudaFuncSetAttribute(k_xf_cl<0, LD_U64, EP_STORE, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));
    CU(cudaOccupancyMaxActiveClusters(clusters, k_xf_cl<0, LD_U64, EP_STORE, 1>, &cfg));
    return HC_OK;
}

static int configure_kernels() {
    if (kernels_configured) return HC_OK;
    // cluster transforms: reserve enough (unused) dynamic smem that each CTA
    // of a cluster lands on its own SM -- otherwise the scheduler packs all 8
    // small CTAs onto one or two SMs and nothing is gained
#define XF_CFG(D, L, E)                                                                                    \
    CU(cudaFuncSetAttribute(k_xf<D, L, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, NPOLY * 8));      \
    CU(cudaFuncSetAttribute(k_xf<D, L, E, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, NPOLY * 8));   \
    CU(cudaFuncSetAttribute(k_xf_cl<D, L, E, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));  \
    CU(cudaFuncSetAttribute(k_xf_cl<D, L, E, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));  \
    CU(cudaFuncSetAttribute(k_xf_cl<D, L, E, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));  \
    CU(cudaFuncSetAttribute(k_xf_cl<D, L, E, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SMEM));
    XF_COMBOS(XF_CFG)
#undef XF_CFG
    CU(cudaFuncSetAttribute(k_plain, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * NPOLY * 8));
    CU(cudaFuncSetAttribute(k_cl_intt2<LD_KSFIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SPREAD_SMEM));
    CU(cudaFuncSetAttribute(k_cl_intt2<LD_RED>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SPREAD_SMEM));
    CU(cudaFuncSetAttribute(k_cl16_intt2<LD_KSFIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SPREAD_SMEM));
    CU(cudaFuncSetAttribute(k_cl16_intt2<LD_RED>, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SPREAD_SMEM));
    CU(cudaFuncSetAttribute(k_cl16_intt2<LD_KSFIN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CU(cudaFuncSetAttribute(k_cl16_intt2<LD_RED>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    {  // 16-CTA clusters for the two-prime INTT when the part can co-schedule them
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(CNT);
        cfg.dynamicSmemBytes = CL_SPREAD_SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n16 = 0;
        if (cudaOccupancyMaxActiveClusters(&n16, k_cl16_intt2<LD_KSFIN>, &cfg) != cudaSuccess) n16 = 0;
        cudaGetLastError();
        const char* e = getenv("HC_I2_16");
        g_i2_16 = (e && e[0] == '0') ? 0 : n16;
    }
    {
        int n = 0;
        if (max_active_clusters(&n) == HC_OK && n > 0) g_cl_chunk = std::min(n, CL_MAX / CL_JPC_MAX);
    }
    CU(cudaFuncSetAttribute(k_ksfused, cudaFuncAttributeMaxDynamicSharedMemorySize, KF_SMEM));
    CU(cudaFuncSetAttribute(k_foldchain, cudaFuncAttributeMaxDynamicSharedMemorySize, CL_SPREAD_SMEM));
    CU(cudaFuncSetAttribute(k_foldchain, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(FC_CL);
        cfg.blockDim = dim3(CNT);
        cfg.dynamicSmemBytes = CL_SPREAD_SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = FC_CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_foldchain, &cfg) != cudaSuccess) n = 0;
        cudaGetLastError();
        const char* e = getenv("HC_FOLDCHAIN");
        g_fc_clusters = (e && e[0] == '0') ? 0 : n;
    }
    kernels_configured = 1;
    return HC_OK;
}

extern "C" int hc_ctx_create(int n, int max_level, const uint64_t* primes, uint64_t p, int ksw_base_bits,
                             int device, hc_ctx** out) {
    if (n != NPOLY) return fail(HC_ERR_ARG, "only n = 8192 is supported");
    if (max_level < 1 || max_level > MAXL)
        return fail(HC_ERR_ARG, "max_level must be 1.." + std::to_string(MAXL) + " for this build");
    if (ksw_base_bits != 16) return fail(HC_ERR_ARG, "only ksw_base_bits = 16 is supported");
    if (p >= (1ull << 31) || p % (2 * (u64)n) != 1) return fail(HC_ERR_ARG, "bad plaintext modulus");
    for (int k = 0; k <= max_level; k++) {
        if (primes[k] >= (1ull << 54) || primes[k] < (1ull << 53))
            return fail(HC_ERR_ARG, "chain primes must be 54-bit");
        if (primes[k] % (2 * (u64)n) != 1 || primes[k] % p != 1)
            return fail(HC_ERR_ARG, "chain prime not = 1 mod 2n and mod p");
        if (k && primes[k] <= primes[k - 1]) return fail(HC_ERR_ARG, "primes must be in level order (ascending)");
    }
    std::unique_ptr<hc_ctx> h(new hc_ctx());
    h->dev = device;
    h->L = max_level;
    h->p = p;
    CU(cudaSetDevice(device));
    int rc = configure_kernels();
    if (rc) return rc;
    // blocking stream: ordered after legacy-stream copies (pageable cudaMemcpy
    // may return before its DMA lands)
    CU(cudaStreamCreate(&h->stream));
    for (int i = 0; i < 4; i++) {
        CU(cudaStreamCreateWithFlags(&h->side[i], cudaStreamNonBlocking));
        CU(cudaEventCreateWithFlags(&h->ev_join[i], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    CU(cudaStreamCreateWithFlags(&h->copy_s, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&h->ev_copy0, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h->ev_copy1, cudaEventDisableTiming));

    DevCtx& D = h->hctx;
    std::vector<Tw> twf, twi;
    std::vector<uint16_t> slot_of;
    build_host_ctx(D, twf, twi, slot_of, n, max_level, primes, p, h->digits);
    CU(cudaMalloc(&h->d_twf, twf.size() * sizeof(Tw)));
    CU(cudaMalloc(&h->d_twi, twi.size() * sizeof(Tw)));
    CU(cudaMalloc(&h->d_slot_of, n * sizeof(uint16_t)));
    CU(cudaMemcpy(h->d_twf, twf.data(), twf.size() * sizeof(Tw), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_twi, twi.data(), twi.size() * sizeof(Tw), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(h->d_slot_of, slot_of.data(), n * sizeof(uint16_t), cudaMemcpyHostToDevice));
    D.twf = h->d_twf;
    D.twi = h->d_twi;
    D.slot_of = h->d_slot_of;
    for (int k = 0; k <= std::min(max_level, KEYL); k++)
        build_kfront(h->kfront.k[k], &h->kfront.w32s[k], &twf[(size_t)k * n], primes[k]);
    CU(cudaMalloc(&h->d_ctx, sizeof(DevCtx)));
    CU(cudaMemcpy(h->d_ctx, &D, sizeof(DevCtx), cudaMemcpyHostToDevice));
    *out = h.release();
    return HC_OK;
}

extern "C" int hc_ctx_digits(const hc_ctx* h, int* digits) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    for (int l = 0; l <= h->L; l++) digits[l] = h->digits[l];
    return HC_OK;
}

extern "C" int hc_clear_keys(hc_ctx* h) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    cudaSetDevice(h->dev);
    cudaDeviceSynchronize();
    h->plan.reset();  // captured graphs hold key pointers: re-plan after a key change
    for (auto& kv : h->keys) release_key(kv.second);
    h->keys.clear();
    return HC_OK;
}

static int load_ksk_impl(hc_ctx* h, uint32_t t, const uint64_t* ksk, int dig_have, int rows_have);
extern "C" int hc_load_ksk(hc_ctx* h, uint32_t t, const uint64_t* ksk) {
    if (!h || !ksk) return fail(HC_ERR_ARG, "null argument");
    return load_ksk_impl(h, t, ksk, h->digits[h->L], h->L + 1);
}
extern "C" int hc_load_ksk_slice(hc_ctx* h, uint32_t t, const uint64_t* ksk, int digits, int rows) {
    if (!h || !ksk) return fail(HC_ERR_ARG, "null argument");
    return load_ksk_impl(h, t, ksk, digits, rows);
}
static int load_ksk_impl(hc_ctx* h, uint32_t t, const uint64_t* ksk, int dig_have, int rows_have) {
    if ((t & 1) == 0 || t >= 2u * NPOLY) return fail(HC_ERR_ARG, "galois element must be odd and < 2n");
    CU(cudaSetDevice(h->dev));
    auto it = h->keys.find(t);
    if (it != h->keys.end()) {
        CU(cudaDeviceSynchronize());
        h->plan.reset();  // the plan's graphs point at the key being replaced
        release_key(it->second);
        h->keys.erase(it);
    }
    DevKey k;
    // ksk: [D_L][2][L+1][n] (the key at max level).  The device keeps the
    // digits and primes key switching uses (levels <= KEYL): at max_level 4
    // the first 14 digits on the 4 smallest primes (_KskPair.at_level,
    // bgv.py:304-312, reduces exactly that way).
    // ksk: [dig_have][2][rows_have][n] (rows in level order); the device keeps
    // the first DK digits on the KL1 smallest primes
    const int L1 = rows_have;
    const int KL1 = h->hctx.KL1, DK = h->digits[KL1 - 1];
    if (dig_have < DK || rows_have < KL1) {
        release_key(k);
        return fail(HC_ERR_ARG, "key-switch key slice smaller than the device's levels need");
    }
    const size_t rows = (size_t)DK * 2 * KL1;
    CU(cudaMalloc(&k.key, rows * NPOLY * 8));
    if (KL1 == L1) {
        CU(cudaMemcpyAsync(k.key, ksk, rows * NPOLY * 8, cudaMemcpyHostToDevice, h->stream));
    } else {
        for (int d = 0; d < DK; d++)
            for (int ab = 0; ab < 2; ab++)
                CU(cudaMemcpyAsync(k.key + ((size_t)d * 2 + ab) * KL1 * NPOLY, ksk + ((size_t)d * 2 + ab) * L1 * NPOLY,
                                   (size_t)KL1 * NPOLY * 8, cudaMemcpyHostToDevice, h->stream));
    }
    k_to_mont<<<592, 256, 0, h->stream>>>(h->hctx, k.key, (long long)rows, KL1);
    CU(cudaGetLastError());
    std::vector<uint16_t> gal(NPOLY), perm(NPOLY);
    int rc = hc_galois_tables(NPOLY, t, gal.data(), perm.data());
    if (rc) return rc;
    CU(cudaMalloc(&k.gal, NPOLY * 2));
    CU(cudaMalloc(&k.perm, NPOLY * 2));
    CU(cudaMemcpy(k.gal, gal.data(), NPOLY * 2, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(k.perm, perm.data(), NPOLY * 2, cudaMemcpyHostToDevice));
    {  // the automorphism is a signed bijection of the coefficients: invert it
        std::vector<uint16_t> igal(NPOLY);
        for (int j = 0; j < NPOLY; j++) igal[gal[j] & 0x7FFF] = (uint16_t)(j | (gal[j] & 0x8000));
        CU(cudaMalloc(&k.igal, NPOLY * 2));
        CU(cudaMemcpy(k.igal, igal.data(), NPOLY * 2, cudaMemcpyHostToDevice));
    }
    k.tinv = (gal[1] & 0x7FFF) + ((gal[1] >> 15) ? NPOLY : 0);
    CU(cudaStreamSynchronize(h->stream));
    h->keys[t] = k;
    return HC_OK;
}

// ---------------------------------------------------------------------------
// schedule helpers
// ---------------------------------------------------------------------------
static int upload_jobs(Schedule& S, Step& st, const void* host, size_t bytes) {
    void* d = nullptr;
    CU(cudaMalloc(&d, bytes));
    CU(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice));
    CU(cudaDeviceSynchronize());  // the DMA must land before any stream uses the jobs
    S.allocs.push_back(d);
    st.djobs = d;
    return HC_OK;
}

// one step (launch) per (direction, loader, epilogue, transform-less) group,
// in first-appearance order
static int g_trace_seq = 0;
// One batch of independent transforms, grouped by (dir, loader, epilogue);
// a group too big for one cluster launch (g_cl_chunk = co-resident 8-CTA
// clusters) is split into launches that run as parallel graph branches.
static int add_xf(Schedule& S, const std::vector<XJob>& jobs) {
    // one launch per kernel instantiation (dir, loader, epilogue)
    std::vector<std::vector<XJob>> sets;
    std::vector<int> taken(jobs.size(), 0);
    for (size_t i = 0; i < jobs.size(); i++) {
        if (taken[i]) continue;
        std::vector<XJob> sel;
        for (size_t k = i; k < jobs.size(); k++) {
            const XJob &a = jobs[i], &b = jobs[k];
            if (!taken[k] && a.dir == b.dir && a.ld == b.ld && kernel_ep(a.dir, a.ld, a.ep) == kernel_ep(b.dir, b.ld, b.ep) &&
                a.noxf == b.noxf) {
                sel.push_back(b);
                taken[k] = 1;
            }
        }
        sets.push_back(sel);
    }
    // clusters only for small batches outside parallel lanes (lanes
    // already fill the GPU; single-CTA transforms are more efficient there)
    auto cl_ok = [&](const std::vector<XJob>& sel) {
        return !sel[0].noxf && (int)sel.size() <= CL_MAX_JOBS && (S.cur_lane < 0 || S.cl_in_lane);
    };
    // several cluster batches of one call are independent: run them side by
    // side (parallel graph branches) sharing one wave of co-resident clusters
    int ncl_sets = 0, shared_jpc = 0;
    for (const auto& sel : sets) ncl_sets += cl_ok(sel);
    if (ncl_sets > 1 && !S.cur_group && S.cur_lane < 0) {
        for (int jj = 1; jj <= CL_JPC_MAX && !shared_jpc; jj++) {
            int need = 0;
            for (const auto& sel : sets)
                if (cl_ok(sel)) need += ((int)sel.size() + jj - 1) / jj;
            if (need <= g_cl_chunk) shared_jpc = jj;
        }
    }
    const bool together = shared_jpc > 0;
    if (together) S.par_begin();
    for (const auto& sel : sets) {
        const bool clu = cl_ok(sel);
        // cluster launches: up to CL_JPC_MAX transforms per cluster so that the
        // batch fits one wave of co-resident clusters
        const int jpc = !clu ? 1
                        : together ? shared_jpc
                                   : std::min(CL_JPC_MAX, std::max(1, ((int)sel.size() + g_cl_chunk - 1) / g_cl_chunk));
        const size_t chunk = clu ? (size_t)g_cl_chunk * jpc : sel.size();
        const int saved = S.cur_group;
        if (clu && sel.size() > chunk && !S.cur_group) S.par_begin();
        for (size_t c0 = 0; c0 < sel.size(); c0 += chunk) {
            std::vector<XJob> part(sel.begin() + c0, sel.begin() + std::min(sel.size(), c0 + chunk));
            for (XJob& j : part) j.trace = g_trace_seq;
            g_trace_seq++;
            Step st;
            st.kind = ST_XF;
            st.gy = part[0].dir;
            st.cl = clu;
            st.jpc = jpc;
            st.njobs = (int)part.size();
            st.hjobs = part;
            st.group = S.cur_group;
            st.lane = S.cur_lane;
            int rc = upload_jobs(S, st, part.data(), part.size() * sizeof(XJob));
            if (rc) return rc;
            S.steps.push_back(st);
        }
        if (!saved) S.par_end();
    }
    if (together) S.par_end();
    return HC_OK;
}
static int add_co(Schedule& S, const std::vector<CJob>& jobs) {
    if (jobs.empty()) return HC_OK;
    Step st;
    st.kind = ST_CO;
    st.group = S.cur_group;
    st.lane = S.cur_lane;
    st.njobs = (int)jobs.size();
    int rc = upload_jobs(S, st, jobs.data(), jobs.size() * sizeof(CJob));
    if (rc) return rc;
    S.steps.push_back(st);
    return HC_OK;
}
static int add_ma(Schedule& S, std::vector<MJob> jobs, int nprime) {
    if (jobs.empty()) return HC_OK;
    // throughput regime: single-term jobs that share a key (one rotation or
    // the column swap over several blocks) go out in groups of MB_MAX, each
    // key digit loaded once per group (k_ksmac_mb; HC_KSMAC_MB=0: off)
    static int mb_on = -1;
    if (mb_on < 0) {
        const char* e = getenv("HC_KSMAC_MB");
        mb_on = (e && e[0] == '0') ? 0 : 1;
    }
    bool single = true;
    for (const MJob& m : jobs) single = single && m.nterm == 1;
    // blocks per group: 2 (48 registers, 5 CTAs/SM) measured best -- N=2^20:
    // 5.68 ms vs 5.77 with 4 and 7.08 with 8 (HC_KSMAC_MB_N=4 for A/B)
    static int mb_n = -1;
    if (mb_n < 0) {
        const char* e = getenv("HC_KSMAC_MB_N");
        mb_n = (e && atoi(e) >= 4) ? 4 : 2;
    }
    if (mb_on && single && jobs.size() > 16) {
        std::vector<MBJob> mb;
        std::vector<int> used(jobs.size(), 0);
        for (size_t i = 0; i < jobs.size(); i++) {
            if (used[i]) continue;
            MBJob g{};
            g.level = jobs[i].level;
            g.key = jobs[i].t[0].key;
            g.perm = jobs[i].t[0].perm;
            for (size_t k2 = i; k2 < jobs.size() && g.nb < mb_n; k2++) {
                const MJob& m = jobs[k2];
                if (used[k2] || m.t[0].key != g.key || m.t[0].perm != g.perm || m.level != g.level) continue;
                used[k2] = 1;
                g.dntt[g.nb] = m.t[0].dntt;
                g.c0src[g.nb] = m.t[0].c0src;
                g.add0[g.nb] = m.add0;
                g.add1[g.nb] = m.add1;
                g.out0[g.nb] = m.out0;
                g.out1[g.nb] = m.out1;
                g.nb++;
            }
            g.trace = g_trace_seq;
            mb.push_back(g);
        }
        g_trace_seq++;
        Step st;
        st.kind = ST_MB;
        st.group = S.cur_group;
        st.lane = S.cur_lane;
        st.njobs = (int)mb.size();
        st.gy = nprime;
        st.jpc = mb_n;  // group width -> instantiation
        int rc = upload_jobs(S, st, mb.data(), mb.size() * sizeof(MBJob));
        if (rc) return rc;
        S.steps.push_back(st);
        return HC_OK;
    }
    for (MJob& j : jobs) j.trace = g_trace_seq;
    g_trace_seq++;
    Step st;
    st.kind = ST_MA;
    st.group = S.cur_group;
    st.lane = S.cur_lane;
    st.njobs = (int)jobs.size();
    st.gy = nprime;
    int rc = upload_jobs(S, st, jobs.data(), jobs.size() * sizeof(MJob));
    if (rc) return rc;
    S.steps.push_back(st);
    return HC_OK;
}
static int add_dx(Schedule& S, std::vector<DXJob> jobs, int nprime) {
    if (jobs.empty()) return HC_OK;
    for (DXJob& j : jobs) j.trace = g_trace_seq;
    g_trace_seq++;
    Step st;
    st.kind = ST_DX;
    st.group = S.cur_group;
    st.lane = S.cur_lane;
    st.njobs = (int)jobs.size();
    st.gy = nprime;
    int rc = upload_jobs(S, st, jobs.data(), jobs.size() * sizeof(DXJob));
    if (rc) return rc;
    S.steps.push_back(st);
    return HC_OK;
}
// fused key switches (k_ksfused): one job per (block, rotation)
static int add_kf(Schedule& S, std::vector<KFJob> jobs, int nprime) {
    if (jobs.empty()) return HC_OK;
    for (KFJob& j : jobs) j.trace = g_trace_seq;
    g_trace_seq++;
    Step st;
    st.kind = ST_KF;
    st.group = S.cur_group;
    st.lane = S.cur_lane;
    st.njobs = (int)jobs.size();
    st.gy = nprime;
    int rc = upload_jobs(S, st, jobs.data(), jobs.size() * sizeof(KFJob));
    if (rc) return rc;
    S.steps.push_back(st);
    return HC_OK;
}
// two-prime INTT + CRT digits (k_cl_intt2), <= I2_MAX jobs per launch
static int add_i2(Schedule& S, std::vector<Intt2Job> jobs) {
    for (size_t c0 = 0; c0 < jobs.size(); c0 += I2_MAX) {
        Step st;
        st.kind = ST_I2;
        st.group = S.cur_group;
        st.lane = S.cur_lane;
        st.i2jobs.assign(jobs.begin() + c0, jobs.begin() + std::min(jobs.size(), c0 + (size_t)I2_MAX));
        for (Intt2Job& j : st.i2jobs) j.j[0].trace = j.j[1].trace = g_trace_seq;
        g_trace_seq++;
        st.njobs = (int)st.i2jobs.size();
        S.steps.push_back(st);
    }
    return HC_OK;
}

static int add_add(Schedule& S, const std::vector<AddJob>& jobs, int rows, int nprime) {
    if (jobs.empty()) return HC_OK;
    Step st;
    st.kind = ST_ADD;
    st.group = S.cur_group;
    st.lane = S.cur_lane;
    st.njobs = (int)jobs.size();
    st.rows = rows;
    st.gy = nprime;
    int rc = upload_jobs(S, st, jobs.data(), jobs.size() * sizeof(AddJob));
    if (rc) return rc;
    S.steps.push_back(st);
    return HC_OK;
}

// Job lists of single ring operations on device buffers (used by the
// single-op entry points and by the mixed-level pack_pair schedule).
// mul_plain + modulus switch at level l (bgv.py:717-733, 579-608):
//   c [2][l+1][n] x ptm [l+1][n] (plaintext in Montgomery form with q_l^-1
//   folded into rows k < l) -> o [2][l][n]; corr: scratch [2][l][n].
static void jobs_mul_plain(std::vector<XJob>& inv, std::vector<XJob>& fwd, int l, const u64* c, const u64* ptm,
                           u64* corr, u64* o) {
    const size_t NB = NPOLY;
    const int P1 = l + 1;
    for (int poly = 0; poly < 2; poly++) {
        XJob j{};
        j.dir = 1; j.k = l; j.ld = LD_MONT; j.ep = l > KEYL ? EP_RESCALE4 : EP_RESCALE; j.level = l;
        j.a = c + ((size_t)poly * P1 + l) * NB;
        j.b = ptm + (size_t)l * NB;
        j.out = corr + (size_t)poly * l * NB;
        j.ostride = NB;
        inv.push_back(j);
        for (int k = 0; k < l; k++) {
            XJob f{};
            f.dir = 0; f.k = k; f.ld = LD_U64; f.ep = EP_ADDMONT;
            f.a = corr + ((size_t)poly * l + k) * NB;
            f.ea = c + ((size_t)poly * P1 + k) * NB;
            f.eb = ptm + (size_t)k * NB;
            f.out = o + ((size_t)poly * l + k) * NB;
            fwd.push_back(f);
        }
    }
}
// rotation by Galois element `key` at level l <= KEYL (bgv.py:735-770,
// 616-647): c [2][l+1][n] -> o [2][l+1][n] (+ add [2][l+1][n] when given);
// scratch coef [l+1][n], dig [D_l][n], dntt [D_l][l+1][n].
static void jobs_rotate(std::vector<XJob>& inv, std::vector<CJob>& co, std::vector<XJob>& fwd, std::vector<MJob>& ma,
                        int l, int D, const DevKey* key, const u64* c, u64* coef, uint16_t* dig, u64* dntt, u64* o,
                        const u64* add = nullptr) {
    const size_t NB = NPOLY;
    const int P1 = l + 1;
    for (int k = 0; k < P1; k++) {
        XJob j{};
        j.dir = 1; j.k = k; j.ld = LD_U64; j.ep = EP_STORE;
        j.a = c + ((size_t)1 * P1 + k) * NB;
        j.out = coef + (size_t)k * NB;
        inv.push_back(j);
    }
    CJob cj{};
    cj.level = l; cj.mode = 0;
    cj.x = coef;
    cj.xstride = NB;
    cj.gal = key->gal;
    cj.dig = dig;
    co.push_back(cj);
    for (int jj = 0; jj < D; jj++)
        for (int k = 0; k < P1; k++) {
            XJob j{};
            j.dir = 0; j.k = k; j.ld = LD_DIG; j.ep = EP_STORE_LAZY;  // feeds k_ksmac (<= 14 lazy terms < q 2^64)
            j.a = (const u64*)(dig + (size_t)jj * NB);
            j.out = dntt + ((size_t)jj * P1 + k) * NB;
            fwd.push_back(j);
        }
    MJob mj{};
    mj.level = l; mj.nterm = 1;
    mj.t[0].dntt = dntt;
    mj.t[0].key = key->key;
    mj.t[0].c0src = c;
    mj.t[0].perm = key->perm;
    if (add) {
        mj.add0 = add;
        mj.add1 = add + (size_t)P1 * NB;
    }
    mj.out0 = o;
    mj.out1 = o + (size_t)P1 * NB;
    ma.push_back(mj);
}

static void add_memset(Schedule& S, void* p, size_t bytes) {
    Step st;
    st.kind = ST_MEMSET;
    st.out = (u64*)p;
    st.bytes = bytes;
    S.steps.push_back(st);
}

// PDL for launches of about one wave or less (the latency path); a multi-wave
// launch gains nothing from an early successor and measured slower with one
// (its CTAs park on SMs the last wave could use): N=2^20 6.12 -> 6.40 ms.
static int g_pdl_maxcta = -1;  // HC_PDL_MAXCTA: elementwise-launch CTA bound for PDL
static bool step_one_wave(const Step& st) {
    const int sms = 148;
    if (g_pdl_maxcta < 0) {
        const char* e = getenv("HC_PDL_MAXCTA");
        g_pdl_maxcta = e ? atoi(e) : 0;  // measured: PDL on elementwise launches helps nowhere
    }
    switch (st.kind) {
        case ST_XF:
            if (st.hjobs[0].noxf) return st.njobs * (NPOLY / 256) <= g_pdl_maxcta;
            if (st.cl && st.njobs <= CL_MAX) return true;
            return st.njobs < g_vt2_jobs && st.njobs <= std::min(sms, g_pdl_maxcta);
        case ST_MA:
        case ST_MB: return (NPOLY / 256) * st.gy * st.njobs <= g_pdl_maxcta;
        case ST_DX: return (NPOLY / 256) * st.njobs <= g_pdl_maxcta;
        case ST_KF: return CL * st.gy * st.njobs <= g_pdl_maxcta;
        case ST_CO: return (NPOLY / 256) * st.njobs <= std::max(g_pdl_maxcta, 148);  // small composes (latency path)
        default: return true;
    }
}

// CTA size of the throughput regime's memory-bound MAC kernels.  The VT = 4
// transform kernels take 3 x 256 threads x 72 registers of an SM; a
// 128-thread MAC CTA fits in what they leave (10 K registers), so a chunk's
// MACs run beside another chunk's transforms instead of waiting for a slot.
static int mac_threads() {
    static int mt = 0;
    if (!mt) {
        const char* e = getenv("HC_MAC_THREADS");
        mt = e ? atoi(e) : 128;
        if (mt != 64 && mt != 128 && mt != 256) mt = 128;
    }
    return mt;
}

static int enqueue_step(const hc_ctx* h, const Step& st, cudaStream_t s) {
    g_step_pdl = st.group == 0 && step_one_wave(st);
    {
        switch (st.kind) {
            case ST_XF: {
                const XJob& j0 = st.hjobs[0];
                if (j0.noxf) {
                    if (j0.ld != LD_KSFIN) return fail(HC_ERR_STATE, "transform-less job needs LD_KSFIN");
                    CU(launch(k_elem<LD_KSFIN>, dim3(NPOLY / 256, st.njobs), 128, 0, s, h->hctx, (const XJob*)st.djobs));
                    break;
                }
                const bool clu = st.cl && st.njobs <= CL_MAX;  // latency path: 8-CTA clusters, jpc transforms each
                const int ncl = (st.njobs + st.jpc - 1) / st.jpc;
                ClJobs cj;
                if (clu) {
                    memset(&cj, 0, sizeof cj);
                    memcpy(cj.j, st.hjobs.data(), st.njobs * sizeof(XJob));
                    cj.n = st.njobs;
                    if (!st.side.empty()) {
                        if (ncl * st.jpc < 8 || st.side.size() != 2 || j0.ep != EP_KSACC)
                            return fail(HC_ERR_STATE, "side finish needs a KSACC cluster launch of >= 8 job slots");
                        cj.nside = 2;
                        cj.side[0] = st.side[0];
                        cj.side[1] = st.side[1];
                    }
                }
                bool done = false;
#define XF_LAUNCH(D, L, E)                                                                               \
    if (!done && j0.dir == D && j0.ld == L && kernel_ep(j0.dir, j0.ld, j0.ep) == E) {                    \
        if (clu) {                                                                                       \
            switch (st.jpc) {                                                                            \
                case 1: CU(launch(k_xf_cl<D, L, E, 1>, ncl * CL, CNT, CL_SMEM, s, h->hctx, cj)); break;     \
                case 2: CU(launch(k_xf_cl<D, L, E, 2>, ncl * CL, 2 * CNT, CL_SMEM, s, h->hctx, cj)); break; \
                case 3: CU(launch(k_xf_cl<D, L, E, 3>, ncl * CL, 3 * CNT, CL_SMEM, s, h->hctx, cj)); break; \
                default: CU(launch(k_xf_cl<D, L, E, 4>, ncl * CL, 4 * CNT, CL_SMEM, s, h->hctx, cj)); break; \
            }                                                                                            \
        }                                                                                                \
        else if (st.njobs >= g_vt2_jobs)                                                                 \
            CU(launch(k_xf<D, L, E, 4>, st.njobs, NT / 4, NPOLY * 8, s, h->hctx, (const XJob*)st.djobs)); \
        else CU(launch(k_xf<D, L, E>, st.njobs, NT, NPOLY * 8, s, h->hctx, (const XJob*)st.djobs));       \
        done = true;                                                                                     \
    }
                XF_COMBOS(XF_LAUNCH)
#undef XF_LAUNCH
                if (!done) return fail(HC_ERR_STATE, "transform job combination not instantiated");
                break;
            }
            case ST_CO:
                CU(launch(k_compose, dim3(NPOLY / 256, st.njobs), 256, 0, s, h->hctx, (const CJob*)st.djobs));
                break;
            case ST_MA:
                if (st.njobs > 16)  // throughput: occupancy
                    CU(launch(k_ksmac<1, 1>, dim3(NPOLY / 256, st.gy, st.njobs), 256, 0, s, h->hctx, (const MJob*)st.djobs));
                else  // small (latency path): 4 digits' loads in flight per thread
                    CU(launch(k_ksmac<1, 4>, dim3(NPOLY / 256, st.gy, st.njobs), 256, 0, s, h->hctx, (const MJob*)st.djobs));
                break;
            case ST_MB: {
                const int mt = mac_threads();
                if (st.jpc == 4)
                    CU(launch(k_ksmac_mb<4>, dim3(NPOLY / mt, st.gy, st.njobs), mt, 0, s, h->hctx, (const MBJob*)st.djobs));
                else
                    CU(launch(k_ksmac_mb<2>, dim3(NPOLY / mt, st.gy, st.njobs), mt, 0, s, h->hctx, (const MBJob*)st.djobs));
                break;
            }
            case ST_DX: {
                const int mt = st.group ? mac_threads() : 256;  // pipelined chunks: beside transform CTAs
                CU(launch(k_diagx, dim3(NPOLY / mt, 1, st.njobs), mt, 0, s, h->hctx, (const DXJob*)st.djobs));
                break;
            }
            case ST_KF:
                CU(launch(k_ksfused, dim3(CL, st.gy, st.njobs), CNT, KF_SMEM, s, h->hctx, h->kfront, (const KFJob*)st.djobs));
                break;
            case ST_MEMSET:
                CU(cudaMemsetAsync(st.out, 0, st.bytes, s));
                break;
            case ST_ADD:
                CU(launch(k_addmod, dim3(NPOLY / 256, st.rows, st.njobs), 256, 0, s, h->hctx, (const AddJob*)st.djobs, st.gy));
                break;
            case ST_FOLD:
                // k_foldchain never triggers its dependents early: the next
                // launch starts when the chain (which spins on grid barriers,
                // all clusters co-resident) is complete
                CU(launch_cl(k_foldchain, FC_CL, st.fc.D * FC_CL, CNT, CL_SPREAD_SMEM, s, h->hctx, st.fc));
                break;
            case ST_I2: {
                Intt2Jobs jj;
                memset(&jj, 0, sizeof jj);
                memcpy(jj.j, st.i2jobs.data(), st.i2jobs.size() * sizeof(Intt2Job));
                const int n = (int)st.i2jobs.size();
                const bool ksfin = st.i2jobs[0].j[0].ld == LD_KSFIN;
                if (n <= g_i2_16) {  // one 16-CTA cluster per job (a prime per 8 CTAs)
                    if (ksfin) CU(launch_cl(k_cl16_intt2<LD_KSFIN>, 16, n * 16, CNT, CL_SPREAD_SMEM, s, h->hctx, jj));
                    else CU(launch_cl(k_cl16_intt2<LD_RED>, 16, n * 16, CNT, CL_SPREAD_SMEM, s, h->hctx, jj));
                } else if (ksfin) {
                    CU(launch(k_cl_intt2<LD_KSFIN>, n * CL, 2 * CNT, CL_SPREAD_SMEM, s, h->hctx, jj));
                } else {
                    CU(launch(k_cl_intt2<LD_RED>, n * CL, 2 * CNT, CL_SPREAD_SMEM, s, h->hctx, jj));
                }
                break;
            }
        }
        CU(cudaGetLastError());
    }
    return HC_OK;
}

// Steps of one nonzero group are independent: fork them onto side streams
// (parallel branches under graph capture) and join back on `s`.
static int enqueue(const hc_ctx* h, const Schedule& S, cudaStream_t s) {
    const size_t n = S.steps.size();
    for (size_t i = 0; i < n;) {
        size_t e = i + 1;
        if (S.steps[i].group)
            while (e < n && S.steps[e].group == S.steps[i].group) e++;
        if (e - i == 1) {
            int rc = enqueue_step(h, S.steps[i], s);
            if (rc) return rc;
        } else {
            CU(cudaEventRecord(h->ev_fork, s));
            size_t nb = std::min<size_t>(e - i, 4);
            for (size_t k = i; k < e; k++)
                if (S.steps[k].lane >= 0) nb = std::max<size_t>(nb, std::min(4, S.steps[k].lane + 1));
            for (size_t b = 0; b < nb; b++) CU(cudaStreamWaitEvent(h->side[b], h->ev_fork, 0));
            for (size_t k = i; k < e; k++) {
                const int lane = S.steps[k].lane >= 0 ? S.steps[k].lane : (int)(k - i);
                int rc = enqueue_step(h, S.steps[k], h->side[lane % 4]);
                if (rc) return rc;
            }
            for (size_t b = 0; b < nb; b++) {
                CU(cudaEventRecord(h->ev_join[b], h->side[b]));
                CU(cudaStreamWaitEvent(s, h->ev_join[b], 0));
            }
        }
        i = e;
    }
    return HC_OK;
}

static int count_launches(const Schedule& S) {
    int c = 0;
    for (const Step& st : S.steps) c += st.kind != ST_MEMSET;
    return c;
}

static int run_now(hc_ctx* h, const Schedule& S) {
    int rc = enqueue(h, S, h->stream);
    if (rc) return rc;
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

static int capture(hc_ctx* h, Schedule& S) {
    cudaGraph_t g = nullptr;
    CU(cudaDeviceSynchronize());  // job/pointer arrays fully uploaded
    CU(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    int rc = enqueue(h, S, h->stream);
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (rc) {
        if (g) cudaGraphDestroy(g);
        return rc;
    }
    if (e != cudaSuccess) return fail(HC_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&S.exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HC_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    S.launches = count_launches(S);
    return HC_OK;
}

// ---------------------------------------------------------------------------
// Comp plan (compress.py:198-367 on the BGV semantics of bgv.py:579-770)
// ---------------------------------------------------------------------------
// The plan's plaintexts (pack masks, diagonals, output mask), reference
// counted: a plan built with hc_plan_shared points at another context's
// (config 5: one database, many queries with their own keys).
struct PlainBufs {
    u64* mask = nullptr;   // [2][4][n]
    u64* diag = nullptr;   // [blocks of the plan's range][s_pad][3][n]
    u64* omask = nullptr;  // [2][n]
    ~PlainBufs() {
        cudaFree(mask);
        cudaFree(diag);
        cudaFree(omask);
    }
};
struct Plan {
    long long N = 0;
    int s = 0, s_pad = 0, baby = 0, giant = 0, m = 0, F = 0, CB = 0, ncopy = 1;
    long long B = 0, C = 0;
    int D1 = 0, D2 = 0;
    bool masked = false;  // comp_masked plan (row-1 diagonals scaled by the DB)
    // block range the plan covers (hc_plan_range; the whole matrix otherwise):
    // diagonals of blocks [rb0, rb1), input ciphertexts [rc0, rc1)
    long long rb0 = 0, rb1 = 0, rc0 = 0, rc1 = 0;
    bool full_range() const { return rb0 == 0 && rb1 == B; }
    std::shared_ptr<PlainBufs> plain;
    std::vector<int> fold;
    std::vector<uint8_t> live;      // [B][s_pad]
    std::vector<uint8_t> acc_live;  // [giant]
    long long live_count = 0;
    // Galois elements
    uint32_t t_col = 0;
    std::vector<uint32_t> t_baby, t_giant, t_fold;
    // device buffers
    std::vector<void*> allocs;
    u64 *cv = nullptr, *cd = nullptr, *mask = nullptr, *diag = nullptr, *omask = nullptr;
    // per-chunk scratch of the block segment (S1..S10); two sets when wide
    // chunks are pipelined (chunk c uses set c % 2, see build_partial)
    struct Scratch {
        u64 *ecor = nullptr, *rc1raw = nullptr, *pn = nullptr, *rc0n = nullptr, *dnttR = nullptr;
        u64 *U = nullptr, *Ucoef = nullptr, *dnttB = nullptr, *ROT = nullptr, *Eslot = nullptr;
        uint16_t *digR = nullptr, *digU = nullptr;
    } scr[4];
    int nsets = 1;
    u64* PX = nullptr;
    u64 *A0 = nullptr, *A1 = nullptr, *A1coef = nullptr, *dnttG = nullptr, *RES = nullptr;
    u64 *rc1coef = nullptr, *dnttF = nullptr, *corr = nullptr, *OUT = nullptr, *ACC = nullptr;
    uint16_t *digG = nullptr, *digF = nullptr;
    u64* uin = nullptr;  // hc_comp_packed: caller's pack_pair outputs u_t, [B][2][3][n] at level 2
    // hc_comp_mixed: inputs at levels (ld, lv), pack_pair on the device
    int mix_ld = -1, mix_lv = -1, mix_mask = -1;
    u64* ans_pt = nullptr;  // hc_answer_db: mask plaintexts [C][ans_level+1][n]
    uint32_t* ans_db = nullptr;  // hc_answer_db: the database mod p
    int ans_level = -1;
    u64 *mix_cd = nullptr, *mix_cv = nullptr, *mix_pt = nullptr, *mix_buf = nullptr, *mix_mcorr = nullptr;
    uint16_t* mix_dig = nullptr;
    std::unique_ptr<Schedule> full, fin, full_u, full_mix;
    std::map<std::pair<long long, long long>, std::unique_ptr<Schedule>> partials;
    ~Plan() {
        full.reset();
        fin.reset();
        full_u.reset();
        full_mix.reset();
        partials.clear();
        for (void* p : allocs) cudaFree(p);
    }
    size_t px_words() const { return (size_t)2 * giant * 2 * 2 * NPOLY; }
};

template <typename T>
static int palloc(Plan& P, T** ptr, size_t count) {
    void* d = nullptr;
    CU(cudaMalloc(&d, count * sizeof(T)));
    P.allocs.push_back(d);
    *ptr = (T*)d;
    return HC_OK;
}

static int bsgs_shape(int s, int* baby, int* giant, int* s_pad) {
    int sp = 1;
    while (sp < s) sp <<= 1;  // 1 << (s-1).bit_length()
    int bl = 0;
    while ((1 << bl) <= 2 * sp) bl++;  // (2*s_pad).bit_length()
    double log_target = (bl - 1) / 2.0;
    int b = 1 << (int)log_target;
    b = std::min(std::max(b, 1), sp);
    *baby = b;
    *giant = sp / b;
    *s_pad = sp;
    return 0;
}

static uint32_t rot_t(long long r, int n) {
    const long long two_n = 2LL * n;
    long long t = 1, b = 3, e = r;
    while (e) {
        if (e & 1) t = t * b % two_n;
        b = b * b % two_n;
        e >>= 1;
    }
    return (uint32_t)t;
}

static const DevKey* need_key(hc_ctx* h, uint32_t t) {
    auto it = h->keys.find(t);
    return it == h->keys.end() ? nullptr : &it->second;
}

// b0 < 0: the whole matrix; else blocks [b0, b1) only (a rank's shard).
// share: take the plaintexts of another context's plan (same chain, N, s).
static int plan_impl(hc_ctx* h, int64_t N, int s, int chunk_blocks, const uint64_t* db, int64_t b0 = -1,
                     int64_t b1 = -1, const Plan* share = nullptr) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    if (h->L < 3) return fail(HC_ERR_ARG, "Comp needs max_level >= 3 (SURVEY F3)");
    const int n = NPOLY, m = n / 2;
    if (N < 1 || s < 1) return fail(HC_ERR_ARG, "N and s must be positive");
    if ((u64)N >= h->p) return fail(HC_ERR_ARG, "p must exceed N (compress.py:52-53)");
    if (2 * s > n) return fail(HC_ERR_ARG, "2s must fit the slots of one ciphertext");
    CU(cudaSetDevice(h->dev));
    h->plan.reset();
    std::unique_ptr<Plan> P(new Plan());
    P->N = N;
    P->s = s;
    P->m = m;
    bsgs_shape(s, &P->baby, &P->giant, &P->s_pad);
    P->B = (N + m - 1) / m;
    P->C = (P->B + 1) / 2;
    if (b0 < 0) {
        b0 = 0;
        b1 = P->B;
    }
    if (b0 > b1 || b1 > P->B) return fail(HC_ERR_ARG, "block range out of bounds");
    P->rb0 = b0;
    P->rb1 = b1;
    P->rc0 = b0 / 2;
    P->rc1 = (b1 + 1) / 2;
    for (int step = P->s_pad; step < m; step <<= 1) P->fold.push_back(step);
    P->F = (int)P->fold.size();
    P->D1 = h->digits[1];
    P->D2 = h->digits[2];
    // wide chunks: 64 blocks, 128 from 256 blocks on (launches twice the size,
    // still >= 2 chunks to pipeline: N=2^20 s=16 5.26 -> 5.11 ms, N=2^22 20.4 -> 20.0)
    P->CB = chunk_blocks > 0 ? chunk_blocks : (int)std::min<long long>(P->B, P->B >= 256 ? 128 : 64);
    // k_diagx sums CB*baby Montgomery products (each < q^2) before one REDC,
    // which needs the sum < q * 2^64, i.e. at most 1024 terms for 54-bit q
    P->CB = std::max(1, std::min(P->CB, 1024 / std::max(1, P->baby)));
    P->ncopy = (int)std::max<long long>(1, (P->B * P->baby + 999) / 1000);
    // live diagonals: only the last block can have all-zero diagonals
    P->live.assign((size_t)P->B * P->s_pad, 1);
    {
        const long long t = P->B - 1;
        for (int g = 0; g < P->giant; g++)
            for (int b = 0; b < P->baby; b++) {
                bool any = false;
                for (int pos = 0; pos < m && !any; pos++) {
                    int row = ((pos - g * P->baby) % P->s_pad + P->s_pad) % P->s_pad;
                    int col = (pos + b) % m;
                    any = row < s && t * m + col + 1 <= N;
                }
                P->live[(size_t)t * P->s_pad + g * P->baby + b] = any;
            }
    }
    P->acc_live.assign(P->giant, 0);
    P->live_count = 0;
    for (long long t = 0; t < P->B; t++)
        for (int i = 0; i < P->s_pad; i++)
            if (P->live[(size_t)t * P->s_pad + i]) {
                P->acc_live[i / P->baby] = 1;
                P->live_count++;
            }
    if (!P->acc_live[0]) {
        bool any = false;
        for (int g = 0; g < P->giant; g++) any |= P->acc_live[g];
        if (!any) return fail(HC_ERR_ARG, "matrix plan had no nonzero diagonals");
    }
    // keys (plan_rotation_amounts, compress.py:87-100)
    P->t_col = 2 * n - 1;
    if (!need_key(h, P->t_col)) return fail(HC_ERR_KEY, "column-swap key was not declared at keygen");
    P->t_baby.assign(P->baby, 1);
    for (int b = 1; b < P->baby; b++) {
        P->t_baby[b] = rot_t(b, n);
        if (!need_key(h, P->t_baby[b])) return fail(HC_ERR_KEY, "rotation by " + std::to_string(b) + " was not declared at keygen");
    }
    P->t_giant.assign(P->giant, 1);
    for (int g = 1; g < P->giant; g++) {
        long long r = ((long long)g * P->baby) % m;
        P->t_giant[g] = rot_t(r, n);
        if (P->acc_live[g] && r != 0 && !need_key(h, P->t_giant[g]))
            return fail(HC_ERR_KEY, "rotation by " + std::to_string(r) + " was not declared at keygen");
    }
    for (int a : P->fold) {
        P->t_fold.push_back(rot_t(a, n));
        if (!need_key(h, P->t_fold.back())) return fail(HC_ERR_KEY, "rotation by " + std::to_string(a) + " was not declared at keygen");
    }

    const size_t NB = NPOLY;
    const int CB = P->CB, bm1 = std::max(P->baby - 1, 0), G = P->giant;
    int rc = 0;
#define PA(ptr, cnt)                    \
    do {                                \
        rc = palloc(*P, &(ptr), (cnt)); \
        if (rc) return rc;              \
    } while (0)
    // inputs and diagonals of the plan's block range only
    const size_t ncts = (size_t)std::max<long long>(1, P->rc1 - P->rc0);
    const size_t nblk = (size_t)std::max<long long>(1, P->rb1 - P->rb0);
    PA(P->cv, ncts * 2 * 4 * NB);
    PA(P->cd, ncts * 2 * 4 * NB);
    if (share) {
        P->plain = share->plain;
    } else {
        P->plain = std::make_shared<PlainBufs>();
        CU(cudaMalloc(&P->plain->mask, (size_t)2 * 4 * NB * 8));
        CU(cudaMalloc(&P->plain->diag, nblk * P->s_pad * 3 * NB * 8));
        CU(cudaMalloc(&P->plain->omask, (size_t)2 * NB * 8));
    }
    P->mask = P->plain->mask;
    P->diag = P->plain->diag;
    P->omask = P->plain->omask;
    // wide chunks (throughput regime) pipeline over up to four scratch sets
    // when the range has several: chunk c+1's transforms overlap chunk c's
    // memory-bound MACs.  N=2^20, s=16: 5.67 ms (one set) -> 5.39 (two) ->
    // 5.28 (four); N=2^22, s=16: 22.19 -> 20.92 -> 20.61 ms
    // (profiles/r02_ab_chunk_pipelining*.txt).  HC_CHUNK_LANES=1: one set.
    {
        static int chunk_lanes = -1;  // HC_CHUNK_LANES: graph lanes for wide chunks (0/1: none, <= 4)
        if (chunk_lanes < 0) {
            const char* e = getenv("HC_CHUNK_LANES");
            chunk_lanes = e ? std::max(1, std::min(4, atoi(e))) : 4;
        }
        const long long nchunks = (P->rb1 - P->rb0 + CB - 1) / CB;
        P->nsets = (chunk_lanes > 1 && CB > g_lane_max_blocks && nchunks >= 2 && nchunks <= 64)
                       ? (int)std::min<long long>(chunk_lanes, nchunks) : 1;
    }
    for (int si = 0; si < P->nsets; si++) {
        Plan::Scratch& X = P->scr[si];
        PA(X.ecor, (size_t)CB * 4 * 3 * NB);
        PA(X.rc1raw, (size_t)CB * 3 * NB);
        PA(X.pn, (size_t)CB * 2 * 3 * NB);
        PA(X.rc0n, (size_t)CB * 3 * NB);
        PA(X.digR, (size_t)CB * P->D2 * NB);
        PA(X.dnttR, (size_t)CB * P->D2 * 3 * NB);
        PA(X.U, (size_t)CB * 2 * 3 * NB);
        PA(X.Ucoef, (size_t)CB * 3 * NB);
        PA(X.digU, (size_t)CB * 2 * P->D2 * NB);
        PA(X.dnttB, (size_t)std::max(1, CB * bm1) * P->D2 * 3 * NB);
        PA(X.ROT, (size_t)std::max(1, CB * bm1) * 2 * 3 * NB);
        PA(X.Eslot, (size_t)CB * P->baby * G * 2 * 2 * NB);
    }
    PA(P->PX, P->px_words());
    PA(P->A0, (size_t)G * 2 * NB);
    PA(P->A1, (size_t)2 * NB);
    PA(P->A1coef, (size_t)G * 2 * NB);
    PA(P->digG, (size_t)G * 2 * P->D1 * NB);
    PA(P->dnttG, (size_t)G * P->D1 * 2 * NB);
    PA(P->RES, (size_t)2 * 2 * 2 * NB);
    PA(P->rc1coef, (size_t)2 * NB);
    PA(P->digF, (size_t)2 * P->D1 * NB);
    PA(P->dnttF, (size_t)P->D1 * 2 * NB);
    PA(P->corr, (size_t)2 * NB);
    PA(P->OUT, (size_t)2 * NB);
    PA(P->ACC, (size_t)3 * 2 * 2 * NB + 8);  // three [poly][prime][n] buffers (folds rotate) + k_foldchain's barrier counter
#undef PA

    // ---- plaintexts on device (K6) ----
    if (!share) {
        std::vector<PJob> pj;
        PJob j{};
        j.kind = PT_TOP; j.level = 3; j.out = P->mask; pj.push_back(j);
        j.kind = PT_BOT; j.level = 3; j.out = P->mask + 4 * NB; pj.push_back(j);
        j.kind = PT_OUTMASK; j.level = 1; j.out = P->omask; pj.push_back(j);
        for (long long t = P->rb0; t < P->rb1; t++)
            for (int g = 0; g < P->giant; g++)
                for (int b = 0; b < P->baby; b++) {
                    int i = g * P->baby + b;
                    if (!P->live[(size_t)t * P->s_pad + i]) continue;
                    PJob d{};
                    d.kind = PT_DIAG; d.t = (int)t; d.g = g; d.b = b; d.level = 2;
                    d.out = P->diag + ((size_t)(t - P->rb0) * P->s_pad + i) * 3 * NB;
                    pj.push_back(d);
                }
        PlanShape S{N, s, P->s_pad, P->baby, m, nullptr};
        if (db) {
            std::vector<uint32_t> dbv((size_t)N);
            for (long long i = 0; i < N; i++) {
                if (db[i] >= h->p) return fail(HC_ERR_ARG, "database values must be reduced mod p");
                dbv[i] = (uint32_t)db[i];
            }
            uint32_t* ddb = nullptr;
            rc = palloc(*P, &ddb, (size_t)N);
            if (rc) return rc;
            CU(cudaMemcpy(ddb, dbv.data(), (size_t)N * 4, cudaMemcpyHostToDevice));
            S.db = ddb;
            P->masked = true;
        }
        PJob* dj = nullptr;
        const size_t maxb = 65535;
        CU(cudaMalloc(&dj, pj.size() * sizeof(PJob)));
        CU(cudaMemcpy(dj, pj.data(), pj.size() * sizeof(PJob), cudaMemcpyHostToDevice));
        for (size_t off = 0; off < pj.size(); off += maxb) {
            int cnt = (int)std::min(maxb, pj.size() - off);
            k_plain<<<cnt, NT, 2 * NPOLY * 8, h->stream>>>(h->hctx, dj + off, S);
        }
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        cudaFree(dj);
        if (e != cudaSuccess) return fail(HC_ERR_CUDA, std::string("plaintext generation: ") + cudaGetErrorString(e));
    }
    h->plan = std::move(P);
    return HC_OK;
}

extern "C" int hc_plan(hc_ctx* h, int64_t N, int s, int chunk_blocks) { return plan_impl(h, N, s, chunk_blocks, nullptr); }

extern "C" int hc_plan_range(hc_ctx* h, int64_t N, int s, int chunk_blocks, int64_t b0, int64_t b1) {
    if (b0 < 0) return fail(HC_ERR_ARG, "block range out of bounds");
    return plan_impl(h, N, s, chunk_blocks, nullptr, b0, b1);
}

extern "C" int hc_plan_shared(hc_ctx* h, const hc_ctx* src, int chunk_blocks) {
    if (!h || !src) return fail(HC_ERR_ARG, "null context");
    if (!src->plan) return fail(HC_ERR_STATE, "the source context has no plan");
    const Plan& S = *src->plan;
    if (!S.full_range() || S.masked) return fail(HC_ERR_ARG, "only whole-matrix hint-path plans are shared");
    if (src->dev != h->dev || src->L != h->L || src->p != h->p) return fail(HC_ERR_MISMATCH, "contexts differ");
    for (int k = 0; k <= h->L; k++)
        if (src->hctx.pc[k].q != h->hctx.pc[k].q) return fail(HC_ERR_MISMATCH, "contexts have different chains");
    return plan_impl(h, S.N, S.s, chunk_blocks, nullptr, -1, -1, &S);
}

extern "C" int hc_plan_masked(hc_ctx* h, int64_t N, int s, int chunk_blocks, const uint64_t* db_mod_p) {
    if (!db_mod_p) return fail(HC_ERR_ARG, "null database");
    return plan_impl(h, N, s, chunk_blocks, db_mod_p);
}

extern "C" int hc_plan_info(const hc_ctx* h, int64_t* info) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "no plan");
    const Plan& P = *h->plan;
    info[0] = P.B;
    info[1] = P.C;
    info[2] = P.baby;
    info[3] = P.giant;
    info[4] = P.F;
    info[5] = P.s_pad;
    info[6] = P.live_count;
    // kernel launches per Comp: the one-graph path, else (sharded mode,
    // hc_comp_partial + hc_comp_finish) the partial graphs this rank has
    // captured plus the root's finish graph; -1 before any capture
    long long launches = -1;
    if (P.full) {
        launches = P.full->launches;
    } else if (!P.partials.empty() || P.fin) {
        launches = P.fin ? P.fin->launches : 0;
        for (const auto& kv : P.partials) launches += kv.second->launches;
    }
    info[7] = launches;
    return HC_OK;
}

extern "C" int64_t hc_partial_words(const hc_ctx* h) {
    if (!h || !h->plan) return -1;
    return (int64_t)h->plan->px_words();
}

// the level-2 ciphertext multiplied by diagonal (t, g, b): u_t for b = 0,
// the baby rotation ROT[t][b] otherwise
static const u64* rot_src(const Plan& P, const Plan::Scratch& X, const u64* U, int tl, int b, int poly) {
    const size_t NB = NPOLY;
    return b == 0 ? U + ((size_t)tl * 2 + poly) * 3 * NB
                  : X.ROT + (((size_t)tl * (P.baby - 1) + (b - 1)) * 2 + poly) * 3 * NB;
}
// correction slot of product (tl, b) for accumulator (g, poly): [2 primes][n]
static u64* eslot(const Plan& P, const Plan::Scratch& X, int tl, int b, int g, int poly) {
    const size_t NB = NPOLY;
    return X.Eslot + ((((size_t)tl * P.baby + b) * P.giant + g) * 2 + poly) * 2 * NB;
}

// HC_KSFUSED=1: the throughput regime's key switches as k_ksfused (one kernel
// per rotation, no digit NTTs in HBM) instead of digit-NTT launches +
// k_ksmac_mb.  Off by default: the transforms are instruction-bound, the
// fused form executes the same butterflies plus the MACs on the same pipes,
// while the multi-launch form hides its memory-bound MACs under another
// chunk's transforms (measured: DESIGN.md section 9)
static int g_ksfused = -1;
static bool ksfused_on() {
    if (g_ksfused < 0) {
        const char* e = getenv("HC_KSFUSED");
        g_ksfused = (e && e[0] == '1') ? 1 : 0;
    }
    return g_ksfused == 1;
}
extern "C" int hc_set_ksfused(int on) {
    g_ksfused = on ? 1 : 0;
    return HC_OK;
}

// Steps S1..S10 for blocks [b0, b1): pack_pair (compress.py:338-367), baby
// rotations and the diagonal products (compress.py:286-297), accumulated
// into the partial PX = [E | X].  Blocks are independent until the
// accumulation, so each chunk runs as up to 4 parallel lanes (graph
// branches) of per-block pipelines S1..S9, joined by S10.  `from_u`: the
// pack_pair outputs u_t are the caller's (P.uin, level 2; the mixed-level
// answer() inputs), so S1..S4 are skipped.
static int build_partial(hc_ctx* h, Plan& P, long long b0, long long b1, Schedule& S, bool from_u = false) {
    const size_t NB = NPOLY;
    const int D2 = P.D2, baby = P.baby, G = P.giant, sp = P.s_pad;
    const DevKey* kcol = need_key(h, P.t_col);
    int rc;
    add_memset(S, P.PX, P.px_words() * 8);
    // pipelined wide chunks: chunk i on graph lane i % nsets with scratch set
    // i % nsets, the lanes' diagonal MACs adding into PX with atomics (words
    // stay < nchunks * q <= 64 q < 2^60; every consumer reduces them)
    const long long nchunks = (b1 - b0 + P.CB - 1) / P.CB;
    const bool pipe = P.nsets >= 2 && nchunks >= 2;
    if (pipe) S.par_begin();
    for (long long c0 = b0; c0 < b1; c0 += P.CB) {
        const int cb = (int)std::min<long long>(P.CB, b1 - c0);
        const int ci = (int)((c0 - b0) / P.CB);
        const Plan::Scratch& X = P.scr[pipe ? ci % P.nsets : 0];
        if (pipe) S.cur_lane = ci % P.nsets;
        const u64* Ub = from_u ? P.uin + (size_t)c0 * 2 * 3 * NB : X.U;  // u_t of chunk block tl at Ub[tl]
        // S1..S6 (pack, u = P + rot_col(R), hoisted baby INTT + digits) run as
        // one stream over the chunk (narrow levels may use cluster transforms);
        // the wide baby segment S7 (digit NTTs) -> S8 (MAC) -> S9 (diagonal
        // INTTs) runs as up to 4 parallel lanes of blocks so the memory-bound
        // MAC of one block overlaps the NTTs of the next.
        std::vector<XJob> s1, s2, s3, s5;
        std::vector<CJob> s2c, s6;
        std::vector<MJob> s4;
        std::vector<std::vector<XJob>> s7(cb), s9(cb);
        std::vector<std::vector<MJob>> s8(cb);
        // throughput regime: each key switch (digit NTTs + key MAC) as one
        // fused job (k_ksfused) instead of S3 -> S4 and S7 -> S8
        const bool fusedks = ksfused_on() && cb > g_lane_max_blocks;
        std::vector<KFJob> kf3, kf7;
        for (int tl = 0; tl < cb; tl++) {
                const long long t = c0 + tl;
                const long long src = t / 2;
                const int par = (int)(t % 2);
                const u64* mk = P.mask + (size_t)par * 4 * NB;
                const u64* cv = P.cv + (size_t)(src - P.rc0) * 2 * 4 * NB;
                const u64* cd = P.cd + (size_t)(src - P.rc0) * 2 * 4 * NB;
                // even block: u = mp(cv, top) + rot_col(mp(cd, top)); odd: rot_col(mp(cv, bot)) + mp(cd, bot)
                const u64* ctP = par == 0 ? cv : cd;
                const u64* ctR = par == 0 ? cd : cv;
                u64* ecor = X.ecor + (size_t)tl * 4 * 3 * NB;  // [P0,P1,R0,R1][3][n]
                if (!from_u) {
                // S1: the pack mul_plains' dropped-prime INTTs (+ modulus-switch
                //     correction) and R.c1's kept-prime INTTs
                for (int mm = 0; mm < 2; mm++)
                    for (int poly = 0; poly < 2; poly++) {
                        const u64* ct = mm == 0 ? ctP : ctR;
                        XJob j{};
                        j.dir = 1; j.k = 3; j.ld = LD_MONT; j.ep = EP_RESCALE; j.level = 3;
                        j.a = ct + ((size_t)poly * 4 + 3) * NB;
                        j.b = mk + 3 * NB;
                        j.out = ecor + (size_t)(mm * 2 + poly) * 3 * NB;
                        j.ostride = NB;
                        s1.push_back(j);
                    }
                for (int k = 0; k < 3; k++) {
                    XJob j{};
                    j.dir = 1; j.k = k; j.ld = LD_MONT; j.ep = EP_STORE;
                    j.a = ctR + ((size_t)1 * 4 + k) * NB;
                    j.b = mk + (size_t)k * NB;
                    j.out = X.rc1raw + ((size_t)tl * 3 + k) * NB;
                    s1.push_back(j);
                }
                // S2: NTT of corrections + plaintext-product combine
                for (int which = 0; which < 3; which++) {  // P.c0, P.c1, R.c0
                    const int mm = which < 2 ? 0 : 1, poly = which < 2 ? which : 0;
                    const u64* ct = mm == 0 ? ctP : ctR;
                    for (int k = 0; k < 3; k++) {
                        XJob j{};
                        j.dir = 0; j.k = k; j.ld = LD_U64; j.ep = EP_ADDMONT;
                        j.a = ecor + ((size_t)(mm * 2 + poly) * 3 + k) * NB;
                        j.ea = ct + ((size_t)poly * 4 + k) * NB;
                        j.eb = mk + (size_t)k * NB;
                        j.out = which < 2 ? X.pn + (((size_t)tl * 2 + poly) * 3 + k) * NB : X.rc0n + ((size_t)tl * 3 + k) * NB;
                        s2.push_back(j);
                    }
                }
                {
                    CJob c{};
                    c.level = 2; c.mode = 0;
                    c.x = X.rc1raw + (size_t)tl * 3 * NB;
                    c.xadd = ecor + (size_t)3 * 3 * NB;
                    c.xstride = NB;
                    c.gal = kcol->gal;
                    c.dig = X.digR + (size_t)tl * D2 * NB;
                    s2c.push_back(c);
                }
                // S3/S4: column-swap key switch of R, u = P + rot_col(R)
                for (int jj = 0; jj < D2; jj++)
                    for (int k = 0; k < 3; k++) {
                        XJob j{};
                        j.dir = 0; j.k = k; j.ld = LD_DIG; j.ep = EP_STORE_LAZY;  // feeds k_ksmac only
                        j.a = (const u64*)(X.digR + ((size_t)tl * D2 + jj) * NB);
                        j.out = X.dnttR + (((size_t)tl * D2 + jj) * 3 + k) * NB;
                        s3.push_back(j);
                    }
                {
                    MJob mj{};
                    mj.level = 2; mj.nterm = 1;
                    mj.t[0].dntt = X.dnttR + (size_t)tl * D2 * 3 * NB;
                    mj.t[0].key = kcol->key;
                    mj.t[0].c0src = X.rc0n + (size_t)tl * 3 * NB;
                    mj.t[0].perm = kcol->perm;
                    mj.add0 = X.pn + ((size_t)tl * 2 + 0) * 3 * NB;
                    mj.add1 = X.pn + ((size_t)tl * 2 + 1) * 3 * NB;
                    mj.out0 = X.U + ((size_t)tl * 2 + 0) * 3 * NB;
                    mj.out1 = X.U + ((size_t)tl * 2 + 1) * 3 * NB;
                    s4.push_back(mj);
                    if (fusedks) {
                        KFJob f{};
                        f.level = 2; f.tinv = 1;  // digR is composed through the column swap's gather
                        f.dpos = X.digR + (size_t)tl * D2 * NB;
                        f.key = kcol->key;
                        f.perm = kcol->perm;
                        f.c0src = mj.t[0].c0src;
                        f.add0 = mj.add0; f.add1 = mj.add1;
                        f.out0 = mj.out0; f.out1 = mj.out1;
                        kf3.push_back(f);
                    }
                }
                }  // !from_u
                // S5..S8: baby-step rotations of u (hoisted INTT + CRT digits)
                if (baby > 1) {
                    for (int k = 0; k < 3; k++) {
                        XJob j{};
                        j.dir = 1; j.k = k; j.ld = LD_U64; j.ep = EP_STORE;
                        j.a = Ub + (((size_t)tl * 2 + 1) * 3 + k) * NB;
                        j.out = X.Ucoef + ((size_t)tl * 3 + k) * NB;
                        s5.push_back(j);
                    }
                    CJob c{};
                    c.level = 2; c.mode = 1;
                    c.x = X.Ucoef + (size_t)tl * 3 * NB;
                    c.xstride = NB;
                    c.dig = X.digU + (size_t)tl * 2 * D2 * NB;
                    s6.push_back(c);
                    for (int b = 1; b < baby; b++) {
                        const DevKey* kb = need_key(h, P.t_baby[b]);
                        const size_t rb = (size_t)tl * (baby - 1) + (b - 1);
                        for (int jj = 0; jj < D2; jj++)
                            for (int k = 0; k < 3; k++) {
                                XJob j{};
                                j.dir = 0; j.k = k; j.ld = LD_DIGGAL; j.ep = EP_STORE_LAZY;  // feeds k_ksmac only
                                j.a = (const u64*)(X.digU + ((size_t)tl * 2 * D2 + jj) * NB);
                                j.b = (const u64*)(X.digU + ((size_t)tl * 2 * D2 + D2 + jj) * NB);
                                j.gal = kb->gal;
                                j.out = X.dnttB + ((rb * D2 + jj) * 3 + k) * NB;
                                s7[tl].push_back(j);
                            }
                        MJob mj{};
                        mj.level = 2; mj.nterm = 1;
                        mj.t[0].dntt = X.dnttB + rb * D2 * 3 * NB;
                        mj.t[0].key = kb->key;
                        mj.t[0].c0src = Ub + ((size_t)tl * 2 + 0) * 3 * NB;
                        mj.t[0].perm = kb->perm;
                        mj.out0 = X.ROT + (rb * 2 + 0) * 3 * NB;
                        mj.out1 = X.ROT + (rb * 2 + 1) * 3 * NB;
                        s8[tl].push_back(mj);
                        if (fusedks) {
                            KFJob f{};
                            f.level = 2; f.tinv = kb->tinv;
                            f.dpos = X.digU + (size_t)tl * 2 * D2 * NB;
                            f.dneg = X.digU + ((size_t)tl * 2 * D2 + D2) * NB;
                            f.key = kb->key;
                            f.perm = kb->perm;
                            f.c0src = mj.t[0].c0src;
                            f.out0 = mj.out0; f.out1 = mj.out1;
                            kf7.push_back(f);
                        }
                    }
                }
                // S9: dropped-prime half of each diagonal product: INTT + the
                //     (r, d) integers of its rescale correction into the
                //     block's slot of Eslot (summed and multiplied by S10)
                for (int g = 0; g < G; g++)
                    for (int b = 0; b < baby; b++) {
                        const int i = g * baby + b;
                        if (!P.live[(size_t)t * sp + i]) continue;
                        const u64* dg = P.diag + ((size_t)(t - P.rb0) * sp + i) * 3 * NB;
                        for (int poly = 0; poly < 2; poly++) {
                            XJob j{};
                            j.dir = 1; j.k = 2; j.ld = LD_MONT; j.ep = EP_RESCALE_RD; j.level = 2;
                            j.a = rot_src(P, X, Ub, tl, b, poly) + 2 * NB;
                            j.b = dg + 2 * NB;
                            j.out = eslot(P, X, tl, b, g, poly);
                            j.ostride = NB;
                            s9[tl].push_back(j);
                        }
                    }
        }
        // S10 job lists for the blocks [tl0, tl1) of the chunk; `atomic`: the
        // lanes' per-block launches run concurrently and add their sums into
        // PX with atomics (PX words stay < 4q: every consumer reduces them)
        auto build_dx = [&](int tl0, int tl1, bool atomic) -> int {
            std::vector<DXJob> dx;
            std::vector<const u64*> srcs, dgs, ess;
            struct Rng { size_t off, cnt; int g, poly; };
            std::vector<Rng> rngs;
            for (int g = 0; g < G; g++)
                for (int poly = 0; poly < 2; poly++) {
                    size_t off = srcs.size();
                    for (int tl = tl0; tl < tl1; tl++) {
                        const long long t = c0 + tl;
                        for (int b = 0; b < baby; b++) {
                            const int i = g * baby + b;
                            if (!P.live[(size_t)t * sp + i]) continue;
                            srcs.push_back(rot_src(P, X, Ub, tl, b, poly));
                            dgs.push_back(P.diag + ((size_t)(t - P.rb0) * sp + i) * 3 * NB);
                            ess.push_back(eslot(P, X, tl, b, g, poly));
                        }
                    }
                    rngs.push_back({off, srcs.size() - off, g, poly});
                }
            if (srcs.empty()) return HC_OK;
            const u64** dsrc = nullptr;
            const u64** ddg = nullptr;
            const u64** des = nullptr;
            CU(cudaMalloc(&dsrc, srcs.size() * sizeof(u64*)));
            S.allocs.push_back(dsrc);
            CU(cudaMalloc(&ddg, dgs.size() * sizeof(u64*)));
            S.allocs.push_back(ddg);
            CU(cudaMalloc(&des, ess.size() * sizeof(u64*)));
            S.allocs.push_back(des);
            CU(cudaMemcpy(dsrc, srcs.data(), srcs.size() * sizeof(u64*), cudaMemcpyHostToDevice));
            CU(cudaMemcpy(ddg, dgs.data(), dgs.size() * sizeof(u64*), cudaMemcpyHostToDevice));
            CU(cudaMemcpy(des, ess.data(), ess.size() * sizeof(u64*), cudaMemcpyHostToDevice));
            for (const Rng& r : rngs) {
                if (!r.cnt) continue;
                DXJob d{};
                d.nterm = (int)r.cnt;
                d.level = 2;
                d.atomic = atomic ? 1 : 0;
                d.src = dsrc + r.off;
                d.dg = ddg + r.off;
                d.es = des + r.off;
                d.X = P.PX + (size_t)1 * G * 2 * 2 * NB + (((size_t)r.g * 2 + r.poly) * 2) * NB;
                d.E = P.PX + (((size_t)r.g * 2 + r.poly) * 2) * NB;
                dx.push_back(d);
            }
            return add_dx(S, dx, 2);
        };
        static int lane_dx = -1;  // HC_LANE_DX=0: one S10 launch after all lanes (A/B)
        if (lane_dx < 0) {
            const char* e = getenv("HC_LANE_DX");
            lane_dx = (e && e[0] == '0') ? 0 : 1;
        }
        bool lanes_dx = false;
        if (!from_u) {
        rc = add_xf(S, s1); if (rc) return rc;
        // S2 (P and R.c0 at level 2) is independent of S2c -> S3 (R.c1's
        // digits and their NTTs): at small chunks (latency regime) they run as
        // two graph branches joined before S4; wide chunks fill the GPU anyway
        const bool fork23 = cb <= g_lane_max_blocks;
        if (fork23) {
            S.par_begin();
            S.cur_lane = 0;
            S.cl_in_lane = true;
        }
        rc = add_xf(S, s2); if (rc) return rc;
        if (fork23) {
            S.cl_in_lane = false;
            S.cur_lane = 1;
        }
        rc = add_co(S, s2c); if (rc) return rc;
        if (!fusedks) { rc = add_xf(S, s3); if (rc) return rc; }
        if (fork23) {
            S.cur_lane = -1;
            S.par_end();
        }
        if (fusedks) rc = add_kf(S, kf3, 3);
        else rc = add_ma(S, s4, 3);
        if (rc) return rc;
        }  // !from_u
        rc = add_xf(S, s5); if (rc) return rc;
        rc = add_co(S, s6); if (rc) return rc;
        if (cb > g_lane_max_blocks || cb < 3) {  // lanes pay off from 3 blocks (measured)
            // one wide launch per segment over the chunk (throughput regime, or
            // too few blocks for lanes to overlap anything)
            std::vector<XJob> w7, w9;
            std::vector<MJob> w8;
            for (int tl = 0; tl < cb; tl++) {
                w7.insert(w7.end(), s7[tl].begin(), s7[tl].end());
                w8.insert(w8.end(), s8[tl].begin(), s8[tl].end());
                w9.insert(w9.end(), s9[tl].begin(), s9[tl].end());
            }
            if (fusedks) {
                rc = add_kf(S, kf7, 3); if (rc) return rc;
            } else {
                rc = add_xf(S, w7); if (rc) return rc;
                rc = add_ma(S, w8, 3); if (rc) return rc;
            }
            rc = add_xf(S, w9); if (rc) return rc;
        } else {
        const int nl = std::min(4, cb);
        if (nl > 1) S.par_begin();
        for (int lane = 0; lane < nl; lane++) {
            S.cur_lane = nl > 1 ? lane : -1;
            // per-lane diagonal MACs add into PX with atomics and no reduction
            // in between: only when this chunk is the range's only one, so PX
            // words stay below cb * q < 4q (< 2^56: the sharded uint64 reduce
            // of up to 255 partials is exact)
            lanes_dx = lane_dx && nl > 1 && b1 - b0 <= P.CB;
            for (int tl = lane; tl < cb; tl += nl) {
                rc = add_xf(S, s7[tl]); if (rc) return rc;
                rc = add_ma(S, s8[tl], 3); if (rc) return rc;
                rc = add_xf(S, s9[tl]); if (rc) return rc;
                if (lanes_dx) {  // this block's diagonal MAC inside its lane
                    rc = build_dx(tl, tl + 1, true);
                    if (rc) return rc;
                }
            }
        }
        S.cur_lane = -1;
        if (nl > 1) S.par_end();
        }
        // S10: per (g, poly): X += sum src * diag * q^-1 (kept primes) and
        //      E += sum of the chunk's correction slots
        if (!lanes_dx) {
            rc = build_dx(0, cb, pipe);
            if (rc) return rc;
        }
    }
    if (pipe) {
        S.cur_lane = -1;
        S.par_end();
    }
    return HC_OK;
}

static const KsSpec* upload_spec(Schedule& S, const KsSpec& spec, int* rc) {
    void* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(KsSpec));
    if (e == cudaSuccess) e = cudaMemcpy(d, &spec, sizeof(KsSpec), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        *rc = fail(HC_ERR_CUDA, std::string("spec upload: ") + cudaGetErrorString(e));
        return nullptr;
    }
    S.allocs.push_back(d);
    *rc = HC_OK;
    return (const KsSpec*)d;
}

// Tail: giant steps, folds and the output mask (compress.py:298-310), level 1.
// Key switches finish in the digit-NTT epilogue: each digit transform
// multiplies its output by its key digit and red.add's it into ACC (u64;
// at most (giant-1)*D_1 = 49 addends < 2^60, exact); the consumer's loader
// (LD_KSFIN) adds base + permuted c0 terms + red(ACC) and re-zeroes ACC.
//   T1   acc[g] = X[g] + NTT(E[g]) (c1 of g >= 1 in coefficient domain)
//   T3   giant digit NTTs (CRT/digit split in the loader, KSACC epilogue)
//   per fold f:
//     F1 two-prime INTT of res_f.c1 (k_cl_intt2: LD_KSFIN, side-stores
//        res_f.c1, CRT/digit split fused) + transform-less jobs
//        materialising res_f.c0
//     F3 fold digit NTTs (LD_DIGGAL -> EP_KSACC)
//   D1   INTT of res_F * mask at the dropped prime (LD_KSFIN * mask) + rescale
//   D2   NTT of the correction + res_F * mask * q^-1 at the kept prime
static int build_finish(hc_ctx* h, Plan& P, Schedule& S) {
    const size_t NB = NPOLY;
    const int G = P.giant, D1 = P.D1;
    const u64* E = P.PX;
    const u64* X = P.PX + (size_t)G * 2 * 2 * NB;
    auto ex = [&](const u64* base, int g, int poly, int k) { return base + (((size_t)g * 2 + poly) * 2 + k) * NB; };
    int rc;
    add_memset(S, P.ACC, ((size_t)3 * 2 * 2 * NB + 8) * 8);  // accumulators + k_foldchain's barrier counter
    // T1 (acc[g] c0 transforms; c1 of g >= 1 inverted on both primes with the
    // CRT digit split fused: k_cl_intt2)
    std::vector<XJob> t1;
    std::vector<Intt2Job> t1i;
    for (int g = 0; g < G; g++) {
        if (!P.acc_live[g]) continue;
        for (int k = 0; k < 2; k++) {
            XJob j{};
            j.dir = 0; j.k = k; j.ld = LD_RED; j.ep = EP_ADDRED;
            j.a = ex(E, g, 0, k);
            j.ea = ex(X, g, 0, k);
            j.out = P.A0 + ((size_t)g * 2 + k) * NB;
            t1.push_back(j);
            if (g == 0) {
                XJob c = j;
                c.a = ex(E, g, 1, k);
                c.ea = ex(X, g, 1, k);
                c.out = P.A1 + (size_t)k * NB;
                t1.push_back(c);
            }
        }
        if (g > 0) {
            Intt2Job ij{};
            for (int k = 0; k < 2; k++) {
                ij.j[k].dir = 1; ij.j[k].k = k; ij.j[k].ld = LD_RED; ij.j[k].ep = EP_STORE;
                ij.j[k].a = ex(X, g, 1, k);
            }
            ij.E = ex(E, g, 1, 0);
            ij.dig = P.digG + (size_t)g * 2 * D1 * NB;
            t1i.push_back(ij);
        }
    }
    // in sequence: two different cluster kernels running side by side slow
    // each other down (measured: 14.6 + 8.0 us in parallel vs 5.0 + 7.4)
    rc = add_xf(S, t1); if (rc) return rc;
    rc = add_i2(S, t1i); if (rc) return rc;
    auto digit_jobs = [&](std::vector<XJob>& out, const uint16_t* dig, const DevKey* key, u64* acc) {
        for (int d = 0; d < D1; d++)
            for (int k = 0; k < 2; k++) {
                XJob j{};
                j.dir = 0; j.k = k; j.ld = LD_DIGGAL; j.ep = EP_KSACC;
                j.a = (const u64*)(dig + (size_t)d * NB);
                j.b = (const u64*)(dig + (size_t)(D1 + d) * NB);
                j.gal = key->gal;
                j.ea = key->key + ((size_t)(d * 2 + 0) * 4 + k) * NB;  // b_d at prime k
                j.eb = key->key + ((size_t)(d * 2 + 1) * 4 + k) * NB;  // a_d at prime k
                j.out = acc + (size_t)k * NB;                           // c0 row; c1 row at +2n
                j.ostride = 2 * NB;
                out.push_back(j);
            }
    };
    // T3 + the specs of res_0 = acc[0] + sum_g rot(acc[g], g*baby)
    KsSpec s0{}, s1{};
    s0.level = s1.level = 1;
    s0.D = s1.D = D1;
    s0.ab = 0;
    s1.ab = 1;
    s0.acc = P.ACC;
    s1.acc = P.ACC + 2 * NB;
    if (P.acc_live[0]) {
        s0.base = P.A0;
        s1.base = P.A1;
    }
    std::vector<XJob> t3;
    for (int g = 1; g < G; g++) {
        if (!P.acc_live[g]) continue;
        const DevKey* kg = need_key(h, P.t_giant[g]);
        digit_jobs(t3, P.digG + (size_t)g * 2 * D1 * NB, kg, P.ACC);
        if (s0.nterm == MAXTERM_KS) return fail(HC_ERR_ARG, "too many giant steps");
        KsTerm T{};
        T.c0src = P.A0 + (size_t)g * 2 * NB;
        T.perm = kg->perm;
        s0.t[s0.nterm++] = T;
    }
    rc = add_xf(S, t3); if (rc) return rc;
    u64* res[2] = {P.RES, P.RES + (size_t)2 * 2 * NB};  // [poly][prime][n] each
    // the fold chain as one persistent kernel (foldchain.cuh) when D_1
    // 16-CTA clusters can be co-resident; else two launches per fold
    const bool chain = g_fc_clusters >= D1 && D1 <= 8 && P.F >= 1 && P.F <= FC_MAXF;
    const int nacc = chain ? 3 : 2;  // accumulator buffers the folds rotate over
    Step fst;
    if (chain) {
        fst.kind = ST_FOLD;
        fst.njobs = P.F;
        fst.fc.F = P.F;
        fst.fc.D = D1;
        fst.fc.bar = reinterpret_cast<unsigned*>(P.ACC + (size_t)3 * 2 * 2 * NB);
    }
    for (int f = 0; f < P.F; f++) {
        u64* cur = res[f % 2];
        const DevKey* ka = need_key(h, P.t_fold[f]);
        const KsSpec* d0 = upload_spec(S, s0, &rc); if (rc) return rc;
        const KsSpec* d1 = upload_spec(S, s1, &rc); if (rc) return rc;
        // the fold's digit products go to the next ACC buffer, so the res_f.c0
        // finish (which reads and re-zeroes this fold's buffer) can ride in the
        // digit-NTT launch; the chain is INTT2 -> digit NTTs, one stream
        u64* acc_next = P.ACC + (size_t)((f + 1) % nacc) * 2 * 2 * NB;
        std::vector<XJob> f3, f1;
        Intt2Job ij{};
        for (int k = 0; k < 2; k++) {
            ij.j[k].dir = 1; ij.j[k].k = k; ij.j[k].ld = LD_KSFIN; ij.j[k].ep = EP_STORE;
            ij.j[k].ks = d1;
            ij.j[k].aux = cur + (size_t)(2 + k) * NB;  // res_f.c1
            XJob e{};
            e.dir = 1; e.k = k; e.ld = LD_KSFIN; e.noxf = 1;
            e.ks = d0;
            e.aux = cur + (size_t)k * NB;  // res_f.c0
            f1.push_back(e);
        }
        ij.dig = P.digF;
        if (chain) {
            FcFold& F = fst.fc.f[f];
            F.base1 = s1.base;  // res_{f-1}.c1, or acc[0].c1 for fold 0 (null when acc[0] is empty)
            F.accf = s0.acc;    // ACC[f % 3]: c0 rows, then c1 rows at +2n
            F.cur = cur;
            F.igal = ka->igal;
            F.key = ka->key;
            F.acc_next = acc_next;
            F.acc_zero = P.ACC + (size_t)((f + 2) % 3) * 2 * 2 * NB;
            // res_f.c0's finish, decoded for the kernel (every term of s0 has a c0 source)
            F.c0n = s0.nterm;
            F.c0base = s0.base;
            F.c0acc = s0.acc;
            for (int i = 0; i < s0.nterm; i++) {
                if (!s0.t[i].c0src || !s0.t[i].perm) return fail(HC_ERR_STATE, "fold chain: key-switch term without a c0 source");
                F.c0src[i] = s0.t[i].c0src;
                F.c0perm[i] = s0.t[i].perm;
            }
        } else {
            digit_jobs(f3, P.digF, ka, acc_next);
            rc = add_i2(S, std::vector<Intt2Job>{ij}); if (rc) return rc;
            const size_t n0 = S.steps.size();
            rc = add_xf(S, f3); if (rc) return rc;
            if (S.steps[n0].cl && S.steps[n0].njobs >= 8) {
                S.steps[n0].side = f1;
            } else {  // no cluster launch to ride in: a separate transform-less launch
                rc = add_xf(S, f1); if (rc) return rc;
            }
        }
        // res_{f+1} = res_f + rot(res_f, a)
        s0 = KsSpec{};
        s1 = KsSpec{};
        s0.level = s1.level = 1;
        s0.D = s1.D = D1;
        s0.ab = 0;
        s1.ab = 1;
        s0.acc = acc_next;
        s1.acc = acc_next + 2 * NB;
        s0.base = cur;
        s1.base = cur + 2 * NB;
        s0.nterm = 1;
        s0.t[0].c0src = cur;
        s0.t[0].perm = ka->perm;
    }
    if (chain) S.steps.push_back(fst);
    // D1/D2: mul_plain(res_F, output_mask) level 1 -> 0
    u64* fin = res[P.F % 2];
    const KsSpec* d0 = upload_spec(S, s0, &rc); if (rc) return rc;
    const KsSpec* d1 = upload_spec(S, s1, &rc); if (rc) return rc;
    std::vector<XJob> dd1, dd2;
    for (int poly = 0; poly < 2; poly++) {
        const KsSpec* sp = poly == 0 ? d0 : d1;
        XJob j{};
        j.dir = 1; j.k = 1; j.ld = LD_KSFIN; j.ep = EP_RESCALE; j.level = 1;
        j.ks = sp;
        j.b = P.omask + NB;
        j.aux = fin + ((size_t)poly * 2 + 1) * NB;
        j.out = P.corr + (size_t)poly * NB;
        j.ostride = NB;
        dd1.push_back(j);
        XJob e{};
        e.dir = 1; e.k = 0; e.ld = LD_KSFIN; e.noxf = 1;
        e.ks = sp;
        e.aux = fin + ((size_t)poly * 2 + 0) * NB;
        dd1.push_back(e);
        XJob o{};
        o.dir = 0; o.k = 0; o.ld = LD_U64; o.ep = EP_ADDMONT;
        o.a = P.corr + (size_t)poly * NB;
        o.ea = fin + ((size_t)poly * 2 + 0) * NB;
        o.eb = P.omask;
        o.out = P.OUT + (size_t)poly * NB;
        dd2.push_back(o);
    }
    S.par_begin();
    rc = add_xf(S, dd1); if (rc) return rc;
    S.par_end();
    rc = add_xf(S, dd2); if (rc) return rc;
    return HC_OK;
}

static int need_full_range(const Plan& P) {
    if (P.full_range()) return HC_OK;
    return fail(HC_ERR_STATE, "the plan covers blocks [" + std::to_string(P.rb0) + ", " + std::to_string(P.rb1) +
                                  ") only: use hc_comp_partial");
}

static int ensure_full(hc_ctx* h) {
    Plan& P = *h->plan;
    if (P.full) return HC_OK;
    if (int rc = need_full_range(P)) return rc;
    std::unique_ptr<Schedule> S(new Schedule());
    int rc = build_partial(h, P, 0, P.B, *S);
    if (rc) return rc;
    rc = build_finish(h, P, *S);
    if (rc) return rc;
    rc = capture(h, *S);
    if (rc) return rc;
    P.full = std::move(S);
    return HC_OK;
}

extern "C" int hc_comp_set_inputs(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    if (int rc = need_full_range(P)) return rc;
    CU(cudaSetDevice(h->dev));
    const size_t bytes = (size_t)C * 2 * 4 * NPOLY * 8;
    CU(cudaMemcpyAsync(P.cd, cd, bytes, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(P.cv, cv, bytes, cudaMemcpyHostToDevice, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

extern "C" int hc_comp_set_inputs_device(hc_ctx* h, const uint64_t* cd_dev, const uint64_t* cv_dev, int C,
                                         void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    if (int rc = need_full_range(P)) return rc;
    CU(cudaSetDevice(h->dev));
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    const size_t bytes = (size_t)C * 2 * 4 * NPOLY * 8;
    CU(cudaMemcpyAsync(P.cd, cd_dev, bytes, cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(P.cv, cv_dev, bytes, cudaMemcpyDeviceToDevice, s));
    return HC_OK;
}

extern "C" int hc_comp_set_inputs_range(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int c0, int c1,
                                        void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (c0 < P.rc0 || c1 > P.rc1 || c0 > c1) return fail(HC_ERR_ARG, "ciphertext range out of bounds");
    if (c0 == c1) return HC_OK;
    CU(cudaSetDevice(h->dev));
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    const size_t ct = (size_t)2 * 4 * NPOLY;
    const size_t bytes = (size_t)(c1 - c0) * ct * 8;
    CU(cudaMemcpyAsync(P.cd + (size_t)(c0 - P.rc0) * ct, cd, bytes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(P.cv + (size_t)(c0 - P.rc0) * ct, cv, bytes, cudaMemcpyHostToDevice, s));
    return HC_OK;
}

extern "C" int hc_comp_launch(hc_ctx* h, void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    CU(cudaSetDevice(h->dev));
    int rc = ensure_full(h);
    if (rc) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    CU(cudaGraphLaunch(h->plan->full->exec, s));
    return HC_OK;
}

extern "C" int hc_comp_get_output(hc_ctx* h, uint64_t* out) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    CU(cudaSetDevice(h->dev));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(out, h->plan->OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost));
    return HC_OK;
}

extern "C" int hc_comp_get_output_async(hc_ctx* h, uint64_t* out, void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    CU(cudaSetDevice(h->dev));
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    // cudaMemcpyDefault: `out` may be pinned host memory or a device buffer
    // (a staging slot of a double-buffered serving loop)
    CU(cudaMemcpyAsync(out, h->plan->OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDefault, s));
    return HC_OK;
}

// H2D of the two input lists on two copy engines: cd on `s`, cv on the
// context's copy stream, joined back into `s` (pinned host buffers: measured
// 22 -> 32 GB/s for the headline's 2 MiB on a B200's PCIe Gen5 x16 link)
static int upload_inputs(hc_ctx* h, u64* dcd, const uint64_t* cd, u64* dcv, const uint64_t* cv, size_t bytes,
                         cudaStream_t s) {
    CU(cudaEventRecord(h->ev_copy0, s));
    CU(cudaStreamWaitEvent(h->copy_s, h->ev_copy0, 0));
    CU(cudaMemcpyAsync(dcd, cd, bytes, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(dcv, cv, bytes, cudaMemcpyHostToDevice, h->copy_s));
    CU(cudaEventRecord(h->ev_copy1, h->copy_s));
    CU(cudaStreamWaitEvent(s, h->ev_copy1, 0));
    return HC_OK;
}

extern "C" int hc_comp(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, uint64_t* out) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    CU(cudaSetDevice(h->dev));
    int rc = ensure_full(h);
    if (rc) return rc;
    const size_t bytes = (size_t)C * 2 * 4 * NPOLY * 8;
    rc = upload_inputs(h, P.cd, cd, P.cv, cv, bytes, h->stream);
    if (rc) return rc;
    CU(cudaGraphLaunch(P.full->exec, h->stream));
    CU(cudaMemcpyAsync(out, P.OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

extern "C" int hc_comp_async(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, uint64_t* out,
                             void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    CU(cudaSetDevice(h->dev));
    int rc = ensure_full(h);
    if (rc) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    const size_t bytes = (size_t)C * 2 * 4 * NPOLY * 8;
    rc = upload_inputs(h, P.cd, cd, P.cv, cv, bytes, s);
    if (rc) return rc;
    CU(cudaGraphLaunch(P.full->exec, s));
    CU(cudaMemcpyAsync(out, P.OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost, s));
    return HC_OK;
}

extern "C" int hc_comp_upload_async(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    if (int rc = need_full_range(P)) return rc;
    CU(cudaSetDevice(h->dev));
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    return upload_inputs(h, P.cd, cd, P.cv, cv, (size_t)C * 2 * 4 * NPOLY * 8, s);
}

// Comp from the caller's pack_pair outputs (answer()'s mixed-level inputs:
// pack_pair runs through hc_mul_plain / hc_rotate / the add's modulus
// switch): u: [B][2][3][n] at level 2, NTT domain,
// canonical residues.  Same BSGS graph as hc_comp from the baby steps on.
extern "C" int hc_comp_packed(hc_ctx* h, const uint64_t* u, int64_t B, uint64_t* out) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (B != P.B) return fail(HC_ERR_ARG, "expected one packed ciphertext per block");
    if (int rc = need_full_range(P)) return rc;
    CU(cudaSetDevice(h->dev));
    const size_t words = (size_t)P.B * 2 * 3 * NPOLY;
    if (!P.uin) {
        int rc = palloc(P, &P.uin, words);
        if (rc) return rc;
    }
    if (!P.full_u) {
        std::unique_ptr<Schedule> S(new Schedule());
        int rc = build_partial(h, P, 0, P.B, *S, true);
        if (!rc) rc = build_finish(h, P, *S);
        if (!rc) rc = capture(h, *S);
        if (rc) return rc;
        P.full_u = std::move(S);
    }
    CU(cudaMemcpyAsync(P.uin, u, words * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaGraphLaunch(P.full_u->exec, h->stream));
    CU(cudaMemcpyAsync(out, P.OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

static int gen_plain(hc_ctx* h, const std::vector<PJob>& pj, const PlanShape& sh) {
    PJob* dj = nullptr;
    CU(cudaMalloc(&dj, pj.size() * sizeof(PJob)));
    CU(cudaMemcpy(dj, pj.data(), pj.size() * sizeof(PJob), cudaMemcpyHostToDevice));
    for (size_t off = 0; off < pj.size(); off += 65535) {
        const int cnt = (int)std::min<size_t>(65535, pj.size() - off);
        k_plain<<<cnt, NT, 2 * NPOLY * 8, h->stream>>>(h->hctx, dj + off, sh);
    }
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(dj);
    if (e != cudaSuccess) return fail(HC_ERR_CUDA, std::string("plaintext generation: ") + cudaGetErrorString(e));
    return HC_OK;
}

// pack_pair (compress.py:338-367) for inputs at levels ld (cd) and lv (cv),
// min = 3, into P.uin at level 2: per block a P term mul_plain(ctP, mask) and
// an R term rot_col(mul_plain(ctR, mask)), each switched down to level 2
// when it lands at level 3 (add's _at_level, bgv.py:610-614, 656-658:
// mul_plain by the constant 1), then u = P + R.  Batched over blocks: one
// launch per stage.
static int build_mixed_pack(hc_ctx* h, Plan& P, Schedule& S, int with_mask) {
    const size_t NB = NPOLY;
    const int ld = P.mix_ld, lv = P.mix_lv, D3 = h->digits[3], D2 = P.D2;
    const DevKey* kcol = need_key(h, P.t_col);
    // plaintexts: mask rows at level 4 ([2][5][n]) and 3 ([2][4][n]), one at level 3 ([4][n])
    const u64* mk4 = P.mix_pt;
    const u64* mk3 = P.mask;
    const u64* one3 = P.mix_pt + (size_t)2 * 5 * NB;
    const size_t SLOT = (size_t)2 * 4 * NB;  // one [2][<=4][n] ciphertext
    // per block: Pm, Rm, Rr, P2, R2, cP, cR, cP2, cR2, coef, dntt
    const size_t per = (size_t)9 * SLOT + (size_t)4 * NB + (size_t)D3 * 4 * NB;
    // two independent chains (graph lanes): terms derived from cd (lane 0,
    // after Mask when it is fused) and from cv (lane 1); each runs
    // mul_plain -> rot_col (its R terms) -> modulus switch (terms at level 3)
    struct Lane {
        std::vector<XJob> i1, f1, i2, f2, i3, f3;
        std::vector<CJob> co;
        std::vector<MJob> ma3, ma2;
    } ln[2];
    std::vector<AddJob> adds;
    for (long long t = 0; t < P.B; t++) {
        const long long src = t / 2;
        const int par = (int)(t % 2);
        const u64* cvp = P.mix_cv + (size_t)src * 2 * (lv + 1) * NB;
        const u64* cdp = P.mix_cd + (size_t)src * 2 * (ld + 1) * NB;
        // even: P = mp(cv, top), R = mp(cd, top); odd: P = mp(cd, bot), R = mp(cv, bot)
        const u64* ctP = par == 0 ? cvp : cdp;
        const u64* ctR = par == 0 ? cdp : cvp;
        const int lP = par == 0 ? lv : ld, lR = par == 0 ? ld : lv;
        Lane& LP = ln[par == 0 ? 1 : 0];  // the lane of the P term's source
        Lane& LR = ln[par == 0 ? 0 : 1];
        auto mask = [&](int l) { return l == 4 ? mk4 + (size_t)par * 5 * NB : mk3 + (size_t)par * 4 * NB; };
        u64* b = P.mix_buf + (size_t)t * per;
        u64 *Pm = b, *Rm = b + SLOT, *Rr = b + 2 * SLOT, *P2 = b + 3 * SLOT, *R2 = b + 4 * SLOT;
        u64 *cP = b + 5 * SLOT, *cR = b + 6 * SLOT, *cP2 = b + 7 * SLOT, *cR2 = b + 8 * SLOT;
        u64* coef = b + 9 * SLOT;
        u64* dntt = coef + (size_t)4 * NB;
        uint16_t* dig = P.mix_dig + (size_t)t * D3 * NB;
        jobs_mul_plain(LP.i1, LP.f1, lP, ctP, mask(lP), cP, Pm);  // level lP - 1
        jobs_mul_plain(LR.i1, LR.f1, lR, ctR, mask(lR), cR, Rm);  // level lR - 1
        const int lr = lR - 1;  // rotation level
        jobs_rotate(LR.i2, LR.co, LR.f2, lr == 3 ? LR.ma3 : LR.ma2, lr, lr == 3 ? D3 : D2, kcol, Rm, coef, dig, dntt, Rr);
        const u64* pf = Pm;
        const u64* rf = Rr;
        if (lP - 1 == 3) {
            jobs_mul_plain(LP.i3, LP.f3, 3, Pm, one3, cP2, P2);
            pf = P2;
        }
        if (lr == 3) {
            jobs_mul_plain(LR.i3, LR.f3, 3, Rr, one3, cR2, R2);
            rf = R2;
        }
        adds.push_back({pf, rf, P.uin + (size_t)t * 2 * 3 * NB});
    }
    static int lanes_on = -1, cl_lanes = -1;  // HC_MIX_LANES=0: one chain; HC_MIX_CL=0: clusters in lane 0 only
    if (lanes_on < 0) {
        const char* e = getenv("HC_MIX_LANES");
        lanes_on = (e && e[0] == '0') ? 0 : 1;
        e = getenv("HC_MIX_CL");
        cl_lanes = (e && e[0] == '0') ? 0 : 1;
    }
    int rc = HC_OK;
    if (lanes_on) S.par_begin();
    for (int l = 0; l < 2; l++) {
        if (lanes_on) {
            S.cur_lane = l;
            S.cl_in_lane = l == 0 || cl_lanes;
        }
        Lane& L = ln[l];
        if (l == 0 && with_mask) {
            // pdq.mask (pdq.py:238-245): cd_c = mul_plain(cv_c, DB block c) at level lv
            std::vector<XJob> inv, fwd;
            for (long long c = 0; c < P.C; c++)
                jobs_mul_plain(inv, fwd, lv, P.mix_cv + (size_t)c * 2 * (lv + 1) * NB, P.ans_pt + (size_t)c * (lv + 1) * NB,
                               P.mix_mcorr + (size_t)c * 2 * lv * NB, P.mix_cd + (size_t)c * 2 * lv * NB);
            rc = add_xf(S, inv); if (rc) return rc;
            rc = add_xf(S, fwd); if (rc) return rc;
        }
        if (!lanes_on && l == 1) break;
        auto both = [&](auto Lane::*m) {  // one chain: both lanes' jobs in one launch
            auto v = L.*m;
            if (!lanes_on) v.insert(v.end(), (ln[1].*m).begin(), (ln[1].*m).end());
            return v;
        };
        rc = add_xf(S, both(&Lane::i1)); if (rc) return rc;
        rc = add_xf(S, both(&Lane::f1)); if (rc) return rc;
        rc = add_xf(S, both(&Lane::i2)); if (rc) return rc;
        rc = add_co(S, both(&Lane::co)); if (rc) return rc;
        rc = add_xf(S, both(&Lane::f2)); if (rc) return rc;
        rc = add_ma(S, both(&Lane::ma3), 4); if (rc) return rc;
        rc = add_ma(S, both(&Lane::ma2), 3); if (rc) return rc;
        rc = add_xf(S, both(&Lane::i3)); if (rc) return rc;
        rc = add_xf(S, both(&Lane::f3)); if (rc) return rc;
    }
    if (lanes_on) {
        S.cur_lane = -1;
        S.cl_in_lane = false;
        S.par_end();
    }
    return add_add(S, adds, 6, 3);  // u = P + R, all blocks in one launch
}

static int ensure_mixed(hc_ctx* h, Plan& P, int ld, int lv, int with_mask) {
    const size_t NB = NPOLY;
    if (int rc = need_full_range(P)) return rc;
    if (P.mix_ld != ld || P.mix_lv != lv || P.mix_mask != with_mask) {
        P.full_mix.reset();
        P.mix_ld = ld;
        P.mix_lv = lv;
        P.mix_mask = with_mask;
    }
    if (P.full_mix) return HC_OK;
    int rc = HC_OK;
    const int D3 = h->digits[3];
    const size_t per = (size_t)9 * 2 * 4 * NB + (size_t)4 * NB + (size_t)D3 * 4 * NB;
    if (!P.uin) rc = palloc(P, &P.uin, (size_t)P.B * 2 * 3 * NB);
    if (!rc && !P.mix_cd) rc = palloc(P, &P.mix_cd, (size_t)P.C * 2 * 5 * NB);
    if (!rc && !P.mix_cv) rc = palloc(P, &P.mix_cv, (size_t)P.C * 2 * 5 * NB);
    if (!rc && !P.mix_buf) rc = palloc(P, &P.mix_buf, (size_t)P.B * per);
    if (!rc && !P.mix_dig) rc = palloc(P, &P.mix_dig, (size_t)P.B * D3 * NB);
    if (!rc && !P.mix_mcorr) rc = palloc(P, &P.mix_mcorr, (size_t)P.C * 2 * 4 * NB);  // Mask's switch scratch
    if (!rc && !P.mix_pt) {
        rc = palloc(P, &P.mix_pt, (size_t)(2 * 5 + 4) * NB);
        if (!rc) {
            std::vector<PJob> pj;
            PJob j{};
            if (h->L >= 4) {
                j.kind = PT_TOP; j.level = 4; j.out = P.mix_pt; pj.push_back(j);
                j.kind = PT_BOT; j.level = 4; j.out = P.mix_pt + 5 * NB; pj.push_back(j);
            }
            j.kind = PT_ONE; j.level = 3; j.out = P.mix_pt + 10 * NB; pj.push_back(j);
            PlanShape sh{P.N, P.s, P.s_pad, P.baby, P.m, nullptr};
            rc = gen_plain(h, pj, sh);
        }
    }
    if (rc) return rc;
    std::unique_ptr<Schedule> S(new Schedule());
    rc = build_mixed_pack(h, P, *S, with_mask);
    if (!rc) rc = build_partial(h, P, 0, P.B, *S, true);
    if (!rc) rc = build_finish(h, P, *S);
    if (!rc) rc = capture(h, *S);
    if (rc) return rc;
    P.full_mix = std::move(S);
    return HC_OK;
}

// Comp with inputs at different levels (answer(): cd = mask(cv) one level
// below cv): cd = uint64[C][2][ld+1][n], cv =
// uint64[C][2][lv+1][n], min(ld, lv) = 3, max <= max_level.  pack_pair runs
// on the device (build_mixed_pack), then the BSGS graph of hc_comp_packed;
// one graph launch.  out = uint64[2][1][n].  Synchronous.
extern "C" int hc_comp_mixed(hc_ctx* h, const uint64_t* cd, int ld, const uint64_t* cv, int lv, int C, uint64_t* out) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    if (std::min(ld, lv) < 3) return fail(HC_ERR_LEVEL, "plaintext multiply at level 0 (Comp inputs below level 3)");
    if (std::min(ld, lv) != 3 || std::max(ld, lv) > h->L)
        return fail(HC_ERR_ARG, "mixed-level Comp takes inputs at levels 3 and <= max_level with min 3");
    CU(cudaSetDevice(h->dev));
    const size_t NB = NPOLY;
    int rc = ensure_mixed(h, P, ld, lv, 0);
    if (rc) return rc;
    CU(cudaMemcpyAsync(P.mix_cd, cd, (size_t)C * 2 * (ld + 1) * NB * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(P.mix_cv, cv, (size_t)C * 2 * (lv + 1) * NB * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaGraphLaunch(P.full_mix->exec, h->stream));
    CU(cudaMemcpyAsync(out, P.OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

// pdq.mask's plaintexts for the current plan: the cleartext database
// (uint64[N], reduced mod p) as C block plaintexts at `level`
// (_db_block_matrices, pdq.py:207-208), generated on the device.
extern "C" int hc_answer_db(hc_ctx* h, int level, const uint64_t* db_mod_p) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    if (!db_mod_p) return fail(HC_ERR_ARG, "null database");
    if (level < 4 || level > h->L) return fail(HC_ERR_ARG, "answer() on the device takes the index vector at level 4");
    Plan& P = *h->plan;
    CU(cudaSetDevice(h->dev));
    const size_t NB = NPOLY;
    std::vector<uint32_t> dbv((size_t)P.N);
    for (long long i = 0; i < P.N; i++) {
        if (db_mod_p[i] >= h->p) return fail(HC_ERR_ARG, "database values must be reduced mod p");
        dbv[i] = (uint32_t)db_mod_p[i];
    }
    int rc = HC_OK;
    if (!P.ans_db) rc = palloc(P, &P.ans_db, (size_t)P.N);  // reused by later databases
    if (rc) return rc;
    uint32_t* ddb = P.ans_db;
    CU(cudaMemcpy(ddb, dbv.data(), (size_t)P.N * 4, cudaMemcpyHostToDevice));
    if (!P.ans_pt || P.ans_level < level) {  // sized for the highest level asked so far
        rc = palloc(P, &P.ans_pt, (size_t)P.C * (level + 1) * NB);
        if (rc) return rc;
        P.full_mix.reset();  // a captured Mask graph read the old buffer
    }
    P.ans_level = level;
    std::vector<PJob> pj;
    for (long long c = 0; c < P.C; c++) {
        PJob j{};
        j.kind = PT_DBVEC; j.t = (int)c; j.level = level; j.out = P.ans_pt + (size_t)c * (level + 1) * NB;
        pj.push_back(j);
    }
    PlanShape sh{P.N, P.s, P.s_pad, P.baby, P.m, ddb};
    return gen_plain(h, pj, sh);
}

// pdq.answer after Match (pdq.py:248-256): mask (cv x the hc_answer_db
// plaintexts) then comp(cd, index_hint=cv), cv = uint64[C][2][lv+1][n] at
// level lv = 4; one graph launch.  out = uint64[2][1][n].  Synchronous.
extern "C" int hc_answer(hc_ctx* h, const uint64_t* cv, int lv, int C, uint64_t* out) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (C != P.C) return fail(HC_ERR_ARG, "expected standard-layout ciphertext lists");
    if (!P.ans_pt || P.ans_level != lv) return fail(HC_ERR_STATE, "hc_answer_db must run first at this level");
    CU(cudaSetDevice(h->dev));
    int rc = ensure_mixed(h, P, lv - 1, lv, 1);
    if (rc) return rc;
    CU(cudaMemcpyAsync(P.mix_cv, cv, (size_t)C * 2 * (lv + 1) * NPOLY * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaGraphLaunch(P.full_mix->exec, h->stream));
    CU(cudaMemcpyAsync(out, P.OUT, (size_t)2 * NPOLY * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

// Device-resident replay of the last hc_comp_mixed / hc_answer graph on
// `stream` (inputs stay in the plan's buffers; timing and serving loops).
extern "C" int hc_mixed_launch(hc_ctx* h, void* stream) {
    if (!h || !h->plan || !h->plan->full_mix) return fail(HC_ERR_STATE, "hc_comp_mixed or hc_answer must run first");
    CU(cudaSetDevice(h->dev));
    CU(cudaGraphLaunch(h->plan->full_mix->exec, stream ? (cudaStream_t)stream : h->stream));
    return HC_OK;
}

extern "C" int hc_comp_partial(hc_ctx* h, int64_t b0, int64_t b1, uint64_t* partial_dev, void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    if (b0 < P.rb0 || b1 > P.rb1 || b0 > b1) return fail(HC_ERR_ARG, "block range outside the plan's");
    CU(cudaSetDevice(h->dev));
    auto key = std::make_pair((long long)b0, (long long)b1);
    auto it = P.partials.find(key);
    if (it == P.partials.end()) {
        std::unique_ptr<Schedule> S(new Schedule());
        int rc = build_partial(h, P, b0, b1, *S);
        if (rc) return rc;
        rc = capture(h, *S);
        if (rc) return rc;
        it = P.partials.emplace(key, std::move(S)).first;
    }
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    CU(cudaGraphLaunch(it->second->exec, s));
    CU(cudaMemcpyAsync(partial_dev, P.PX, P.px_words() * 8, cudaMemcpyDeviceToDevice, s));
    return HC_OK;
}

extern "C" int hc_comp_finish(hc_ctx* h, const uint64_t* partial_dev, void* stream) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    Plan& P = *h->plan;
    CU(cudaSetDevice(h->dev));
    if (!P.fin) {
        std::unique_ptr<Schedule> S(new Schedule());
        int rc = build_finish(h, P, *S);
        if (rc) return rc;
        rc = capture(h, *S);
        if (rc) return rc;
        P.fin = std::move(S);
    }
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    CU(cudaMemcpyAsync(P.PX, partial_dev, P.px_words() * 8, cudaMemcpyDeviceToDevice, s));
    CU(cudaGraphLaunch(P.fin->exec, s));
    return HC_OK;
}

// ---------------------------------------------------------------------------
// ring helpers and single operations (host buffers)
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    ~DevBuf() { cudaFree(p); }
};

extern "C" int hc_ntt(hc_ctx* h, uint64_t* data, int rows, const int* pidx, int inverse) {
    if (!h || rows < 0) return fail(HC_ERR_ARG, "bad arguments");
    if (rows == 0) return HC_OK;
    CU(cudaSetDevice(h->dev));
    DevBuf buf;
    const size_t bytes = (size_t)rows * NPOLY * 8;
    CU(cudaMalloc(&buf.p, bytes));
    CU(cudaMemcpy(buf.p, data, bytes, cudaMemcpyHostToDevice));
    std::vector<XJob> jobs;
    for (int r = 0; r < rows; r++) {
        if (pidx[r] < 0 || pidx[r] >= NPR || (pidx[r] > h->L && pidx[r] != PIDX))
            return fail(HC_ERR_ARG, "bad prime index");
        XJob j{};
        j.dir = inverse ? 1 : 0;
        j.k = pidx[r];
        j.ld = LD_RED;
        j.ep = EP_STORE;
        j.a = (u64*)buf.p + (size_t)r * NPOLY;
        j.out = (u64*)buf.p + (size_t)r * NPOLY;
        jobs.push_back(j);
    }
    Schedule S;
    int rc = add_xf(S, jobs);
    if (rc) return rc;
    rc = run_now(h, S);
    if (rc) return rc;
    CU(cudaMemcpy(data, buf.p, bytes, cudaMemcpyDeviceToHost));
    return HC_OK;
}

extern "C" int hc_pointwise(hc_ctx* h, const uint64_t* a, const uint64_t* b, uint64_t* out, int rows,
                            const int* pidx, int op) {
    if (!h || rows < 0 || op < 0 || op > 2) return fail(HC_ERR_ARG, "bad arguments");
    if (rows == 0) return HC_OK;
    CU(cudaSetDevice(h->dev));
    const size_t bytes = (size_t)rows * NPOLY * 8;
    DevBuf da, db, dp;
    CU(cudaMalloc(&da.p, bytes));
    CU(cudaMalloc(&db.p, bytes));
    CU(cudaMalloc(&dp.p, rows * sizeof(int)));
    CU(cudaMemcpy(da.p, a, bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(db.p, b, bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dp.p, pidx, rows * sizeof(int), cudaMemcpyHostToDevice));
    k_pointwise<<<592, 256, 0, h->stream>>>(h->hctx, (u64*)da.p, (u64*)db.p, (u64*)da.p, rows, (int*)dp.p, op);
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(h->stream));
    CU(cudaMemcpy(out, da.p, bytes, cudaMemcpyDeviceToHost));
    return HC_OK;
}

// ---------------------------------------------------------------------------
// decrypt (bgv.py:559-575) on the device: phase = c0 + c1 s (NTT domain),
// INTT, the exact integer in [0, Q_l) (CRT compose), centred, reduced mod p,
// slot_decode (NTT mod p + slot gather, bgv.py:387-394)
// ---------------------------------------------------------------------------
// s (ternary, int64) -> residues [l+1][n]
__global__ void k_ternary_res(const __grid_constant__ DevCtx C, const int64_t* s, int P1, u64* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (j >= NPOLY || k >= P1) return;
    const int64_t v = s[j];
    const u64 q = C.pc[k].q;
    out[(size_t)k * NPOLY + j] = v >= 0 ? (u64)v : q - (u64)(-v);
}
// phase = c0 + c1 * s_ntt per prime (canonical residues)
__global__ void k_phase(const __grid_constant__ DevCtx C, const u64* ct, const u64* sn, int P1, u64* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (j >= NPOLY || k >= P1) return;
    const PrimeC& P = C.pc[k];
    const size_t o = (size_t)k * NPOLY + j;
    // c1 * s mod q: Montgomery product then * R (Shoup) back to the plain residue
    u64 hi, lo;
    mul128(hi, lo, ct[(size_t)P1 * NPOLY + o], sn[o]);
    const u64 m = mul_shoup(redc(hi, lo, P.q, P.qneg), P.rmod, P.rmod_s, P.q);
    out[o] = add_mod(ct[o], m, P.q);
}
// coefficient residues [l+1][n] -> centred integer mod p  (l <= KEYL)
template <int L>
__device__ __forceinline__ u64 lift_one(const DevCtx& C, const u64* x, int j) {
    u64 X[NLIMB];
    if constexpr (L == 0) {
        X[0] = x[j];
        X[1] = X[2] = X[3] = 0;
    } else {
        u64 xr[L + 1];
        HC_UNROLL
        for (int k = 0; k <= L; k++) xr[k] = x[(size_t)k * NPOLY + j];
        crt_compose<L>(C.lv(L), C.pc, xr, X);
    }
    // Q_l and X as limbs; centred: X > Q/2 -> X - Q (negative)
    u64 Q[NLIMB];
    if constexpr (L == 0) {
        Q[0] = C.pc[0].q;
        Q[1] = Q[2] = Q[3] = 0;
    } else {
        HC_UNROLL
        for (int i = 0; i < NLIMB; i++) Q[i] = C.lv(L).Q[i];
    }
    // X > floor(Q / 2)  <=>  2X > Q  (X < Q < 2^216, so 2X fits 4 limbs)
    u64 X2[NLIMB];
    u64 carry = 0;
    HC_UNROLL
    for (int i = 0; i < NLIMB; i++) {
        X2[i] = (X[i] << 1) | carry;
        carry = X[i] >> 63;
    }
    int gt = 0, decided = 0;
    HC_UNROLL
    for (int i = NLIMB - 1; i >= 0; i--) {
        if (!decided && X2[i] != Q[i]) {
            gt = X2[i] > Q[i];
            decided = 1;
        }
    }
    const u64 p = C.p;
    auto modp = [&](const u64 (&V)[NLIMB]) {
        unsigned __int128 acc = 0;
        HC_UNROLL
        for (int i = NLIMB - 1; i >= 0; i--) acc = ((acc << 64) | V[i]) % p;
        return (u64)acc;
    };
    const u64 xm = modp(X);
    if (!gt) return xm;
    const u64 qm = modp(Q);
    return xm >= qm ? xm - qm : xm + p - qm;  // (X - Q) mod p
}
__global__ void k_lift(const __grid_constant__ DevCtx C, const u64* x, int level, u64* out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= NPOLY) return;
    u64 v = 0;
    switch (level) {
        case 0: v = lift_one<0>(C, x, j); break;
        case 1: v = lift_one<1>(C, x, j); break;
        case 2: v = lift_one<2>(C, x, j); break;
        default: v = lift_one<KEYL>(C, x, j); break;
    }
    out[j] = v;
}
// evaluations mod p (NTT index order) -> slot matrix [2][n/2]
__global__ void k_slot_gather(const __grid_constant__ DevCtx C, const u64* ev, int64_t* rows) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= NPOLY) return;
    const unsigned so = C.slot_of[j];
    rows[(size_t)(so >> 12) * (NPOLY / 2) + (so & 4095)] = (int64_t)ev[j];
}

extern "C" int hc_decrypt(hc_ctx* h, const uint64_t* ct, int level, const int64_t* secret, int64_t* slots) {
    if (!h || !ct || !secret || !slots) return fail(HC_ERR_ARG, "null argument");
    if (level < 0 || level > KEYL || level > h->L) return fail(HC_ERR_ARG, "device decrypt takes levels 0..3");
    CU(cudaSetDevice(h->dev));
    const int P1 = level + 1;
    const size_t NB = NPOLY;
    DevBuf dct, ds, dsn, dph, dlift, drows;
    CU(cudaMalloc(&dct.p, (size_t)2 * P1 * NB * 8));
    CU(cudaMalloc(&ds.p, NB * 8));
    CU(cudaMalloc(&dsn.p, (size_t)P1 * NB * 8));
    CU(cudaMalloc(&dph.p, (size_t)P1 * NB * 8));
    CU(cudaMalloc(&dlift.p, NB * 8));
    CU(cudaMalloc(&drows.p, NB * 8));
    CU(cudaMemcpyAsync(dct.p, ct, (size_t)2 * P1 * NB * 8, cudaMemcpyHostToDevice, h->stream));
    CU(cudaMemcpyAsync(ds.p, secret, NB * 8, cudaMemcpyHostToDevice, h->stream));
    k_ternary_res<<<dim3(NB / 256, P1), 256, 0, h->stream>>>(h->hctx, (const int64_t*)ds.p, P1, (u64*)dsn.p);
    CU(cudaGetLastError());
    {  // NTT(s) per prime
        std::vector<XJob> jobs;
        for (int k = 0; k < P1; k++) {
            XJob j{};
            j.dir = 0; j.k = k; j.ld = LD_U64; j.ep = EP_STORE;
            j.a = (u64*)dsn.p + (size_t)k * NB;
            j.out = (u64*)dsn.p + (size_t)k * NB;
            jobs.push_back(j);
        }
        Schedule S;
        int rc = add_xf(S, jobs);
        if (!rc) rc = enqueue(h, S, h->stream);
        if (rc) return rc;
        k_phase<<<dim3(NB / 256, P1), 256, 0, h->stream>>>(h->hctx, (const u64*)dct.p, (const u64*)dsn.p, P1, (u64*)dph.p);
        CU(cudaGetLastError());
        std::vector<XJob> inv;
        for (int k = 0; k < P1; k++) {
            XJob j{};
            j.dir = 1; j.k = k; j.ld = LD_U64; j.ep = EP_STORE;
            j.a = (u64*)dph.p + (size_t)k * NB;
            j.out = (u64*)dph.p + (size_t)k * NB;
            inv.push_back(j);
        }
        Schedule S2;
        rc = add_xf(S2, inv);
        if (!rc) rc = enqueue(h, S2, h->stream);
        if (rc) return rc;
        k_lift<<<NB / 256, 256, 0, h->stream>>>(h->hctx, (const u64*)dph.p, level, (u64*)dlift.p);
        CU(cudaGetLastError());
        std::vector<XJob> fp(1);
        fp[0].dir = 0; fp[0].k = PIDX; fp[0].ld = LD_U64; fp[0].ep = EP_STORE;
        fp[0].a = (u64*)dlift.p;
        fp[0].out = (u64*)dlift.p;
        Schedule S3;
        rc = add_xf(S3, fp);
        if (!rc) rc = enqueue(h, S3, h->stream);
        if (rc) return rc;
        k_slot_gather<<<NB / 256, 256, 0, h->stream>>>(h->hctx, (const u64*)dlift.p, (int64_t*)drows.p);
        CU(cudaGetLastError());
    }
    CU(cudaMemcpyAsync(slots, drows.p, NB * 8, cudaMemcpyDeviceToHost, h->stream));
    CU(cudaStreamSynchronize(h->stream));
    return HC_OK;
}

// modulus-switch correction of a deep level (l > LVC): per kept prime k,
// e_k = (d - r q_l^-1) mod q_k from the dropped prime's (r, d) integers
// (EP_RESCALE_RD); the constants of (l, k) come in `qk` = [qinv, qinv_s]
// grid (n/256, l, 2 polys)
__global__ void k_deep_corr(const __grid_constant__ DevCtx C, const u64* rd, const u64* qk, int l, u64* corr) {
    const int j = blockIdx.x * 256 + threadIdx.x;
    const int k = blockIdx.y, poly = blockIdx.z;
    const u64* s = rd + (size_t)poly * 2 * NPOLY;
    const PrimeC& P = C.pc[k];
    corr[((size_t)poly * l + k) * NPOLY + j] =
        corr_from_sums((long long)s[j], (long long)s[NPOLY + j], P.q, qk[2 * k], qk[2 * k + 1], P.one_s);
}

extern "C" int hc_mul_plain(hc_ctx* h, const uint64_t* ct, int level, const uint64_t* pt, uint64_t* out) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    if (level < 1) return fail(HC_ERR_LEVEL, "plaintext multiply at level 0");
    if (level > h->L) return fail(HC_ERR_ARG, "level above max_level");
    CU(cudaSetDevice(h->dev));
    const int l = level, P1 = l + 1;
    const size_t NB = NPOLY;
    // plaintext in Montgomery form with the modulus-switch factor folded in
    std::vector<u64> ptm((size_t)P1 * NB), qk((size_t)2 * l);
    for (int k = 0; k <= l; k++) {
        const PrimeC& pc = h->hctx.pc[k];
        u64 w = pc.rmod;
        if (k < l) {
            const u64 qi = inv_mod(h->hctx.pc[l].q % pc.q, pc.q);  // q_l^-1 mod q_k
            qk[2 * k] = qi;
            qk[2 * k + 1] = shoup_const(qi, pc.q);
            w = mulmod_slow(qi, pc.rmod, pc.q);
        }
        for (size_t j = 0; j < NB; j++) ptm[k * NB + j] = mulmod_slow(pt[k * NB + j] % pc.q, w, pc.q);
    }
    if (l > LVC) {  // deep level of a protocol chain: (r, d) -> per-prime corrections -> NTTs
        DevBuf dct, dpt, drd, dqk, dcorr, dout;
        CU(cudaMalloc(&dct.p, (size_t)2 * P1 * NB * 8));
        CU(cudaMalloc(&dpt.p, (size_t)P1 * NB * 8));
        CU(cudaMalloc(&drd.p, (size_t)2 * 2 * NB * 8));
        CU(cudaMalloc(&dqk.p, qk.size() * 8));
        CU(cudaMalloc(&dcorr.p, (size_t)2 * l * NB * 8));
        CU(cudaMalloc(&dout.p, (size_t)2 * l * NB * 8));
        CU(cudaMemcpy(dct.p, ct, (size_t)2 * P1 * NB * 8, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dpt.p, ptm.data(), (size_t)P1 * NB * 8, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dqk.p, qk.data(), qk.size() * 8, cudaMemcpyHostToDevice));
        const u64* c = (const u64*)dct.p;
        const u64* p = (const u64*)dpt.p;
        std::vector<XJob> inv, fwd;
        for (int poly = 0; poly < 2; poly++) {
            XJob j{};
            j.dir = 1; j.k = l; j.ld = LD_MONT; j.ep = EP_RESCALE_RD; j.level = l;
            j.a = c + ((size_t)poly * P1 + l) * NB;
            j.b = p + (size_t)l * NB;
            j.out = (u64*)drd.p + (size_t)poly * 2 * NB;
            j.ostride = NB;
            inv.push_back(j);
            for (int k = 0; k < l; k++) {
                XJob f{};
                f.dir = 0; f.k = k; f.ld = LD_U64; f.ep = EP_ADDMONT;
                f.a = (u64*)dcorr.p + ((size_t)poly * l + k) * NB;
                f.ea = c + ((size_t)poly * P1 + k) * NB;
                f.eb = p + (size_t)k * NB;
                f.out = (u64*)dout.p + ((size_t)poly * l + k) * NB;
                fwd.push_back(f);
            }
        }
        Schedule S1, S2;
        int rc = add_xf(S1, inv);
        if (!rc) rc = run_now(h, S1);
        if (rc) return rc;
        k_deep_corr<<<dim3(NB / 256, l, 2), 256, 0, h->stream>>>(h->hctx, (const u64*)drd.p, (const u64*)dqk.p, l, (u64*)dcorr.p);
        CU(cudaGetLastError());
        rc = add_xf(S2, fwd);
        if (!rc) rc = run_now(h, S2);
        if (rc) return rc;
        CU(cudaMemcpy(out, dout.p, (size_t)2 * l * NB * 8, cudaMemcpyDeviceToHost));
        return HC_OK;
    }
    DevBuf dct, dpt, dcorr, dout;
    CU(cudaMalloc(&dct.p, (size_t)2 * P1 * NB * 8));
    CU(cudaMalloc(&dpt.p, (size_t)P1 * NB * 8));
    CU(cudaMalloc(&dcorr.p, (size_t)2 * l * NB * 8));
    CU(cudaMalloc(&dout.p, (size_t)2 * l * NB * 8));
    CU(cudaMemcpy(dct.p, ct, (size_t)2 * P1 * NB * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(dpt.p, ptm.data(), (size_t)P1 * NB * 8, cudaMemcpyHostToDevice));
    const u64* c = (const u64*)dct.p;
    const u64* p = (const u64*)dpt.p;
    u64* corr = (u64*)dcorr.p;
    u64* o = (u64*)dout.p;
    std::vector<XJob> a, b;
    jobs_mul_plain(a, b, l, c, p, corr, o);
    Schedule S;
    int rc = add_xf(S, a);
    if (!rc) rc = add_xf(S, b);
    if (!rc) rc = run_now(h, S);
    if (rc) return rc;
    CU(cudaMemcpy(out, o, (size_t)2 * l * NB * 8, cudaMemcpyDeviceToHost));
    return HC_OK;
}

extern "C" int hc_rotate(hc_ctx* h, const uint64_t* ct, int level, uint32_t t, uint64_t* out) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    if (level < 1 || level > h->L) return fail(HC_ERR_ARG, "rotation level must be 1..max_level");
    if (level > KEYL) return fail(HC_ERR_ARG, "device key switching runs at levels <= 3");
    const DevKey* key = need_key(h, t);
    if (!key) return fail(HC_ERR_KEY, "rotation key was not declared at keygen");
    CU(cudaSetDevice(h->dev));
    const int l = level, P1 = l + 1, D = h->digits[l];
    const size_t NB = NPOLY;
    DevBuf dct, dcoef, ddig, dntt, dout;
    CU(cudaMalloc(&dct.p, (size_t)2 * P1 * NB * 8));
    CU(cudaMalloc(&dcoef.p, (size_t)P1 * NB * 8));
    CU(cudaMalloc(&ddig.p, (size_t)D * NB * 2));
    CU(cudaMalloc(&dntt.p, (size_t)D * P1 * NB * 8));
    CU(cudaMalloc(&dout.p, (size_t)2 * P1 * NB * 8));
    CU(cudaMemcpy(dct.p, ct, (size_t)2 * P1 * NB * 8, cudaMemcpyHostToDevice));
    const u64* c = (const u64*)dct.p;
    std::vector<XJob> inv, fwd;
    std::vector<CJob> co;
    std::vector<MJob> ma;
    jobs_rotate(inv, co, fwd, ma, l, D, key, c, (u64*)dcoef.p, (uint16_t*)ddig.p, (u64*)dntt.p, (u64*)dout.p);
    Schedule S;
    int rc = add_xf(S, inv);
    if (!rc) rc = add_co(S, co);
    if (!rc) rc = add_xf(S, fwd);
    if (!rc) rc = add_ma(S, ma, P1);
    if (!rc) rc = run_now(h, S);
    if (rc) return rc;
    CU(cudaMemcpy(out, dout.p, (size_t)2 * P1 * NB * 8, cudaMemcpyDeviceToHost));
    return HC_OK;
}

// ---------------------------------------------------------------------------
// measurement helpers
// ---------------------------------------------------------------------------
static int comp_profile(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind, int* step_jobs,
                        int* step_tag);
extern "C" int hc_comp_profile(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind,
                               int* step_jobs) {
    return comp_profile(h, stream, max_steps, step_ms, step_kind, step_jobs, nullptr);
}
extern "C" int hc_comp_profile_ex(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind,
                                  int* step_jobs, int* step_tag) {
    return comp_profile(h, stream, max_steps, step_ms, step_kind, step_jobs, step_tag);
}
static int comp_profile(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind, int* step_jobs,
                        int* step_tag) {
    if (!h || !h->plan) return fail(HC_ERR_STATE, "hc_plan must run first");
    CU(cudaSetDevice(h->dev));
    int rc = ensure_full(h);
    if (rc) return rc;
    const Schedule& S = *h->plan->full;
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    const int ns = (int)S.steps.size();
    std::vector<cudaEvent_t> ev(ns + 1);
    for (auto& e : ev) CU(cudaEventCreate(&e));
    CU(cudaEventRecord(ev[0], s));
    g_pdl_suspended = true;  // each launch timed on its own, no early start
    for (int i = 0; i < ns; i++) {
        Schedule one;
        one.steps.push_back(S.steps[i]);
        rc = enqueue(h, one, s);
        one.steps.clear();
        if (rc) {
            g_pdl_suspended = false;
            return rc;
        }
        CU(cudaEventRecord(ev[i + 1], s));
    }
    g_pdl_suspended = false;
    CU(cudaStreamSynchronize(s));
    int k = 0;
    for (int i = 0; i < ns && k < max_steps; i++, k++) {
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        step_ms[k] = ms;
        step_kind[k] = S.steps[i].kind;
        step_jobs[k] = S.steps[i].njobs;
        if (step_tag) {  // transform launches: which instantiation ran
            const Step& st = S.steps[i];
            int tag = 0;
            if (st.kind == ST_XF && !st.hjobs.empty()) {
                const XJob& j = st.hjobs[0];
                const bool clu = st.cl && st.njobs <= CL_MAX;
                const int vt = clu ? st.jpc : (st.njobs >= g_vt2_jobs ? 4 : 1);
                tag = (clu ? 1 << 20 : 0) | (j.dir << 16) | (j.ld << 12) | (kernel_ep(j.dir, j.ld, j.ep) << 8) | (j.noxf << 4) | vt;
            }
            step_tag[k] = tag;
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    return k;
}

// Butterfly-throughput ceiling: the CT butterfly of the NTT kernels
// (Harvey lazy Shoup, bf_ct) in registers at full occupancy, no memory
// traffic.  Returns butterflies per second; the integer-ALU roofline
// denominator for the transform kernels (k_xf, k_xf_cl, k_cl_intt2).
__global__ void __launch_bounds__(256) k_bf_peak(const __grid_constant__ DevCtx C, int iters, u64* sink) {
    const PrimeC P = C.pc[0];
    u64 x[16];
    for (int i = 0; i < 16; i++) x[i] = (threadIdx.x * 977 + i * 131 + blockIdx.x) % P.q;
    u64 w = C.twf[5].w, ws = C.twf[5].ws;
    for (int it = 0; it < iters; it++) {
        HC_UNROLL
        for (int i = 0; i < 8; i++) bf_ct_lazy(x[i], x[i + 8], w, ws, P.q, 2 * P.q2);
        HC_UNROLL
        for (int i = 0; i < 16; i += 2) bf_ct_lazy(x[i], x[i + 1], w, ws, P.q, 2 * P.q2);
    }
    u64 acc = 0;
    for (int i = 0; i < 16; i++) acc ^= x[i];
    if (acc == 0x12345) sink[0] = acc;
}

extern "C" int hc_bf_peak(hc_ctx* h, double* bfly_per_s) {
    if (!h) return fail(HC_ERR_ARG, "null context");
    CU(cudaSetDevice(h->dev));
    int nsm = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
    DevBuf sink;
    CU(cudaMalloc(&sink.p, 8));
    const int blocks = nsm * 8, iters = 4096;
    k_bf_peak<<<blocks, 256, 0, h->stream>>>(h->hctx, 64, (u64*)sink.p);  // warm-up
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    CU(cudaEventRecord(a, h->stream));
    k_bf_peak<<<blocks, 256, 0, h->stream>>>(h->hctx, iters, (u64*)sink.p);
    CU(cudaEventRecord(b, h->stream));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *bfly_per_s = (double)blocks * 256 * iters * 16 / (ms * 1e-3);
    return HC_OK;
}

// INT32 multiply-pipe ceilings, independent of the kernels' code: streams of
// one instruction kind (mad.lo.u32 -> IMAD, mad.wide.u32 -> IMAD.WIDE.U32,
// mad.hi.u32 -> IMAD.HI.U32; 8 independent accumulator chains per thread,
// 2048 threads per SM), no memory traffic.  Writes ops/s for the three kinds.
__global__ void __launch_bounds__(256) k_imad_peak(int mode, int iters, uint32_t seed, u64* sink) {
    uint32_t a[8], b = seed ^ (threadIdx.x * 2654435761u), c = blockIdx.x * 40503u + 7u;
    u64 w[8];
    HC_UNROLL
    for (int i = 0; i < 8; i++) {
        a[i] = b + 977u * i;
        w[i] = a[i];
    }
    if (mode == 0) {
        for (int it = 0; it < iters; it++) {
            HC_UNROLL
            for (int i = 0; i < 8; i++) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        }
    } else if (mode == 1) {
        for (int it = 0; it < iters; it++) {
            HC_UNROLL
            for (int i = 0; i < 8; i++) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[i]) : "r"(a[i]), "r"(b));
        }
    } else {
        for (int it = 0; it < iters; it++) {
            HC_UNROLL
            for (int i = 0; i < 8; i++) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b), "r"(c));
        }
    }
    u64 acc = 0;
    HC_UNROLL
    for (int i = 0; i < 8; i++) acc ^= a[i] ^ w[i];
    if (acc == 0x1234567ull) sink[0] = acc;
}

extern "C" int hc_imad_peak(hc_ctx* h, double* ops_per_s) {
    if (!h || !ops_per_s) return fail(HC_ERR_ARG, "bad arguments");
    CU(cudaSetDevice(h->dev));
    int nsm = 0;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev));
    DevBuf sink;
    CU(cudaMalloc(&sink.p, 8));
    const int blocks = nsm * 8, iters = 8192;
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    for (int mode = 0; mode < 3; mode++) {
        k_imad_peak<<<blocks, 256, 0, h->stream>>>(mode, 256, 1u, (u64*)sink.p);  // warm-up
        CU(cudaEventRecord(a, h->stream));
        k_imad_peak<<<blocks, 256, 0, h->stream>>>(mode, iters, 1u, (u64*)sink.p);
        CU(cudaEventRecord(b, h->stream));
        CU(cudaEventSynchronize(b));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, a, b));
        ops_per_s[mode] = (double)blocks * 256 * iters * 8 / (ms * 1e-3);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return HC_OK;
}

// Transform microbenchmark: `njobs` independent plain transforms (LD_U64 /
// EP_STORE) per launch, `iters` back-to-back launches; returns us/launch.
extern "C" int hc_set_cluster_threshold(int max_jobs) {
    CL_MAX_JOBS = max_jobs;
    return HC_OK;
}

extern "C" int hc_max_active_clusters(hc_ctx* h, int* clusters) {
    if (!h || !clusters) return fail(HC_ERR_ARG, "bad arguments");
    CU(cudaSetDevice(h->dev));
    return max_active_clusters(clusters);
}

extern "C" int hc_set_vt2_jobs(int jobs) {
    g_vt2_jobs = jobs;
    return HC_OK;
}

extern "C" int hc_set_lane_blocks(int max_blocks) {
    g_lane_max_blocks = max_blocks;
    return HC_OK;
}

extern "C" int hc_bench_xform(hc_ctx* h, int njobs, int dir, int iters, double* us_per_launch) {
    if (!h || njobs < 1 || iters < 1) return fail(HC_ERR_ARG, "bad arguments");
    CU(cudaSetDevice(h->dev));
    DevBuf buf;
    CU(cudaMalloc(&buf.p, (size_t)njobs * NPOLY * 8));
    CU(cudaMemset(buf.p, 0, (size_t)njobs * NPOLY * 8));
    std::vector<XJob> jobs;
    for (int i = 0; i < njobs; i++) {
        XJob j{};
        j.dir = dir; j.k = i % (h->L + 1); j.ld = LD_U64; j.ep = EP_STORE;
        j.a = (u64*)buf.p + (size_t)i * NPOLY;
        j.out = (u64*)buf.p + (size_t)i * NPOLY;
        jobs.push_back(j);
    }
    Schedule S;
    int rc = add_xf(S, jobs);
    if (rc) return rc;
    for (int w = 0; w < 3; w++) {
        rc = enqueue(h, S, h->stream);
        if (rc) return rc;
    }
    cudaEvent_t a, b;
    CU(cudaEventCreate(&a));
    CU(cudaEventCreate(&b));
    CU(cudaEventRecord(a, h->stream));
    for (int i = 0; i < iters; i++) {
        rc = enqueue(h, S, h->stream);
        if (rc) return rc;
    }
    CU(cudaEventRecord(b, h->stream));
    CU(cudaEventSynchronize(b));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *us_per_launch = 1e3 * ms / iters;
    return HC_OK;
}

// HC_TRACE builds: reset the launch numbering / read back the per-CTA
// %globaltimer stamps [launch][block][point] (128 x 512 x 8 u64).
extern "C" int hc_trace_reset(void) {
    g_trace_seq = 0;
#ifdef HC_TRACE
    static unsigned long long zero[TR_LAUNCH][TR_BLK][TR_PT];
    CU(cudaMemcpyToSymbol(g_trace, zero, sizeof(zero)));
#endif
    return HC_OK;
}
extern "C" int hc_trace_read_tail(uint64_t* out) {
#ifdef HC_TRACE
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpyFromSymbol(out, g_fc_trace, sizeof(g_fc_trace)));
    return HC_OK;
#else
    (void)out;
    return fail(HC_ERR_STATE, "library built without HC_TRACE");
#endif
}
extern "C" int hc_trace_read(uint64_t* out) {
#ifdef HC_TRACE
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace)));
    return HC_OK;
#else
    return fail(HC_ERR_STATE, "library built without HC_TRACE");
#endif
}

extern "C" void hc_ctx_destroy(hc_ctx* h) {
    if (!h) return;
    cudaSetDevice(h->dev);
    cudaDeviceSynchronize();
    h->plan.reset();
    for (auto& kv : h->keys) release_key(kv.second);
    cudaFree(h->d_twf);
    cudaFree(h->d_twi);
    cudaFree(h->d_slot_of);
    cudaFree(h->d_ctx);
    if (h->stream) cudaStreamDestroy(h->stream);
    for (int i = 0; i < 4; i++) {
        if (h->side[i]) cudaStreamDestroy(h->side[i]);
        if (h->ev_join[i]) cudaEventDestroy(h->ev_join[i]);
    }
    if (h->ev_fork) cudaEventDestroy(h->ev_fork);
    if (h->copy_s) cudaStreamDestroy(h->copy_s);
    if (h->ev_copy0) cudaEventDestroy(h->ev_copy0);
    if (h->ev_copy1) cudaEventDestroy(h->ev_copy1);
    delete h;
}

// ---------------------------------------------------------------------------
// Host sampling with the reference's random.Random stream (pyrng.hpp):
// keygen / encrypt (bgv.py:398-557) run their samplers natively, consuming
// exactly the values the reference would.
// ---------------------------------------------------------------------------
struct hc_rng {
    PyMT mt;
};

extern "C" int hc_rng_create(const uint32_t* key, int len, hc_rng** out) {
    if (!key || len < 1 || !out) return fail(HC_ERR_ARG, "bad seed words");
    hc_rng* r = new hc_rng();
    r->mt.init_by_array(key, len);
    *out = r;
    return HC_OK;
}

extern "C" void hc_rng_destroy(hc_rng* r) { delete r; }

extern "C" int hc_rng_getrandbits(hc_rng* r, int k, uint32_t* words) {
    if (!r || k < 0 || !words) return fail(HC_ERR_ARG, "bad arguments");
    r->mt.getrandbits(k, words);
    return HC_OK;
}

// [randrange(3) - 1 for _ in range(n)]  (bgv.py _sample_ternary)
extern "C" int hc_rng_ternary(hc_rng* r, int n, int64_t* out) {
    if (!r || n < 0 || !out) return fail(HC_ERR_ARG, "bad arguments");
    for (int i = 0; i < n; i++) out[i] = (int64_t)r->mt.randbelow32(3) - 1;
    return HC_OK;
}

// getrandbits(k).bit_count() - getrandbits(k).bit_count()  (centered binomial)
extern "C" int hc_rng_cbd(hc_rng* r, int n, int k, int64_t* out) {
    if (!r || n < 0 || k < 1 || k > 32 || !out) return fail(HC_ERR_ARG, "bad arguments");
    for (int i = 0; i < n; i++) {
        uint32_t a, b;
        r->mt.getrandbits(k, &a);
        r->mt.getrandbits(k, &b);
        out[i] = (int64_t)__builtin_popcount(a) - (int64_t)__builtin_popcount(b);
    }
    return HC_OK;
}

// [randrange(Q) for _ in range(n)] reduced mod each prime: out[np][n]
extern "C" int hc_rng_uniform(hc_rng* r, int n, const uint32_t* q, int nw, int kbits, const uint64_t* primes, int np,
                              uint64_t* out) {
    if (!r || n < 0 || !q || nw < 1 || nw > 48 || kbits < 1 || kbits > 32 * nw || !primes || np < 1 || !out)
        return fail(HC_ERR_ARG, "bad arguments");
    uint32_t w[48];
    // 2^(32 j) mod q_k: a draw's residue is sum_j w_j (2^(32 j) mod q_k) with
    // one reduction (48 terms < 2^86 each stay below 2^92)
    std::vector<uint64_t> pw((size_t)np * nw);
    for (int k = 0; k < np; k++) {
        unsigned __int128 v = 1;
        for (int j = 0; j < nw; j++) {
            pw[(size_t)k * nw + j] = (uint64_t)v;
            v = (v << 32) % primes[k];
        }
    }
    for (int i = 0; i < n; i++) {
        r->mt.randbelow_words(q, nw, kbits, w);
        for (int k = 0; k < np; k++) {
            unsigned __int128 acc = 0;
            const uint64_t* pk = &pw[(size_t)k * nw];
            for (int j = 0; j < nw; j++) acc += (unsigned __int128)w[j] * pk[j];
            out[(size_t)k * n + i] = (uint64_t)(acc % primes[k]);
        }
    }
    return HC_OK;
}
