// sm_100a kernels of the Comp path.  All are job-list kernels: a launch
// carries an array of descriptors, so one launch batches every independent
// transform / CRT / MAC of a schedule step (hcomp.cu builds the lists once
// per plan and replays them in a CUDA graph).
//
//   k_xf       one 8192-point NTT or INTT per CTA (1024 threads, or 256
//              threads running the 1024-thread schedule 4x, three CTAs per
//              SM), 64 KiB smem tile, with a fused loader (pointwise
//              Montgomery product, digit gather through a Galois table,
//              key-switch finish, ...) and a fused epilogue (plaintext-
//              multiply combine, modulus-switch correction, key MAC, ...).
//   k_xf_cl    the same jobs on 8-CTA clusters, 1-4 transforms per cluster
//              (latency path); k_cl_intt2 the two-prime INTT + CRT digits of
//              a level-1 key switch on one cluster.
//   k_compose  exact CRT + base-2^16 digit split (optionally through the
//              coefficient-domain Galois gather), one thread per coefficient.
//   k_ksmac    key-switch inner product sum_j NTT(digit_j) * ksk_j with
//              128-bit lazy accumulation and one Montgomery reduction, fused
//              with the automorphism of c0 and the ciphertext additions.
//   k_diagx    diagonal multiply-accumulate of the BSGS matvec (kept primes).
//   k_plain    on-device plaintext generation (Vandermonde diagonals and
//              masks: slot values -> INTT mod p -> NTT mod q_k -> Montgomery).
#pragma once
#include <cooperative_groups.h>

#include "elem.cuh"
#include "ntt1k.cuh"

namespace hc {

// Checked builds (-DHC_CHECK, libhcomp_check.so): device-side assertions of
// the value-range invariants the exact arithmetic relies on -- lazy ranges of
// transform inputs/outputs, Galois gather indices, REDC preconditions
// (128-bit sums below q * 2^64) and the no-overflow bounds of every red.add
// accumulator.  A violated invariant traps (kernel error) instead of
// producing a silently wrong residue.  Release builds compile them away.
#ifdef HC_CHECK
#define HC_ASSERT(c)          \
    do {                      \
        if (!(c)) __trap();   \
    } while (0)
#else
#define HC_ASSERT(c) \
    do {             \
    } while (0)
#endif
// red.add into an accumulator whose words must stay below `bound`
__device__ __forceinline__ void acc_add(u64* p, u64 v, u64 bound) {
#ifdef HC_CHECK
    const u64 old = atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
    HC_ASSERT(old + v >= old && old + v < bound);
#else
    (void)bound;
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
#endif
}
constexpr u64 KSACC_BOUND = 1ull << 62;  // <= 49 digit products < q < 2^54 per word (+ slack)
constexpr u64 PX_BOUND = 1ull << 61;     // diagonal-MAC atomics: < 4q (block lanes) or < 64q (pipelined chunks) per word

// ---------------------------------------------------------------------------
// transform jobs: loaders and epilogues
// ---------------------------------------------------------------------------
enum : int {
    LD_U64 = 0,    // a[j]
    LD_MONT = 1,   // a[j] * b[j] (b in Montgomery form), in [0, 2q): inverse transforms only
    LD_ADD = 2,    // a[j] + b[j] mod q
    LD_RED = 3,    // a[j] reduced from any u64 (+ b[j] likewise if b)
    LD_DIG = 4,    // u16 digit a[j]
    LD_DIGGAL = 5, // u16 digit gathered: gal[j] -> (neg ? b : a)[src]
    LD_KSFIN = 8,  // base + sum_t c0src_t[perm_t] + red(acc) (KsSpec.acc, zeroed) [* b], aux
};

// Key-switch finish for one output poly (c0: ab = 0, c1: ab = 1) at prime k:
//   v = base[k][j] + sum_t ( c0src_t[k][perm_t[j]] (ab = 0 only)
//                            + REDC(sum_d dntt_t[d][k][j] * key_t[d][ab][k][j]) )
// = the k_ksmac computation, fused into the consumer's loader.
constexpr int MAXTERM_KS = 8;
struct KsTerm {
    const u64* dntt;  // [D][P][n]
    const u64* key;   // [D_L][2][L+1][n] Montgomery
    const u64* c0src; // [P][n] (ab = 0)
    const uint16_t* perm;
};
struct KsSpec {
    int level, nterm, ab, D;  // D = digits at `level`
    const u64* base;  // [P][n] or null
    KsTerm t[MAXTERM_KS];
    u64* acc;         // LD_KSFIN: [P][n] digit-product accumulator (EP_KSACC), zeroed after use
};
enum : int {
    EP_STORE = 0,          // out[j] = x
    EP_ADDMONT = 1,        // out[j] = x + ea[j]*eb[j]   (eb Montgomery)
    EP_ADD = 2,            // out[j] = x + ea[j]
    EP_ADDRED = 3,         // out[j] = x + red(ea[j])
    EP_RESCALE = 4,        // out[k*ostride + j] = e_k (k < level)
    EP_RESCALE_RD = 5,     // out[j] = r, out[ostride + j] = d (int64; summed by k_diagx)
    EP_KSACC = 6,          // key-switch digit product: out[j] += x*ea[j], out[ostride+j] += x*eb[j]
    EP_STORE_LAZY = 7,     // out[j] = x, x < 2^60 not canonicalised (forward NTT feeding k_ksmac)
    EP_RESCALE4 = 8,       // EP_RESCALE from level 4 (answer()'s Mask / pack products; 4 kept primes)
    // kernel instantiation only (never a job's ep): EP_RESCALE and EP_STORE jobs
    // of one step in ONE launch, the job's own ep picked per CTA -- pack_pair's
    // dropped-prime and kept-prime INTTs (S1) as one launch instead of two
    // cluster kernels side by side
    EP_RS = 9,
};
// the instantiation a job's epilogue runs in
__host__ __device__ inline int kernel_ep(int dir, int ld, int ep) {
    return (dir == 1 && ld == LD_MONT && (ep == EP_RESCALE || ep == EP_STORE)) ? EP_RS : ep;
}

struct XJob {
    int dir;    // 0 forward, 1 inverse
    int k;      // RNS prime index of the transform
    int ld, ep;
    int level;  // EP_RESCALE*: level switched from (k == level)
    int noxf;   // 1: loader + side store only (no transform, no epilogue)
    int trace;  // HC_TRACE builds: launch sequence number
    const KsSpec* ks;    // LD_KSFIN
    u64* aux;            // LD_KSFIN side store of the pre-transform value
    const u64* a;
    const u64* b;
    const uint16_t* gal;
    const u64* ea;
    const u64* eb;
    u64* out;
    long long ostride;
};

// Programmatic dependent launch (schedule kernels outside parallel graph
// branches are launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// a kernel may start while its predecessor still runs.  pdl_wait() blocks until
// the predecessor grid has completed and its writes are visible, so it precedes
// every global access to data another kernel of the Comp writes or reads (job
// tables, key-switch specs, Galois tables, keys and twiddles are constant for
// the plan's lifetime and are read before it).  Right after the wait the kernel
// lets ITS successor launch: the successor's CTAs run their constant-operand
// prologue on the SMs this kernel leaves free, and at most two kernels of a
// chain are resident at once (no cascade of idle CTAs).  HC_PDL_LATE moves the
// trigger to just before the epilogue instead (A/B builds).
#ifndef HC_PDL_LATE
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {}
#else
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
#endif

#ifdef HC_TRACE
constexpr int TR_LAUNCH = 128, TR_BLK = 512, TR_PT = 8;
__device__ unsigned long long g_trace[TR_LAUNCH][TR_BLK][TR_PT];
#define TRACE(pt)                                                                    \
    do {                                                                             \
        if (threadIdx.x == 0 && J.trace < TR_LAUNCH && blockIdx.x < TR_BLK) {       \
            unsigned long long tnow;                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));                 \
            g_trace[J.trace][blockIdx.x][pt] = tnow;                                 \
        }                                                                            \
    } while (0)
#else
#define TRACE(pt) \
    do {          \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// Loaders and epilogues, compile-time specialised (one kernel instantiation
// per (direction, loader, epilogue) used by the schedule -- no unused code
// paths, no register spills).  Each handles N coefficients j0 + e*stride per
// thread and issues every round of global loads for all N before any use.
// ---------------------------------------------------------------------------

// Loaders run in two phases around pdl_wait(): load_pre issues the loads of
// operands that are constant for the plan's lifetime (Galois gather tables,
// key-switch specs and their permutations, plaintext multipliers), so they
// overlap the predecessor kernel's tail; load_post reads the data the
// predecessor produced.
template <int LD, int N>
struct LdPre {};
template <int N>
struct LdPre<LD_DIGGAL, N> {
    unsigned g[N];
};
template <int N>
struct LdPre<LD_KSFIN, N> {
    const u64* base;
    u64* acc;
    const u64* c0;  // term 0's c0src (null: none)
    int nterm;
    unsigned pe[N];  // term 0's permutation
    u64 b[N];        // J.b multiplier (if J.b)
};

template <int N>
__device__ __forceinline__ void ksfin_pre(const XJob& J, int j0, int stride, LdPre<LD_KSFIN, N>& pre) {
    const KsSpec& S = *J.ks;
    pre.base = S.base;
    pre.acc = S.acc;
    pre.nterm = S.nterm;
    pre.c0 = S.nterm > 0 ? S.t[0].c0src : nullptr;
    if (pre.c0) {
        const uint16_t* pm = S.t[0].perm;
        HC_UNROLL
        for (int e = 0; e < N; e++) pre.pe[e] = pm[j0 + e * stride];
    }
    if (J.b) {
        HC_UNROLL
        for (int e = 0; e < N; e++) pre.b[e] = J.b[j0 + e * stride];
    }
}

// key-switch finish, loads (no stores: two finishes' loads can be in flight together)
template <int N>
struct KsLd {
    u64 x[N], acc[N], c[N];
};
template <int N>
__device__ __forceinline__ void ksfin_load(const XJob& J, const PrimeC& P, int j0, int stride,
                                           const LdPre<LD_KSFIN, N>& pre, KsLd<N>& v) {
    const size_t kofs = (size_t)J.k * NPOLY;
    HC_UNROLL
    for (int e = 0; e < N; e++) {
        v.x[e] = pre.base ? pre.base[kofs + j0 + e * stride] : 0;
        v.acc[e] = pre.acc ? pre.acc[kofs + j0 + e * stride] : 0;
        v.c[e] = pre.c0 ? pre.c0[kofs + pre.pe[e]] : 0;
    }
    // further terms (the giant-step sum): permutation, then gather
    for (int t = 1; t < pre.nterm; t++) {
        const KsTerm T = J.ks->t[t];
        if (!T.c0src) continue;
        unsigned pe[N];
        HC_UNROLL
        for (int e = 0; e < N; e++) pe[e] = T.perm[j0 + e * stride];
        HC_UNROLL
        for (int e = 0; e < N; e++) v.c[e] = add_mod(v.c[e], T.c0src[kofs + pe[e]], P.q);
    }
}
// v = base + sum_t c0src_t[perm_t] + red(acc); zero acc; aux store; [* b]
template <int N>
__device__ __forceinline__ void ksfin_finish(const XJob& J, const PrimeC& P, int j0, int stride,
                                             const LdPre<LD_KSFIN, N>& pre, const KsLd<N>& v, u64 (&x)[N]) {
    const size_t kofs = (size_t)J.k * NPOLY;
    HC_UNROLL
    for (int e = 0; e < N; e++) x[e] = add_mod(add_mod(v.x[e], v.c[e], P.q), red64(v.acc[e], P.q, P.one_s), P.q);
    if (pre.acc) {
        HC_UNROLL
        for (int e = 0; e < N; e++) pre.acc[kofs + j0 + e * stride] = 0;
    }
    if (J.aux) {
        HC_UNROLL
        for (int e = 0; e < N; e++) J.aux[j0 + e * stride] = x[e];
    }
    if (J.b) {
        HC_UNROLL
        for (int e = 0; e < N; e++) x[e] = mul_mont(x[e], pre.b[e], P.q, P.qneg);
    }
}

template <int LD, int N>
__device__ __forceinline__ void load_pre(const XJob& J, int j0, int stride, LdPre<LD, N>& pre) {
    if constexpr (LD == LD_DIGGAL) {
        HC_UNROLL
        for (int e = 0; e < N; e++) pre.g[e] = J.gal[j0 + e * stride];
    } else if constexpr (LD == LD_KSFIN) {
        ksfin_pre<N>(J, j0, stride, pre);
    }
}

template <int LD, int N>
__device__ __forceinline__ void load_post(const DevCtx& C, const XJob& J, const PrimeC& P, int j0, int stride,
                                          const LdPre<LD, N>& pre, u64 (&x)[N]) {
    if constexpr (LD == LD_MONT || LD == LD_ADD) {
        u64 b[N];
        HC_UNROLL
        for (int e = 0; e < N; e++) { x[e] = J.a[j0 + e * stride]; b[e] = J.b[j0 + e * stride]; }
        HC_UNROLL
        // LD_MONT feeds inverse transforms only (XF_COMBOS), whose first stage takes [0, 2q)
        for (int e = 0; e < N; e++) x[e] = LD == LD_MONT ? mul_mont_lazy(x[e], b[e], P.q, P.qneg) : add_mod(x[e], b[e], P.q);
    } else if constexpr (LD == LD_RED) {
        HC_UNROLL
        for (int e = 0; e < N; e++) x[e] = J.a[j0 + e * stride];
        HC_UNROLL
        for (int e = 0; e < N; e++) x[e] = red64(x[e], P.q, P.one_s);
    } else if constexpr (LD == LD_DIG) {
        const uint16_t* d = reinterpret_cast<const uint16_t*>(J.a);
        HC_UNROLL
        for (int e = 0; e < N; e++) x[e] = d[j0 + e * stride];
    } else if constexpr (LD == LD_DIGGAL) {
        const uint16_t* dp = reinterpret_cast<const uint16_t*>(J.a);
        const uint16_t* dn = reinterpret_cast<const uint16_t*>(J.b);
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            HC_ASSERT((pre.g[e] & 0x7FFF) < NPOLY);
            x[e] = ((pre.g[e] >> 15) ? dn : dp)[pre.g[e] & 0x7FFF];
        }
    } else if constexpr (LD == LD_KSFIN) {
        KsLd<N> v;
        ksfin_load<N>(J, P, j0, stride, pre, v);
        ksfin_finish<N>(J, P, j0, stride, pre, v, x);
    } else {  // LD_U64
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            x[e] = J.a[j0 + e * stride];
            HC_ASSERT(x[e] < (J.dir ? 2 * P.q : 4 * P.q));  // lazy input ranges of the GS / CT transforms
        }
    }
}

template <int LD, int N>
__device__ __forceinline__ void load_n(const DevCtx& C, const XJob& J, const PrimeC& P, int j0, int stride, u64 (&x)[N]) {
    LdPre<LD, N> pre;
    load_pre<LD, N>(J, j0, stride, pre);
    load_post<LD, N>(C, J, P, j0, stride, pre, x);
}

template <int EP, int N>
__device__ __forceinline__ void store_n(const DevCtx& D, const XJob& J, const PrimeC& P, int j0, int stride,
                                        const u64 (&x)[N]) {
    if constexpr (EP == EP_RS) {  // uniform per CTA (per thread group in cluster launches)
        if (J.ep == EP_STORE) store_n<EP_STORE, N>(D, J, P, j0, stride, x);
        else store_n<EP_RESCALE, N>(D, J, P, j0, stride, x);
    } else if constexpr (EP == EP_ADDMONT || EP == EP_KSACC) {
        u64 a[N], b[N];
        HC_UNROLL
        for (int e = 0; e < N; e++) { a[e] = J.ea[j0 + e * stride]; b[e] = J.eb[j0 + e * stride]; }
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            const int j = j0 + e * stride;
            if constexpr (EP == EP_ADDMONT) {
                J.out[j] = add_mod(x[e], mul_mont(a[e], b[e], P.q, P.qneg), P.q);
            } else {
                acc_add(J.out + j, mul_mont(x[e], a[e], P.q, P.qneg), KSACC_BOUND);
                acc_add(J.out + J.ostride + j, mul_mont(x[e], b[e], P.q, P.qneg), KSACC_BOUND);
            }
        }
    } else if constexpr (EP == EP_ADD || EP == EP_ADDRED) {
        u64 a[N];
        HC_UNROLL
        for (int e = 0; e < N; e++) a[e] = J.ea[j0 + e * stride];
        HC_UNROLL
        for (int e = 0; e < N; e++)
            J.out[j0 + e * stride] = add_mod(x[e], EP == EP_ADD ? a[e] : red64(a[e], P.q, P.one_s), P.q);
    } else if constexpr (EP == EP_RESCALE_RD) {
        const RescaleK R = rescale_consts_rd(D, J.level);
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            long long r, d;
            rescale_rd(R, x[e], r, d);
            J.out[j0 + e * stride] = (u64)r;
            J.out[J.ostride + j0 + e * stride] = (u64)d;
        }
    } else if constexpr (EP == EP_RESCALE || EP == EP_RESCALE4) {
        constexpr int NQ = EP == EP_RESCALE4 ? LVC : KEYL;
        const int l = J.level;
        const RescaleKT<NQ> R = rescale_consts<NQ>(D, l);
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            u64 ek[NQ];
            rescale_corr(R, x[e], ek);
            HC_UNROLL
            for (int k = 0; k < NQ; k++) {
                if (k >= l) break;
                J.out[(size_t)k * J.ostride + j0 + e * stride] = ek[k];
            }
        }
    } else {  // EP_STORE, EP_STORE_LAZY
        HC_UNROLL
        for (int e = 0; e < N; e++) {
            HC_ASSERT(EP == EP_STORE ? x[e] < P.q : x[e] < (1ull << 60));
            J.out[j0 + e * stride] = x[e];
        }
    }
}

// ---------------------------------------------------------------------------
// k_xf: one transform job per CTA (512 threads, 64 KiB smem tile), throughput path
// ---------------------------------------------------------------------------
// VT = 1: one 1024-thread transform per SM (latency); VT = 4: 256-thread CTAs,
// three per SM (64 KiB smem each), whose independent barriers keep the IMAD
// pipe busy while other transforms load, store or synchronise (throughput).
#ifndef HC_XF4_BOUND
#define HC_XF4_BOUND 288
#endif
template <int DIR, int LD, int EP, int VT = 1>
__global__ void __launch_bounds__(VT == 4 ? HC_XF4_BOUND : NT / VT, VT == 4 ? 3 : VT) k_xf(const __grid_constant__ DevCtx C, const XJob* __restrict__ jobs) {
    extern __shared__ u64 sm[];
    const XJob J = jobs[blockIdx.x];
    const PrimeC& P = C.pc[J.k];
    TRACE(0);
    // The bit-0 stage runs in registers at the kernel's edge (ntt1k.cuh): the
    // inverse transform's loader and the forward transform's epilogue own the
    // coefficient pairs (j, j + 1), j = 2t + 2048m; the other side keeps the
    // coefficients t + 1024e.
    const Tw* tw = (DIR ? C.twi : C.twf) + (size_t)J.k * NPOLY;
    if constexpr (DIR == 1) {
        if constexpr (VT == 1) {
            const int t = threadIdx.x;
            u64 xe[4], xo[4];
            LdPre<LD, 4> pe, po;
            load_pre<LD, 4>(J, 2 * t, 2048, pe);
            load_pre<LD, 4>(J, 2 * t + 1, 2048, po);
            pdl_wait();
            load_post<LD, 4>(C, J, P, 2 * t, 2048, pe, xe);
            load_post<LD, 4>(C, J, P, 2 * t + 1, 2048, po, xo);
            inv_first_stage(xe, xo, tw, t, P);
            HC_UNROLL
            for (int m = 0; m < 4; m++)
                *reinterpret_cast<ulonglong2*>(sm + pair_index(t, m)) = make_ulonglong2(xe[m], xo[m]);
        } else {
            pdl_wait();
            HC_NOUNROLL
            for (int v = 0; v < VT; v++) {
                const int t = threadIdx.x + v * (NT / VT);
                u64 xe[4], xo[4];
                load_n<LD, 4>(C, J, P, 2 * t, 2048, xe);
                load_n<LD, 4>(C, J, P, 2 * t + 1, 2048, xo);
                inv_first_stage(xe, xo, tw, t, P);
                HC_UNROLL
                for (int m = 0; m < 4; m++)
                    *reinterpret_cast<ulonglong2*>(sm + pair_index(t, m)) = make_ulonglong2(xe[m], xo[m]);
            }
        }
    } else if constexpr (VT == 1) {
        const int t = threadIdx.x;
        u64 x[EPT];  // coefficients t + 1024 e
        LdPre<LD, EPT> pre;
        load_pre<LD, EPT>(J, t, NT, pre);
        pdl_wait();
        load_post<LD, EPT>(C, J, P, t, NT, pre, x);
        // one schedule thread per thread: the loader's coefficients are pass
        // 0's, so stages 0..2 run before the first trip through the tile
        r8_ct(x, TwG{tw}, 0, 0, P.q, 2 * P.q2);
        HC_UNROLL
        for (int e = 0; e < EPT; e++) sm[swz(t) + NT * e] = x[e];
    } else {
        pdl_wait();
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const int t = threadIdx.x + v * (NT / VT);
            u64 x[EPT];  // coefficients t + 1024 e
            load_n<LD, EPT>(C, J, P, t, NT, x);
            HC_UNROLL
            for (int e = 0; e < EPT; e++) sm[swz(t) + NT * e] = x[e];
        }
    }
    __syncthreads();
    TRACE(1);
    // forward outputs that only feed Montgomery products stay lazy (< 2^60)
    constexpr bool lazy = EP == EP_KSACC || EP == EP_STORE_LAZY;
    if (DIR == 0) cta_ntt_fwd_core<VT, VT == 1 ? 1 : 0>(tw, P, sm);
    else cta_ntt_inv_core<VT, VT == 1>(tw, P, sm);
    TRACE(4);
    pdl_trigger();
    HC_NOUNROLL
    for (int v = 0; v < VT; v++) {
        const int t = threadIdx.x + v * (NT / VT);
        if constexpr (DIR == 0) {
            u64 xe[4], xo[4];
            HC_UNROLL
            for (int m = 0; m < 4; m++) {
                const ulonglong2 pr = *reinterpret_cast<const ulonglong2*>(sm + pair_index(t, m));
                xe[m] = pr.x;
                xo[m] = pr.y;
            }
            fwd_last_stage(xe, xo, tw, t, P, lazy);
            store_n<EP, 4>(C, J, P, 2 * t, 2048, xe);
            store_n<EP, 4>(C, J, P, 2 * t + 1, 2048, xo);
        } else {
            u64 x[EPT];
            HC_UNROLL
            for (int e = 0; e < EPT; e++) x[e] = sm[swz(t) + NT * e];
            if constexpr (VT == 1) c_phaseA_inv(x, tw, P);  // the last pass, in the epilogue's registers
            store_n<EP, EPT>(C, J, P, t, NT, x);
        }
    }
    TRACE(5);
}

// ---------------------------------------------------------------------------
// k_elem: transform-less jobs (loader with side store only), e.g. the c0
// half of a key-switch finish.  grid (NPOLY / 256, njobs), 128 threads x 2.
// ---------------------------------------------------------------------------
template <int LD>
__global__ void __launch_bounds__(128) k_elem(const __grid_constant__ DevCtx C, const XJob* __restrict__ jobs) {
    const XJob J = jobs[blockIdx.y];
    const PrimeC& P = C.pc[J.k];
    const int j0 = blockIdx.x * 256 + threadIdx.x;
    LdPre<LD, 2> pre;
    load_pre<LD, 2>(J, j0, 128, pre);
    pdl_wait();
    u64 x[2];
    load_post<LD, 2>(C, J, P, j0, 128, pre, x);
}

// ---------------------------------------------------------------------------
// k_xf_cl: latency path, one job per 8-CTA cluster (ntt_cl.cuh)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// DSMEM all-to-all of the cluster transforms.  Default: every value goes out
// as st.async to the peer CTA, whose mbarrier counts the incoming bytes
// (complete_tx); a CTA proceeds once its own receive buffer is full -- no
// cluster-wide release/acquire barrier (the latter costs a GPU-scope MEMBAR
// and an L1 invalidate per exchange).  HC_CLUSTER_BAR builds the barrier form
// (A/B).  Protocol: thread 0 initialises the CTA's mbarrier (one arrival) and
// posts the expected byte count before the kernel's start-of-cluster barrier;
// senders wait on that barrier before their first st.async.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void xch_init(u64* bar, uint32_t bytes) {
#ifndef HC_CLUSTER_BAR
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
#endif
}
// value v into the peer CTA `rank` at the address `dst` has in this CTA
__device__ __forceinline__ void xch_put(cooperative_groups::cluster_group& cl, u64* dst, int rank, u64 v, u64* bar) {
#ifndef HC_CLUSTER_BAR
    uint32_t ra, rb;
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(smem_u32(dst)), "r"(rank));
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];\n" ::"r"(ra), "l"(v), "r"(rb)
                 : "memory");
#else
    cl.map_shared_rank(dst, rank)[0] = v;
#endif
}
// all values destined to this CTA have landed (and are visible to this thread)
__device__ __forceinline__ void xch_wait(u64* bar) {
#ifndef HC_CLUSTER_BAR
    // bounded: a lost transfer traps (kernel error) instead of hanging the GPU
    for (unsigned it = 0;; it++) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar))
            : "memory");
        if (done) break;
        if (it > (1u << 26)) __trap();
    }
#else
    cluster_arrive_release();
    cluster_wait();
#endif
}

constexpr int CL_MAX = 60;  // jobs per cluster launch (passed by value): 15 clusters x 4
constexpr int CL_JPC_MAX = 4;  // transforms per cluster (one per 128-thread group of each CTA)
// dynamic smem of a cluster-transform CTA: JPC groups of [tile | recv (inverse) |
// twiddle slice] (<= 4 x 32 KiB), padded so every CTA of a cluster lands on its
// own SM (the scheduler would otherwise pack small CTAs onto one or two SMs)
constexpr int CL_GROUP_WORDS_FWD = CTILE + 2048, CL_GROUP_WORDS_INV = 2 * CTILE + 2048;
constexpr int CL_SMEM = 150 * 1024;
struct ClJobs {
    XJob j[CL_MAX];
    int n;  // jobs in this launch (the last cluster's spare groups idle)
    // optional transform-less key-switch finishes (LD_KSFIN, noxf; one per
    // prime) spread over every thread of a forward KSACC launch of >= 8 job slots:
    // a fold's res_f.c0 finish rides in the fold's digit-NTT launch instead of
    // a parallel graph branch (the digit products go to the other ACC buffer)
    int nside;
    XJob side[2];
};

// prefetch this CTA's 1023-entry twiddle slice (TwL) into shared memory;
// all 8 loads per thread are issued before the first shared store
// the CTA's twiddle slice: loads issued first (tw_issue, constant tables, so
// they overlap the data loads), stored to smem afterwards (tw_commit)
struct TwPre {
    ulonglong2 v[8];
};
__device__ __forceinline__ void tw_issue(TwPre& pre, const Tw* tw, int c, int t) {
    HC_UNROLL
    for (int i = 0; i < 8; i++) {
        const int L = t + CNT * i;
        const int Lc = L < 1023 ? L : 1022;
        const int e = 31 - __clz(Lc + 1);
        const int m8 = 1 << e;
        pre.v[i] = __ldg(reinterpret_cast<const ulonglong2*>(tw) + ((m8 << 3) + c * m8 + (Lc - (m8 - 1))));
    }
}
__device__ __forceinline__ void tw_commit(Tw* sl, const TwPre& pre, int t) {
    HC_UNROLL
    for (int i = 0; i < 8; i++) {
        const int L = t + CNT * i;
        if (L < 1023) reinterpret_cast<ulonglong2*>(sl)[L] = pre.v[i];
    }
}

// JPC transforms per cluster: thread group g = threadIdx.x / 128 of every CTA
// runs job (cluster * JPC + g) with its own tile / receive buffer / twiddle
// slice; the groups share the CTA and cluster barriers.  A small launch thus
// fits in one wave of co-resident clusters (e.g. 42 giant-step digit NTTs:
// 14 clusters of 3 instead of three sequential launches of <= 15), and the
// extra warps per SM hide the butterflies' latency.
template <int DIR, int LD, int EP, int JPC>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(CNT * JPC)
    k_xf_cl(const __grid_constant__ DevCtx C, const __grid_constant__ ClJobs jobs) {
    extern __shared__ __align__(16) u64 csm[];
    constexpr int GW = DIR ? CL_GROUP_WORDS_INV : CL_GROUP_WORDS_FWD;
    const int grp = JPC == 1 ? 0 : (int)(threadIdx.x >> 7);
    u64* tile = csm + grp * GW;
    u64* recv = tile + CTILE;  // inverse only
    Tw* twsl = reinterpret_cast<Tw*>(tile + (DIR ? 2 : 1) * CTILE);
    u64* xbar = csm + JPC * GW;  // exchange mbarrier (one per CTA)
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    const int c = (int)cl.block_rank();
    const int t = threadIdx.x & (CNT - 1);
    xch_init(xbar, JPC * CTILE * 8);  // every group receives 1024 values
    cluster_arrive_relaxed();  // "this CTA has started" (waited on before DSMEM stores)
    const int jid = (blockIdx.x / CL) * JPC + grp;
    const bool valid = jid < jobs.n;  // spare group of the last cluster: barriers only
    const XJob& J = jobs.j[valid ? jid : jobs.n - 1];
    TRACE(0);
    const PrimeC& P = C.pc[J.k];
    const TwL twl{twsl, c};
    u64 x[CEPT];
    if (DIR == 0) {
        const Tw* tw = C.twf + (size_t)J.k * NPOLY;
        TwPre pre;
        tw_issue(pre, tw, c, t);
        Tw wa[8];
        HC_UNROLL
        for (int i = 1; i < 8; i++) wa[i] = ldtw(tw, i);  // phase-A twiddles tbl[1..7]
        const int b = 128 * c + t;
        LdPre<LD, CEPT> lpre;
        if (valid) load_pre<LD, CEPT>(J, b, CTILE, lpre);
        // key digits of the KSACC epilogue: constant, fetched before the wait
        u64 ka[EP == EP_KSACC ? CEPT : 1], kb[EP == EP_KSACC ? CEPT : 1];
        if constexpr (EP == EP_KSACC) {
            if (valid) {
                HC_UNROLL
                for (int v = 0; v < CEPT; v++) {
                    ka[v] = J.ea[c * CTILE + t + 128 * v];
                    kb[v] = J.eb[c * CTILE + t + 128 * v];
                }
            }
        }
        constexpr bool SIDE = EP == EP_KSACC;
        const bool side = SIDE && jobs.nside;
        const int gt = blockIdx.x * blockDim.x + threadIdx.x, gT = gridDim.x * blockDim.x;  // gT >= n (host-checked)
        LdPre<LD_KSFIN, 1> sp[2];
        KsLd<1> sv[2];
        if constexpr (SIDE) {
            if (side) {
                HC_UNROLL
                for (int i = 0; i < 2; i++) {
                    const int e = gt + i * gT;
                    if (e < 2 * NPOLY) ksfin_pre<1>(jobs.side[e >> 13], e & (NPOLY - 1), 0, sp[i]);
                }
            }
        }
        pdl_wait();
        if (valid) load_post<LD, CEPT>(C, J, P, b, CTILE, lpre, x);
        else
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) x[v] = 0;
        if constexpr (SIDE) {
            if (side) {
                HC_UNROLL
                for (int i = 0; i < 2; i++) {
                    const int e = gt + i * gT;
                    if (e < 2 * NPOLY) ksfin_load<1>(jobs.side[e >> 13], C.pc[jobs.side[e >> 13].k], e & (NPOLY - 1), 0, sp[i], sv[i]);
                }
            }
        }
        TRACE(6);
        tw_commit(twsl, pre, t);
        TRACE(7);
        r8_ct(x, TwR{wa}, 0, 0, P.q, 2 * P.q2);
        if constexpr (SIDE) {
            if (side) {
                HC_UNROLL
                for (int i = 0; i < 2; i++) {
                    const int e = gt + i * gT;
                    if (e < 2 * NPOLY) {
                        u64 y[1];
                        ksfin_finish<1>(jobs.side[e >> 13], C.pc[jobs.side[e >> 13].k], e & (NPOLY - 1), 0, sp[i], sv[i], y);
                    }
                }
            }
        }
        TRACE(1);
        cluster_wait();
        TRACE(2);
        HC_UNROLL
        for (int r = 0; r < CEPT; r++) xch_put(cl, tile + cswz(b), r, x[r], xbar);
        xch_wait(xbar);
        __syncthreads();  // this CTA's twiddle-slice stores
        TRACE(3);
        HC_UNROLL
        for (int p = 0; p < 3; p++) {
            const CPass I = cpass(p, c, t);
            c_load(x, tile, I);
            r8_ct(x, twl, I.s0, I.G, P.q, 2 * P.q2);
            if (p == 2) c_st12<EP == EP_KSACC || EP == EP_STORE_LAZY>(c, t, x, twl, P.q, 2 * P.q2, P.one_s);
            c_store(x, tile, I);
            __syncthreads();
        }
        TRACE(4);
        pdl_trigger();
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) x[v] = tile[cswz(t) + 128 * v];
        if (!valid) {
        } else if constexpr (EP == EP_KSACC) {
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) {
                const int j = c * CTILE + t + 128 * v;
                acc_add(J.out + j, mul_mont(x[v], ka[v], P.q, P.qneg), KSACC_BOUND);
                acc_add(J.out + J.ostride + j, mul_mont(x[v], kb[v], P.q, P.qneg), KSACC_BOUND);
            }
        } else {
            store_n<EP, CEPT>(C, J, P, c * CTILE + t, 128, x);
        }
        TRACE(5);
    } else {
        const Tw* tw = C.twi + (size_t)J.k * NPOLY;
        TwPre pre;
        tw_issue(pre, tw, c, t);
        LdPre<LD, CEPT> lpre;
        if (valid) load_pre<LD, CEPT>(J, c * CTILE + t, 128, lpre);
        pdl_wait();
        if (valid) load_post<LD, CEPT>(C, J, P, c * CTILE + t, 128, lpre, x);
        else
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) x[v] = 0;
        tw_commit(twsl, pre, t);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) tile[cswz(t) + 128 * v] = x[v];
        __syncthreads();
        TRACE(1);
        HC_UNROLL
        for (int p = 0; p < 3; p++) {
            const CPass I = cpass(2 - p, c, t);
            c_load(x, tile, I);
            if (p == 0) c_st0(c, t, x, twl, P.q, P.q2);
            r8_gs(x, twl, 1 + 3 * p, I.G, P.q, 2 * P.q2);
            if (p < 2) {
                c_store(x, tile, I);
                __syncthreads();
            }
        }
        // all-to-all: element (row c, column t + 128 v) -> CTA v, slot c*128 + t
        TRACE(4);
        pdl_trigger();
        cluster_wait();
        TRACE(2);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) xch_put(cl, recv + c * 128 + t, v, x[v], xbar);
        xch_wait(xbar);
        TRACE(3);
        HC_UNROLL
        for (int r = 0; r < CEPT; r++) x[r] = recv[r * 128 + t];
        c_phaseA_inv(x, tw, P);
        if (valid) store_n<EP, CEPT>(C, J, P, 128 * c + t, CTILE, x);
        TRACE(5);
    }
}

// ---------------------------------------------------------------------------
// k_cl_intt2: level-1 key-switch front end on one 8-CTA cluster.  Inverts
// BOTH primes of a c1 polynomial (the two INTTs of a tail key switch,
// interleaved per thread for ILP), then splits each coefficient's CRT
// integer into base-2^16 digits of X and of Q - X (k_compose mode 1) in the
// epilogue, so the following digit NTTs only gather u16 digits (LD_DIGGAL)
// instead of re-composing every coefficient 14 times.
//   j[0] / j[1]: the two primes' loader jobs (k = 0, 1; LD_KSFIN or LD_RED,
//   optional aux side store); E: optional coefficient-domain addend
//   ([2][n], reduced with red64) applied before the split (T1 of the tail:
//   acc[g].c1 = INTT(X) + E).
// ---------------------------------------------------------------------------
struct Intt2Job {
    XJob j[2];
    const u64* E;
    uint16_t* dig;  // [2 * D_1][n]: digits of X, then of Q - X
};
constexpr int I2_MAX = 8;
struct Intt2Jobs {
    Intt2Job j[I2_MAX];
};

template <int LD>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(2 * CNT)
    k_cl_intt2(const __grid_constant__ DevCtx C, const __grid_constant__ Intt2Jobs jobs) {
    // threads [0,128) invert prime 0, [128,256) prime 1 (one INTT chain per
    // thread, as in k_xf_cl); the CRT/digit split is then shared by all 256
    extern __shared__ u64 dsm[];  // 2 tiles, 2 receive buffers, 2 twiddle slices
    const int pr = threadIdx.x >> 7;
    const int t = threadIdx.x & 127;
    u64* tile = dsm + pr * CTILE;
    u64* recvb = dsm + (2 + pr) * CTILE;
    Tw* twsl = reinterpret_cast<Tw*>(dsm + 4 * CTILE) + pr * 1024;
    u64* xbar = dsm + 8 * CTILE;  // after the two twiddle slices
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    const int c = (int)cl.block_rank();
    xch_init(xbar, 2 * CTILE * 8);
    cluster_arrive_relaxed();
    const Intt2Job& JJ = jobs.j[blockIdx.x / CL];
    const XJob& J = JJ.j[pr];
    TRACE(0);
    const PrimeC& P = C.pc[pr];
    const Tw* tw = C.twi + (size_t)pr * NPOLY;
    u64 x[CEPT];
    TwPre pre;
    tw_issue(pre, tw, c, t);
    const int jl = c * CTILE + t;
    LdPre<LD, CEPT> lpre;
    load_pre<LD, CEPT>(J, jl, 128, lpre);
    pdl_wait();
    load_post<LD, CEPT>(C, J, P, jl, 128, lpre, x);
    tw_commit(twsl, pre, t);
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) tile[cswz(t) + 128 * v] = x[v];
    __syncthreads();
    TRACE(1);
    const TwL twl{twsl, c};
    HC_UNROLL
    for (int p = 0; p < 3; p++) {
        const CPass I = cpass(2 - p, c, t);
        c_load(x, tile, I);
        if (p == 0) c_st0(c, t, x, twl, P.q, P.q2);
        r8_gs(x, twl, 1 + 3 * p, I.G, P.q, 2 * P.q2);
        if (p < 2) {
            c_store(x, tile, I);
            __syncthreads();
        }
    }
    TRACE(4);
    pdl_trigger();
    cluster_wait();
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) xch_put(cl, recvb + c * 128 + t, v, x[v], xbar);
    xch_wait(xbar);
    TRACE(3);
    HC_UNROLL
    for (int r = 0; r < CEPT; r++) x[r] = recvb[r * 128 + t];
    c_phaseA_inv(x, tw, P);
    // x[r] = coefficient r*1024 + 128c + t mod q_pr; park it (local index r*128 + t)
    HC_UNROLL
    for (int r = 0; r < CEPT; r++) tile[r * 128 + t] = x[r];
    __syncthreads();
    const LevelC& LV = C.lv(1);
    const int D = LV.D;
    const u64* E = JJ.E;
    uint16_t* dig = JJ.dig;
    u64* out0 = JJ.j[0].out;
    u64* out1 = JJ.j[1].out;
    const u64* tile0 = dsm;
    const u64* tile1 = dsm + CTILE;
    // each thread: 4 adjacent coefficients (local L = 4 tt + i), so every
    // digit index is one 8-byte store of 4 digits (coalesced across the warp)
    const int L0 = 4 * threadIdx.x;
    const int j0 = (L0 >> 7) * CTILE + 128 * c + (L0 & 127);
    u64 a[4], b[4];
    HC_UNROLL
    for (int i = 0; i < 4; i++) {
        a[i] = tile0[L0 + i];
        b[i] = tile1[L0 + i];
    }
    if (E) {
        HC_UNROLL
        for (int i = 0; i < 4; i++) {
            a[i] = add_mod(a[i], red64(E[j0 + i], C.pc[0].q, C.pc[0].one_s), C.pc[0].q);
            b[i] = add_mod(b[i], red64(E[NPOLY + j0 + i], C.pc[1].q, C.pc[1].one_s), C.pc[1].q);
        }
    }
    if (out0) {  // optional coefficient side store
        HC_UNROLL
        for (int i = 0; i < 4; i++) {
            out0[j0 + i] = a[i];
            out1[j0 + i] = b[i];
        }
    }
    u64 X[4][NLIMB];
    HC_UNROLL
    for (int i = 0; i < 4; i++) compose2(LV, C.pc, a[i], b[i], X[i]);
    HC_UNROLL
    for (int d = 0; d < 8; d++)
        if (d < D)
            *reinterpret_cast<ushort4*>(dig + (size_t)d * NPOLY + j0) =
                make_ushort4(digit16(X[0], d), digit16(X[1], d), digit16(X[2], d), digit16(X[3], d));
    HC_UNROLL
    for (int i = 0; i < 4; i++) neg_mod_Q<1>(LV, X[i]);
    HC_UNROLL
    for (int d = 0; d < 8; d++)
        if (d < D)
            *reinterpret_cast<ushort4*>(dig + (size_t)(D + d) * NPOLY + j0) =
                make_ushort4(digit16(X[0], d), digit16(X[1], d), digit16(X[2], d), digit16(X[3], d));
    TRACE(5);
}

// ---------------------------------------------------------------------------
// k_cl16_intt2: the same job on a 16-CTA cluster (non-portable size, launched
// with a runtime cluster dimension): CTAs 0-7 invert prime 0, CTAs 8-15 prime
// 1, one INTT per CTA group as in k_xf_cl (128 threads x 8 coefficients), so
// each SM carries half the butterflies of k_cl_intt2 (whose passes ran at
// ~0.77 of the butterfly peak of one SM -- throughput-, not latency-bound).
// Then CTA (0, c) and CTA (1, c), which hold the same coefficients mod the
// two primes, swap halves over DSMEM and each composes 512 of them.
// ---------------------------------------------------------------------------
template <int LD>
__global__ void __launch_bounds__(CNT) k_cl16_intt2(const __grid_constant__ DevCtx C, const __grid_constant__ Intt2Jobs jobs) {
    extern __shared__ u64 dsm[];  // tile | recv | twiddle slice | half-exchange buffer | 2 mbarriers
    u64* tile = dsm;
    u64* recvb = dsm + CTILE;
    Tw* twsl = reinterpret_cast<Tw*>(dsm + 2 * CTILE);
    u64* half = dsm + 4 * CTILE;        // 4 x 128 values from the partner CTA
    u64* xbar = dsm + 4 * CTILE + 512;  // INTT all-to-all
    u64* hbar = xbar + 1;               // half exchange
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    const int rank = (int)cl.block_rank();
    const int pr = rank >> 3, c = rank & 7;
    const int t = threadIdx.x;
    xch_init(xbar, CTILE * 8);
    xch_init(hbar, 4 * CNT * 8);
    cluster_arrive_relaxed();
    const Intt2Job& JJ = jobs.j[blockIdx.x / 16];
    const XJob& J = JJ.j[pr];
    TRACE(0);
    const PrimeC& P = C.pc[pr];
    const Tw* tw = C.twi + (size_t)pr * NPOLY;
    u64 x[CEPT];
    TwPre pre;
    tw_issue(pre, tw, c, t);
    Tw wa[8];
    HC_UNROLL
    for (int i = 1; i < 8; i++) wa[i] = ldtw(tw, i);
    const int jl = c * CTILE + t;
    LdPre<LD, CEPT> lpre;
    load_pre<LD, CEPT>(J, jl, 128, lpre);
    pdl_wait();
    load_post<LD, CEPT>(C, J, P, jl, 128, lpre, x);
    tw_commit(twsl, pre, t);
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) tile[cswz(t) + 128 * v] = x[v];
    __syncthreads();
    TRACE(1);
    const TwL twl{twsl, c};
    HC_UNROLL
    for (int p = 0; p < 3; p++) {
        const CPass I = cpass(2 - p, c, t);
        c_load(x, tile, I);
        if (p == 0) c_st0(c, t, x, twl, P.q, P.q2);
        r8_gs(x, twl, 1 + 3 * p, I.G, P.q, 2 * P.q2);
        if (p < 2) {
            c_store(x, tile, I);
            __syncthreads();
        }
    }
    TRACE(4);
    pdl_trigger();
    cluster_wait();
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) xch_put(cl, recvb + c * 128 + t, pr * 8 + v, x[v], xbar);
    xch_wait(xbar);
    HC_UNROLL
    for (int r = 0; r < CEPT; r++) x[r] = recvb[r * 128 + t];
    c_phaseA_inv_w(x, wa, P);
    // x[r] = coefficient r*1024 + 128c + t mod q_pr.  Prime-0 CTAs compose
    // r = 0..3, prime-1 CTAs r = 4..7: send the other half to the partner.
    const int partner = (1 - pr) * 8 + c;
    const int mine0 = pr ? 4 : 0, theirs0 = pr ? 0 : 4;
    HC_UNROLL
    for (int i = 0; i < 4; i++) xch_put(cl, half + i * CNT + t, partner, x[theirs0 + i], hbar);
    xch_wait(hbar);
    TRACE(3);
    const LevelC& LV = C.lv(1);
    const int D = LV.D;
    const u64* E = JJ.E;
    uint16_t* dig = JJ.dig;
    u64* out0 = JJ.j[0].out;
    u64* out1 = JJ.j[1].out;
    u64 a[4], b[4];
    int jj[4];
    HC_UNROLL
    for (int i = 0; i < 4; i++) {
        const u64 mine = x[mine0 + i], other = half[i * CNT + t];
        a[i] = pr ? other : mine;  // residue mod q0
        b[i] = pr ? mine : other;  // residue mod q1
        jj[i] = (mine0 + i) * CTILE + 128 * c + t;
    }
    if (E) {
        HC_UNROLL
        for (int i = 0; i < 4; i++) {
            a[i] = add_mod(a[i], red64(E[jj[i]], C.pc[0].q, C.pc[0].one_s), C.pc[0].q);
            b[i] = add_mod(b[i], red64(E[NPOLY + jj[i]], C.pc[1].q, C.pc[1].one_s), C.pc[1].q);
        }
    }
    if (out0) {  // optional coefficient side store
        HC_UNROLL
        for (int i = 0; i < 4; i++) {
            out0[jj[i]] = a[i];
            out1[jj[i]] = b[i];
        }
    }
    u64 X[4][NLIMB];
    HC_UNROLL
    for (int i = 0; i < 4; i++) compose2(LV, C.pc, a[i], b[i], X[i]);
    HC_UNROLL
    for (int d = 0; d < 8; d++)
        if (d < D)
            HC_UNROLL
            for (int i = 0; i < 4; i++) dig[(size_t)d * NPOLY + jj[i]] = digit16(X[i], d);
    HC_UNROLL
    for (int i = 0; i < 4; i++) neg_mod_Q<1>(LV, X[i]);
    HC_UNROLL
    for (int d = 0; d < 8; d++)
        if (d < D)
            HC_UNROLL
            for (int i = 0; i < 4; i++) dig[(size_t)(D + d) * NPOLY + jj[i]] = digit16(X[i], d);
    TRACE(5);
}
constexpr int CL16_SMEM = (4 * CTILE + 512 + 2) * 8;

// ---------------------------------------------------------------------------
// k_compose: grid (n/256, njobs)
// ---------------------------------------------------------------------------
struct CJob {
    int level;
    int mode;  // 0: digits of (gathered, signed) X -> dig[D][n]; 1: X and Q-X -> dig[2][D][n]
    const u64* x;      // [P][xstride]
    const u64* xadd;   // optional addend, same layout
    long long xstride;
    const uint16_t* gal;  // mode 0: optional coefficient-domain gather
    uint16_t* dig;
};

template <int L>
__device__ __forceinline__ void compose_one(const DevCtx& C, const CJob& J, int pos, unsigned e) {
    const LevelC& LV = C.lv(L);
    constexpr int P = L + 1;
    const int D = LV.D;
    int src = pos, neg = 0;
    if (J.mode == 0 && J.gal) {
        src = e & 0x7FFF;
        neg = e >> 15;
    }
    u64 xr[P];
    HC_UNROLL
    for (int k = 0; k < P; k++) {
        u64 v = J.x[(size_t)k * J.xstride + src];
        if (J.xadd) v = add_mod(v, J.xadd[(size_t)k * J.xstride + src], C.pc[k].q);
        xr[k] = v;
    }
    u64 X[NLIMB];
    crt_compose<L>(LV, C.pc, xr, X);
    constexpr int DMAX = 4 * (L + 1);
    if (J.mode == 0) {
        if (neg) neg_mod_Q<L>(LV, X);
        HC_UNROLL
        for (int j = 0; j < DMAX; j++)
            if (j < D) J.dig[(size_t)j * NPOLY + pos] = digit16(X, j);
    } else {
        HC_UNROLL
        for (int j = 0; j < DMAX; j++)
            if (j < D) J.dig[(size_t)j * NPOLY + pos] = digit16(X, j);
        neg_mod_Q<L>(LV, X);
        HC_UNROLL
        for (int j = 0; j < DMAX; j++)
            if (j < D) J.dig[(size_t)(D + j) * NPOLY + pos] = digit16(X, j);
    }
}

__global__ void __launch_bounds__(256) k_compose(const __grid_constant__ DevCtx C, const CJob* __restrict__ jobs) {
    const CJob J = jobs[blockIdx.y];
    const int pos = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned e = (J.mode == 0 && J.gal) ? J.gal[pos] : 0u;  // constant gather table: before the wait
    pdl_wait();
    switch (J.level) {
        case 1: compose_one<1>(C, J, pos, e); break;
        case 2: compose_one<2>(C, J, pos, e); break;
        case 3: compose_one<3>(C, J, pos, e); break;
        default: break;
    }
}

// ---------------------------------------------------------------------------
// k_ksmac<CPT>: grid (n/(256 CPT), P, njobs)
//   out0 = add0 + sum_t ( c0src_t[perm_t[j]] + sum_j dntt_t[j] * b_t[j] )
//   out1 = add1 + sum_t ( sum_j dntt_t[j] * a_t[j] )
// dntt: [D][P][n]; key: [D_L][2][L+1][n] (Montgomery form).
// ---------------------------------------------------------------------------
constexpr int MAXTERM = 8;
struct MTerm {
    const u64* dntt;
    const u64* key;
    const u64* c0src;     // [P][n] NTT domain (nullable)
    const uint16_t* perm; // NTT-domain Galois permutation for c0src
};
struct MJob {
    int level, nterm;
    int trace, pad;  // HC_TRACE builds: launch sequence number
    MTerm t[MAXTERM];
    const u64* add0;
    const u64* add1;
    u64* out0;
    u64* out1;
};

// CPT adjacent coefficients per thread: 1 at scale (low register count, the
// digit loads of many warps in flight), 2 for small launches that share the
// SMs with transform CTAs (fewer CTAs).  Digits are loaded KSB at a time
// (every load of a batch in flight before its MACs: the loop is bound by
// memory latency, not bandwidth, at the latency-path launch sizes); the
// Galois permutation of the c0 term is constant and read before pdl_wait().
template <int CPT, int KSB>
__global__ void __launch_bounds__(256, KSB == 1 ? 5 : 3) k_ksmac(const __grid_constant__ DevCtx C, const MJob* __restrict__ jobs) {
    const MJob& J = jobs[blockIdx.z];
    TRACE(0);
    const int k = blockIdx.y;
    const int j = CPT * (blockIdx.x * blockDim.x + threadIdx.x);
    const LevelC& LV = C.lv(J.level);
    const int P = LV.P, D = LV.D, L1 = C.KL1;
    const PrimeC pc = C.pc[k];
    const size_t kn = (size_t)k * NPOLY + j;
    const int nt = J.nterm;
    unsigned pe0[CPT];  // term 0's c0 permutation (constant)
    if (J.t[0].c0src) {
        HC_UNROLL
        for (int c = 0; c < CPT; c++) pe0[c] = J.t[0].perm[j + c];
    }
    pdl_wait();
    u64 o0[CPT], o1[CPT];
    HC_UNROLL
    for (int c = 0; c < CPT; c++) {
        o0[c] = J.add0 ? J.add0[kn + c] : 0;
        o1[c] = J.add1 ? J.add1[kn + c] : 0;
    }
    const size_t vstep = (size_t)P * NPOLY, kstep = (size_t)2 * L1 * NPOLY, astep = (size_t)L1 * NPOLY;
    for (int t = 0; t < nt; t++) {
        const MTerm T = J.t[t];
        u64 h0[CPT], l0[CPT], h1[CPT], l1[CPT];
        HC_UNROLL
        for (int c = 0; c < CPT; c++) h0[c] = l0[c] = h1[c] = l1[c] = 0;
        const u64* vp = T.dntt + kn;
        const u64* bp = T.key + kn;
        u64 c0v[CPT];
#pragma unroll(KSB == 1 ? 4 : 1)  // batched digits: one batch body (registers); single digits: unrolled
        for (int d0 = 0; d0 < D; d0 += KSB) {
            u64 v[KSB][CPT], kb[KSB][CPT], ka[KSB][CPT];
            HC_UNROLL
            for (int i = 0; i < KSB; i++) {
                if (d0 + i < D) {
                    const int d = d0 + i;
                    if constexpr (CPT == 2) {
                        const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(vp + d * vstep));
                        const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(bp + d * kstep));
                        const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(bp + d * kstep + astep));
                        v[i][0] = a.x; v[i][1] = a.y; kb[i][0] = b.x; kb[i][1] = b.y; ka[i][0] = e.x; ka[i][1] = e.y;
                    } else {
                        v[i][0] = __ldcs(vp + d * vstep);
                        kb[i][0] = __ldg(bp + d * kstep);
                        ka[i][0] = __ldg(bp + d * kstep + astep);
                    }
                }
            }
            if (d0 == 0 && T.c0src) {  // the c0 gather, in flight with the first batch
                const u64* c0 = T.c0src + (size_t)k * NPOLY;
                HC_UNROLL
                for (int c = 0; c < CPT; c++) c0v[c] = c0[t == 0 ? pe0[c] : T.perm[j + c]];
            }
            HC_UNROLL
            for (int i = 0; i < KSB; i++) {
                if (d0 + i < D) {
                    HC_UNROLL
                    for (int c = 0; c < CPT; c++) {
                        mac128(h0[c], l0[c], v[i][c], kb[i][c]);
                        mac128(h1[c], l1[c], v[i][c], ka[i][c]);
                    }
                }
            }
        }
        HC_UNROLL
        for (int c = 0; c < CPT; c++) {
            HC_ASSERT(h0[c] < pc.q && h1[c] < pc.q);  // REDC precondition of the digit MAC
            o0[c] = add_mod(o0[c], redc(h0[c], l0[c], pc.q, pc.qneg), pc.q);
            o1[c] = add_mod(o1[c], redc(h1[c], l1[c], pc.q, pc.qneg), pc.q);
        }
        TRACE(1);
        if (T.c0src) {
            HC_UNROLL
            for (int c = 0; c < CPT; c++) o0[c] = add_mod(o0[c], c0v[c], pc.q);
        }
    }
    TRACE(4);
    HC_UNROLL
    for (int c = 0; c < CPT; c++) {
        J.out0[kn + c] = o0[c];
        J.out1[kn + c] = o1[c];
    }
    TRACE(5);
}

// ---------------------------------------------------------------------------
// k_ksmac_mb<NB>: the throughput-regime key-switch MAC over up to NB blocks
// that share one key (the same rotation or the column swap of different
// blocks): each thread loads a key digit pair once and applies it to every
// block's digit NTT, so the key stream is read once per group instead of once
// per block.  Same sums and output as k_ksmac with nterm = 1.
// grid (n/256, P, ngroups).
// ---------------------------------------------------------------------------
constexpr int MB_MAX = 4;
struct MBJob {
    int level, nb;
    int trace, pad;             // HC_TRACE builds: launch sequence number
    const u64* key;             // [D_L][2][L+1][n] Montgomery, shared by the group
    const uint16_t* perm;       // c0 permutation (shared), with c0src
    const u64* dntt[MB_MAX];    // [D][P][n] per block
    const u64* c0src[MB_MAX];   // [P][n] (nullable)
    const u64* add0[MB_MAX];
    const u64* add1[MB_MAX];
    u64* out0[MB_MAX];
    u64* out1[MB_MAX];
};

template <int NB>
__global__ void __launch_bounds__(256) k_ksmac_mb(const __grid_constant__ DevCtx C, const MBJob* __restrict__ jobs) {
    const MBJob& J = jobs[blockIdx.z];
    TRACE(0);
    const int k = blockIdx.y;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const LevelC& LV = C.lv(J.level);
    const int P = LV.P, D = LV.D, L1 = C.KL1;
    const PrimeC pc = C.pc[k];
    const size_t kn = (size_t)k * NPOLY + j;
    const unsigned pe = J.perm ? J.perm[j] : 0u;
    const int nb = J.nb;
    pdl_wait();
    u64 h0[NB], l0[NB], h1[NB], l1[NB];
    HC_UNROLL
    for (int b = 0; b < NB; b++) h0[b] = l0[b] = h1[b] = l1[b] = 0;
    const u64* bp = J.key + kn;
    const size_t vstep = (size_t)P * NPOLY, kstep = (size_t)2 * L1 * NPOLY, astep = (size_t)L1 * NPOLY;
#pragma unroll 2
    for (int d = 0; d < D; d++) {
        const u64 kb = __ldg(bp + d * kstep);
        const u64 ka = __ldg(bp + d * kstep + astep);
        u64 v[NB];
        HC_UNROLL
        for (int b = 0; b < NB; b++) v[b] = b < nb ? __ldcs(J.dntt[b] + kn + d * vstep) : 0;
        HC_UNROLL
        for (int b = 0; b < NB; b++) {
            mac128(h0[b], l0[b], v[b], kb);
            mac128(h1[b], l1[b], v[b], ka);
        }
    }
    TRACE(4);
    HC_UNROLL
    for (int b = 0; b < NB; b++) {
        if (b >= nb) break;
        HC_ASSERT(h0[b] < pc.q && h1[b] < pc.q);
        u64 o0 = redc(h0[b], l0[b], pc.q, pc.qneg), o1 = redc(h1[b], l1[b], pc.q, pc.qneg);
        if (J.add0[b]) o0 = add_mod(o0, J.add0[b][kn], pc.q);
        if (J.add1[b]) o1 = add_mod(o1, J.add1[b][kn], pc.q);
        if (J.c0src[b]) o0 = add_mod(o0, J.c0src[b][(size_t)k * NPOLY + pe], pc.q);
        J.out0[b][kn] = o0;
        J.out1[b][kn] = o1;
    }
    TRACE(5);
}

// ---------------------------------------------------------------------------
// k_diagx: grid (n/256, 1, njobs), the two kept primes per thread.  X[k][j] += sum_t src_t[k][j] * dg_t[k][j]
// (dg Montgomery with q^-1 folded in) -- the kept-prime half of each
// plaintext product -- and E[k][j] += sum_t d_t - (sum_t r_t) q_l^-1 from the
// (r, d) slots the dropped-prime INTTs wrote (EP_RESCALE_RD).
// ---------------------------------------------------------------------------
struct DXJob {
    int nterm, level;       // level: of the dropped prime behind the (r, d) slots
    int trace;              // HC_TRACE builds: launch sequence number
    int atomic;             // 1: add into X / E with atomics (concurrent launches; words < 4q)
    const u64* const* src;  // nterm pointers, each [>=nprime][n]
    const u64* const* dg;   // nterm pointers, each [>=nprime][n]
    const u64* const* es;   // nterm (r, d) slots [2][n] int64 (EP_RESCALE_RD), or null
    u64* X;                 // [nprime][n], canonical, updated in place
    u64* E;                 // [nprime][n], += sum of the slots' corrections (mod q)
};

// one coefficient per thread, both kept primes, so every (r, d) slot is read
// once; terms in batches of DXB (pointers, then all loads, then the MACs)
constexpr int DXB = 4;
__global__ void __launch_bounds__(256) k_diagx(const __grid_constant__ DevCtx C, const DXJob* __restrict__ jobs) {
    const DXJob& J = jobs[blockIdx.z];
    TRACE(0);
    pdl_wait();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const u64 q0 = C.pc[0].q, q1 = C.pc[1].q;
    u64 h0 = 0, l0 = 0, h1 = 0, l1 = 0;
    long long sr = 0, sd = 0;
    const int nt = J.nterm;
    const u64* const* src = J.src;
    const u64* const* dg = J.dg;
    const u64* const* es = J.es;
    for (int t0 = 0; t0 < nt; t0 += DXB) {
        u64 a0[DXB], a1[DXB], b0[DXB], b1[DXB], r[DXB], d[DXB];
        HC_UNROLL
        for (int i = 0; i < DXB; i++)
            if (t0 + i < nt) {
                const u64* sp = src[t0 + i];
                const u64* gp = dg[t0 + i];
                a0[i] = __ldcs(sp + j);
                a1[i] = __ldcs(sp + NPOLY + j);
                b0[i] = __ldg(gp + j);
                b1[i] = __ldg(gp + NPOLY + j);
                if (es) {
                    r[i] = __ldcs(es[t0 + i] + j);
                    d[i] = __ldcs(es[t0 + i] + NPOLY + j);
                }
            }
        HC_UNROLL
        for (int i = 0; i < DXB; i++)
            if (t0 + i < nt) {
                mac128(h0, l0, a0[i], b0[i]);
                mac128(h1, l1, a1[i], b1[i]);
                if (es) {  // |r| < 2^53, nterm <= 1024: exact in int64
                    sr += (long long)r[i];
                    sd += (long long)d[i];
                }
            }
    }
    TRACE(1);
    HC_ASSERT(nt <= 1024 && h0 < q0 && h1 < q1);  // one REDC of the 128-bit sums (sum < q 2^64)
    const u64 x0 = redc(h0, l0, q0, C.pc[0].qneg), x1 = redc(h1, l1, q1, C.pc[1].qneg);
    u64 e0 = 0, e1 = 0;
    if (es) {
        const LevelC& LV = C.lv(J.level);
        e0 = corr_from_sums(sr, sd, q0, LV.qinv[0], LV.qinv_s[0], C.pc[0].one_s);
        e1 = corr_from_sums(sr, sd, q1, LV.qinv[1], LV.qinv_s[1], C.pc[1].one_s);
    }
    if (J.atomic) {
        acc_add(J.X + j, x0, PX_BOUND);
        acc_add(J.X + NPOLY + j, x1, PX_BOUND);
        if (es) {
            acc_add(J.E + j, e0, PX_BOUND);
            acc_add(J.E + NPOLY + j, e1, PX_BOUND);
        }
    } else {
        J.X[j] = add_mod(J.X[j], x0, q0);
        J.X[NPOLY + j] = add_mod(J.X[NPOLY + j], x1, q1);
        if (es) {
            J.E[j] = add_mod(J.E[j], e0, q0);
            J.E[NPOLY + j] = add_mod(J.E[NPOLY + j], e1, q1);
        }
    }
    TRACE(4);
    TRACE(5);
}

// ---------------------------------------------------------------------------
// k_plain: on-device plaintext encoding, one CTA per plaintext.
// Slot values (compress.py:186-195 diagonals / :242-243,351-352 masks) ->
// slot_encode (INTT mod p, bgv.py:379-385) -> NTT mod q_k (bgv.py:452-460)
// -> Montgomery form with the modulus-switch factor folded in:
//   k == level (dropped prime): pt * R;  k < level: pt * q_level^-1 * R.
// ---------------------------------------------------------------------------
// PT_ONE: the modulus switch of add's _at_level; PT_DBVEC: block t of the
// cleartext database vector (pdq.mask's _db_block_matrices, pdq.py:207-208)
enum : int { PT_DIAG = 0, PT_TOP = 1, PT_BOT = 2, PT_OUTMASK = 3, PT_ONE = 4, PT_DBVEC = 5 };
struct PJob {
    int kind, t, g, b, level, pad;
    u64* out;  // [level+1][n]
};
struct PlanShape {
    long long N;
    int s, s_pad, baby, m;
    const uint32_t* db;  // comp_masked: cleartext DB mod p scaling row 1 (D = C diag(DB)), or null
};

HD u64 powmod_small(u64 b, int e, u64 p, double pinv) {
    u64 r = 1;
    while (e) {
        if (e & 1) r = mod_small(r * b, p, pinv);
        b = mod_small(b * b, p, pinv);
        e >>= 1;
    }
    return r;
}

HD u64 plain_slot_value(const PJob& J, const PlanShape& S, int r, int c, u64 p, double pinv) {
    switch (J.kind) {
        case PT_DIAG: {
            // entry[pos=c] = M[(c - g*baby) mod s_pad][(c + b) mod m], M[row][col] = (t*m+col+1)^(row+1)
            int row = ((c - J.g * S.baby) % S.s_pad + S.s_pad) % S.s_pad;
            int col = (c + J.b) % S.m;
            long long idx = (long long)J.t * S.m + col + 1;
            if (row >= S.s || idx > S.N) return 0;
            const u64 v = powmod_small((u64)(idx % (long long)p), row + 1, p, pinv);
            // precompute_masked_matrix (compress.py:154-157,131-135): the bottom
            // lane's table is column-scaled by the cleartext database
            return (r == 1 && S.db) ? mod_small(v * S.db[idx - 1], p, pinv) : v;
        }
        case PT_TOP: return r == 0 ? 1 : 0;
        case PT_BOT: return r == 1 ? 1 : 0;
        case PT_ONE: return 1;
        case PT_DBVEC: {  // SlotMatrix.from_vector: first m entries in row 0, the next m in row 1
            const long long pos = (long long)J.t * 2 * S.m + (long long)r * S.m + c;
            return pos < S.N ? S.db[pos] : 0;
        }
        default: return c < S.s ? 1 : 0;  // PT_OUTMASK
    }
}

__global__ void __launch_bounds__(NT, 1) k_plain(const __grid_constant__ DevCtx C, const PJob* __restrict__ jobs, PlanShape S) {
    extern __shared__ u64 sm[];
    u64* coef = sm + NPOLY;
    const PJob J = jobs[blockIdx.x];
    const int tid = threadIdx.x;
    HC_NOUNROLL
    for (int j = tid; j < NPOLY; j += NT) {
        const unsigned so = C.slot_of[j];
        sm[swz(j)] = plain_slot_value(J, S, so >> 12, so & 4095, C.p, C.pinv);
    }
    __syncthreads();
    cta_ntt_inv(C.twi + (size_t)PIDX * NPOLY, C.pc[PIDX], sm);
    HC_NOUNROLL
    for (int j = tid; j < NPOLY; j += NT) coef[j] = sm[swz(j)];
    const LevelC& LV = C.lv(J.level);
    for (int k = 0; k <= J.level; k++) {
        const PrimeC P = C.pc[k];
        __syncthreads();
        HC_NOUNROLL
        for (int j = tid; j < NPOLY; j += NT) sm[swz(j)] = coef[j];
        __syncthreads();
        cta_ntt_fwd(C.twf + (size_t)k * NPOLY, P, sm);
        const u64 w = (k == J.level) ? P.rmod : LV.qinv_r[k];
        const u64 ws = (k == J.level) ? P.rmod_s : LV.qinv_rs[k];
        HC_NOUNROLL
        for (int j = tid; j < NPOLY; j += NT) J.out[(size_t)k * NPOLY + j] = mul_shoup(sm[swz(j)], w, ws, P.q);
    }
}

// ---------------------------------------------------------------------------
// small utility kernels
// ---------------------------------------------------------------------------

// in-place x -> x*R mod q (Montgomery form); prime of row r = r % period
__global__ void k_to_mont(const __grid_constant__ DevCtx C, u64* data, long long rows, int period) {
    const long long total = rows * NPOLY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int k = (int)((i / NPOLY) % period);
        const PrimeC P = C.pc[k];
        data[i] = mul_shoup(data[i], P.rmod, P.rmod_s, P.q);
    }
}

// pointwise op over rows; prime of row r = pidx[r]
// out = a + b mod q_k over rows of n, row r modulo prime r % P: the add of
// pack_pair's two terms (bgv.py:651-670) in the mixed-level schedule
struct AddJob {
    const u64* a;
    const u64* b;
    u64* out;
};
// grid (n/256, rows, jobs)
__global__ void __launch_bounds__(256) k_addmod(const __grid_constant__ DevCtx C, const AddJob* __restrict__ jobs, int P) {
    const AddJob J = jobs[blockIdx.z];
    const size_t i = (size_t)blockIdx.y * NPOLY + blockIdx.x * 256 + threadIdx.x;
    const u64 q = C.pc[blockIdx.y % P].q;
    pdl_wait();
    J.out[i] = add_mod(J.a[i], J.b[i], q);
}

__global__ void k_pointwise(const __grid_constant__ DevCtx C, const u64* a, const u64* b, u64* out, int rows,
                            const int* pidx, int op) {
    const long long total = (long long)rows * NPOLY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const PrimeC P = C.pc[pidx[i / NPOLY]];
        const u64 x = a[i], y = b[i];
        u64 r;
        if (op == 0) {
            u64 hi, lo;
            mul128(hi, lo, x, y);
            // x*y mod q via Montgomery twice: redc(x*y) = x*y*R^-1; then * R^2 ... use
            // x*y*R^-1 then multiply by R^2 mod q = (R mod q)^2 through two Shoup steps
            u64 t = redc(hi, lo, P.q, P.qneg);             // x*y*R^-1
            t = mul_shoup(t, P.rmod, P.rmod_s, P.q);        // x*y
            r = t;
        } else if (op == 1) {
            r = add_mod(x, y, P.q);
        } else {
            r = sub_mod(x, y, P.q);
        }
        out[i] = r;
    }
}

}  // namespace hc
