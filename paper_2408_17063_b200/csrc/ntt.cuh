// Negacyclic NTT / INTT for n = 8192 over one 54-bit prime, one CTA of 256
// threads per polynomial, 32 coefficients per thread held in registers.
//
// Semantics (must match the reference bit-for-bit after canonicalisation):
//   forward  = NttContext.fwd  (bgv.py:178-199): Cooley-Tukey, natural-order
//              input, bit-reversed output, twiddle tbl[m+i] = psi^bitrev(m+i);
//   inverse  = NttContext.inv  (bgv.py:201-225): Gentleman-Sande with
//              inv_tbl[h+i] = psi^-bitrev(h+i), then * n^-1.
// Modular arithmetic is exact, so any schedule of the same butterflies gives
// the reference's values; the schedule here is radix-32/16/16 in registers
// with two swizzled shared-memory transposes between register passes.
//
// Register layout in and out of both transforms ("canonical layout"):
//   thread tid holds x[i] = a[tid + 256*i], i = 0..31   (coalesced in HBM).
//
// Every pass is a __host__ __device__ function of (tid, registers, smem) so
// the CPU self-test can run the exact device schedule thread by thread
// (passes are separated by __syncthreads on the device, by a loop over all
// 256 tids on the host).
#pragma once
#include "arith.cuh"

#if defined(__CUDACC__)
#define HC_UNROLL _Pragma("unroll")
#else
#define HC_UNROLL
#endif

namespace hc {

constexpr int LOGN = 13;
constexpr int NPOLY = 1 << LOGN;  // ring degree n
constexpr int NT = 256;           // threads per transform CTA
constexpr int EPT = NPOLY / NT;   // 32 coefficients per thread

struct alignas(16) Tw {
    u64 w, ws;  // twiddle and its Shoup constant
};

// Per-prime constants.
struct PrimeC {
    u64 q, q2, qneg;       // q, 2q, -q^-1 mod 2^64
    u64 ninv, ninv_s;      // n^-1 (Shoup)
    u64 ninvw, ninvw_s;    // inv_tbl[1] * n^-1 (Shoup): last GS stage
    u64 rmod, rmod_s;      // 2^64 mod q (Shoup): to Montgomery form
    u64 one_s;             // floor(2^64 / q): full reduction of any u64
};

HD Tw ldtw(const Tw* t, int i) {
#if defined(__CUDA_ARCH__)
    ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(t) + i);
    Tw r;
    r.w = v.x;
    r.ws = v.y;
    return r;
#else
    return t[i];
#endif
}

// shared-memory swizzle: conflict-free for all four access patterns below
HD int swz(int j) { return j ^ ((j >> 4) & 15); }

// ---------------- forward -------------------------------------------------

// stages 0..4 (bits 12..8), registers only
HD void fwd_p1(u64 (&x)[EPT], const Tw* tw, u64 q, u64 q2) {
    HC_UNROLL
    for (int s = 0; s < 5; s++) {
        const int half = 16 >> s;
        HC_UNROLL
        for (int i = 0; i < 32; i++) {
            if (!(i & half)) {
                Tw w = ldtw(tw, (1 << s) + (i >> (5 - s)));
                bf_ct(x[i], x[i + half], w.w, w.ws, q, q2);
            }
        }
    }
}

HD void st_canon(int tid, const u64 (&x)[EPT], u64* sm) {
    HC_UNROLL
    for (int i = 0; i < 32; i++) sm[swz(tid + NT * i)] = x[i];
}
HD void ld_canon(int tid, u64 (&x)[EPT], const u64* sm) {
    HC_UNROLL
    for (int i = 0; i < 32; i++) x[i] = sm[swz(tid + NT * i)];
}

// "mid" groups: fixed bits 12..8 and 3..0, v = bits 7..4
HD int mid_index(int G, int v) { return ((G >> 4) << 8) | (v << 4) | (G & 15); }
HD void ld_mid(int tid, u64 (&x)[EPT], const u64* sm) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        HC_UNROLL
        for (int v = 0; v < 16; v++) x[g * 16 + v] = sm[swz(mid_index(tid + NT * g, v))];
    }
}
HD void st_mid(int tid, const u64 (&x)[EPT], u64* sm) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        HC_UNROLL
        for (int v = 0; v < 16; v++) sm[swz(mid_index(tid + NT * g, v))] = x[g * 16 + v];
    }
}
// "low" groups: fixed bits 12..4, v = bits 3..0
HD void ld_low(int tid, u64 (&x)[EPT], const u64* sm) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        HC_UNROLL
        for (int v = 0; v < 16; v++) x[g * 16 + v] = sm[swz(((tid + NT * g) << 4) | v)];
    }
}
HD void st_low(int tid, const u64 (&x)[EPT], u64* sm) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        HC_UNROLL
        for (int v = 0; v < 16; v++) sm[swz(((tid + NT * g) << 4) | v)] = x[g * 16 + v];
    }
}

// stages 5..8 (bits 7..4)
HD void fwd_p2(int tid, u64 (&x)[EPT], const Tw* tw, u64 q, u64 q2) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        const int hi5 = (tid + NT * g) >> 4;
        HC_UNROLL
        for (int s = 5; s < 9; s++) {
            const int half = 8 >> (s - 5);
            HC_UNROLL
            for (int v = 0; v < 16; v++) {
                if (!(v & half)) {
                    Tw w = ldtw(tw, (1 << s) + ((hi5 << (s - 5)) | (v >> (9 - s))));
                    bf_ct(x[g * 16 + v], x[g * 16 + v + half], w.w, w.ws, q, q2);
                }
            }
        }
    }
}

// stages 9..12 (bits 3..0); leaves values canonical in [0, q)
HD void fwd_p3(int tid, u64 (&x)[EPT], const Tw* tw, u64 q, u64 q2) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        const int G = tid + NT * g;
        HC_UNROLL
        for (int s = 9; s < 13; s++) {
            const int half = 8 >> (s - 9);
            HC_UNROLL
            for (int v = 0; v < 16; v++) {
                if (!(v & half)) {
                    Tw w = ldtw(tw, (1 << s) + ((G << (s - 9)) | (v >> (13 - s))));
                    bf_ct(x[g * 16 + v], x[g * 16 + v + half], w.w, w.ws, q, q2);
                }
            }
        }
    }
    HC_UNROLL
    for (int i = 0; i < 32; i++) x[i] = canon4(x[i], q, q2);
}

// ---------------- inverse -------------------------------------------------

// bits 0..3; input in [0, 2q)
HD void inv_pa(int tid, u64 (&x)[EPT], const Tw* tw, u64 q, u64 q2) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        const int G = tid + NT * g;
        HC_UNROLL
        for (int b = 0; b < 4; b++) {
            const int half = 1 << b;
            HC_UNROLL
            for (int v = 0; v < 16; v++) {
                if (!(v & half)) {
                    Tw w = ldtw(tw, (1 << (12 - b)) + ((G << (3 - b)) | (v >> (b + 1))));
                    bf_gs(x[g * 16 + v], x[g * 16 + v + half], w.w, w.ws, q, q2);
                }
            }
        }
    }
}

// bits 4..7
HD void inv_pb(int tid, u64 (&x)[EPT], const Tw* tw, u64 q, u64 q2) {
    HC_UNROLL
    for (int g = 0; g < 2; g++) {
        const int hi5 = (tid + NT * g) >> 4;
        HC_UNROLL
        for (int b = 4; b < 8; b++) {
            const int half = 1 << (b - 4);
            HC_UNROLL
            for (int v = 0; v < 16; v++) {
                if (!(v & half)) {
                    Tw w = ldtw(tw, (1 << (12 - b)) + ((hi5 << (7 - b)) | (v >> (b - 3))));
                    bf_gs(x[g * 16 + v], x[g * 16 + v + half], w.w, w.ws, q, q2);
                }
            }
        }
    }
}

// bits 8..12 in canonical layout; the last stage folds in n^-1.
// Output canonical in [0, q).
HD void inv_pc(u64 (&x)[EPT], const Tw* tw, const PrimeC& P) {
    const u64 q = P.q, q2 = P.q2;
    HC_UNROLL
    for (int b = 8; b < 12; b++) {
        const int half = 1 << (b - 8);
        HC_UNROLL
        for (int i = 0; i < 32; i++) {
            if (!(i & half)) {
                Tw w = ldtw(tw, (1 << (12 - b)) + (i >> (b - 7)));
                bf_gs(x[i], x[i + half], w.w, w.ws, q, q2);
            }
        }
    }
    HC_UNROLL
    for (int i = 0; i < 16; i++) {
        u64 u = x[i], v = x[i + 16];
        x[i] = reduce_once(mul_shoup_lazy(u + v, P.ninv, P.ninv_s, q), q);
        x[i + 16] = reduce_once(mul_shoup_lazy(u - v + q2, P.ninvw, P.ninvw_s, q), q);
    }
}

#if defined(__CUDACC__)
// Device CTA transforms (blockDim.x == 256).  `sm` = 8192 u64 of shared memory.
// In/out in canonical layout.  fwd input < 4q; inv input < 2q.  Output < q.
__device__ __forceinline__ void cta_ntt_fwd(u64 (&x)[EPT], const Tw* tw, const PrimeC& P, u64* sm) {
    const int tid = threadIdx.x;
    fwd_p1(x, tw, P.q, P.q2);
    st_canon(tid, x, sm);
    __syncthreads();
    ld_mid(tid, x, sm);
    fwd_p2(tid, x, tw, P.q, P.q2);
    st_mid(tid, x, sm);
    __syncthreads();
    ld_low(tid, x, sm);
    fwd_p3(tid, x, tw, P.q, P.q2);
    st_low(tid, x, sm);
    __syncthreads();
    ld_canon(tid, x, sm);
    __syncthreads();  // smem reusable by the caller
}

__device__ __forceinline__ void cta_ntt_inv(u64 (&x)[EPT], const Tw* tw, const PrimeC& P, u64* sm) {
    const int tid = threadIdx.x;
    st_canon(tid, x, sm);
    __syncthreads();
    ld_low(tid, x, sm);
    inv_pa(tid, x, tw, P.q, P.q2);
    st_low(tid, x, sm);
    __syncthreads();
    ld_mid(tid, x, sm);
    inv_pb(tid, x, tw, P.q, P.q2);
    st_mid(tid, x, sm);
    __syncthreads();
    ld_canon(tid, x, sm);
    inv_pc(x, tw, P);
    __syncthreads();
}
#endif

// Host emulation of the device schedule (CPU self-test only): a[n] in/out.
inline void host_emulate_fwd(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    for (int t = 0; t < NT; t++)
        for (int i = 0; i < EPT; i++) regs[t][i] = a[t + NT * i];
    for (int t = 0; t < NT; t++) { fwd_p1(regs[t], tw, P.q, P.q2); st_canon(t, regs[t], sm); }
    for (int t = 0; t < NT; t++) { ld_mid(t, regs[t], sm); fwd_p2(t, regs[t], tw, P.q, P.q2); }
    for (int t = 0; t < NT; t++) st_mid(t, regs[t], sm);
    for (int t = 0; t < NT; t++) { ld_low(t, regs[t], sm); fwd_p3(t, regs[t], tw, P.q, P.q2); }
    for (int t = 0; t < NT; t++) st_low(t, regs[t], sm);
    for (int t = 0; t < NT; t++) ld_canon(t, regs[t], sm);
    for (int t = 0; t < NT; t++)
        for (int i = 0; i < EPT; i++) a[t + NT * i] = regs[t][i];
}

inline void host_emulate_inv(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    for (int t = 0; t < NT; t++)
        for (int i = 0; i < EPT; i++) regs[t][i] = a[t + NT * i];
    for (int t = 0; t < NT; t++) st_canon(t, regs[t], sm);
    for (int t = 0; t < NT; t++) { ld_low(t, regs[t], sm); inv_pa(t, regs[t], tw, P.q, P.q2); }
    for (int t = 0; t < NT; t++) st_low(t, regs[t], sm);
    for (int t = 0; t < NT; t++) { ld_mid(t, regs[t], sm); inv_pb(t, regs[t], tw, P.q, P.q2); }
    for (int t = 0; t < NT; t++) st_mid(t, regs[t], sm);
    for (int t = 0; t < NT; t++) { ld_canon(t, regs[t], sm); inv_pc(regs[t], tw, P); }
    for (int t = 0; t < NT; t++)
        for (int i = 0; i < EPT; i++) a[t + NT * i] = regs[t][i];
}

}  // namespace hc
