// Single-CTA negacyclic NTT / INTT for n = 8192 (throughput path): one CTA
// of 1024 threads per transform, 8 coefficients per thread, radix-8
// register passes (the building blocks of ntt_cl.cuh) through a swizzled
// 64 KiB shared-memory tile.  13 stages = 3 + 3 + 3 + 3 + 1 (the bit-0 stage
// across lane pairs by warp shuffle).  At <= 64 registers per thread this
// keeps 32 warps per SM resident (the 512-thread radix-16 version had 16 and
// was latency-bound: ncu issue-active 42%).
//
// Tile convention: coefficient j at sm[swz(j)]; the caller fills the tile
// (natural order), syncs, calls the transform, and reads the result back in
// natural order.  Forward input < 4q (lazy CT, output canonical); inverse
// input < 2q (GS, output canonical).  Semantics: NttContext.fwd/inv
// (bgv.py:178-225).
#pragma once
#include "ntt_cl.cuh"

namespace hc {

// 64-bit, 16-lane phases: XOR index bits 1..3 with bits 4..6 (conflict-free
// for the four affine layouts below)
HD int swz(int j) { return cswz(j); }

// forward pass p covers bits 12-3p .. 10-3p: thread t's coefficients are
// j(v) = base + v*stride, G = index bits above the pass
HD CPass pass1k(int p, int t) {
    CPass r;
    if (p == 0) {
        r.base = t; r.stride = 1024; r.G = 0; r.s0 = 0;
    } else if (p == 1) {
        r.base = ((t >> 7) << 10) | (t & 127); r.stride = 128; r.G = t >> 7; r.s0 = 3;
    } else if (p == 2) {
        r.base = ((t >> 4) << 7) | (t & 15); r.stride = 16; r.G = t >> 4; r.s0 = 6;
    } else {
        r.base = ((t >> 1) << 4) | (t & 1); r.stride = 2; r.G = t >> 1; r.s0 = 9;
    }
    return r;
}

HD void t_load(u64 (&x)[EPT], const u64* sm, const CPass& I) {
    HC_UNROLL
    for (int v = 0; v < EPT; v++) x[v] = sm[cswz_elem(I.base, I.stride, v)];
}
HD void t_store(const u64 (&x)[EPT], u64* sm, const CPass& I) {
    HC_UNROLL
    for (int v = 0; v < EPT; v++) sm[cswz_elem(I.base, I.stride, v)] = x[v];
}

#if defined(__CUDACC__)
// VT virtual threads per thread: a CTA of NT / VT threads runs the 1024-thread
// schedule, each thread taking threads t, t + NT / VT, ... in turn within every
// pass (their coefficients are disjoint, so no extra synchronisation).  VT = 4
// puts three independent transforms (CTAs, barriers) on each SM.
template <bool LAZY = false, int VT = 1>
__device__ __forceinline__ void cta_ntt_fwd(const Tw* tw, const PrimeC& P, u64* sm) {
    const TwG tg{tw};
    u64 x[EPT];
    HC_UNROLL
    for (int p = 0; p < 4; p++) {
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const int t = threadIdx.x + v * (NT / VT);
            const CPass I = pass1k(p, t);
            t_load(x, sm, I);
            r8_ct(x, tg, I.s0, I.G, P.q, 2 * P.q2);
            if (p == 3) c_st12<LAZY>(0, t, x, tg, P.q, 2 * P.q2, P.one_s);
            t_store(x, sm, I);
        }
        __syncthreads();
    }
}

template <int VT = 1>
__device__ __forceinline__ void cta_ntt_inv(const Tw* tw, const PrimeC& P, u64* sm) {
    const TwG tg{tw};
    u64 x[EPT];
    HC_UNROLL
    for (int p = 0; p < 3; p++) {
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const int t = threadIdx.x + v * (NT / VT);
            const CPass I = pass1k(3 - p, t);
            t_load(x, sm, I);
            if (p == 0) c_st0(0, t, x, tg, P.q, P.q2);
            r8_gs(x, tg, 1 + 3 * p, I.G, P.q, 2 * P.q2);
            t_store(x, sm, I);
        }
        __syncthreads();
    }
    HC_NOUNROLL
    for (int v = 0; v < VT; v++) {
        const CPass I = pass1k(0, threadIdx.x + v * (NT / VT));
        t_load(x, sm, I);
        c_phaseA_inv(x, tw, P);  // bits 10..12 (element v*1024 + t), n^-1 folded
        t_store(x, sm, I);
    }
    __syncthreads();
}
#endif

// k_xf's form of the same transforms: the bit-0 stage runs in REGISTERS at
// the edge of the kernel instead of across lane pairs -- the forward
// transform's epilogue (the inverse transform's loader) owns the four
// coefficient pairs (j, j + 1), j = 2t + 2048m, so the stage needs no shuffle
// and none of c_st12 / c_st0's even/odd selects (~100 of ~1400 instructions
// per schedule thread), and the pairs move as 128-bit shared-memory accesses.
HD void fwd_last_stage(u64 (&xe)[4], u64 (&xo)[4], const Tw* tw, int t, const PrimeC& P, bool lazy) {
    Tw w[4];
    HC_UNROLL
    for (int m = 0; m < 4; m++) w[m] = ldtw(tw, 4096 + t + 1024 * m);  // tbl[4096 + (j >> 1)]
    edge_fwd(xe, xo, w, P, lazy);
}
// inverse bit-0 stage on loader outputs in [0, 2q): sums < 4q, products < 4q
HD void inv_first_stage(u64 (&xe)[4], u64 (&xo)[4], const Tw* tw, int t, const PrimeC& P) {
    Tw w[4];
    HC_UNROLL
    for (int m = 0; m < 4; m++) w[m] = ldtw(tw, 4096 + t + 1024 * m);
    edge_inv(xe, xo, w, P);
}
// tile index of the pair (2t + 2048m, +1): swz leaves bit 0 alone and 2048m
// leaves bits 1..6 alone, so one swizzled base and immediate offsets
HD int pair_index(int t, int m) { return swz(2 * t) + 2048 * m; }

#if defined(__CUDACC__)
// P0: first pass to run (1: the caller did pass 0 -- stages 0..2 on the
// coefficients t + 1024e its loader holds -- in registers and stored them)
template <int VT = 1, int P0 = 0>
__device__ __forceinline__ void cta_ntt_fwd_core(const Tw* tw, const PrimeC& P, u64* sm) {  // stages 0..11
    const TwG tg{tw};
    u64 x[EPT];
    HC_UNROLL
    for (int p = P0; p < 4; p++) {
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const CPass I = pass1k(p, threadIdx.x + v * (NT / VT));
            t_load(x, sm, I);
            r8_ct(x, tg, I.s0, I.G, P.q, 2 * P.q2);
            t_store(x, sm, I);
        }
        __syncthreads();
    }
}
// LASTREG: the last pass (stages 10..12, n^-1 folded) is left to the caller,
// which runs it in registers on the coefficients t + 1024e its epilogue owns
template <int VT = 1, bool LASTREG = false>
__device__ __forceinline__ void cta_ntt_inv_core(const Tw* tw, const PrimeC& P, u64* sm) {  // stages 1..12 (bit 0 done)
    const TwG tg{tw};
    u64 x[EPT];
    HC_UNROLL
    for (int p = 0; p < 3; p++) {
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const CPass I = pass1k(3 - p, threadIdx.x + v * (NT / VT));
            t_load(x, sm, I);
            r8_gs(x, tg, 1 + 3 * p, I.G, P.q, 2 * P.q2);
            t_store(x, sm, I);
        }
        __syncthreads();
    }
    if constexpr (!LASTREG) {
        HC_NOUNROLL
        for (int v = 0; v < VT; v++) {
            const CPass I = pass1k(0, threadIdx.x + v * (NT / VT));
            t_load(x, sm, I);
            c_phaseA_inv(x, tw, P);
            t_store(x, sm, I);
        }
        __syncthreads();
    }
}
#endif

// ---- host emulation of the 1024-thread schedule (CPU self-test only) ------
inline void host_emulate_fwd(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    const TwG tg{tw};
    for (int j = 0; j < NPOLY; j++) sm[swz(j)] = a[j];
    for (int p = 0; p < 4; p++) {
        for (int t = 0; t < NT; t++) {
            CPass I = pass1k(p, t);
            t_load(regs[t], sm, I);
            r8_ct(regs[t], tg, I.s0, I.G, P.q, 2 * P.q2);
        }
        if (p == 3) host_st12(0, NT, regs, tg, P.q, 2 * P.q2, P.one_s);
        for (int t = 0; t < NT; t++) t_store(regs[t], sm, pass1k(p, t));
    }
    for (int j = 0; j < NPOLY; j++) a[j] = sm[swz(j)];
}

inline void host_emulate_inv(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    const TwG tg{tw};
    for (int j = 0; j < NPOLY; j++) sm[swz(j)] = a[j];
    for (int p = 0; p < 3; p++) {
        for (int t = 0; t < NT; t++) t_load(regs[t], sm, pass1k(3 - p, t));
        if (p == 0) host_st0(0, NT, regs, tg, P.q, P.q2);
        for (int t = 0; t < NT; t++) {
            CPass I = pass1k(3 - p, t);
            r8_gs(regs[t], tg, 1 + 3 * p, I.G, P.q, 2 * P.q2);
            t_store(regs[t], sm, I);
        }
    }
    for (int t = 0; t < NT; t++) {
        CPass I = pass1k(0, t);
        t_load(regs[t], sm, I);
        c_phaseA_inv(regs[t], tw, P);
        t_store(regs[t], sm, I);
    }
    for (int j = 0; j < NPOLY; j++) a[j] = sm[swz(j)];
}


// host emulation of k_xf's edge-stage form (fwd_last_stage / inv_first_stage)
inline void host_emulate_fwd_edge(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    const TwG tg{tw};
    for (int j = 0; j < NPOLY; j++) sm[swz(j)] = a[j];
    for (int p = 0; p < 4; p++) {
        for (int t = 0; t < NT; t++) {
            CPass I = pass1k(p, t);
            t_load(regs[t], sm, I);
            r8_ct(regs[t], tg, I.s0, I.G, P.q, 2 * P.q2);
        }
        for (int t = 0; t < NT; t++) t_store(regs[t], sm, pass1k(p, t));
    }
    for (int t = 0; t < NT; t++) {
        u64 xe[4], xo[4];
        for (int m = 0; m < 4; m++) {
            xe[m] = sm[pair_index(t, m)];
            xo[m] = sm[pair_index(t, m) + 1];
        }
        fwd_last_stage(xe, xo, tw, t, P, false);
        for (int m = 0; m < 4; m++) {
            a[2 * t + 2048 * m] = xe[m];
            a[2 * t + 2048 * m + 1] = xo[m];
        }
    }
}
inline void host_emulate_inv_edge(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT];
    static u64 sm[NPOLY];
    const TwG tg{tw};
    for (int t = 0; t < NT; t++) {
        u64 xe[4], xo[4];
        for (int m = 0; m < 4; m++) {
            xe[m] = a[2 * t + 2048 * m];
            xo[m] = a[2 * t + 2048 * m + 1];
        }
        inv_first_stage(xe, xo, tw, t, P);
        for (int m = 0; m < 4; m++) {
            sm[pair_index(t, m)] = xe[m];
            sm[pair_index(t, m) + 1] = xo[m];
        }
    }
    for (int p = 0; p < 3; p++) {
        for (int t = 0; t < NT; t++) {
            CPass I = pass1k(3 - p, t);
            t_load(regs[t], sm, I);
            r8_gs(regs[t], tg, 1 + 3 * p, I.G, P.q, 2 * P.q2);
        }
        for (int t = 0; t < NT; t++) t_store(regs[t], sm, pass1k(3 - p, t));
    }
    for (int t = 0; t < NT; t++) {
        CPass I = pass1k(0, t);
        t_load(regs[t], sm, I);
        c_phaseA_inv(regs[t], tw, P);
        t_store(regs[t], sm, I);
    }
    for (int j = 0; j < NPOLY; j++) a[j] = sm[swz(j)];
}

}  // namespace hc
