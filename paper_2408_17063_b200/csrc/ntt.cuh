// Negacyclic NTT / INTT for n = 8192 over one 54-bit prime: one CTA of 512
// threads per polynomial, 16 coefficients per thread in registers.
//
// Semantics (bit-for-bit after canonicalisation):
//   forward = NttContext.fwd (bgv.py:178-199): Cooley-Tukey, natural-order
//             input, bit-reversed output, twiddle tbl[m+i] = psi^bitrev(m+i);
//   inverse = NttContext.inv (bgv.py:201-225): Gentleman-Sande with
//             inv_tbl[h+i] = psi^-bitrev(h+i), then * n^-1.
// Modular arithmetic is exact, so any schedule of the same butterflies gives
// the reference's values.  Schedule (13 stages = 4 + 4 + 4 + 1):
//   three radix-16 register passes over coefficient index bits 12..9, 8..5
//   and 4..1 -- ONE inlined radix-16 routine run in a rolled loop, because
//   each pass's index pattern is affine, j(v) = base + v*stride -- and the
//   bit-0 stage across lane pairs with a warp shuffle.  Between passes the
//   data goes through a swizzled 64 KiB shared-memory tile.  Compact code is
//   deliberate: the fully unrolled first version (468 KiB of SASS) stalled
//   on instruction fetch.
//
// Register layout in/out of both transforms ("canonical layout"):
//   thread t holds x[v] = a[t + 512*v], v = 0..15  (coalesced in HBM).
//
// The passes are __host__ __device__ functions of (tid, registers, smem), so
// the CPU self-test runs this exact schedule thread by thread.
#pragma once
#include "arith.cuh"

#if defined(__CUDACC__)
#define HC_UNROLL _Pragma("unroll")
#define HC_NOUNROLL _Pragma("unroll 1")
#else
#define HC_UNROLL
#define HC_NOUNROLL
#endif

namespace hc {

constexpr int LOGN = 13;
constexpr int NPOLY = 1 << LOGN;  // ring degree n
constexpr int NT = 512;           // threads per transform CTA
constexpr int EPT = NPOLY / NT;   // 16 coefficients per thread

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

// shared-memory swizzle (XOR index bits 1..4 with bits 5..8): conflict-free
// for the three affine patterns below (64-bit accesses, 16 lanes per phase)
HD int swz(int j) { return j ^ (((j >> 5) & 15) << 1); }

// Forward pass p covers index bits 12-4p .. 9-4p; thread t's 16 coefficients
// are j(v) = base + v*stride, "hi" = the index bits above the pass.
struct PassIdx {
    int base, stride, hi, s0;
};
HD PassIdx pass_idx(int p, int t) {
    PassIdx r;
    if (p == 0) {
        r.base = t; r.stride = 512; r.hi = 0; r.s0 = 0;
    } else if (p == 1) {
        r.base = ((t >> 5) << 9) | (t & 31); r.stride = 32; r.hi = t >> 5; r.s0 = 4;
    } else {
        r.base = ((t >> 1) << 5) | (t & 1); r.stride = 2; r.hi = t >> 1; r.s0 = 8;
    }
    return r;
}

HD void sm_load(u64 (&x)[EPT], const u64* sm, int base, int stride) {
    HC_UNROLL
    for (int v = 0; v < EPT; v++) x[v] = sm[swz(base + v * stride)];
}
HD void sm_store(const u64 (&x)[EPT], u64* sm, int base, int stride) {
    HC_UNROLL
    for (int v = 0; v < EPT; v++) sm[swz(base + v * stride)] = x[v];
}

// 4 Cooley-Tukey stages s0..s0+3 on a 16-point group: stage s0+u pairs v and
// v + (8 >> u), twiddle tbl[2^(s0+u) + (hi << u | v >> (4-u))].  Lazy
// (bf_ct_lazy): q2 here carries 4q.
HD void r16_ct(u64 (&x)[EPT], const Tw* tw, int s0, int hi, u64 q, u64 q2) {
    HC_UNROLL
    for (int u = 0; u < 4; u++) {
        const int half = 8 >> u;
        const int tbase = (1 << (s0 + u)) + (hi << u);
        HC_UNROLL
        for (int v = 0; v < EPT; v++) {
            if (!(v & half)) {
                Tw w = ldtw(tw, tbase + (v >> (4 - u)));
                bf_ct_lazy(x[v], x[v + half], w.w, w.ws, q, q2);
            }
        }
    }
}

// 4 Gentleman-Sande stages b0..b0+3 on a 16-point group: stage b0+u pairs v
// and v + (1 << u), twiddle inv_tbl[2^(12-b0-u) + (hi << (3-u) | v >> (u+1))].
HD void r16_gs(u64 (&x)[EPT], const Tw* tw, int b0, int hi, u64 q, u64 q2) {
    HC_UNROLL
    for (int u = 0; u < 4; u++) {
        const int half = 1 << u;
        const int tbase = (1 << (12 - b0 - u)) + (hi << (3 - u));
        HC_UNROLL
        for (int v = 0; v < EPT; v++) {
            if (!(v & half)) {
                Tw w = ldtw(tw, tbase + (v >> (u + 1)));
                bf_gs(x[v], x[v + half], w.w, w.ws, q, q2);
            }
        }
    }
}

// Forward stage 12 (index bit 0) across the lane pair (t, t^1): even lane
// keeps X + w*Y, odd lane X - w*Y, w = tbl[4096 + ((t >> 1) << 4 | v)].
// Lazy inputs (< 52q), outputs canonical.  `other` = the partner lane's
// registers; q2 carries 4q, one_s the full-reduction constant.
HD void st12_ct(int t, u64 (&x)[EPT], const u64 (&other)[EPT], const Tw* tw, u64 q, u64 q2, u64 one_s) {
    const int odd = t & 1;
    const int tb = 4096 + ((t >> 1) << 4);
    HC_UNROLL
    for (int v = 0; v < EPT; v++) {
        u64 X = odd ? other[v] : x[v];
        u64 Y = odd ? x[v] : other[v];
        Tw w = ldtw(tw, tb + v);
        bf_ct_lazy(X, Y, w.w, w.ws, q, q2);
        x[v] = canon_any(odd ? Y : X, q, one_s);
    }
}

// First inverse stage (bit 0) across the lane pair: even lane X + Y, odd
// lane (X - Y) * w, w = inv_tbl[4096 + ((t >> 1) << 4 | v)].  [0,2q) in/out.
HD void st0_gs(int t, u64 (&x)[EPT], const u64 (&other)[EPT], const Tw* tw, u64 q, u64 q2) {
    const int odd = t & 1;
    const int tb = 4096 + ((t >> 1) << 4);
    HC_UNROLL
    for (int v = 0; v < EPT; v++) {
        const u64 X = odd ? other[v] : x[v];
        const u64 Y = odd ? x[v] : other[v];
        if (odd) {
            Tw w = ldtw(tw, tb + v);
            x[v] = mul_shoup_lazy(X - Y + q2, w.w, w.ws, q);
        } else {
            u64 s = X + Y;
            x[v] = s >= q2 ? s - q2 : s;
        }
    }
}

// Inverse stages 9..11 in the canonical layout, then the bit-12 stage folded
// with n^-1.  Output canonical.
HD void inv_tail(u64 (&x)[EPT], const Tw* tw, const PrimeC& P) {
    const u64 q = P.q, q2 = P.q2;
    HC_UNROLL
    for (int u = 0; u < 3; u++) {
        const int half = 1 << u;
        const int tbase = 1 << (3 - u);
        HC_UNROLL
        for (int v = 0; v < EPT; v++) {
            if (!(v & half)) {
                Tw w = ldtw(tw, tbase + (v >> (u + 1)));
                bf_gs(x[v], x[v + half], w.w, w.ws, q, q2);
            }
        }
    }
    HC_UNROLL
    for (int v = 0; v < 8; v++) {
        u64 a = x[v], b = x[v + 8];
        x[v] = reduce_once(mul_shoup_lazy(a + b, P.ninv, P.ninv_s, q), q);
        x[v + 8] = reduce_once(mul_shoup_lazy(a - b + q2, P.ninvw, P.ninvw_s, q), q);
    }
}

#if defined(__CUDACC__)
__device__ __forceinline__ void shfl_pair(const u64 (&x)[EPT], u64 (&o)[EPT]) {
    HC_UNROLL
    for (int v = 0; v < EPT; v++) o[v] = __shfl_xor_sync(0xffffffffu, x[v], 1);
}

// Device CTA transforms (blockDim.x == 512) on a 64 KiB smem tile holding
// coefficient j at sm[swz(j)] (natural index order in and out; the caller
// writes/reads it with rolled per-coefficient loops).  fwd input < 4q,
// inv input < 2q; output canonical < q.  The caller must __syncthreads()
// after filling the tile; the functions end with a barrier.
// In any one access pattern every smem word belongs to exactly one thread,
// so one barrier between a store pattern and the next load pattern suffices.
__device__ __forceinline__ void cta_ntt_fwd(const Tw* tw, const PrimeC& P, u64* sm) {
    const int t = threadIdx.x;
    u64 x[EPT];
    HC_NOUNROLL
    for (int p = 0; p < 3; p++) {
        const PassIdx I = pass_idx(p, t);
        sm_load(x, sm, I.base, I.stride);
        r16_ct(x, tw, I.s0, I.hi, P.q, 2 * P.q2);
        if (p == 2) {
            u64 o[EPT];
            shfl_pair(x, o);
            st12_ct(t, x, o, tw, P.q, 2 * P.q2, P.one_s);
        }
        sm_store(x, sm, I.base, I.stride);
        __syncthreads();
    }
}

__device__ __forceinline__ void cta_ntt_inv(const Tw* tw, const PrimeC& P, u64* sm) {
    const int t = threadIdx.x;
    u64 x[EPT];
    HC_NOUNROLL
    for (int p = 0; p < 3; p++) {
        const PassIdx I = pass_idx(2 - p, t);
        sm_load(x, sm, I.base, I.stride);
        if (p == 0) {
            u64 o[EPT];
            shfl_pair(x, o);
            st0_gs(t, x, o, tw, P.q, P.q2);
        }
        if (p < 2) {
            r16_gs(x, tw, 1 + 4 * p, I.hi, P.q, P.q2);
            sm_store(x, sm, I.base, I.stride);
            __syncthreads();
        }
    }
    inv_tail(x, tw, P);
    sm_store(x, sm, t, NT);
    __syncthreads();
}
#endif

// ---- host emulation of the device schedule (CPU self-test only) ----------
inline void host_emulate_fwd(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT], other[NT][EPT];
    static u64 sm[NPOLY];
    for (int j = 0; j < NPOLY; j++) sm[swz(j)] = a[j];
    for (int p = 0; p < 3; p++) {
        for (int t = 0; t < NT; t++) {
            PassIdx I = pass_idx(p, t);
            sm_load(regs[t], sm, I.base, I.stride);
            r16_ct(regs[t], tw, I.s0, I.hi, P.q, 2 * P.q2);
        }
        if (p == 2) {
            for (int t = 0; t < NT; t++)
                for (int v = 0; v < EPT; v++) other[t][v] = regs[t ^ 1][v];
            for (int t = 0; t < NT; t++) st12_ct(t, regs[t], other[t], tw, P.q, 2 * P.q2, P.one_s);
        }
        for (int t = 0; t < NT; t++) {
            PassIdx I = pass_idx(p, t);
            sm_store(regs[t], sm, I.base, I.stride);
        }
    }
    for (int j = 0; j < NPOLY; j++) a[j] = sm[swz(j)];
}

inline void host_emulate_inv(u64* a, const Tw* tw, const PrimeC& P) {
    static u64 regs[NT][EPT], other[NT][EPT];
    static u64 sm[NPOLY];
    for (int j = 0; j < NPOLY; j++) sm[swz(j)] = a[j];
    for (int p = 0; p < 3; p++) {
        for (int t = 0; t < NT; t++) {
            PassIdx I = pass_idx(2 - p, t);
            sm_load(regs[t], sm, I.base, I.stride);
        }
        if (p == 0) {
            for (int t = 0; t < NT; t++)
                for (int v = 0; v < EPT; v++) other[t][v] = regs[t ^ 1][v];
            for (int t = 0; t < NT; t++) st0_gs(t, regs[t], other[t], tw, P.q, P.q2);
        }
        if (p < 2) {
            for (int t = 0; t < NT; t++) {
                PassIdx I = pass_idx(2 - p, t);
                r16_gs(regs[t], tw, 1 + 4 * p, I.hi, P.q, P.q2);
                sm_store(regs[t], sm, I.base, I.stride);
            }
        }
    }
    for (int t = 0; t < NT; t++) {
        inv_tail(regs[t], tw, P);
        sm_store(regs[t], sm, t, NT);
    }
    for (int j = 0; j < NPOLY; j++) a[j] = sm[swz(j)];
}

}  // namespace hc
