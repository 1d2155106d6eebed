// Cluster NTT: one 8192-point transform per thread-block CLUSTER of 8 CTAs
// (8 SMs), 128 threads x 8 coefficients per CTA.  Latency path of the Comp
// (giant steps, folds, output mask) runs chains of 1-14 transforms; a
// single-CTA transform occupies one SM for ~18 us, the cluster form spreads
// it over 8 SMs.  Same arithmetic and semantics as ntt.cuh (bgv.py:178-225).
//
// Index j = a*1024 + b, a = bits 12..10 (CTA "row"), b = bits 9..0.
// Forward (CT, natural in, bit-reversed out):
//   phase A  CTA c, thread t owns column b = 128c + t, rows a = 0..7
//            (global loads coalesced); stages 0..2 (bits 12..10) in registers;
//            element (a, b) is stored into CTA a's shared tile at b (DSMEM);
//   cluster barrier;
//   phase B  CTA c owns j = c*1024 + b, b = 0..1023: three radix-8 register
//            passes over bits 9..7, 6..4, 3..1 through the local tile, then
//            bit 0 across lane pairs (shuffle); output coalesced.
// Inverse (GS): phase B' on CTA c's own rows (bit 0, then bits 1..9), DSMEM
// all-to-all into column layout, cluster barrier, phase A' = bits 10..12 in
// registers with n^-1 folded into the last stage.
#pragma once
#include "ntt.cuh"

namespace hc {

constexpr int CL = 8;       // CTAs per transform
constexpr int CNT = 128;    // threads per CTA
constexpr int CEPT = 8;     // coefficients per thread
constexpr int CTILE = 1024; // coefficients per CTA

// Twiddle access for stage "level" M (M = 2^s for CT stage s, 2^(12-b) for
// GS stage b).  TwG reads the global table; TwL reads the CTA's prefetched
// slice: for M >= 8, CTA c only touches indices [M + c*M/8, M + (c+1)*M/8),
// stored at local offset (M/8 - 1) + (idx - M - c*M/8): 1023 entries.
struct TwG {
    const Tw* t;
    HD Tw operator()(int idx, int M) const { return ldtw(t, idx); }
};
struct TwL {
    const Tw* sm;  // 1023 entries
    int c;
    HD Tw operator()(int idx, int M) const {
        const int m8 = M >> 3;
        const Tw* p = sm + (idx - M - c * m8 + m8 - 1);
#if defined(__CUDA_ARCH__)
        ulonglong2 v = *reinterpret_cast<const ulonglong2*>(p);
        Tw r;
        r.w = v.x;
        r.ws = v.y;
        return r;
#else
        return *p;
#endif
    }
};
// register-held twiddles tbl[1..7] (forward phase A)
struct TwR {
    const Tw* r;
    HD Tw operator()(int idx, int M) const { return r[idx]; }
};
// global index of local slice entry L (0..1022) of CTA c
HD int tw_slice_index(int L, int c) {
    int e = 0;
    while ((2 << e) - 1 <= L) e++;  // level with M/8 = 2^e entries: offsets [2^e - 1, 2^(e+1) - 1)
    const int m8 = 1 << e, M = m8 << 3;
    return M + c * m8 + (L - (m8 - 1));
}

// local tile swizzle for the three radix-8 patterns (64-bit, 16 lanes/phase):
// XOR bits 1..3 with bits 4..6
HD int cswz(int b) { return b ^ (((b >> 4) & 7) << 1); }

// phase-B pass p (0: bits 9..7, 1: bits 6..4, 2: bits 3..1) of CTA c:
// b(v) = base + v*stride; G = all index bits of j above the pass.
struct CPass {
    int base, stride, G, s0;
};
HD CPass cpass(int p, int c, int t) {
    CPass r;
    if (p == 0) {
        r.base = t; r.stride = 128; r.G = c; r.s0 = 3;
    } else if (p == 1) {
        r.base = ((t >> 4) << 7) | (t & 15); r.stride = 16; r.G = (c << 3) | (t >> 4); r.s0 = 6;
    } else {
        r.base = ((t >> 1) << 4) | (t & 1); r.stride = 2; r.G = (c << 6) | (t >> 1); r.s0 = 9;
    }
    return r;
}

// Swizzled index of element v of a pass, cswz(base + v * stride), in the form
// that costs the fewest address instructions (the stride is a compile-time
// constant wherever a pass is unrolled):
//   stride >= 128: v * stride leaves bits 1..6 alone, so cswz(base) + v * stride
//                  -- one address per pass, immediate offsets per element;
//   stride 16:     base has bits 4..6 clear (pass layouts), so bits 4..6 = v and
//                  the index is (base ^ 2v) + 16v -- one logic op per element;
//   stride 2:      base has bits 1..3 clear, bits 4..6 fixed: base | (2v ^ T).
HD int cswz_elem(int base, int stride, int v) {
    if (stride >= 128) return cswz(base) + v * stride;
    if (stride == 16) return (base ^ (2 * v)) + 16 * v;
    if (stride == 2) return base | ((2 * v) ^ (((base >> 4) & 7) << 1));
    return cswz(base + v * stride);
}
HD void c_load(u64 (&x)[CEPT], const u64* sm, const CPass& I) {
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) x[v] = sm[cswz_elem(I.base, I.stride, v)];
}
HD void c_store(const u64 (&x)[CEPT], u64* sm, const CPass& I) {
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) sm[cswz_elem(I.base, I.stride, v)] = x[v];
}

// 3 CT stages s0..s0+2 on 8 points: stage s0+u pairs v, v + (4 >> u),
// twiddle tbl[2^(s0+u) + (G << u | v >> (3-u))]
template <class TW>
HD void r8_ct(u64 (&x)[CEPT], const TW& tw, int s0, int G, u64 q, u64 q2) {
    HC_UNROLL
    for (int u = 0; u < 3; u++) {
        const int half = 4 >> u;
        const int tb = (1 << (s0 + u)) + (G << u);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            if (!(v & half)) {
                Tw w = tw(tb + (v >> (3 - u)), 1 << (s0 + u));
                bf_ct_lazy(x[v], x[v + half], w.w, w.ws, q, q2);
            }
        }
    }
}

// 3 GS stages b0..b0+2 on 8 points: stage b0+u pairs v, v + (1 << u),
// twiddle inv_tbl[2^(12-b0-u) + (G << (2-u) | v >> (u+1))].
// Inputs in [0, 4q).  The sums are NOT reduced inside the pass: a sum output
// doubles its operands' bound (compile-time per register: after the three
// stages x0 < 32q, x1 < 16q, x2, x3 < 8q; every product output is < 4q), the
// differences take the matching multiple of q as offset (4q / 8q / 16q), and
// seven conditional subtractions at the end (instead of one per butterfly,
// twelve) bring every output back below 4q.  q < 2^54, so 32q < 2^59.
HD void gs_csub(u64& x, u64 c) {  // x in [0, 2c) -> [0, c): the sign of x - c decides
    const u64 d = x - c;
    x = (long long)d < 0 ? x : d;
}
template <class TW>
HD void r8_gs(u64 (&x)[CEPT], const TW& tw, int b0, int G, u64 q, u64 q4) {
    const u64 q8 = 2 * q4, q16 = 4 * q4;
    HC_UNROLL
    for (int u = 0; u < 3; u++) {
        const int half = 1 << u;
        const int tb = (1 << (12 - b0 - u)) + (G << (2 - u));
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            if (!(v & half)) {
                Tw w = tw(tb + (v >> (u + 1)), 1 << (12 - b0 - u));
                // bound of both operands: 4q << (number of low bits of v below `half` that are 0 ... )
                // u = 0: 4q; u = 1: v even -> 8q, v odd -> 4q; u = 2: v = 0 -> 16q, v = 1 -> 8q, v = 2, 3 -> 4q
                const u64 off = u == 0 ? q4 : u == 1 ? ((v & 1) ? q4 : q8) : (v == 0 ? q16 : v == 1 ? q8 : q4);
                const u64 a = x[v], b = x[v + half];
                x[v] = a + b;
                x[v + half] = mul_shoup_approx(a - b + off, w.w, w.ws, q);
            }
        }
    }
    gs_csub(x[0], q16);
    gs_csub(x[0], q8);
    gs_csub(x[0], q4);
    gs_csub(x[1], q8);
    gs_csub(x[1], q4);
    gs_csub(x[2], q4);
    gs_csub(x[3], q4);
}

// forward bit-0 stage across lanes (t, t^1) in pass-2 layout:
// w = tbl[4096 + (j >> 1)], j >> 1 = (c << 9) | ((t >> 1) << 3) | v.
// The even lane holds X_v, the odd lane Y_v of 8 butterflies; each lane
// computes 4 of them (even: v = 4..7, odd: v = 0..3), so the stage costs
// half a pass of modmuls, with two exchanges of 4 values:
//   st12_send1 -> exchange -> st12_compute (-> 4 sends) -> exchange -> st12_recv2.
// Outputs canonical, or (LAZY) below 2^60 for consumers that only feed them
// to Montgomery products.
HD void st12_send1(int odd, const u64 (&x)[CEPT], u64 (&s)[4]) {
    HC_UNROLL
    for (int i = 0; i < 4; i++) s[i] = odd ? x[4 + i] : x[i];
}
template <bool LAZY = false, class TW>
HD void st12_compute(int c, int t, const u64 (&x)[CEPT], const u64 (&r)[4], const TW& tw, u64 q, u64 q4,
                     u64 one_s, u64 (&A)[4], u64 (&B)[4], u64 (&s)[4]) {
    const int odd = t & 1;
    const int tb = 4096 + (c << 9) + ((t >> 1) << 3);
    HC_UNROLL
    for (int i = 0; i < 4; i++) {
        u64 X = odd ? r[i] : x[4 + i];
        u64 Y = odd ? x[i] : r[i];
        Tw w = tw(tb + (odd ? i : 4 + i), 4096);
        bf_ct_lazy(X, Y, w.w, w.ws, q, q4);
        A[i] = LAZY ? X : canon_any(X, q, one_s);  // LAZY: < 2^60 (13 stages of < 4q growth)
        B[i] = LAZY ? Y : canon_any(Y, q, one_s);
        s[i] = odd ? A[i] : B[i];  // the partner's outputs
    }
}
HD void st12_recv2(int odd, u64 (&x)[CEPT], const u64 (&r)[4], const u64 (&A)[4], const u64 (&B)[4]) {
    HC_UNROLL
    for (int i = 0; i < 4; i++) {
        x[i] = odd ? B[i] : r[i];
        x[4 + i] = odd ? r[i] : A[i];
    }
}
#if defined(__CUDACC__)
template <bool LAZY = false, class TW>
__device__ __forceinline__ void c_st12(int c, int t, u64 (&x)[CEPT], const TW& tw, u64 q, u64 q4, u64 one_s) {
    const int odd = t & 1;
    u64 s[4], r[4], A[4], B[4];
    st12_send1(odd, x, s);
    HC_UNROLL
    for (int i = 0; i < 4; i++) r[i] = __shfl_xor_sync(0xffffffffu, s[i], 1);
    st12_compute<LAZY>(c, t, x, r, tw, q, q4, one_s, A, B, s);
    HC_UNROLL
    for (int i = 0; i < 4; i++) r[i] = __shfl_xor_sync(0xffffffffu, s[i], 1);
    st12_recv2(odd, x, r, A, B);
}
#endif
// host emulation of c_st12 over lane pairs: regs[t] for t in [0, n)
template <class TW>
inline void host_st12(int c, int n, u64 (*regs)[CEPT], const TW& tw, u64 q, u64 q4, u64 one_s) {
    static u64 snd[1024][4], A[1024][4], B[1024][4];
    for (int t = 0; t < n; t++) st12_send1(t & 1, regs[t], snd[t]);
    static u64 rcv[1024][4];
    for (int t = 0; t < n; t++)
        for (int i = 0; i < 4; i++) rcv[t][i] = snd[t ^ 1][i];
    for (int t = 0; t < n; t++) st12_compute(c, t, regs[t], rcv[t], tw, q, q4, one_s, A[t], B[t], snd[t]);
    for (int t = 0; t < n; t++)
        for (int i = 0; i < 4; i++) rcv[t][i] = snd[t ^ 1][i];
    for (int t = 0; t < n; t++) st12_recv2(t & 1, regs[t], rcv[t], A[t], B[t]);
}

// inverse bit-0 stage across lanes: the even lane keeps X + Y, the odd lane
// (X - Y) w; as for the forward stage each lane computes 4 butterflies
// (st12_send1 -> exchange -> st0_compute -> exchange -> st12_recv2).
// Inputs (loader output) in [0, 2q), outputs in [0, 4q).
template <class TW>
HD void st0_compute(int c, int t, const u64 (&x)[CEPT], const u64 (&r)[4], const TW& tw, u64 q, u64 q2,
                    u64 (&A)[4], u64 (&B)[4], u64 (&s)[4]) {
    const int odd = t & 1;
    const int tb = 4096 + (c << 9) + ((t >> 1) << 3);
    HC_UNROLL
    for (int i = 0; i < 4; i++) {
        const u64 X = odd ? r[i] : x[4 + i];
        const u64 Y = odd ? x[i] : r[i];
        Tw w = tw(tb + (odd ? i : 4 + i), 4096);
        const u64 d = X - Y + q2;
        A[i] = X + Y;
        B[i] = mul_shoup_approx(d, w.w, w.ws, q);
        s[i] = odd ? A[i] : B[i];
    }
}
#if defined(__CUDACC__)
template <class TW>
__device__ __forceinline__ void c_st0(int c, int t, u64 (&x)[CEPT], const TW& tw, u64 q, u64 q2) {
    const int odd = t & 1;
    u64 s[4], r[4], A[4], B[4];
    st12_send1(odd, x, s);
    HC_UNROLL
    for (int i = 0; i < 4; i++) r[i] = __shfl_xor_sync(0xffffffffu, s[i], 1);
    st0_compute(c, t, x, r, tw, q, q2, A, B, s);
    HC_UNROLL
    for (int i = 0; i < 4; i++) r[i] = __shfl_xor_sync(0xffffffffu, s[i], 1);
    st12_recv2(odd, x, r, A, B);
}
#endif
template <class TW>
inline void host_st0(int c, int n, u64 (*regs)[CEPT], const TW& tw, u64 q, u64 q2) {
    static u64 snd[1024][4], rcv[1024][4], A[1024][4], B[1024][4];
    for (int t = 0; t < n; t++) st12_send1(t & 1, regs[t], snd[t]);
    for (int t = 0; t < n; t++)
        for (int i = 0; i < 4; i++) rcv[t][i] = snd[t ^ 1][i];
    for (int t = 0; t < n; t++) st0_compute(c, t, regs[t], rcv[t], tw, q, q2, A[t], B[t], snd[t]);
    for (int t = 0; t < n; t++)
        for (int i = 0; i < 4; i++) rcv[t][i] = snd[t ^ 1][i];
    for (int t = 0; t < n; t++) st12_recv2(t & 1, regs[t], rcv[t], A[t], B[t]);
}

// k_ksfused's front (ksfused.cuh): output r of the three leading forward
// stages on a column whose inputs are base-2^16 digits, as the linear form
// sum_a K[r][a] * dg[a] (K = r8_ct at s0 = 0, G = 0 on the unit vectors, split
// into 32-bit halves klo / khi): 16 products of 16 x 32 bits, two 64-bit sums
// (< 2^51 and < 2^41), one Shoup reduction of the high part by 2^32.
// Result in [0, 2q + 2^32) -- a valid lazy input of the remaining ten stages.
HD u64 kf_front(const u32 (&dg)[CEPT], const u32 (&klo)[CEPT], const u32 (&khi)[CEPT], u64 w32s, u64 q) {
    u64 lo = 0, hi = 0;
    HC_UNROLL
    for (int a = 0; a < CEPT; a++) {
        lo += (u64)dg[a] * klo[a];  // IMAD.WIDE.U32 with 64-bit accumulate
        hi += (u64)dg[a] * khi[a];
    }
    const u64 H = hi + (lo >> 32);  // value = H * 2^32 + (u32)lo, H < 2^42
    return (H << 32) - mulhi(H, w32s) * q + (u32)lo;
}

// The bit-0 stage at the EDGE of a transform, in registers: the thread owns
// four coefficient pairs (j, j + 1) and w[m] = tbl[4096 + (j_m >> 1)].  The
// forward transform ends with it (epilogue side), the inverse starts with it
// (loader side); no lane exchange, none of c_st12 / c_st0's even/odd selects.
// Forward outputs canonical, or (lazy) below 2^60; inverse inputs in [0, 2q),
// outputs in [0, 4q).
HD void edge_fwd(u64 (&xe)[4], u64 (&xo)[4], const Tw (&w)[4], const PrimeC& P, bool lazy) {
    HC_UNROLL
    for (int m = 0; m < 4; m++) {
        bf_ct_lazy(xe[m], xo[m], w[m].w, w[m].ws, P.q, 2 * P.q2);
        if (!lazy) {
            xe[m] = canon_any(xe[m], P.q, P.one_s);
            xo[m] = canon_any(xo[m], P.q, P.one_s);
        }
    }
}
HD void edge_inv(u64 (&xe)[4], u64 (&xo)[4], const Tw (&w)[4], const PrimeC& P) {
    HC_UNROLL
    for (int m = 0; m < 4; m++) {
        const u64 X = xe[m], Y = xo[m];
        xe[m] = X + Y;
        xo[m] = mul_shoup_approx(X - Y + P.q2, w[m].w, w[m].ws, P.q);
    }
}
// cluster schedule: CTA c's thread t owns the local pairs 2t + 256m (tile
// index cswz(2t) + 256m: bit 0 and bits >= 7 are outside the swizzle), global
// coefficient c*1024 + 2t + 256m, twiddle index 4096 + 512c + t + 128m
HD int cpair_index(int t, int m) { return cswz(2 * t) + 256 * m; }
HD int cpair_tw(int c, int t, int m) { return 4096 + (c << 9) + t + 128 * m; }

// forward phase A: stages 0..2 on the column (x[a] = coefficient a*1024 + b)
HD void c_phaseA_fwd(u64 (&x)[CEPT], const Tw* tw, u64 q, u64 q4) { r8_ct(x, TwG{tw}, 0, 0, q, q4); }

// inverse phase A': GS stages 10, 11 on the column, then bit 12 folded with n^-1;
// wa = inv_tbl[1..7] (stages 10, 11 use indices 2..7), preloadable by the
// caller (constant)
HD void c_phaseA_inv_w(u64 (&x)[CEPT], const Tw (&wa)[8], const PrimeC& P) {
    const u64 q = P.q, q4 = 2 * P.q2;
    HC_UNROLL
    for (int u = 0; u < 2; u++) {
        const int half = 1 << u;
        const int tb = 1 << (2 - u);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            if (!(v & half)) {
                Tw w = wa[tb + (v >> (u + 1))];
                bf_gs_lazy(x[v], x[v + half], w.w, w.ws, q, q4);
            }
        }
    }
    // bit 12 with n^-1 folded in: exact Shoup takes any 64-bit input (< 8q here)
    HC_UNROLL
    for (int v = 0; v < 4; v++) {
        u64 a = x[v], b = x[v + 4];
        x[v] = reduce_once(mul_shoup_lazy(a + b, P.ninv, P.ninv_s, q), q);
        x[v + 4] = reduce_once(mul_shoup_lazy(a - b + q4, P.ninvw, P.ninvw_s, q), q);
    }
}
HD void c_phaseA_inv(u64 (&x)[CEPT], const Tw* tw, const PrimeC& P) {
    Tw wa[8];
    HC_UNROLL
    for (int i = 1; i < 8; i++) wa[i] = ldtw(tw, i);
    c_phaseA_inv_w(x, wa, P);
}

// ---- host emulation of the cluster schedule (CPU self-test only) ----------
inline void host_tw_slices(const Tw* tw, Tw (*sl)[1023]) {
    for (int c = 0; c < CL; c++)
        for (int L = 0; L < 1023; L++) sl[c][L] = tw[tw_slice_index(L, c)];
}

inline void host_emulate_cl_fwd(u64* a, const Tw* tw, const PrimeC& P) {
    static Tw sl[CL][1023];
    host_tw_slices(tw, sl);
    static u64 tile[CL][CTILE];
    static u64 regs[CL][CNT][CEPT];
    for (int c = 0; c < CL; c++)
        for (int t = 0; t < CNT; t++) {
            u64 x[CEPT];
            const int b = 128 * c + t;
            for (int r = 0; r < CEPT; r++) x[r] = a[r * CTILE + b];
            c_phaseA_fwd(x, tw, P.q, 2 * P.q2);
            for (int r = 0; r < CEPT; r++) tile[r][cswz(b)] = x[r];
        }
    for (int p = 0; p < 3; p++) {
        for (int c = 0; c < CL; c++)
            for (int t = 0; t < CNT; t++) {
                CPass I = cpass(p, c, t);
                c_load(regs[c][t], tile[c], I);
                r8_ct(regs[c][t], TwL{sl[c], c}, I.s0, I.G, P.q, 2 * P.q2);
            }
        if (p == 2)
            for (int c = 0; c < CL; c++) host_st12(c, CNT, regs[c], TwL{sl[c], c}, P.q, 2 * P.q2, P.one_s);
        for (int c = 0; c < CL; c++)
            for (int t = 0; t < CNT; t++) c_store(regs[c][t], tile[c], cpass(p, c, t));
    }
    for (int c = 0; c < CL; c++)
        for (int b = 0; b < CTILE; b++) a[c * CTILE + b] = tile[c][cswz(b)];
}

inline void host_emulate_cl_inv(u64* a, const Tw* tw, const PrimeC& P) {
    static Tw sl[CL][1023];
    host_tw_slices(tw, sl);
    static u64 tile[CL][CTILE], recv[CL][CTILE];
    static u64 regs[CL][CNT][CEPT];
    for (int c = 0; c < CL; c++)
        for (int b = 0; b < CTILE; b++) tile[c][cswz(b)] = a[c * CTILE + b];
    for (int p = 0; p < 3; p++) {
        for (int c = 0; c < CL; c++)
            for (int t = 0; t < CNT; t++) c_load(regs[c][t], tile[c], cpass(2 - p, c, t));
        if (p == 0) {
            for (int c = 0; c < CL; c++) host_st0(c, CNT, regs[c], TwL{sl[c], c}, P.q, P.q2);
        }
        for (int c = 0; c < CL; c++)
            for (int t = 0; t < CNT; t++) {
                CPass I = cpass(2 - p, c, t);
                r8_gs(regs[c][t], TwL{sl[c], c}, 1 + 3 * p, I.G, P.q, 2 * P.q2);
                if (p < 2) c_store(regs[c][t], tile[c], I);
            }
    }
    // all-to-all: element (a=c, b) -> CTA b>>7, slot a*128 + (b & 127)
    for (int c = 0; c < CL; c++)
        for (int t = 0; t < CNT; t++) {
            CPass I = cpass(0, c, t);
            for (int v = 0; v < CEPT; v++) {
                const int b = I.base + v * I.stride;
                recv[b >> 7][c * 128 + (b & 127)] = regs[c][t][v];
            }
        }
    for (int c = 0; c < CL; c++)
        for (int t = 0; t < CNT; t++) {
            u64 x[CEPT];
            for (int r = 0; r < CEPT; r++) x[r] = recv[c][r * 128 + t];
            c_phaseA_inv(x, tw, P);
            for (int r = 0; r < CEPT; r++) a[r * CTILE + 128 * c + t] = x[r];
        }
}

}  // namespace hc
