// Per-coefficient building blocks of the Comp path (host+device so the CPU
// self-test can check them against the oracle):
//   crt_compose   exact CRT of RNS residues to the integer in [0, Q_l)
//                 (the reference keeps that integer natively, bgv.py:622)
//   digits16      its base-2^16 digits (bgv.py:627-629)
//   rescale_corr  the per-coefficient part of the modulus switch
//                 (bgv.py:592-603), in the linear-split form used on the GPU:
//                   out_k = x_k * q^-1 + e_k,  e_k = (d - r * q^-1) mod q_k
//                 with r = centered(x mod q), d = centered_p(r mod p);
//                 e_k depends only on the dropped prime's residue.
#pragma once
#include "ctx.cuh"

namespace hc {

// X = CRT(x_0..x_L) in [0, Q_L), x_k canonical residues; Q_L has L+1 limbs
// (every chain prime is 54 bits).  Compile-time L keeps arrays in registers.
template <int L>
HD void crt_compose(const LevelC& C, const PrimeC* pc, const u64* x, u64 (&X)[NLIMB]) {
    constexpr int P = L + 1, nl = L + 1;
    u64 y[P];
    double f = 0.0;
    HC_UNROLL
    for (int k = 0; k < P; k++) {
        y[k] = mul_shoup(x[k], C.Minv[k], C.Minv_s[k], pc[k].q);
        f += (double)y[k] * C.qrecip[k];
    }
    u64 S[nl];
    HC_UNROLL
    for (int i = 0; i < nl; i++) S[i] = 0;
    HC_UNROLL
    for (int k = 0; k < P; k++) {
        u64 carry = 0;
        HC_UNROLL
        for (int i = 0; i < nl; i++) {
            u128 t = (u128)y[k] * C.M[k][i] + S[i] + carry;
            S[i] = (u64)t;
            carry = (u64)(t >> 64);
        }
    }
    // X = S - kappa*Q with kappa = floor(sum y_k/q_k) (estimated, then fixed)
    const u64 kappa = (u64)f;
    u64 borrow = 0, carry = 0;
    HC_UNROLL
    for (int i = 0; i < nl; i++) {
        u128 t = (u128)kappa * C.Q[i] + carry;
        u64 tl = (u64)t;
        carry = (u64)(t >> 64);
        u64 s = S[i];
        u64 d = s - tl - borrow;
        borrow = (s < tl) || (s - tl < borrow) ? 1 : 0;
        X[i] = d;
    }
    HC_UNROLL
    for (int i = nl; i < NLIMB; i++) X[i] = 0;
    if (borrow) {  // went negative: add Q back
        u64 c = 0;
        HC_UNROLL
        for (int i = 0; i < nl; i++) {
            u128 t = (u128)X[i] + C.Q[i] + c;
            X[i] = (u64)t;
            c = (u64)(t >> 64);
        }
    } else {  // may be >= Q: subtract once
        int ge = 1, done = 0;
        HC_UNROLL
        for (int i = nl - 1; i >= 0; i--) {
            if (!done && X[i] != C.Q[i]) {
                ge = X[i] > C.Q[i];
                done = 1;
            }
        }
        if (ge) {
            u64 b = 0;
            HC_UNROLL
            for (int i = 0; i < nl; i++) {
                u64 s = X[i];
                u64 d = s - C.Q[i] - b;
                b = (s < C.Q[i]) || (s - C.Q[i] < b) ? 1 : 0;
                X[i] = d;
            }
        }
    }
}

// Two-prime CRT by Garner's formula (level 1): X = x0 + q0 * t with
// t = (x1 - x0) * q0^-1 mod q1, which lands in [0, q0 q1) directly -- one
// Shoup multiply and one 64x64 product instead of crt_compose<1>'s general
// sum-and-correct.  x0 < q0, x1 < q1 canonical.
HD void compose2(const LevelC& C, const PrimeC* pc, u64 x0, u64 x1, u64 (&X)[NLIMB]) {
    const u64 q0 = pc[0].q, q1 = pc[1].q;
    const u64 a = x0 >= q1 ? x0 - q1 : x0;  // x0 mod q1
    const u64 t = mul_shoup(sub_mod(x1, a, q1), C.g01, C.g01_s, q1);
    u64 hi, lo;
    mul128(hi, lo, q0, t);
    lo += x0;
    hi += lo < x0 ? 1 : 0;
    X[0] = lo;
    X[1] = hi;
    X[2] = 0;
    X[3] = 0;
}

// Q - X for X != 0 (0 stays 0): the coefficient a negated automorphism
// image carries (coeff_automorphism, bgv.py:273-284)
template <int L>
HD void neg_mod_Q(const LevelC& C, u64 (&X)[NLIMB]) {
    int nz = 0;
    HC_UNROLL
    for (int i = 0; i < L + 1; i++) nz |= X[i] != 0;
    if (!nz) return;
    u64 b = 0;
    HC_UNROLL
    for (int i = 0; i < L + 1; i++) {
        u64 q = C.Q[i], x = X[i];
        u64 d = q - x - b;
        b = (q < x) || (q - x < b) ? 1 : 0;
        X[i] = d;
    }
}

HD uint16_t digit16(const u64 (&X)[NLIMB], int j) {
    const int l = j >> 2;  // select chain: keeps X in registers for runtime j
    const u64 w = l == 0 ? X[0] : l == 1 ? X[1] : l == 2 ? X[2] : X[3];
    return (uint16_t)(w >> (16 * (j & 3)));
}

// Modulus-switch correction (see file header).  The constants of the
// switch from level l are gathered once (RescaleK) so the per-coefficient
// path touches registers only.
// NQ: kept primes the switch can produce (KEYL for the Comp's levels <= 3;
// MAXL only for the level-4 products of answer(), EP_RESCALE4).
template <int NQ = KEYL>
struct RescaleKT {
    int l;
    u64 ql, half_qd, p, half_p, pbar;
    u64 q[NQ], qinv[NQ], qinv_s[NQ];
};
using RescaleK = RescaleKT<KEYL>;
template <int NQ = KEYL>
HD RescaleKT<NQ> rescale_consts(const DevCtx& D, int l) {
    RescaleKT<NQ> R;
    R.l = l;
    R.ql = D.pc[l].q;
    R.half_qd = D.lv(l).half_qd;
    R.p = D.p;
    R.half_p = D.half_p;
    R.pbar = D.pbar;
    HC_UNROLL
    for (int k = 0; k < NQ; k++) {
        R.q[k] = D.pc[k].q;
        R.qinv[k] = D.lv(l).qinv[k];
        R.qinv_s[k] = D.lv(l).qinv_s[k];
    }
    return R;
}

// the constants rescale_rd reads, at any level (deep protocol chains: no LevelC)
HD RescaleK rescale_consts_rd(const DevCtx& D, int l) {
    RescaleK R;
    R.l = l;
    R.ql = D.pc[l].q;
    R.half_qd = D.pc[l].q >> 1;
    R.p = D.p;
    R.half_p = D.half_p;
    R.pbar = D.pbar;
    return R;
}

// x = canonical residue of the coefficient modulo the dropped prime q_l;
// writes e_k for k < l.
template <int NQ>
HD void rescale_corr(const RescaleKT<NQ>& R, u64 x, u64* e) {
    const bool neg = x > R.half_qd;
    const u64 mag = neg ? R.ql - x : x;  // |r| <= q_l / 2 < 2^53 <= q_k
    // d = centered_p(r mod p), r = x - neg (mod p) since q_l = 1 (mod p); 32-bit
    const u64 xm = x - mulhi(x, R.pbar) * R.p;  // Barrett: [0, 2p)
    const u32 p = (u32)R.p;
    u32 m = (u32)xm;
    m = m >= p ? m - p : m;
    m = neg ? (m ? m - 1 : p - 1) : m;
    const long long d = m > (u32)R.half_p ? (long long)m - (long long)p : (long long)m;
    HC_UNROLL
    for (int k = 0; k < NQ; k++) {
        if (k >= R.l) break;
        const u64 q = R.q[k];
        // e_k = d - r q_l^-1 = d -+ |r| q_l^-1 (mod q_k), from residues in [0, q)
        const u64 u = mul_shoup(mag, R.qinv[k], R.qinv_s[k], q);
        const u64 dk = d < 0 ? q + (u64)d : (u64)d;  // d mod q_k (|d| < p / 2)
        e[k] = reduce_once(dk + (neg ? u : q - u), q);  // q - u = q when u = 0: the sum stays < 2q
    }
}

HD void rescale_corr(const DevCtx& D, int l, u64 x, u64* e) { rescale_corr(rescale_consts(D, l), x, e); }

// any 64-bit value -> [0, q)
HD u64 red64(u64 a, u64 q, u64 one_s) { return reduce_once(mul_shoup_lazy(a, 1, one_s, q), q); }

// The integers behind rescale_corr: r = centered(x mod q_l) (|r| < q_l / 2)
// and d = centered_p(r mod p).  e_k = d - r q_l^-1 (mod q_k) is linear in
// (r, d), so a sum of corrections is formed from the sums of r and d (exact in
// int64 for up to 1024 terms) with one multiply per coefficient (k_diagx).
HD void rescale_rd(const RescaleK& R, u64 x, long long& r, long long& d) {
    const bool neg = x > R.half_qd;
    r = (long long)(x - (neg ? R.ql : 0));  // centered residue, |r| <= q_l / 2
    // r mod p: every chain prime is 1 mod p (hc_ctx_create checks), so
    // r = x - neg * q_l = x - neg (mod p); p < 2^31, 32-bit from here on
    const u64 xm = x - mulhi(x, R.pbar) * R.p;  // Barrett: [0, 2p)
    const u32 p = (u32)R.p;
    u32 m = (u32)xm;
    m = m >= p ? m - p : m;                      // x mod p
    m = neg ? (m ? m - 1 : p - 1) : m;           // r mod p in [0, p)
    d = m > (u32)R.half_p ? (long long)m - (long long)p : (long long)m;
}

// signed 64-bit -> [0, q)
HD u64 smod(long long v, u64 q, u64 one_s) {
    if (v >= 0) return red64((u64)v, q, one_s);
    const u64 m = red64((u64)(-(v + 1)) + 1, q, one_s);
    return m ? q - m : 0;
}

// e_k of a sum of rescale_rd terms: (sum d) - (sum r) q_l^-1 mod q_k
HD u64 corr_from_sums(long long sr, long long sd, u64 q, u64 qinv, u64 qinv_s, u64 one_s) {
    return sub_mod(smod(sd, q, one_s), mul_shoup(smod(sr, q, one_s), qinv, qinv_s, q), q);
}

}  // namespace hc
