// Modular arithmetic for 54-bit RNS primes (q < 2^54, so 4q < 2^56 and
// Harvey-style lazy ranges fit a 64-bit word).  Host+device: the same code
// is compiled by nvcc for sm_100a and by g++ for the CPU self-tests
// (tests/test_csrc_host.py), so the GPU arithmetic is checked bit-for-bit
// on the build machine, which has no GPU.
//
// Reference semantics being implemented: BgvBackend._pointwise (bgv.py:431-437),
// NttContext butterflies (bgv.py:185-198, 207-225), _mod_switch_once
// (bgv.py:579-608) and the _key_switch digit split (bgv.py:622-631).
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HD __host__ __device__ __forceinline__
#else
#define HD inline
#endif

namespace hc {

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

// high 64 bits of a*b
HD u64 mulhi(u64 a, u64 b) {
#if defined(__CUDA_ARCH__)
    return __umul64hi(a, b);
#else
    return (u64)(((u128)a * b) >> 64);
#endif
}

// Shoup constant for multiplication by w mod q: floor(w * 2^64 / q)
HD u64 shoup_const(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

// a * w mod q, result in [0, 2q) for any 64-bit a (w < q, ws = shoup_const(w))
HD u64 mul_shoup_lazy(u64 a, u64 w, u64 ws, u64 q) {
    u64 qh = mulhi(a, ws);
    return a * w - qh * q;
}

HD u64 reduce_once(u64 a, u64 q) { return a >= q ? a - q : a; }

HD u64 mul_shoup(u64 a, u64 w, u64 ws, u64 q) { return reduce_once(mul_shoup_lazy(a, w, ws, q), q); }

HD u64 add_mod(u64 a, u64 b, u64 q) { return reduce_once(a + b, q); }       // a,b < q
HD u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }  // a,b < q

// Montgomery reduction with R = 2^64: (hi:lo) < q * 2^64  ->  (hi:lo) * R^-1 mod q,
// result in [0, 2q).  qneg = -q^-1 mod 2^64.
HD u64 redc_lazy(u64 hi, u64 lo, u64 q, u64 qneg) {
    u64 m = lo * qneg;
    return hi + mulhi(m, q) + (lo != 0 ? 1 : 0);
}
HD u64 redc(u64 hi, u64 lo, u64 q, u64 qneg) { return reduce_once(redc_lazy(hi, lo, q, qneg), q); }

// 128-bit multiply-accumulate: (hi:lo) += a*b
HD void mac128(u64& hi, u64& lo, u64 a, u64 b) {
#if defined(__CUDA_ARCH__)
    asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;"
        : "+l"(lo), "+l"(hi)
        : "l"(a), "l"(b));
#else
    u128 t = ((u128)hi << 64 | lo) + (u128)a * b;
    lo = (u64)t;
    hi = (u64)(t >> 64);
#endif
}

HD void mul128(u64& hi, u64& lo, u64 a, u64 b) {
    lo = a * b;
    hi = mulhi(a, b);
}

// a * b mod q where bm = b * R mod q (Montgomery form), a < 2^64 with a*b < q*2^64
HD u64 mul_mont(u64 a, u64 bm, u64 q, u64 qneg) {
    u64 hi, lo;
    mul128(hi, lo, a, bm);
    return redc(hi, lo, q, qneg);
}

// the same without the final conditional subtraction: result in [0, 2q)
// (loader outputs of the inverse transforms, whose first stage takes < 2q)
HD u64 mul_mont_lazy(u64 a, u64 bm, u64 q, u64 qneg) {
    u64 hi, lo;
    mul128(hi, lo, a, bm);
    return redc_lazy(hi, lo, q, qneg);
}

// -q^-1 mod 2^64 (q odd)
HD u64 mont_qneg(u64 q) {
    u64 x = 1;
    for (int i = 0; i < 7; i++) x *= 2 - q * x;  // Newton: x = q^-1 mod 2^64
    return (u64)0 - x;
}

// host-only helpers (table construction)
inline u64 mulmod_slow(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
inline u64 powmod_slow(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod_slow(r, b, q);
        b = mulmod_slow(b, b, q);
        e >>= 1;
    }
    return r;
}

// ---------------------------------------------------------------------------
// Butterflies (Harvey lazy reduction)
// ---------------------------------------------------------------------------

// Cooley-Tukey forward butterfly, bgv.py:194-197.  In/out in [0, 4q).
HD void bf_ct(u64& X, u64& Y, u64 w, u64 ws, u64 q, u64 q2) {
    u64 x = X >= q2 ? X - q2 : X;
    u64 t = mul_shoup_lazy(Y, w, ws, q);
    X = x + t;
    Y = x - t + q2;
}

// Lazy forward butterfly used by the transforms: no reduction of X and a
// 3-product approximate Shoup quotient.  mulhi_approx(a, b) drops the
// lo x lo product and the low halves of the cross products, so it returns
// floor(a*b / 2^64) - {0, 1, 2}; hence t = Y*w - qhat*q lies in [0, 4q) for
// any 64-bit Y.  Each stage adds < 4q to the value range: from inputs < 4q,
// 13 stages stay below 56q < 2^60, and the caller canonicalises once.
#if defined(__CUDA_ARCH__)
// 32x32 -> 64-bit product as IMAD.WIDE.U32: full rate on the IMAD pipe,
// where IMAD.HI.U32 issues at half rate (hc_imad_peak: 17.2 vs 8.8 T/s)
__device__ __forceinline__ u64 mul_wide32(u32 x, u32 y) {
    u64 r;
    asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(x), "r"(y));
    return r;
}
#endif
HD u64 mulhi_approx(u64 a, u64 b) {
#if defined(__CUDA_ARCH__)
    const u32 al = (u32)a, ah = (u32)(a >> 32), bl = (u32)b, bh = (u32)(b >> 32);
    u64 r = mul_wide32(ah, bh);
    r += mul_wide32(ah, bl) >> 32;
    r += mul_wide32(al, bh) >> 32;
    return r;
#else
    const u64 al = (u32)a, ah = a >> 32, bl = (u32)b, bh = b >> 32;
    return ah * bh + ((ah * bl) >> 32) + ((al * bh) >> 32);
#endif
}

// a * w - mulhi_approx(a, ws) * q (mod 2^64): the lazy Shoup product, in
// [0, 4q) for any 64-bit a.  On the device the 64-bit expression is spelled
// out in 32-bit pieces so that ptxas emits the minimum: five IMAD.WIDE (three
// for the approximate quotient, one each for the low words of a * w and of
// qhat * (-q), the second accumulating onto the first), four IMAD for the
// cross terms chained into one 32-bit high-word sum, and two carry-chained
// add pairs -- 18 instructions per butterfly instead of the 23 the plain
// 64-bit C expression compiles to (no negation of qhat * q, no register moves
// to widen the quotient's addends, one add for the high word).
HD u64 mul_shoup_approx(u64 a, u64 w, u64 ws, u64 q) {
#if defined(__CUDA_ARCH__)
    const u64 nq = 0 - q;  // loop-invariant
    const u32 al = (u32)a, ah = (u32)(a >> 32), wl = (u32)w, wh = (u32)(w >> 32), sl = (u32)ws, sh = (u32)(ws >> 32);
    const u32 nl = (u32)nq, nh = (u32)(nq >> 32);
    const u64 p1 = mul_wide32(ah, sh), p2 = mul_wide32(ah, sl), p3 = mul_wide32(al, sh);
    u32 rl, rh;  // qhat = p1 + hi(p2) + hi(p3) = mulhi_approx(a, ws)
    asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;\n\tadd.cc.u32 %0, %0, %5;\n\taddc.u32 %1, %1, 0;"
        : "=&r"(rl), "=&r"(rh)
        : "r"((u32)p1), "r"((u32)(p2 >> 32)), "r"((u32)(p1 >> 32)), "r"((u32)(p3 >> 32)));
    u32 hi = ah * wl;
    hi = al * wh + hi;
    hi = rh * nl + hi;
    hi = rl * nh + hi;
    u64 t = mul_wide32(al, wl);
    asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(t) : "r"(rl), "r"(nl));
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"((u32)t), "r"((u32)(t >> 32) + hi));
    return r;
#else
    return a * w - mulhi_approx(a, ws) * q;
#endif
}

HD void bf_ct_lazy(u64& X, u64& Y, u64 w, u64 ws, u64 q, u64 q4) {
    const u64 t = mul_shoup_approx(Y, w, ws, q);  // [0, 4q)
    const u64 x = X;
    X = x + t;
    Y = x - t + q4;
}

// Lazy Gentleman-Sande inverse butterfly (bgv.py:217-220): X + Y and
// (X - Y) * w with the 3-product quotient; in/out in [0, 4q) (q4 = 4q < 2^56,
// so X + Y and X - Y + 4q stay below 2^57).
HD void bf_gs_lazy(u64& X, u64& Y, u64 w, u64 ws, u64 q, u64 q4) {
    const u64 x = X, y = Y;
    const u64 s = x + y;
    X = s >= q4 ? s - q4 : s;
    Y = mul_shoup_approx(x - y + q4, w, ws, q);  // [0, 4q)
}

// any value < 2^64 -> [0, q) (final canonicalisation of lazy transforms)
HD u64 canon_any(u64 x, u64 q, u64 one_s) { return reduce_once(x - mulhi(x, one_s) * q, q); }

// [0, 4q) -> [0, q)
HD u64 canon4(u64 x, u64 q, u64 q2) {
    x = x >= q2 ? x - q2 : x;
    return x >= q ? x - q : x;
}

// ---------------------------------------------------------------------------
// Small-modulus helpers for the plaintext prime p (< 2^31)
// ---------------------------------------------------------------------------

// a mod p for a < 2^53 using a double reciprocal and one fix-up each side
HD u64 mod_small(u64 a, u64 p, double pinv) {
    u64 qt = (u64)((double)a * pinv);
    int64_t r = (int64_t)(a - qt * p);
    while (r < 0) r += (int64_t)p;
    while (r >= (int64_t)p) r -= (int64_t)p;
    return (u64)r;
}

}  // namespace hc
