// Host-side table construction shared by libhcomp (hcomp.cu) and the CPU
// self-test (hosttest.cpp): twiddles (bgv.py:156-166), roots (bgv.py:120-126),
// per-level rescale / CRT constants, slot map (bgv.py:367-377), Galois
// index tables (bgv.py:258-261, 273-284).
#pragma once
#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.cuh"

namespace hc {

// ---------------------------------------------------------------------------
// host number theory
// ---------------------------------------------------------------------------
static inline int bitrev13(int i, int logn) {
    int r = 0;
    for (int b = 0; b < logn; b++) r |= ((i >> b) & 1) << (logn - 1 - b);
    return r;
}

// bgv.py:120-126: smallest g >= 2 whose (q-1)/2n power has order 2n
static inline uint64_t prim_root_2n_host(uint64_t q, int n) {
    for (u64 g = 2; g < q; g++) {
        u64 w = powmod_slow(g, (q - 1) / (2 * (u64)n), q);
        if (powmod_slow(w, (u64)n, q) == q - 1) return w;
    }
    return 0;
}

static inline u64 inv_mod(u64 a, u64 q) { return powmod_slow(a % q, q - 2, q); }

// Galois tables for X -> X^t (t odd, n = 2^logn)
static inline int galois_tables_host(int n, uint32_t t, uint16_t* coef, uint16_t* perm) {
    if (n != NPOLY || (t & 1) == 0) return 1;
    const int two_n = 2 * n;
    const int logn = LOGN;
    // t^-1 mod 2n
    int tinv = -1;
    for (int c = 1; c < two_n; c += 2)
        if ((long long)c * t % two_n == 1) {
            tinv = c;
            break;
        }
    if (tinv < 0) return 1;
    for (int pos = 0; pos < n; pos++) {
        // output coefficient pos receives +-c_i with i*t = pos (mod 2n) or pos+n
        int i = (int)((long long)pos * tinv % two_n);
        if (coef) coef[pos] = (uint16_t)(i < n ? i : ((i - n) | 0x8000));
        // NTT index k evaluates at psi^{e_k}, e_k = 2*bitrev(k)+1 (bgv.py:170-174)
        int e = 2 * bitrev13(pos, logn) + 1;
        int et = (int)((long long)e * t % two_n);
        if (perm) perm[pos] = (uint16_t)bitrev13((et - 1) / 2, logn);
    }
    return 0;
}

// limbs of a product of primes
static inline void limbs_mul(u64* a, int nl, u64 m) {
    u128 carry = 0;
    for (int i = 0; i < nl; i++) {
        u128 t = (u128)a[i] * m + carry;
        a[i] = (u64)t;
        carry = t >> 64;
    }
}
static inline u64 limbs_mod(const u64* a, int nl, u64 q) {
    u128 r = 0;
    for (int i = nl - 1; i >= 0; i--) r = ((r << 64) | a[i]) % q;
    return (u64)r;
}
static inline int bitlen_limbs(const u64* a, int nl) {
    for (int i = nl - 1; i >= 0; i--)
        if (a[i]) return 64 * i + (64 - __builtin_clzll(a[i]));
    return 0;
}

static inline void fill_prime(PrimeC& P, Tw* twf, Tw* twi, u64 q, int n) {
    const int logn = LOGN;
    u64 psi = prim_root_2n_host(q, n);
    u64 psi_inv = inv_mod(psi, q);
    for (int i = 0; i < n; i++) {
        int e = bitrev13(i, logn);
        u64 w = powmod_slow(psi, (u64)e, q);
        u64 wi = powmod_slow(psi_inv, (u64)e, q);
        twf[i].w = w;
        twf[i].ws = shoup_const(w, q);
        twi[i].w = wi;
        twi[i].ws = shoup_const(wi, q);
    }
    P.q = q;
    P.q2 = 2 * q;
    P.qneg = mont_qneg(q);
    P.ninv = inv_mod((u64)n, q);
    P.ninv_s = shoup_const(P.ninv, q);
    P.ninvw = mulmod_slow(twi[1].w, P.ninv, q);
    P.ninvw_s = shoup_const(P.ninvw, q);
    P.rmod = (u64)(((u128)1 << 64) % q);
    P.rmod_s = shoup_const(P.rmod, q);
    P.one_s = shoup_const(1, q);
}

// k_ksfused's front constants (ksfused.cuh): K[r][a] = output r of the three
// leading forward stages (ntt_cl.cuh phase A: r8_ct at s0 = 0, G = 0) applied
// to the unit vector e_a, as a canonical residue; w32s = Shoup(2^32)
static inline void build_kfront(u64 (*K)[8], u64* w32s, const Tw* twf, u64 q) {
    for (int a = 0; a < 8; a++) {
        u64 x[CEPT] = {0, 0, 0, 0, 0, 0, 0, 0};
        x[a] = 1;
        r8_ct(x, TwG{twf}, 0, 0, q, 4 * q);
        for (int r = 0; r < 8; r++) K[r][a] = x[r] % q;
    }
    *w32s = shoup_const(1ull << 32, q);
}

// Fill the device context (host copy; device pointers are set by the caller)
static inline void build_host_ctx(DevCtx& D, std::vector<Tw>& twf, std::vector<Tw>& twi,
                                  std::vector<uint16_t>& slot_of, int n, int max_level,
                                  const uint64_t* primes, uint64_t p, int* digits_out) {
    memset(&D, 0, sizeof D);
    memset(&D, 0, sizeof D);
    D.L = max_level;
    D.p = p;
    D.half_p = p >> 1;
    D.pinv = 1.0 / (double)p;
    D.pbar = (u64)(((u128)1 << 64) / p);
    twf.assign((size_t)NPR * n, Tw{});
    twi.assign((size_t)NPR * n, Tw{});
    // chain primes at RNS rows 0..L; unused rows (L < 3) get a copy of prime 0
    for (int k = 0; k < NPR; k++) {
        u64 q = (k == PIDX) ? p : (k <= max_level ? primes[k] : primes[0]);
        fill_prime(D.pc[k], &twf[(size_t)k * n], &twi[(size_t)k * n], q, n);
    }
    D.KL1 = std::min(max_level, KEYL) + 1;
    for (int l = 0; l <= max_level; l++) {
        LevelC scratch;  // level 0 and levels > LVC: digit count only
        LevelC& C = (l && l <= LVC) ? D.lvs[l - 1] : scratch;
        C.P = l + 1;
        C.nlimb = l + 1;
        u64 Qw[MAXL + 1] = {1};  // Q_l over l+1 limbs (digit count at every level)
        for (int k = 0; k <= l; k++) limbs_mul(Qw, MAXL + 1, primes[k]);
        C.D = (bitlen_limbs(Qw, MAXL + 1) + 15) / 16;
        digits_out[l] = C.D;
        if (l > LVC) continue;  // deep protocol levels: digit count only (no LevelC)
        C.half_qd = primes[l] >> 1;
        for (int k = 0; k < l; k++) {
            u64 qi = inv_mod(primes[l], primes[k]);
            C.qinv[k] = qi;
            C.qinv_s[k] = shoup_const(qi, primes[k]);
            C.qinv_r[k] = mulmod_slow(qi, D.pc[k].rmod, primes[k]);
            C.qinv_rs[k] = shoup_const(C.qinv_r[k], primes[k]);
        }
        if (l > KEYL) continue;  // level 4: modulus switch only (no compose on the device)
        memcpy(C.Q, Qw, sizeof C.Q);
        for (int k = 0; k <= l; k++) {
            u64 M[NLIMB] = {1, 0, 0, 0};
            for (int i = 0; i <= l; i++)
                if (i != k) limbs_mul(M, NLIMB, primes[i]);
            memcpy(C.M[k], M, sizeof M);
            u64 mi = inv_mod(limbs_mod(M, NLIMB, primes[k]), primes[k]);
            C.Minv[k] = mi;
            C.Minv_s[k] = shoup_const(mi, primes[k]);
            C.qrecip[k] = 1.0 / (double)primes[k];
        }
        if (l >= 1) {
            C.g01 = inv_mod(primes[0] % primes[1], primes[1]);
            C.g01_s = shoup_const(C.g01, primes[1]);
        }
    }
    // slot_of: NTT index -> (row << 12 | col)  (bgv.py:367-377)
    slot_of.assign(n, 0);
    {
        const int two_n = 2 * n, half = n / 2;
        long long e = 1;
        for (int c = 0; c < half; c++) {
            int i0 = bitrev13((int)((e - 1) / 2), LOGN);
            int i1 = bitrev13((int)((two_n - e - 1) / 2), LOGN);
            slot_of[i0] = (uint16_t)(0 << 12 | c);
            slot_of[i1] = (uint16_t)(1 << 12 | c);
            e = e * 3 % two_n;
        }
    }
}

}  // namespace hc
