/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement (RNS form) of the reference
 * BGV ring arithmetic on the Comp hot path.  This is the parity checker and
 * the `--impl reference` CPU arm of bench.py; the product library
 * (paper_2408_17063_b200/csrc) never links it and the product Python path
 * never loads it.
 *
 * Every routine follows a reference function; all arithmetic is exact.
 * The reference computes over the composite modulus Q_l with big integers;
 * per SURVEY.md F8 the residues of its composite-modulus NTT are exactly
 * the per-prime NTTs below, because psi_full = CRT(psi_i) (bgv.py:343-348).
 *
 *   orc_ntt_tables   <- NttContext.__init__        bgv.py:150-166
 *   orc_ntt_fwd      <- NttContext.fwd             bgv.py:178-199
 *   orc_ntt_inv      <- NttContext.inv             bgv.py:201-225
 *   orc_rescale      <- BgvBackend._mod_switch_once  bgv.py:579-608 (A.4)
 *   orc_digits       <- BgvBackend._key_switch digit loop bgv.py:622-631 (A.5)
 *   orc_mac_digits   <- BgvBackend._key_switch MAC  bgv.py:632-639
 *   orc_pointwise    <- BgvBackend._pointwise       bgv.py:431-437
 *
 * Built by oracle/Makefile into oracle/liboracle.so (gcc -O2 -fopenmp).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }

static u64 powmod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = mulmod(r, b, q);
        b = mulmod(b, b, q);
        e >>= 1;
    }
    return r;
}

static int bitrev(int i, int logn) {
    int r = 0;
    for (int b = 0; b < logn; b++) r |= ((i >> b) & 1) << (logn - 1 - b);
    return r;
}

/* bgv.py:156-166: tbl[i] = psi^bitrev(i), inv_tbl[i] = psi^-bitrev(i),
 * n_inv = n^-1 mod q.  (psi itself is _prim_root_2n, computed by the caller.) */
void orc_ntt_tables(u64 q, u64 psi, int n, u64 *tbl, u64 *inv_tbl, u64 *n_inv) {
    int logn = 0;
    while ((1 << logn) < n) logn++;
    u64 psi_inv = powmod(psi, q - 2, q);
    for (int i = 0; i < n; i++) {
        int e = bitrev(i, logn);
        tbl[i] = powmod(psi, (u64)e, q);
        inv_tbl[i] = powmod(psi_inv, (u64)e, q);
    }
    *n_inv = powmod((u64)n % q, q - 2, q);
}

/* bgv.py:178-199 (Cooley-Tukey, natural in / bit-reversed out). */
static void ntt_fwd_one(u64 *a, int n, u64 q, const u64 *tbl) {
    int t = n;
    for (int m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            int j1 = 2 * i * t;
            u64 S = tbl[m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 V = mulmod(a[j + t], S, q);
                u64 U = a[j];
                a[j] = (U + V) % q;
                a[j + t] = (U + q - V) % q;
            }
        }
    }
}

/* bgv.py:201-225 (Gentleman-Sande, then * n^-1). */
static void ntt_inv_one(u64 *a, int n, u64 q, const u64 *inv_tbl, u64 n_inv) {
    int t = 1;
    for (int m = n; m > 1; m >>= 1) {
        int j1 = 0;
        int h = m >> 1;
        for (int i = 0; i < h; i++) {
            u64 S = inv_tbl[h + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = (U + V) % q;
                a[j + t] = mulmod((U + q - V) % q, S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < n; j++) a[j] = mulmod(a[j], n_inv, q);
}

/* Batched transforms: a[count][n]; prime/table index per row via `which`
 * (row r uses q[which[r]], tbl + which[r]*n).  Inputs must be < q. */
void orc_ntt_fwd(u64 *a, int count, int n, const u64 *q, const u64 *tbls, const int *which) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < count; r++) {
        int w = which[r];
        ntt_fwd_one(a + (size_t)r * n, n, q[w], tbls + (size_t)w * n);
    }
}

void orc_ntt_inv(u64 *a, int count, int n, const u64 *q, const u64 *inv_tbls,
                 const u64 *n_invs, const int *which) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < count; r++) {
        int w = which[r];
        ntt_inv_one(a + (size_t)r * n, n, q[w], inv_tbls + (size_t)w * n, n_invs[w]);
    }
}

/* bgv.py:431-437: op 0 = mul, 1 = add, 2 = sub, over `rows` rows of n,
 * row r modulo q[r % P]. */
void orc_pointwise(const u64 *x, const u64 *y, u64 *out, int rows, int P, int n,
                   const u64 *q, int op) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < rows; r++) {
        u64 m = q[r % P];
        const u64 *a = x + (size_t)r * n, *b = y + (size_t)r * n;
        u64 *o = out + (size_t)r * n;
        for (int j = 0; j < n; j++) {
            if (op == 0) o[j] = mulmod(a[j], b[j], m);
            else if (op == 1) o[j] = (a[j] + b[j]) % m;
            else o[j] = (a[j] + m - b[j]) % m;
        }
    }
}

/* ---------------- multi-limb helpers (little-endian u64 limbs) ------------ */
#define ML 6 /* enough for 4 x 54-bit primes times a 64-bit factor */

static void ml_zero(u64 *a) { memset(a, 0, ML * sizeof(u64)); }

static void ml_mul_small(const u64 *a, u64 b, u64 *out) { /* out = a*b */
    u128 carry = 0;
    for (int i = 0; i < ML; i++) {
        u128 t = (u128)a[i] * b + carry;
        out[i] = (u64)t;
        carry = t >> 64;
    }
}

static void ml_add(u64 *a, const u64 *b) { /* a += b */
    u128 carry = 0;
    for (int i = 0; i < ML; i++) {
        u128 t = (u128)a[i] + b[i] + carry;
        a[i] = (u64)t;
        carry = t >> 64;
    }
}

static int ml_cmp(const u64 *a, const u64 *b) {
    for (int i = ML - 1; i >= 0; i--) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

static void ml_sub(u64 *a, const u64 *b) { /* a -= b, requires a >= b */
    u64 borrow = 0;
    for (int i = 0; i < ML; i++) {
        u64 bi = b[i] + borrow;
        u64 nb = (bi < borrow) || (a[i] < bi);
        a[i] = a[i] - bi;
        borrow = nb;
    }
}

static u64 ml_mod_small(const u64 *a, u64 q) {
    u128 r = 0;
    for (int i = ML - 1; i >= 0; i--) r = ((r << 64) | a[i]) % q;
    return (u64)r;
}

/* Exact CRT (bgv.py:129-137): constants for the modulus q[0..P). */
typedef struct {
    int P;
    u64 q[8];
    u64 Q[ML];      /* prod q_i */
    u64 M[8][ML];   /* Q / q_i */
    u64 Minv[8];    /* (Q / q_i)^-1 mod q_i */
} crt_t;

static void crt_init(crt_t *c, const u64 *q, int P) {
    u64 tmp[ML];
    c->P = P;
    ml_zero(c->Q);
    c->Q[0] = 1;
    for (int i = 0; i < P; i++) {
        c->q[i] = q[i];
        ml_mul_small(c->Q, q[i], tmp);
        memcpy(c->Q, tmp, sizeof tmp);
    }
    for (int i = 0; i < P; i++) {
        ml_zero(c->M[i]);
        c->M[i][0] = 1;
        for (int k = 0; k < P; k++) {
            if (k == i) continue;
            ml_mul_small(c->M[i], q[k], tmp);
            memcpy(c->M[i], tmp, sizeof tmp);
        }
        c->Minv[i] = powmod(ml_mod_small(c->M[i], q[i]), q[i] - 2, q[i]);
    }
}

/* the unique X in [0, Q) with X = x_i (mod q_i) */
static void crt_compose(const crt_t *c, const u64 *x, u64 *X) {
    u64 tmp[ML];
    ml_zero(X);
    for (int i = 0; i < c->P; i++) {
        u64 coef = mulmod(x[i] % c->q[i], c->Minv[i], c->q[i]);
        ml_mul_small(c->M[i], coef, tmp);
        ml_add(X, tmp);
        while (ml_cmp(X, c->Q) >= 0) ml_sub(X, c->Q);
    }
}

/* bgv.py:579-608, evaluated literally on the composed
 * integer.  x: coefficient-domain residues [P][n] of a level-(P-1)
 * polynomial in level-prime order (index P-1 = the prime divided out).
 * out: [P-1][n].  For each coefficient X in [0, Q_l):
 *   r = X mod q (centered), y = (X - r)/q, d = (X - y) mod p (centered),
 *   out = (y + d) mod Q_{l-1}. */
void orc_rescale(const u64 *x, u64 *out, int P, int n, const u64 *q, u64 p) {
    u64 qd = q[P - 1];
    crt_t crt;
    crt_init(&crt, q, P);
#pragma omp parallel for schedule(static)
    for (int j = 0; j < n; j++) {
        u64 res[8];
        for (int i = 0; i < P; i++) res[i] = x[(size_t)i * n + j];
        u64 X[ML], Xm[ML], rv[ML], y[ML];
        crt_compose(&crt, res, X);
        u64 rr = ml_mod_small(X, qd);
        int neg = rr > (qd >> 1); /* r = rr - qd when negative */
        memcpy(Xm, X, sizeof Xm);
        ml_zero(rv);
        if (!neg) {
            rv[0] = rr;
            ml_sub(Xm, rv);
        } else {
            rv[0] = qd - rr;
            ml_add(Xm, rv);
        }
        u128 rem = 0;
        for (int i = ML - 1; i >= 0; i--) {
            u128 cur = (rem << 64) | Xm[i];
            y[i] = (u64)(cur / qd);
            rem = cur % qd;
        }
        if (rem != 0) abort(); /* X - r is a multiple of q by construction */
        u64 xm = ml_mod_small(X, p), ym = ml_mod_small(y, p);
        u64 dd = (xm + p - ym) % p;
        int64_t d = (int64_t)dd;
        if (dd > (p >> 1)) d -= (int64_t)p;
        for (int i = 0; i < P - 1; i++) {
            u64 yi = ml_mod_small(y, q[i]);
            u64 v;
            if (d >= 0) v = (yi + (u64)d) % q[i];
            else v = (yi + q[i] - (u64)(-d)) % q[i];
            out[(size_t)i * n + j] = v;
        }
    }
}

/* bgv.py:622-631: coefficients x (RNS [P][n], canonical) -> the exact integer
 * in [0, Q_l), then D base-2^w digits: dig[j][k] = (X >> (w*j)) & (2^w - 1). */
void orc_digits(const u64 *x, u64 *dig, int P, int n, const u64 *q, int D, int w) {
    crt_t crt;
    crt_init(&crt, q, P);
#pragma omp parallel for schedule(static)
    for (int k = 0; k < n; k++) {
        u64 res[8];
        for (int i = 0; i < P; i++) res[i] = x[(size_t)i * n + k];
        u64 X[ML];
        crt_compose(&crt, res, X);
        u64 mask = (w == 64) ? ~0ull : ((1ull << w) - 1);
        for (int j = 0; j < D; j++) {
            int bit = w * j;
            int limb = bit >> 6, off = bit & 63;
            u64 v = 0;
            if (limb < ML) {
                v = X[limb] >> off;
                if (off && limb + 1 < ML) v |= X[limb + 1] << (64 - off);
            }
            dig[(size_t)j * n + k] = v & mask;
        }
    }
}

/* bgv.py:632-639: out0 = sum_j dig_ntt[j] * b_j mod Q, out1 = sum_j dig_ntt[j] * a_j.
 * dig_ntt: [D][P][n]; b, a: [D][P][n] (key already reduced to the level's primes);
 * out0/out1: [P][n]. */
void orc_mac_digits(const u64 *dig_ntt, const u64 *b, const u64 *a, u64 *out0, u64 *out1,
                    int D, int P, int n, const u64 *q) {
#pragma omp parallel for schedule(static)
    for (int i = 0; i < P; i++) {
        for (int k = 0; k < n; k++) {
            u64 s0 = 0, s1 = 0;
            for (int j = 0; j < D; j++) {
                size_t idx = ((size_t)j * P + i) * n + k;
                s0 = (s0 + mulmod(dig_ntt[idx], b[idx], q[i])) % q[i];
                s1 = (s1 + mulmod(dig_ntt[idx], a[idx], q[i])) % q[i];
            }
            out0[(size_t)i * n + k] = s0;
            out1[(size_t)i * n + k] = s1;
        }
    }
}

/* Exact composition to little-endian bytes of width 8*W (serialization,
 * bgv.py:787-789, and decrypt's centering bgv.py:571-575). out: [n][W] u64. */
void orc_compose(const u64 *x, u64 *out, int P, int n, const u64 *q, int W) {
    crt_t crt;
    crt_init(&crt, q, P);
#pragma omp parallel for schedule(static)
    for (int k = 0; k < n; k++) {
        u64 res[8];
        for (int i = 0; i < P; i++) res[i] = x[(size_t)i * n + k];
        u64 X[ML];
        crt_compose(&crt, res, X);
        for (int w = 0; w < W; w++) out[(size_t)k * W + w] = X[w];
    }
}

/* thread count for the calling thread's later parallel regions (torchrun
 * exports OMP_NUM_THREADS=1 to every rank; the CPU baseline wants them all) */
void orc_set_num_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_num_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
