// CPU self-test shim (tests/test_csrc_host.py): compiles the device-side
// arithmetic, the 256-thread NTT schedule (emulated thread by thread), the
// CRT/digit split and the modulus-switch correction for the host with g++,
// so the exact code the GPU runs is checked against the oracle on a machine
// without a GPU.  Not part of the product library.
#include <cstring>
#include <cstdint>
#include <vector>

#include "elem.cuh"
#include "ntt1k.cuh"
#include "host_tables.hpp"

using namespace hc;

static DevCtx g_ctx;
static std::vector<Tw> g_twf, g_twi;
static std::vector<uint16_t> g_slot;
static int g_digits[MAXL + 1];

extern "C" int ht_init(const uint64_t* primes, int max_level, uint64_t p) {
    build_host_ctx(g_ctx, g_twf, g_twi, g_slot, NPOLY, max_level, primes, p, g_digits);
    g_ctx.twf = g_twf.data();
    g_ctx.twi = g_twi.data();
    g_ctx.slot_of = g_slot.data();
    return 0;
}

extern "C" int ht_digits(int level) { return g_digits[level]; }

// exact device NTT schedule on the host; k = RNS index (4 = p)
extern "C" void ht_ntt(int k, uint64_t* a, int inverse) {
    if (inverse) host_emulate_inv(a, g_ctx.twi + (size_t)k * NPOLY, g_ctx.pc[k]);
    else host_emulate_fwd(a, g_ctx.twf + (size_t)k * NPOLY, g_ctx.pc[k]);
}

// k_xf's form: bit-0 stage in registers at the kernel's edge (ntt1k.cuh)
extern "C" void ht_ntt_edge(int k, uint64_t* a, int inverse) {
    if (inverse) host_emulate_inv_edge(a, g_ctx.twi + (size_t)k * NPOLY, g_ctx.pc[k]);
    else host_emulate_fwd_edge(a, g_ctx.twf + (size_t)k * NPOLY, g_ctx.pc[k]);
}

extern "C" void ht_ntt_cl(int k, uint64_t* a, int inverse) {
    if (inverse) host_emulate_cl_inv(a, g_ctx.twi + (size_t)k * NPOLY, g_ctx.pc[k]);
    else host_emulate_cl_fwd(a, g_ctx.twf + (size_t)k * NPOLY, g_ctx.pc[k]);
}

template <int L>
static void compose_all(const uint64_t* x, const uint16_t* gal, int mode, uint16_t* dig) {
    const LevelC& LV = g_ctx.lv(L);
    const int D = LV.D;
    for (int pos = 0; pos < NPOLY; pos++) {
        int src = pos, neg = 0;
        if (mode == 0 && gal) {
            src = gal[pos] & 0x7FFF;
            neg = gal[pos] >> 15;
        }
        u64 xr[L + 1];
        for (int k = 0; k <= L; k++) xr[k] = x[(size_t)k * NPOLY + src];
        u64 X[NLIMB];
        crt_compose<L>(LV, g_ctx.pc, xr, X);
        if (mode == 0) {
            if (neg) neg_mod_Q<L>(LV, X);
            for (int j = 0; j < D; j++) dig[(size_t)j * NPOLY + pos] = digit16(X, j);
        } else {
            for (int j = 0; j < D; j++) dig[(size_t)j * NPOLY + pos] = digit16(X, j);
            neg_mod_Q<L>(LV, X);
            for (int j = 0; j < D; j++) dig[(size_t)(D + j) * NPOLY + pos] = digit16(X, j);
        }
    }
}

// compose2 (Garner, level 1) against crt_compose<1>: number of mismatches
extern "C" int ht_compose2_check(const uint64_t* x0, const uint64_t* x1, int count) {
    const LevelC& LV = g_ctx.lv(1);
    int bad = 0;
    for (int i = 0; i < count; i++) {
        u64 xr[2] = {x0[i], x1[i]};
        u64 A[NLIMB], B[NLIMB];
        crt_compose<1>(LV, g_ctx.pc, xr, A);
        compose2(LV, g_ctx.pc, x0[i], x1[i], B);
        bad += memcmp(A, B, sizeof A) != 0;
    }
    return bad;
}

extern "C" int ht_compose(int level, const uint64_t* x, const uint16_t* gal, int mode, uint16_t* dig) {
    switch (level) {
        case 1: compose_all<1>(x, gal, mode, dig); return 0;
        case 2: compose_all<2>(x, gal, mode, dig); return 0;
        case 3: compose_all<3>(x, gal, mode, dig); return 0;
        default: return 1;
    }
}

// e[k][j] for k < level from the dropped-prime residues x[j]
extern "C" void ht_rescale_corr(int level, const uint64_t* x, uint64_t* e) {
    for (int j = 0; j < NPOLY; j++) {
        u64 ek[MAXL];
        rescale_corr(g_ctx, level, x[j], ek);
        for (int k = 0; k < level; k++) e[(size_t)k * NPOLY + j] = ek[k];
    }
}

// rescale_rd + corr_from_sums (one term) against rescale_corr, and a sum of
// terms against the sum of corrections: number of mismatches
extern "C" int ht_rescale_rd_check(int level, const uint64_t* x, int count) {
    const RescaleK R = rescale_consts(g_ctx, level);
    int bad = 0;
    long long sr = 0, sd = 0;
    u64 se[MAXL] = {0, 0, 0};
    for (int i = 0; i < count; i++) {
        u64 e[MAXL];
        rescale_corr(R, x[i], e);
        long long r, d;
        rescale_rd(R, x[i], r, d);
        sr += r;
        sd += d;
        for (int k = 0; k < level; k++) {
            const PrimeC& P = g_ctx.pc[k];
            const LevelC& LV = g_ctx.lv(level);
            bad += corr_from_sums(r, d, P.q, LV.qinv[k], LV.qinv_s[k], P.one_s) != e[k];
            se[k] = add_mod(se[k], e[k], P.q);
        }
    }
    for (int k = 0; k < level; k++) {
        const PrimeC& P = g_ctx.pc[k];
        const LevelC& LV = g_ctx.lv(level);
        bad += corr_from_sums(sr, sd, P.q, LV.qinv[k], LV.qinv_s[k], P.one_s) != se[k];
    }
    return bad;
}

// Montgomery / Shoup helpers on arrays: op 0 = a*b mod q via mul_mont(a, b*R),
// op 1 = redc(hi, lo) of 128-bit a*b, op 2 = red64(a)
extern "C" void ht_modops(int k, int op, const uint64_t* a, const uint64_t* b, uint64_t* out, int count) {
    const PrimeC& P = g_ctx.pc[k];
    for (int i = 0; i < count; i++) {
        if (op == 0) {
            u64 bm = mul_shoup(b[i], P.rmod, P.rmod_s, P.q);
            out[i] = mul_mont(a[i], bm, P.q, P.qneg);
        } else if (op == 1) {
            u64 hi, lo;
            mul128(hi, lo, a[i], b[i]);
            u64 t = redc(hi, lo, P.q, P.qneg);
            out[i] = mul_shoup(t, P.rmod, P.rmod_s, P.q);
        } else {
            out[i] = red64(a[i], P.q, P.one_s);
        }
    }
}

// k_ksfused's digit NTT on the host (ksfused.cuh): the closed-form Galois
// gather ((j * tinv) mod 2n into [digits of X | digits of Q - X]), the front
// linear form of the three leading stages per output chunk, then the cluster
// schedule's phase B on the chunk; canonical output in natural order
extern "C" void ht_ksfused_ntt(int k, uint32_t t, const uint16_t* dpos, const uint16_t* dneg, uint64_t* out) {
    const PrimeC& P = g_ctx.pc[k];
    const Tw* tw = g_ctx.twf + (size_t)k * NPOLY;
    std::vector<uint16_t> coef(NPOLY);
    galois_tables_host(NPOLY, t, coef.data(), nullptr);
    const unsigned tinv = (coef[1] & 0x7FFF) + ((coef[1] >> 15) ? NPOLY : 0);
    u64 K[8][8], w32s;
    build_kfront(K, &w32s, tw, P.q);
    static Tw sl[CL][1023];
    host_tw_slices(tw, sl);
    static u64 tile[CTILE];
    static u64 regs[CNT][CEPT];
    for (int r = 0; r < CL; r++) {
        u32 klo[8], khi[8];
        for (int a = 0; a < 8; a++) {
            klo[a] = (u32)K[r][a];
            khi[a] = (u32)(K[r][a] >> 32);
        }
        const TwL twl{sl[r], r};
        for (int tt = 0; tt < CNT; tt++) {
            for (int e = 0; e < CEPT; e++) {
                u32 dg[CEPT];
                for (int a = 0; a < 8; a++) {
                    const unsigned i = ((unsigned)(tt + 128 * e + 1024 * a) * tinv) & 16383u;
                    dg[a] = i < (unsigned)NPOLY ? dpos[i] : dneg[i - NPOLY];
                }
                regs[tt][e] = kf_front(dg, klo, khi, w32s, P.q);
            }
            const CPass I = cpass(0, r, tt);
            r8_ct(regs[tt], twl, I.s0, I.G, P.q, 2 * P.q2);
            c_store(regs[tt], tile, I);
        }
        for (int p = 1; p < 3; p++) {
            for (int tt = 0; tt < CNT; tt++) {
                const CPass I = cpass(p, r, tt);
                c_load(regs[tt], tile, I);
                r8_ct(regs[tt], twl, I.s0, I.G, P.q, 2 * P.q2);
            }
            if (p == 2) host_st12(r, CNT, regs, twl, P.q, 2 * P.q2, P.one_s);
            for (int tt = 0; tt < CNT; tt++) c_store(regs[tt], tile, cpass(p, r, tt));
        }
        for (int b = 0; b < CTILE; b++) out[r * CTILE + b] = tile[cswz(b)];
    }
}

extern "C" void ht_galois(uint32_t t, uint16_t* coef, uint16_t* perm) { galois_tables_host(NPOLY, t, coef, perm); }

extern "C" void ht_slot_of(uint16_t* out) {
    for (int i = 0; i < NPOLY; i++) out[i] = g_slot[i];
}
