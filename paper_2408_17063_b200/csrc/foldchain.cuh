// k_foldchain: bsgs_matvec's fold chain (compress.py:306-307) as ONE
// persistent kernel with ONE grid-wide synchronisation per fold.
//
// Each fold res_{f+1} = res_f + rot(res_f, a_f) is a level-1 key switch
// (bgv.py:616-647).  The multi-launch schedule runs it as two kernels -- the
// two-prime INTT of res_f.c1 with the CRT/base-2^16 digit split (one 16-CTA
// cluster), then 2 x D_1 = 14 digit NTTs -- and pays two producer->consumer
// hand-offs through global memory per fold (~2-3 us each: grid completion,
// griddepcontrol release, loads; profiles/r02_trace_*).  Here D_1 = 7
// co-resident 16-CTA clusters stay on the SMs for the whole chain and
// cluster d owns digit d:
//   A  every cluster inverts res_f.c1 itself (CTAs 0-7 prime 0, 8-15
//      prime 1, k_cl16_intt2's schedule) and CRT-composes its 512
//      coefficients per CTA -- the INTT is recomputed by all 7 clusters (the
//      GPU is otherwise idle in the chain) so no cluster waits for another's
//      digits.  Each composed coefficient's digit d (of X, or of Q - X where
//      the automorphism negates) is pushed with st.async straight to the two
//      CTAs (one per prime half) whose forward-NTT column needs it: the
//      rotation's inverse Galois table names the destination;
//   B  each 8-CTA half waits for its 1024 digits (mbarrier byte count),
//      runs the forward NTT at prime = half (k_xf_cl's schedule) and
//      red.adds NTT(digit) * key_d into the next accumulator;
//   then one grid barrier.  The c0 half of the fold (base + perm(c0) +
//   red(acc.c0), bgv.py:643-645) and the zeroing of the accumulator two folds
//   back run in the barrier's slack.  Accumulators rotate over three
//   buffers: fold f reads ACC[f%3] (res_f's key-switch sums, read by all 7
//   clusters, so never zeroed by its readers), writes ACC[(f+1)%3], zeroes
//   ACC[(f+2)%3] (read in fold f-1, next written in fold f+1: both ordered by
//   the barriers).  Every value is computed exactly as in the multi-launch
//   schedule (same loaders, butterflies, CRT, digits and MAC).
#pragma once
#include "kernels.cuh"

namespace hc {

constexpr int FC_MAXF = 12;  // folds: log2(4096 / s_pad)
constexpr int FC_CL = 16;    // CTAs per cluster (non-portable size)
struct FcFold {
    const u64* base1;     // res_{f-1}.c1 (or acc[0].c1 for f = 0) [2 primes][n], nullable
    const u64* accf;      // ACC[f % 3]: [2 polys][2 primes][n] key-switch sums of res_f
    u64* cur;             // res_f: [2 polys][2 primes][n]
    const uint16_t* igal; // inverse coefficient Galois gather of rotation a_f
    const u64* key;       // its KSK [D_L][2][KL1][n], Montgomery
    u64* acc_next;        // ACC[(f+1) % 3]
    u64* acc_zero;        // ACC[(f+2) % 3] (c1 rows zeroed here; c0 rows by their reader)
    // s0 decoded on the host (<= FC_C0T terms: one per fold, up to three
    // giant steps before the first), so the c0 finish needs no dependent load
    // of the spec: res_f.c0 = c0base + sum_i c0src_i[perm_i] + red(c0acc)
    int c0n;              // terms (the host falls back to two launches per fold when s0 does not fit)
    const u64* c0base;    // nullable
    const u64* c0src[MAXTERM_KS];
    const uint16_t* c0perm[MAXTERM_KS];
    u64* c0acc;
};
constexpr int FC_C0T = 3;  // terms whose gathers are prefetched; further ones (fold 0 at giant > 4) load in the slack
struct FcArgs {
    int F, D;
    unsigned* bar;  // grid-barrier arrival counter, zeroed before the launch
    FcFold f[FC_MAXF];
};

__device__ __forceinline__ void fc_arm(u64* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fc_put(u64* dst, unsigned rank, u64 v, u64* bar) {
    uint32_t ra, rb;
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(smem_u32(dst)), "r"(rank));
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];\n" ::"r"(ra), "l"(v), "r"(rb)
                 : "memory");
}
__device__ __forceinline__ void fc_wait(u64* bar, unsigned par) {
    for (unsigned it = 0;; it++) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(par)
            : "memory");
        if (done) break;
        if (it > (1u << 26)) __trap();  // a lost transfer traps instead of hanging
    }
}
__device__ __forceinline__ void fc_put32(uint32_t* dst, unsigned rank, uint32_t v, u64* bar) {
    uint32_t ra, rb;
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(smem_u32(dst)), "r"(rank));
    asm("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(smem_u32(bar)), "r"(rank));
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(ra), "r"(v), "r"(rb)
                 : "memory");
}
__device__ __forceinline__ unsigned fc_ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// grid barrier number `gen` (1, 2, ...) over `ncta` CTAs: every CTA's global
// writes (stores and red.adds) before it are visible to every CTA after it:
// release = gpu-scope fence + arrival by thread 0 after the CTA barrier,
// acquire = thread 0's ld.acquire.gpu poll, extended to the CTA by the
// barrier.  Every load of data another CTA wrote is an L2 load (__ldcg), so
// no L1 invalidation (a second gpu-scope fence) is needed after the wait
__device__ __forceinline__ void fc_grid_bar(unsigned* ctr, unsigned gen, unsigned ncta) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        const unsigned target = gen * ncta;
        for (unsigned it = 0; fc_ld_acquire(ctr) < target; it++)
            if (it > (1u << 24)) __trap();
#ifdef HC_FC_FENCE2
        __threadfence();
#endif
    }
    __syncthreads();
}

#ifdef HC_TRACE
// per-fold phase stamps: [fold][CTA][point] (%globaltimer)
constexpr int FT_F = FC_MAXF, FT_CTA = 128, FT_PT = 12;
__device__ unsigned long long g_fc_trace[FT_F][FT_CTA][FT_PT];
#define FTRACE(f, pt)                                                                \
    do {                                                                             \
        if (threadIdx.x == 0 && blockIdx.x < FT_CTA) {                               \
            unsigned long long tnow;                                                 \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));                 \
            g_fc_trace[f][blockIdx.x][pt] = tnow;                                    \
        }                                                                            \
    } while (0)
#else
#define FTRACE(f, pt) \
    do {              \
    } while (0)
#endif

// smem words: tile | recv | fwd twiddle slice | inv twiddle slice | half |
// received digits (1024 u32) | 4 mbarriers
constexpr int FC_SMEM_WORDS = CTILE + CTILE + 2 * 1024 + 2 * 1024 + 4 * CNT + 512 + 4;

__global__ void __launch_bounds__(CNT, 1) k_foldchain(const __grid_constant__ DevCtx C, const __grid_constant__ FcArgs A) {
    extern __shared__ __align__(16) u64 fsm[];
    u64* tile = fsm;
    u64* recv = fsm + CTILE;
    Tw* twf_sl = reinterpret_cast<Tw*>(fsm + 2 * CTILE);
    Tw* twi_sl = reinterpret_cast<Tw*>(fsm + 2 * CTILE + 2 * 1024);
    u64* half = fsm + 2 * CTILE + 4 * 1024;
    uint32_t* drecv = reinterpret_cast<uint32_t*>(half + 4 * CNT);  // this CTA's NTT inputs, [v][t] (1024 digits)
    u64* xbar = half + 4 * CNT + 512;  // INTT all-to-all (8 KiB per use)
    u64* hbar = xbar + 1;              // INTT half exchange (4 KiB per use)
    u64* fbar = xbar + 2;              // forward NTT all-to-all (8 KiB per use)
    u64* dbar = xbar + 3;              // digits pushed by the composing CTAs (4 KiB per use)
    unsigned rank;
    asm("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
    const int t = threadIdx.x;
    const int k = (int)(rank >> 3);  // prime of this CTA (INTT half and NTT half alike)
    const int c = (int)(rank & 7);
    const int d = blockIdx.x / FC_CL;  // digit of this cluster
    const unsigned ncta = gridDim.x;
    const unsigned hbase = (unsigned)k << 3;
    const unsigned partner = (unsigned)((1 - k) * 8 + c);
    const PrimeC& P = C.pc[k];
    const LevelC& LV = C.lv(1);
    const int KL1 = C.KL1;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(xbar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(hbar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(fbar)) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(dbar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        fc_arm(xbar, CTILE * 8);
        fc_arm(hbar, 4 * CNT * 8);
        fc_arm(fbar, CTILE * 8);
        fc_arm(dbar, CTILE * 4);
    }
    unsigned xuse = 0, huse = 0, fuse = 0, duse = 0;  // completed uses of each barrier (wait parity)
    {   // constants for the whole chain: both twiddle slices of prime k
        TwPre pf, pi;
        tw_issue(pf, C.twf + (size_t)k * NPOLY, c, t);
        tw_issue(pi, C.twi + (size_t)k * NPOLY, c, t);
        tw_commit(twf_sl, pf, t);
        tw_commit(twi_sl, pi, t);
    }
    Tw waf[8], wai[8];
    HC_UNROLL
    for (int i = 1; i < 8; i++) {
        waf[i] = ldtw(C.twf + (size_t)k * NPOLY, i);
        wai[i] = ldtw(C.twi + (size_t)k * NPOLY, i);
    }
    const int b = 128 * c + t;  // forward loader column of this thread
    const int mine0 = k ? 4 : 0, theirs0 = k ? 0 : 4;
    // per-fold constants, fetched a fold ahead: the inverse Galois entries of
    // the 4 coefficients this thread composes, and the key digit pair
    // (b_d, a_d) at prime k at this CTA's NTT outputs
    unsigned ig[4];
    u64 kb[CEPT], ka[CEPT];
    const int gtid = blockIdx.x * CNT + t, gthreads = gridDim.x * CNT;
    unsigned c0pe[2][FC_C0T] = {};  // the c0 finish's permutation entries of this thread's <= 2 elements
    auto fetch = [&](int f) {
        const FcFold& F = A.f[f];
        HC_UNROLL
        for (int i = 0; i < 2; i++) {
            const int e = gtid + i * gthreads;
            HC_UNROLL
            for (int tt = 0; tt < FC_C0T; tt++)
                if (e < 2 * NPOLY && tt < F.c0n) c0pe[i][tt] = F.c0perm[tt][e & (NPOLY - 1)];
        }
        const u64* kbp = F.key + ((size_t)(d * 2 + 0) * KL1 + k) * NPOLY + c * CTILE + t;
        const u64* kap = F.key + ((size_t)(d * 2 + 1) * KL1 + k) * NPOLY + c * CTILE + t;
        HC_UNROLL
        for (int i = 0; i < 4; i++) ig[i] = F.igal[(mine0 + i) * CTILE + 128 * c + t];
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            kb[v] = kbp[128 * v];
            ka[v] = kap[128 * v];
        }
    };
    fetch(0);
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");  // barriers initialised,
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");    // twiddle slices stored
    asm volatile("griddepcontrol.wait;\n" ::: "memory");  // the giant step's accumulators are complete
    const TwL tlf{twf_sl, c}, tli{twi_sl, c};
    unsigned gen = 0;
    for (int f = 0; f < A.F; f++) {
        const FcFold& F = A.f[f];
        // ---- A: INTT of res_f.c1 = base + red(ACC[f%3].c1) at prime k ----
        FTRACE(f, 0);
        u64 x[CEPT];
        {
            const int jl = c * CTILE + t;
            const u64* ac = F.accf + (size_t)(2 + k) * NPOLY;
            const u64* bs = F.base1 ? F.base1 + (size_t)k * NPOLY : nullptr;
            u64 av[CEPT], bv[CEPT];
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) {
                av[v] = __ldcg(ac + jl + 128 * v);
                bv[v] = bs ? __ldcg(bs + jl + 128 * v) : 0;
            }
            u64* aux = (d == 0) ? F.cur + (size_t)(2 + k) * NPOLY : nullptr;  // res_f.c1 (one writer)
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) {
                x[v] = add_mod(bv[v], red64(av[v], P.q, P.one_s), P.q);
                if (aux) aux[jl + 128 * v] = x[v];
            }
        }
        // res_f.c0 = c0base + sum_i c0src_i[perm_i] + red(ACC[f%3].c0) (bgv.py:643-645):
        // its loads go out now (independent: operands decoded on the host,
        // permutation entries fetched a fold ahead), the sums are formed after
        // the NTT (<= 2 elements per thread; its single reader re-zeroes ACC[f%3].c0)
        u64 c0x[2], c0a[2], c0g[2][FC_C0T];
        HC_UNROLL
        for (int i = 0; i < 2; i++) {
            const int e = gtid + i * gthreads;
            if (e < 2 * NPOLY) {
                const size_t kofs = (size_t)(e >> 13) * NPOLY;
                const int j = e & (NPOLY - 1);
                c0x[i] = F.c0base ? __ldcg(F.c0base + kofs + j) : 0;
                c0a[i] = __ldcg(F.c0acc + kofs + j);
                HC_UNROLL
                for (int tt = 0; tt < FC_C0T; tt++) c0g[i][tt] = tt < F.c0n ? __ldcg(F.c0src[tt] + kofs + c0pe[i][tt]) : 0;
            }
        }
        FTRACE(f, 1);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) tile[cswz(t) + 128 * v] = x[v];
        __syncthreads();
        HC_UNROLL
        for (int p = 0; p < 3; p++) {
            const CPass I = cpass(2 - p, c, t);
            c_load(x, tile, I);
            if (p == 0) c_st0(c, t, x, tli, P.q, P.q2);
            r8_gs(x, tli, 1 + 3 * p, I.G, P.q, 2 * P.q2);
            if (p < 2) {
                c_store(x, tile, I);
                __syncthreads();
            }
        }
        FTRACE(f, 2);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) fc_put(recv + c * 128 + t, hbase + v, x[v], xbar);
        fc_wait(xbar, xuse & 1);
        FTRACE(f, 3);
        xuse++;
        if (t == 0) fc_arm(xbar, CTILE * 8);
        HC_UNROLL
        for (int r = 0; r < CEPT; r++) x[r] = recv[r * 128 + t];
        c_phaseA_inv_w(x, wai, P);  // x[r] = coefficient r*1024 + 128c + t mod q_k
        HC_UNROLL
        for (int i = 0; i < 4; i++) fc_put(half + i * CNT + t, partner, x[theirs0 + i], hbar);
        fc_wait(hbar, huse & 1);
        FTRACE(f, 4);
        huse++;
        if (t == 0) fc_arm(hbar, 4 * CNT * 8);
        HC_UNROLL
        for (int i = 0; i < 4; i++) {
            // coefficient (mine0 + i) * 1024 + 128c + t lands at automorphism
            // position dst = ig & 0x7FFF (negated when ig >> 15): NTT column
            // (dst >> 7) & 7, slot (dst >> 10) * 128 + (dst & 127) of both halves
            const u64 mine = x[mine0 + i], other = half[i * CNT + t];
            u64 X[NLIMB];
            compose2(LV, C.pc, k ? other : mine, k ? mine : other, X);  // (mod q0, mod q1)
            if (ig[i] >> 15) neg_mod_Q<1>(LV, X);
            const uint32_t dig = digit16(X, d);
            const unsigned dst = ig[i] & 0x7FFF;
            const unsigned col = (dst >> 7) & 7;
            uint32_t* slot = drecv + (dst >> 10) * CNT + (dst & 127);
            fc_put32(slot, col, dig, dbar);
            fc_put32(slot, 8 + col, dig, dbar);
        }
        FTRACE(f, 5);
        fc_wait(dbar, duse & 1);  // this CTA's 1024 NTT inputs have arrived
        duse++;
        if (t == 0) fc_arm(dbar, CTILE * 4);
        FTRACE(f, 6);
        // ---- B: forward NTT of digit d at prime k ----
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) x[v] = drecv[v * CNT + t];
        u64 kbs[CEPT], kas[CEPT];
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            kbs[v] = kb[v];
            kas[v] = ka[v];
        }
        FTRACE(f, 7);
        if (f + 1 < A.F) fetch(f + 1);  // in flight during the NTT
        r8_ct(x, TwR{waf}, 0, 0, P.q, 2 * P.q2);
        HC_UNROLL
        for (int r = 0; r < CEPT; r++) fc_put(tile + cswz(b), hbase + r, x[r], fbar);
        fc_wait(fbar, fuse & 1);
        FTRACE(f, 8);
        fuse++;
        if (t == 0) fc_arm(fbar, CTILE * 8);
        HC_UNROLL
        for (int p = 0; p < 3; p++) {
            const CPass I = cpass(p, c, t);
            c_load(x, tile, I);
            r8_ct(x, tlf, I.s0, I.G, P.q, 2 * P.q2);
            if (p == 2) c_st12<true>(c, t, x, tlf, P.q, 2 * P.q2, P.one_s);
            c_store(x, tile, I);
            __syncthreads();
        }
        FTRACE(f, 9);
        {
            u64* a0 = F.acc_next + (size_t)k * NPOLY + c * CTILE + t;
            u64* a1 = F.acc_next + (size_t)(2 + k) * NPOLY + c * CTILE + t;
            HC_UNROLL
            for (int v = 0; v < CEPT; v++) {
                const u64 y = tile[cswz(t) + 128 * v];
                acc_add(a0 + 128 * v, mul_mont(y, kbs[v], P.q, P.qneg), KSACC_BOUND);
                acc_add(a1 + 128 * v, mul_mont(y, kas[v], P.q, P.qneg), KSACC_BOUND);
            }
        }
        FTRACE(f, 10);
        // ---- slack: res_f.c0 formed from the loads issued at the fold's
        //      start, ACC[(f+2)%3].c1 cleared for fold f+1's sums ----
        HC_UNROLL
        for (int i = 0; i < 2; i++) {
            const int e = gtid + i * gthreads;
            if (e < 2 * NPOLY) {
                const PrimeC& PC = C.pc[e >> 13];
                const size_t kofs = (size_t)(e >> 13) * NPOLY;
                const int j = e & (NPOLY - 1);
                u64 v = add_mod(c0x[i], red64(c0a[i], PC.q, PC.one_s), PC.q);
                HC_UNROLL
                for (int tt = 0; tt < FC_C0T; tt++) v = add_mod(v, c0g[i][tt], PC.q);  // absent terms are 0
                for (int tt = FC_C0T; tt < F.c0n; tt++)
                    v = add_mod(v, __ldcg(F.c0src[tt] + kofs + F.c0perm[tt][j]), PC.q);
                F.cur[kofs + j] = v;
                F.c0acc[kofs + j] = 0;
                F.acc_zero[2 * NPOLY + e] = 0;
            }
        }
        FTRACE(f, 11);
        if (f + 1 < A.F) fc_grid_bar(A.bar, ++gen, ncta);
    }
}

}  // namespace hc
