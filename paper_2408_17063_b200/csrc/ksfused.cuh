// k_ksfused: the throughput-regime key switch of one rotation as ONE kernel
// (bgv.py:616-647: digit NTTs, key inner product, automorphism of c0, adds).
//
// The multi-launch form materialises every digit NTT in HBM (D x P x 64 KiB
// per rotation, written by k_xf and read back by k_ksmac_mb: ~0.4 GB per
// 64-block chunk at N = 2^20).  Here a CTA owns one 1024-point output chunk
// r of one (rotation, prime k) and walks the D digits itself:
//
//   front   the three leading Cooley-Tukey stages pair coefficients
//           a*1024 + b, a = 0..7 (ntt_cl.cuh phase A).  Their r-th output is
//           a fixed linear form  y_r(b) = sum_a K[k][r][a] * x[a*1024 + b]
//           (KFront: r8_ct applied to the unit vectors, host_tables.hpp), and
//           the inputs are base-2^16 digits, so the form is 8 x 2 IMAD.WIDE
//           (16 x 32-bit products, 64-bit sums < 2^51) and one Shoup
//           reduction -- cheaper than the three butterfly stages it replaces,
//           and chunk r needs no other chunk's data: no cluster, no DSMEM;
//   gather  the digit polynomial of rotation t at coefficient j is the
//           source digit at i = j * t^-1 mod 2n (of X for i < n, of Q - X
//           for i >= n: LD_DIGGAL's table, in closed form).  The CTA stages
//           the source digits [pos | neg] (32 KiB) in shared memory with one
//           bulk copy per digit (mbarrier-counted, issued a digit ahead) and
//           gathers from there: index = (j * tinv) & 16383;
//   local   stages 3..12 on the chunk: ntt_cl.cuh phase B (three radix-8
//           register passes through an 8 KiB tile + the lane-pair stage);
//   mac     acc0 += y * b_d, acc1 += y * a_d in 128-bit register accumulators
//           (<= 14 lazy terms < q 2^64), one REDC after the last digit, then
//           + perm(c0) (+ the pack_pair addends) as k_ksmac.
//
// Every value is the one the multi-launch schedule computes (exact modular
// arithmetic; the same final REDC of the same 128-bit sum).
// grid (8 chunks, P primes, jobs), 128 threads, 41 KiB dynamic smem.
#pragma once
#include "kernels.cuh"

namespace hc {

struct KFront {
    u64 k[KEYL + 1][8][8];  // [prime][chunk r][row a], canonical residues
    u64 w32s[KEYL + 1];     // Shoup constant of 2^32 mod q_k
};

struct KFJob {
    int level;   // P = level + 1 primes, D = digits at `level`
    int tinv;    // t^-1 mod 2n of the coefficient automorphism (1: none)
    int trace, pad;
    const uint16_t* dpos;  // [D][n] digits of X
    const uint16_t* dneg;  // [D][n] digits of Q - X (null when tinv == 1)
    const u64* key;        // [D_L][2][KL1][n] Montgomery
    const uint16_t* perm;  // NTT-domain permutation of c0src
    const u64* c0src;      // [P][n] (nullable)
    const u64* add0;       // [P][n] (nullable)
    const u64* add1;
    u64* out0;             // [P][n]
    u64* out1;
};

// digits [pos | neg] 32 KiB, tile 8 KiB, twiddle slice 1023 x 16 B with the
// mbarrier in its spare slot: 56 KiB, so four CTAs fill an SM's 228 KiB
constexpr int KF_SMEM = 2 * NPOLY * 2 + CTILE * 8 + 1024 * 16;

__device__ __forceinline__ void kf_bulk(void* dst, const void* src, uint32_t bytes, u64* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void kf_wait(u64* bar, unsigned par) {
    for (unsigned it = 0;; it++) {
        uint32_t done;
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(par)
            : "memory");
        if (done) break;
        if (it > (1u << 26)) __trap();  // a lost copy traps instead of hanging
    }
}

__global__ void __launch_bounds__(CNT, 4) k_ksfused(const __grid_constant__ DevCtx C, const __grid_constant__ KFront KF,
                                                     const KFJob* __restrict__ jobs) {
    extern __shared__ __align__(128) unsigned char kfsm[];
    const unsigned char* dig = kfsm;                              // u16 [pos 8192 | neg 8192]
    u64* tile = reinterpret_cast<u64*>(kfsm + 2 * NPOLY * 2);     // 8 KiB
    Tw* twsl = reinterpret_cast<Tw*>(tile + CTILE);               // this chunk's twiddles (TwL)
    u64* bar = reinterpret_cast<u64*>(twsl + 1023);
    const KFJob& J = jobs[blockIdx.z];
    TRACE(0);
    const int r = blockIdx.x, k = blockIdx.y, t = threadIdx.x;
    const PrimeC& P = C.pc[k];
    const int D = C.lv(J.level).D, L1 = C.KL1;
    const u64 q = P.q, q4 = 2 * P.q2;
    {   // constant for the plan: before pdl_wait
        TwPre tp;
        tw_issue(tp, C.twf + (size_t)k * NPOLY, r, t);
        tw_commit(twsl, tp, t);
    }
    const TwL tg{twsl, r};
    u32 klo[8], khi[8];
    HC_UNROLL
    for (int a = 0; a < 8; a++) {
        const u64 kk = KF.k[k][r][a];
        klo[a] = (u32)kk;
        khi[a] = (u32)(kk >> 32);
    }
    const u64 w32s = KF.w32s[k];
    const bool gal = J.dneg != nullptr;
    const uint32_t dbytes = gal ? 2 * NPOLY * 2 : NPOLY * 2;
    if (t == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // byte offsets of the gather: ((t + 128 e + 1024 a) * tinv mod 2n) * 2
    const unsigned tinv = (unsigned)J.tinv;
    const unsigned base2 = ((t * tinv) & 16383u) * 2, s128 = ((128u * tinv) & 16383u) * 2, s1024 = ((1024u * tinv) & 16383u) * 2;
    unsigned arow[8];  // a * s1024 mod 32 KiB (CTA-uniform)
    HC_UNROLL
    for (int a = 0; a < 8; a++) arow[a] = (a * s1024) & 0x7FFEu;
    __syncthreads();
    pdl_wait();  // the digits are the predecessor's (k_compose) output
    if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(dbytes) : "memory");
        kf_bulk(kfsm, J.dpos, NPOLY * 2, bar);
        if (gal) kf_bulk(kfsm + NPOLY * 2, J.dneg, NPOLY * 2, bar);
    }
    u64 h0[CEPT], l0[CEPT], h1[CEPT], l1[CEPT];
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) h0[v] = l0[v] = h1[v] = l1[v] = 0;
    const size_t jn = (size_t)k * NPOLY + r * CTILE + t;  // + 128 v: this thread's outputs
    HC_NOUNROLL
    for (int d = 0; d < D; d++) {
        u64 x[CEPT];
        kf_wait(bar, d & 1);  // digit d has landed
        // ---- front: y_r of columns b = t + 128 e ----
        unsigned cole = base2;
        HC_UNROLL
        for (int e = 0; e < CEPT; e++) {
            if (e) cole = (cole + s128) & 0x7FFEu;
            u32 dg[CEPT];
            HC_UNROLL
            for (int a = 0; a < 8; a++)
                dg[a] = *reinterpret_cast<const uint16_t*>(dig + ((cole + arow[a]) & 0x7FFEu));
            x[e] = kf_front(dg, klo, khi, w32s, q);
        }
        {
            const CPass I = cpass(0, r, t);
            r8_ct(x, tg, I.s0, I.G, q, q4);
            __syncthreads();  // every gather of digit d done (buffer free), every read of the tile done
            if (t == 0 && d + 1 < D) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(dbytes)
                             : "memory");
                kf_bulk(kfsm, J.dpos + (size_t)(d + 1) * NPOLY, NPOLY * 2, bar);
                if (gal) kf_bulk(kfsm + NPOLY * 2, J.dneg + (size_t)(d + 1) * NPOLY, NPOLY * 2, bar);
            }
            c_store(x, tile, I);
            __syncthreads();
        }
        HC_UNROLL
        for (int p = 1; p < 3; p++) {
            const CPass I = cpass(p, r, t);
            c_load(x, tile, I);
            r8_ct(x, tg, I.s0, I.G, q, q4);
            if (p == 2) c_st12<true>(r, t, x, tg, q, q4, P.one_s);
            c_store(x, tile, I);  // in place: the positions this thread loaded
            __syncthreads();
        }
        // ---- mac: outputs j = r*1024 + t + 128 v, keys streamed from L2 ----
        const u64* kp = J.key + (size_t)(d * 2) * L1 * NPOLY + jn;
        u64 kb[CEPT], ka[CEPT];
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) kb[v] = __ldcs(kp + 128 * v);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) ka[v] = __ldcs(kp + (size_t)L1 * NPOLY + 128 * v);
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) {
            const u64 y = tile[cswz(t) + 128 * v];
            mac128(h0[v], l0[v], y, kb[v]);
            mac128(h1[v], l1[v], y, ka[v]);
        }
    }
    TRACE(4);
    unsigned pe[CEPT];
    if (J.c0src) {
        HC_UNROLL
        for (int v = 0; v < CEPT; v++) pe[v] = J.perm[r * CTILE + t + 128 * v];
    }
    HC_UNROLL
    for (int v = 0; v < CEPT; v++) {
        HC_ASSERT(h0[v] < q && h1[v] < q);
        u64 o0 = redc(h0[v], l0[v], q, P.qneg), o1 = redc(h1[v], l1[v], q, P.qneg);
        if (J.add0) o0 = add_mod(o0, J.add0[jn + 128 * v], q);
        if (J.add1) o1 = add_mod(o1, J.add1[jn + 128 * v], q);
        if (J.c0src) o0 = add_mod(o0, J.c0src[(size_t)k * NPOLY + pe[v]], q);
        J.out0[jn + 128 * v] = o0;
        J.out1[jn + 128 * v] = o1;
    }
    TRACE(5);
}

}  // namespace hc
