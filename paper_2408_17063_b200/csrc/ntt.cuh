// Shared definitions of the 8192-point negacyclic NTT / INTT over one 54-bit
// prime (tables, constants).  Schedules: ntt1k.cuh (one CTA of 1024 threads
// per transform, throughput path) and ntt_cl.cuh (one 8-CTA cluster per
// transform, latency path).
//
// Semantics (bit-for-bit after canonicalisation):
//   forward = NttContext.fwd (bgv.py:178-199): Cooley-Tukey, natural-order
//             input, bit-reversed output, twiddle tbl[m+i] = psi^bitrev(m+i);
//   inverse = NttContext.inv (bgv.py:201-225): Gentleman-Sande with
//             inv_tbl[h+i] = psi^-bitrev(h+i), then * n^-1.
// Modular arithmetic is exact, so any schedule of the same butterflies gives
// the reference's values.
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
constexpr int NT = 1024;          // threads per single-CTA transform (ntt1k.cuh)
constexpr int EPT = NPOLY / NT;   // 8 coefficients per thread

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


}  // namespace hc
