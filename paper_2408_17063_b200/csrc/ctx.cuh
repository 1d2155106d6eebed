// Device-visible context: per-prime constants, per-level rescale / CRT
// constants, twiddle tables and slot/Galois index tables.  Built on the host
// by hcomp.cu (HostCtx) from the chain primes; consumed by kernels.cuh.
#pragma once
#include "ntt.cuh"

namespace hc {

// Chains of up to 5 primes (max_level 4).  Comp's fused schedule runs at
// levels <= 3 (the 4 smallest primes); level 4 only carries the Mask /
// pack-pair products of answer() (pdq.py:238-256) down to level 3, so CRT
// compose, digit decomposition and key switching stop at level 3 (KEYL).
#ifndef HC_MAXL
#define HC_MAXL 4  // build.py compiles -DHC_MAXL=3 (libhcomp.so), 4 (libhcomp_l4.so), 22 (libhcomp_deep.so)
#endif
constexpr int MAXL = HC_MAXL;  // max level supported (MAXL + 1 chain primes)
constexpr int KEYL = MAXL < 3 ? MAXL : 3;        // highest level with device key switching / CRT compose
// levels with a LevelC entry: the Comp's levels (<= 4).  Deeper levels of a
// protocol chain (pdq.protocol_max_level = 21) only carry ring transforms and
// the modulus switch of mul_plain, whose per-prime constants travel with the
// call (hcomp.cu, mul_plain_deep) -- the context passed by value to every
// kernel stays small.
constexpr int LVC = MAXL < 4 ? MAXL : 4;
constexpr int NPR = MAXL + 2;  // chain primes + plaintext prime p (index 5)
constexpr int PIDX = MAXL + 1; // RNS index of p in the tables
constexpr int NLIMB = 4;       // limbs for composed integers (216 bits: levels <= KEYL)
constexpr int MAXD = 14;       // digits at level 3 (216-bit modulus, base 2^16)

// Constants for level l (P = l+1 primes at RNS indices 0..l).
struct LevelC {
    int P, D;             // primes, base-2^16 digits of Q_l (bgv.py:360-363)
    int nlimb;            // limbs of Q_l
    int pad;
    // modulus switch l -> l-1 (drops prime l), bgv.py:579-608
    u64 half_qd;          // q_l >> 1
    u64 qinv[KEYL + 1];   // q_l^-1 mod q_k (k < l <= MAXL)
    u64 qinv_s[KEYL + 1];
    u64 qinv_r[KEYL + 1]; // q_l^-1 * R mod q_k (Montgomery, folded into plaintexts)
    u64 qinv_rs[KEYL + 1];
    // CRT compose at level l <= KEYL
    u64 Minv[KEYL + 1], Minv_s[KEYL + 1];  // (Q_l/q_k)^-1 mod q_k
    u64 M[KEYL + 1][NLIMB];                // Q_l/q_k
    u64 Q[NLIMB];                          // Q_l
    double qrecip[KEYL + 1];               // 1/q_k
    u64 g01, g01_s;                        // Garner: q_0^-1 mod q_1 (compose2)
};

struct DevCtx {
    const Tw* twf;       // [NPR][n]
    const Tw* twi;       // [NPR][n]
    const uint16_t* slot_of;  // [n]: NTT index -> (row << 12 | col)
    u64 p, half_p;
    double pinv;
    u64 pbar;  // floor(2^64 / p): integer Barrett for r mod p
    int L;    // max level
    int KL1;  // RNS rows per key digit on the device: min(L, KEYL) + 1
    PrimeC pc[NPR];
    LevelC lvs[LVC];  // levels 1..LVC (kernel parameter space: no level-0 entry)
    HD const LevelC& lv(int l) const { return lvs[l - 1]; }
};

}  // namespace hc
