// Host-side restatement of CPython's random.Random (Modules/_randommodule.c,
// the MT19937 reference generator) with exactly the consumption semantics the
// reference backend's samplers rely on (bgv.py:398-414 via random.Random):
//   seed(int)        init_by_array over |seed| as little-endian 32-bit words
//   getrandbits(k)   k <= 32: one word >> (32 - k); k > 32: words from least
//                    to most significant, the last one truncated to its bits
//   randrange(n)     _randbelow_with_getrandbits: r = getrandbits(bitlen(n))
//                    until r < n
// so keygen/encrypt consume the same stream as the reference and produce
// bit-identical keys and ciphertexts (checked against random.Random itself in
// tests/test_host_logic.py and against the reference goldens).
#pragma once
#include <cstdint>
#include <vector>

namespace hc {

struct PyMT {
    static constexpr int N = 624, M = 397;
    uint32_t mt[N];
    int mti = N + 1;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < N; mti++) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t* key, int len) {
        init_genrand(19650218u);
        int i = 1, j = 0;
        for (int k = N > len ? N : len; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            i++;
            j++;
            if (i >= N) {
                mt[0] = mt[N - 1];
                i = 1;
            }
            if (j >= len) j = 0;
        }
        for (int k = N - 1; k; k--) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            i++;
            if (i >= N) {
                mt[0] = mt[N - 1];
                i = 1;
            }
        }
        mt[0] = 0x80000000u;
        mti = N;
    }
    uint32_t next32() {
        static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
        uint32_t y;
        if (mti >= N) {
            int kk;
            for (kk = 0; kk < N - M; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + M] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < N - 1; kk++) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[N - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ mag01[y & 1u];
            mti = 0;
        }
        y = mt[mti++];
        y ^= (y >> 11);
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= (y >> 18);
        return y;
    }
    // getrandbits(k) into little-endian 32-bit words (ceil(k / 32) of them)
    void getrandbits(int k, uint32_t* words) {
        if (k <= 32) {
            words[0] = k ? next32() >> (32 - k) : 0;
            return;
        }
        const int nw = (k - 1) / 32 + 1;
        for (int i = 0; i < nw; i++, k -= 32) {
            uint32_t r = next32();
            if (k < 32) r >>= (32 - k);
            words[i] = r;
        }
    }
    // randrange(n) for 0 < n < 2^32
    uint32_t randbelow32(uint32_t n) {
        int k = 0;
        while (k < 32 && (n >> k)) k++;  // bit_length
        uint32_t r;
        do {
            getrandbits(k, &r);
        } while (r >= n);
        return r;
    }
    // randrange(Q) for a multi-word Q (little-endian 32-bit words, bit length kbits)
    void randbelow_words(const uint32_t* q, int nw, int kbits, uint32_t* out) {
        for (;;) {
            getrandbits(kbits, out);
            int lt = 0;  // out < q ?
            for (int i = nw - 1; i >= 0; i--)
                if (out[i] != q[i]) {
                    lt = out[i] < q[i];
                    break;
                }
            if (lt) return;
        }
    }
};

}  // namespace hc
