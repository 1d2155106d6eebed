/*
 * hcomp -- B200-native (sm_100a) BGV Comp for arXiv 2408.17063.
 *
 * C ABI of libhcomp.so.  Plain pointers and sizes only; the library owns all
 * device memory tied to a context.  One context per CUDA stream; a context is
 * not re-entrant (the reference backend is not thread-safe either:
 * bgv.py:358-359, heiface.py:174).
 *
 * The reference (Python, /root/reference/pkg/src/hcpdq) has no native ABI;
 * the Python package paper_2408_17063_b200 binds these entry points with
 * ctypes behind the reference's own API (comp / BgvBackend methods).  Each
 * entry point below names the reference interface it replaces.
 *
 * Data layout of every ring element: RNS residues uint64[P][n], row k the
 * residue modulo level_prime(k) (bgv.py:104-106: row 0 = smallest prime,
 * the last row is the prime a modulus switch divides out), values in [0, q_k).
 * A ciphertext at level l is uint64[2][l+1][n] (c0 then c1), NTT domain.
 * Only n = 8192 is supported; max_level <= 3 (libhcomp.so), 4 (libhcomp_l4.so)
 * or up to 22 (libhcomp_deep.so: pdq's protocol chain, whose levels above 4
 * carry ring transforms and mul_plain's modulus switch only).  Key switching, CRT
 * compose and the fused Comp run at levels <= 3 (the 4 smallest primes);
 * level 4 is for the Mask / pack products of answer() (pdq.py:238-256),
 * which enter Comp through hc_comp_packed.
 */
#ifndef HCOMP_H
#define HCOMP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps them onto the reference exceptions */
#define HC_OK 0
#define HC_ERR_ARG 1      /* ValueError            (compress.py:282-283, 348-349) */
#define HC_ERR_LEVEL 2    /* LevelExhausted        (bgv.py:721-722) */
#define HC_ERR_KEY 3      /* MissingRotationKey    (bgv.py:760-761, 767-768) */
#define HC_ERR_MISMATCH 4 /* BackendMismatch       (bgv.py:443-450, 654-655) */
#define HC_ERR_CUDA 5     /* CUDA runtime failure (no reference analogue) */
#define HC_ERR_STATE 6    /* call out of order (e.g. comp before plan) */

typedef struct hc_ctx hc_ctx;

/* last error message of the calling thread (static storage) */
const char* hc_last_error(void);
/* RNS table row of the plaintext prime p in hc_ntt / hc_pointwise prime
 * indices (chain primes occupy rows 0..max_level) */
int hc_plain_row(void);

/* Replaces BgvBackend.__init__ tables (bgv.py:328-363) and NttContext.__init__
 * (bgv.py:150-174).  primes: the L+1 chain primes in LEVEL order
 * (primes[k] = level_prime(k), ascending); p: plaintext modulus;
 * ksw_base_bits must be 16 (bgv.py:333).  device: CUDA ordinal. */
int hc_ctx_create(int n, int max_level, const uint64_t* primes, uint64_t p, int ksw_base_bits,
                  int device, hc_ctx** out);
void hc_ctx_destroy(hc_ctx* h);
/* digits D_l per level (bgv.py:360-363) into digits[0..max_level] */
int hc_ctx_digits(const hc_ctx* h, int* digits);

/* Replaces KeySet.rotation_keys / col_swap_key material (bgv.py:482-509,
 * _KskPair bgv.py:294-312).  Uploads one gadget key-switch key for the
 * Galois element t (3^r mod 2n for rot_row(r), 2n-1 for rot_col):
 * ksk = uint64[D_L][2][L+1][n] = (b_j, a_j) pairs, NTT domain residues.
 * At max_level 4 the device keeps the first D_3 digits on the 4 smallest
 * primes (what _KskPair.at_level yields at levels <= 3). */
int hc_load_ksk(hc_ctx* h, uint32_t galois_t, const uint64_t* ksk);
int hc_clear_keys(hc_ctx* h);
/* The same from a slice of a deep chain's key: ksk = uint64[digits][2][rows][n]
 * holding the first `digits` pairs on the `rows` smallest primes (level
 * order).  A protocol chain (pdq.protocol_max_level = 21: 75 digits x 22
 * primes) only ever key-switches at levels <= 3, where _KskPair.at_level
 * (bgv.py:304-312) reads the first 14 digits on the 4 smallest primes. */
int hc_load_ksk_slice(hc_ctx* h, uint32_t galois_t, const uint64_t* ksk, int digits, int rows);

/* Replaces compress._plan / build_plan (compress.py:198-270, packed mode,
 * no cleartext database): generates every diagonal, the pack masks and the
 * output mask on the device and records the Comp schedule (a CUDA graph).
 * chunk_blocks: blocks processed per pass (0 = automatic).
 * Fails with HC_ERR_KEY if a needed rotation key is not loaded. */
int hc_plan(hc_ctx* h, int64_t N, int s, int chunk_blocks);
/* hc_plan for one rank of a block-sharded Comp: only the
 * diagonals of blocks [b0, b1) are generated and only input ciphertexts
 * [b0/2, (b1+1)/2) are allocated, so a rank's plan memory and generation
 * time are O(N / world); run it with hc_comp_set_inputs_range +
 * hc_comp_partial(h, b', b'', ...) for sub-ranges of [b0, b1) and
 * hc_comp_finish.  The whole-matrix entry points return HC_ERR_STATE. */
int hc_plan_range(hc_ctx* h, int64_t N, int s, int chunk_blocks, int64_t b0, int64_t b1);
/* hc_plan with the plaintexts (pack masks, diagonals, output mask) of
 * another context's current plan on the same device and chain: config 5's
 * independent queries over one database share one copy of the diagonals
 * (the buffers are reference counted and live while any plan uses them).
 * The source plan must be a whole-matrix hint-path plan (hc_plan). */
int hc_plan_shared(hc_ctx* h, const hc_ctx* src, int chunk_blocks);

/* Replaces _plan(params, "packed", masked) for comp_masked (compress.py:
 * 154-157, 521-530): as hc_plan, but the bottom lane evaluates
 * D = C diag(DB) (VandermondeTable with db_values, compress.py:107-135).
 * db_mod_p = uint64[N], the cleartext database reduced mod p (int(v) % p).
 * Run it with hc_comp(h, cv, cv, ...): the index vector is both inputs. */
int hc_plan_masked(hc_ctx* h, int64_t N, int s, int chunk_blocks, const uint64_t* db_mod_p);
/* schedule facts: [B, C, baby, giant, F, s_pad, live_diagonals, kernel_launches];
 * kernel_launches counts the one-graph Comp, or in sharded mode the captured
 * hc_comp_partial graphs plus the hc_comp_finish graph; -1 before a capture */
int hc_plan_info(const hc_ctx* h, int64_t* info8);

/* Replaces compress.comp(cd, ..., index_hint=cv) (compress.py:488-514),
 * host buffers: cd, cv = uint64[C][2][4][n] at level 3; out = uint64[2][1][n]
 * (the level-0 ciphertext of the CompressedAnswer).  Synchronous. */
int hc_comp(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, uint64_t* out);

/* Replaces compress.comp(cd, ..., index_hint=cv) when cd and cv sit at
 * different levels -- answer()'s cd = mask(cv) (pdq.py:238-256) one level
 * below cv, reconciled by add's _at_level (bgv.py:656-658) inside pack_pair
 * (compress.py:338-367).  The caller runs pack_pair with the single-op entry
 * points below and passes its outputs: u = uint64[B][2][3][n], the B packed
 * two-row ciphertexts at level 2 (NTT domain, canonical residues); the
 * baby steps, diagonal products, giant steps, folds and the output mask run
 * as in hc_comp (one graph launch).  out = uint64[2][1][n].  Synchronous. */
int hc_comp_packed(hc_ctx* h, const uint64_t* u, int64_t B, uint64_t* out);
/* The same for answer()'s inputs as they arrive: cd = uint64[C][2][ld+1][n]
 * at level ld, cv = uint64[C][2][lv+1][n] at level lv, min(ld, lv) = 3,
 * max <= max_level (each list at one level).  pack_pair itself runs on the
 * device -- mul_plain at each input's level, rot_col, the modulus switch of
 * add's _at_level, the add -- in the same graph as the BSGS steps.
 * HC_ERR_LEVEL when an input is below level 3 (the reference raises
 * LevelExhausted at the output mask).  Synchronous. */
int hc_comp_mixed(hc_ctx* h, const uint64_t* cd, int ld, const uint64_t* cv, int lv, int C, uint64_t* out);

/* Replaces pdq.answer after Match (pdq.py:248-256): cd = mask(cv, db)
 * (pdq.py:238-245) then comp(cd, index_hint=cv), in one graph launch.
 * hc_answer_db first turns the cleartext database (uint64[N], reduced mod p)
 * into the mask plaintexts at `level` for the current plan (repeat after
 * hc_plan); hc_answer then takes cv = uint64[C][2][lv+1][n] at level
 * lv = 4 (max_level 4) and writes out = uint64[2][1][n].  Synchronous. */
int hc_answer_db(hc_ctx* h, int level, const uint64_t* db_mod_p);
int hc_answer(hc_ctx* h, const uint64_t* cv, int lv, int C, uint64_t* out);
/* Replay the last hc_comp_mixed / hc_answer graph on `stream` with the inputs
 * already on the device (one graph launch; read the output with
 * hc_comp_get_output). */
int hc_mixed_launch(hc_ctx* h, void* stream);

/* Device-resident variant for timing: inputs already uploaded with
 * hc_comp_set_inputs; hc_comp_launch enqueues the whole Comp (one graph
 * launch) on `stream` (a cudaStream_t, NULL = legacy default stream). */
int hc_comp_set_inputs(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C);
/* Sharded use: upload only input ciphertexts [c0, c1) (host buffers hold
 * exactly those c1 - c0 ciphertexts, layout as above), asynchronously on
 * `stream` (pinned host memory for a true async copy).  A rank running
 * blocks [b0, b1) needs ciphertexts [b0/2, (b1+1)/2). */
int hc_comp_set_inputs_range(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int c0, int c1, void* stream);
/* Streamed use: inputs already in device memory (e.g. uploaded on a copy
 * stream while the previous query computes) -> the plan's input buffers,
 * device to device, on `stream`. */
int hc_comp_set_inputs_device(hc_ctx* h, const uint64_t* cd_dev, const uint64_t* cv_dev, int C, void* stream);
int hc_comp_launch(hc_ctx* h, void* stream);
int hc_comp_get_output(hc_ctx* h, uint64_t* out);
/* Enqueue the device->host read of the output on `stream` (pinned `out`). */
int hc_comp_get_output_async(hc_ctx* h, uint64_t* out, void* stream);
/* Asynchronous end-to-end Comp on `stream`: H2D of cd/cv, the Comp graph and
 * D2H of the output, all stream-ordered (pass pinned host buffers for
 * overlap; the caller synchronises). */
int hc_comp_async(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, uint64_t* out, void* stream);
/* The upload half of hc_comp_async alone, for serving loops that pipeline
 * queries: H2D of cd/cv (pinned host buffers) into the plan's input buffers
 * on two copy engines, ordered after the work already on `stream` and joined
 * back into it.  A copy stream runs this for query i+1 while the compute
 * stream runs hc_comp_launch for query i and a third stream drains
 * hc_comp_get_output_async of query i-1 (bench.py, e2e "streamed"). */
int hc_comp_upload_async(hc_ctx* h, const uint64_t* cd, const uint64_t* cv, int C, void* stream);

/* Block-sharded Comp.  hc_comp_partial runs pack + baby
 * steps + diagonal products for blocks [b0, b1) of the database (inputs:
 * the C ciphertexts of hc_comp_set_inputs, i.e. the full standard layout)
 * and writes the partial accumulators to partial_dev, a DEVICE buffer of
 * hc_partial_words() uint64 (every word < 2^54, so up to 1023 partials may
 * be summed as uint64 before hc_comp_finish reduces mod q).  hc_comp_finish
 * runs giant steps, folds and the output mask from a (summed) partial. */
int64_t hc_partial_words(const hc_ctx* h);
int hc_comp_partial(hc_ctx* h, int64_t b0, int64_t b1, uint64_t* partial_dev, void* stream);
int hc_comp_finish(hc_ctx* h, const uint64_t* partial_dev, void* stream);

/* Ring helpers on HOST buffers, executed on the GPU (used by the host-side
 * keygen / encrypt / decrypt / serialization of the backend, bgv.py:464-575,
 * 777-790).  rows of n values; row r uses RNS prime prime_idx[r]
 * (0..max_level = chain primes in level order, 4 = p).
 * hc_ntt: inverse = 0 -> NttContext.fwd, 1 -> NttContext.inv.
 * hc_pointwise: op 0 mul, 1 add, 2 sub (bgv.py:431-437). */
int hc_ntt(hc_ctx* h, uint64_t* data, int rows, const int* prime_idx, int inverse);
int hc_pointwise(hc_ctx* h, const uint64_t* a, const uint64_t* b, uint64_t* out, int rows,
                 const int* prime_idx, int op);

/* Replaces BgvBackend.decrypt (bgv.py:559-575) for levels 0..3, in one
 * device call: phase = c0 + c1 s (ct = uint64[2][level+1][n], NTT domain;
 * secret = the ternary key, int64[n]), INTT, exact integer in [0, Q_level)
 * by CRT, centred, reduced mod p, slot_decode (bgv.py:387-394).
 * slots = int64[2][n/2] (SlotMatrix rows). */
int hc_decrypt(hc_ctx* h, const uint64_t* ct, int level, const int64_t* secret, int64_t* slots);

/* Single backend operations (BgvBackend.mul_plain bgv.py:717-733 and
 * _apply_galois bgv.py:735-747) on host buffers.
 * hc_mul_plain: ct uint64[2][l+1][n] at level l >= 1, pt = NttContext
 * residues of the plaintext at level l, uint64[l+1][n]; out uint64[2][l][n].
 * hc_rotate: key switch by Galois element t at level l (1..3); out [2][l+1][n]. */
int hc_mul_plain(hc_ctx* h, const uint64_t* ct, int level, const uint64_t* pt, uint64_t* out);
int hc_rotate(hc_ctx* h, const uint64_t* ct, int level, uint32_t galois_t, uint64_t* out);

/* Measurement: run the Comp schedule un-graphed with CUDA events around
 * every step (kind: 0 transform, 1 CRT/digits, 2 key-switch MAC, 3 diagonal
 * MAC, 4 copy fold, 5 memset).  Returns the number of steps written. */
int hc_comp_profile(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind, int* step_jobs);
/* The same with step_tag[i] naming a transform launch's kernel instantiation:
 * (cluster << 20) | (dir << 16) | (loader << 12) | (epilogue << 8) |
 * (transform-less << 4) | (VT or transforms per cluster); 0 for other steps. */
int hc_comp_profile_ex(hc_ctx* h, void* stream, int max_steps, float* step_ms, int* step_kind, int* step_jobs,
                       int* step_tag);
/* Measured butterfly-throughput ceiling of this GPU for the NTT butterfly
 * used by the transform kernel (register-only microbenchmark). */
int hc_bf_peak(hc_ctx* h, double* bfly_per_s);
/* INT32 multiply-pipe ceilings of this GPU, independent of the Comp code:
 * ops_per_s[0..2] = IMAD (mad.lo.u32), IMAD.WIDE.U32 (mad.wide.u32) and
 * IMAD.HI.U32 (mad.hi.u32) per second, register-only instruction streams. */
int hc_imad_peak(hc_ctx* h, double* ops_per_s);
/* Transform microbenchmark: njobs plain NTTs (dir 0) or INTTs (dir 1) per
 * launch, iters back-to-back launches; writes microseconds per launch. */
int hc_bench_xform(hc_ctx* h, int njobs, int dir, int iters, double* us_per_launch);
/* Transform launches with <= max_jobs jobs use the 8-CTA cluster kernel
 * (latency path); larger launches use one CTA per transform.  Default 16. */
int hc_set_cluster_threshold(int max_jobs);
/* Tuning: chunks of up to `max_blocks` blocks run the baby-step segment as
 * parallel per-block lanes (latency regime); larger chunks use one wide launch
 * per segment (throughput regime). Applies to plans built afterwards. */
int hc_set_lane_blocks(int max_blocks);
/* Tuning: the throughput regime's key switches (chunks of more than the lane
 * limit) as one fused kernel per rotation (k_ksfused: digit NTTs, key MAC and
 * the c0 automorphism in one CTA per output chunk, no digit NTT reaches HBM;
 * bgv.py:616-647) instead of digit-NTT launches + k_ksmac_mb.  Same answer bit
 * for bit; off by default (HC_KSFUSED=1 or this call enables it; measured
 * slower on B200).  Applies to plans built afterwards. */
int hc_set_ksfused(int on);
/* Tuning: single-CTA transform launches of >= jobs (default 200) use the
 * 256-thread three-per-SM variant.  Applies to schedules built afterwards. */
int hc_set_vt2_jobs(int jobs);
/* Diagnostics: co-resident 8-CTA transform clusters on this device. */
int hc_max_active_clusters(hc_ctx* h, int* clusters);

/* Debug builds compiled with -DHC_TRACE: reset the launch numbering and read
 * per-CTA %globaltimer stamps [128 launches][512 CTAs][8 points]. */
int hc_trace_reset(void);
int hc_trace_read(uint64_t* out);
/* k_foldchain's per-fold phase stamps [12 folds][128 CTAs][12 points] */
int hc_trace_read_tail(uint64_t* out);

/* Pure host helpers (no GPU needed): Galois tables for element t.
 * coef: uint16[n] (source index | negate << 15) realising X -> X^t on
 * coefficients (coeff_automorphism, bgv.py:273-284, as a gather);
 * perm: uint16[n] NTT-domain gather (galois_permutation, bgv.py:258-261). */
int hc_galois_tables(int n, uint32_t galois_t, uint16_t* coef, uint16_t* perm);
/* primitive 2n-th root used by the tables (bgv.py:120-126) */
uint64_t hc_prim_root_2n(uint64_t q, int n);

/* Host samplers on the reference's random.Random stream (keygen / encrypt,
 * bgv.py:398-557; CPython's MT19937, Modules/_randommodule.c):
 * hc_rng_create seeds like random.Random(seed) for an int seed, key = |seed|
 * as little-endian 32-bit words (at least one).  Each call consumes exactly
 * what the named Python expression consumes. */
typedef struct hc_rng hc_rng;
int hc_rng_create(const uint32_t* key, int len, hc_rng** out);
void hc_rng_destroy(hc_rng* r);
/* getrandbits(k) -> little-endian 32-bit words, ceil(k/32) of them */
int hc_rng_getrandbits(hc_rng* r, int k, uint32_t* words);
/* [randrange(3) - 1 for _ in range(n)] */
int hc_rng_ternary(hc_rng* r, int n, int64_t* out);
/* [getrandbits(k).bit_count() - getrandbits(k).bit_count() for _ in range(n)] */
int hc_rng_cbd(hc_rng* r, int n, int k, int64_t* out);
/* [randrange(Q) for _ in range(n)] as residues out[np][n] mod primes[np];
 * Q = nw little-endian 32-bit words of bit length kbits */
int hc_rng_uniform(hc_rng* r, int n, const uint32_t* q, int nw, int kbits, const uint64_t* primes, int np,
                   uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif
