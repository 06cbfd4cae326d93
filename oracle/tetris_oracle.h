/*
 * TEST INFRASTRUCTURE ONLY — the CPU restatement oracle. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and
 * only as the checker. Never linked into the product.
 *
 * Plain-C restatement of the TETRIS reference's RNS-CKKS ring and
 * key-switching arithmetic (/root/reference/proj/include/tetris/*.hpp),
 * written from the published algorithm, one function per reference routine
 * (file:line cited on each). Pinned against golden vectors produced by the
 * compiled, unmodified reference (tests/golden/, tests/golden/gen_golden.py).
 */
#ifndef TETRIS_ORACLE_H
#define TETRIS_ORACLE_H
#include <stdint.h>

/* --- RNG: splitmix64 + mt19937_64 (common.hpp:154-210) --- */
typedef struct {
    uint64_t seed;
    uint64_t mt[312];
    int mti;
    int have_spare;
    double spare;
} or_rng;
void or_rng_init(or_rng* r, uint64_t seed);
uint64_t or_rng_next(or_rng* r);
uint64_t or_rng_uniform(or_rng* r, uint64_t bound);
double or_rng_normal(or_rng* r);
void or_rng_split(const or_rng* r, uint64_t label, or_rng* child);
uint64_t or_splitmix64(uint64_t x);

/* --- primes (common.hpp:103-147) --- */
int or_is_prime(uint64_t n);
/* returns count found (== count unless exhausted) */
int or_find_ntt_primes(int bits, int count, uint64_t modulus, const uint64_t* exclude, int nexclude, uint64_t* out);

/* --- NTT (ring.hpp:25-101) --- */
/* Builds the tables of modulus index `idx` of a ring exactly as RingParams does
 * (Rng(0x7e7215a1d2c3).split(idx) drives the psi search). */
void or_ntt_tables(uint64_t q, uint32_t n, uint32_t idx, uint64_t* psi, uint64_t* w, uint64_t* ws, uint64_t* winv,
                   uint64_t* winvs, uint64_t* ninv2);
void or_ntt_forward(uint64_t* a, uint32_t n, uint64_t q, const uint64_t* w, const uint64_t* ws);
void or_ntt_inverse(uint64_t* a, uint32_t n, uint64_t q, const uint64_t* winv, const uint64_t* winvs,
                    const uint64_t* ninv2);
/* eval_exp/slot_of_exp by transforming X with modulus-0 tables (ring.hpp:165-186) */
void or_eval_order(uint32_t n, uint64_t q0, const uint64_t* w0, const uint64_t* ws0, uint64_t psi0, uint32_t* eval_exp,
                   uint32_t* slot_of_exp);

/* --- element-wise (ring.hpp:250-325); row r uses modulus mod[r] --- */
void or_poly_add(uint64_t* out, const uint64_t* a, const uint64_t* b, const uint64_t* mod, int rows, uint32_t n);
void or_poly_sub(uint64_t* out, const uint64_t* a, const uint64_t* b, const uint64_t* mod, int rows, uint32_t n);
void or_poly_neg(uint64_t* out, const uint64_t* a, const uint64_t* mod, int rows, uint32_t n);
void or_poly_mul(uint64_t* out, const uint64_t* a, const uint64_t* b, const uint64_t* mod, int rows, uint32_t n);
void or_poly_mul_scalar(uint64_t* out, const uint64_t* a, const uint64_t* scalar, const uint64_t* mod, int rows,
                        uint32_t n);
/* automorphism_apply (ring.hpp:410-436); eval form uses the order maps */
void or_automorphism(uint64_t* out, const uint64_t* in, uint64_t g, int eval_form, const uint64_t* mod, int rows,
                     uint32_t n, const uint32_t* eval_exp, const uint32_t* slot_of_exp);
/* rescale_round (ring.hpp:493-518): in has level+1 rows over moduli[0..level], out level rows */
void or_rescale(uint64_t* out, const uint64_t* in, const uint64_t* moduli, int level, uint32_t n);

/* --- key switching (rlwe.hpp:28-206, 501-592) ---
 * moduli = q-chain (nq) followed by K specials. Digit/poly rows are
 * 0..level over q then the K special rows. */
/* GadgetPlan::decompose base conversion (rlwe.hpp:65-101), COEFF-form output
 * (digits back to back, ndig = ceil((level+1)/group)); caller NTTs them. */
int or_modup(uint64_t* digits, const uint64_t* d, const uint64_t* moduli, int nq, int K, int group, int level,
             uint32_t n);
/* ks_inner dot product (rlwe.hpp:514-536), eval form; key_b/key_a point at
 * digit i's full-row key polys (nq+K rows). */
void or_key_inner(uint64_t* acc0, uint64_t* acc1, const uint64_t* digits, int nd, const uint64_t* const* key_b,
                  const uint64_t* const* key_a, const uint64_t* moduli, int nq, int K, int level, uint32_t n);
/* mod_down_p (rlwe.hpp:547-592): coeff in (level+1+K rows) -> coeff out (level+1 rows) */
void or_mod_down(uint64_t* out, const uint64_t* in, const uint64_t* moduli, int nq, int K, int level, uint32_t n);

#endif
