/*
 * tetris_b200.h — C-ABI boundary of the B200-native RNS-CKKS evaluator.
 *
 * This is the thin layer the C++ host API (include/tetris_b200/*.hpp, the
 * drop-in for the reference's proj/include/tetris/ evaluation path) calls into.
 * Plain pointers, sizes and opaque handles only; no C++ or torch types.
 *
 * Data model (mirrors the reference's Poly, ring.hpp:204-374):
 *   a "poly" is rows x N uint64 residues, row-major, rows = level+1+nspecial;
 *   row r is reduced mod moduli[r <= level ? r : q_count + (r-level-1)]
 *   (ring.hpp:227-229). nspecial is 0 or the ring's special count. Every
 *   residue stored at the boundary is canonical in [0, q).
 *   Batched entry points take `npolys` polys of identical shape laid out
 *   back to back (stride rows*N words).
 *
 * All device pointers are device-global memory allocated with tg_alloc (or
 * any cudaMalloc'd memory). `stream` is a cudaStream_t (NULL = legacy
 * default stream). Every call is asynchronous on `stream` unless stated.
 *
 * Errors: every function returns 0 on success or a negative TG_E* code; the
 * message is available from tg_last_error() (thread-local). Contract errors
 * mirror the reference's TetrisError messages ("ring"/"rlwe"/"ckks" tags).
 */
#ifndef TETRIS_B200_H
#define TETRIS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TG_OK 0
#define TG_E_ARG (-1)     /* contract violation (shape/form/level)          */
#define TG_E_CUDA (-2)    /* CUDA runtime error                              */
#define TG_E_NOMEM (-3)   /* device allocation failed                        */
#define TG_E_STATE (-4)   /* no device / context unusable                    */

#define TG_FORM_COEFF 0   /* Form::coeff (ring.hpp:202) */
#define TG_FORM_EVAL 1    /* Form::eval                 */

typedef struct tg_context tg_context; /* RingParams + its NTT tables on device */
typedef struct tg_gadget tg_gadget;   /* GadgetPlan + ModDown constants        */

/* ---- library / errors -------------------------------------------------- */
const char* tg_last_error(void);
/* Number of CUDA devices visible (0 on a host without GPU). Never fails. */
int tg_device_count(void);
/* Library build string (arch, version). */
const char* tg_build_info(void);

/* ---- context: replaces RingParams (ring.hpp:116-195) ------------------- */
/* Uploads the host-built NTT tables verbatim, so psi choice and the
 * bit-reversed evaluation order are exactly the reference's
 * (NttTables::init ring.hpp:25-51, build_eval_order_map ring.hpp:165-186).
 *   tables:   4*nmod*N words: per modulus i, [w | w_shoup | winv | winv_shoup]
 *   n_inv:    2*nmod words:   per modulus i, [n_inv, n_inv_shoup]
 *   eval_exp: N entries; slot_of_exp: 2N entries.
 * Rescale constants (ring.hpp:505-508) are derived from `moduli` here. */
int tg_context_create(tg_context** out, int device, uint32_t degree, const uint64_t* moduli,
                      uint32_t nmod, uint32_t special_count, const uint64_t* tables,
                      const uint64_t* n_inv, const uint32_t* eval_exp,
                      const uint32_t* slot_of_exp);
void tg_context_destroy(tg_context* ctx);
uint32_t tg_context_degree(const tg_context* ctx);

/* ---- memory ------------------------------------------------------------- */
/* Stream-ordered allocation from the context device's memory pool. */
int tg_alloc(tg_context* ctx, void** ptr, size_t bytes, void* stream);
int tg_free(tg_context* ctx, void* ptr, void* stream);
int tg_memcpy_h2d(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream);
int tg_memcpy_d2h(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream);
int tg_memcpy_d2d(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream);
int tg_memset0(tg_context* ctx, void* dst, size_t bytes, void* stream);
int tg_stream_sync(tg_context* ctx, void* stream);
/* A non-blocking stream on the context's device (*stream = cudaStream_t). */
int tg_stream_create(tg_context* ctx, void** stream);
int tg_stream_destroy(tg_context* ctx, void* stream);
/* Events for cross-stream ordering without host synchronisation (staged
 * host->device uploads overlapping compute). */
int tg_event_create(tg_context* ctx, void** event);
int tg_event_destroy(tg_context* ctx, void* event);
int tg_event_record(tg_context* ctx, void* event, void* stream);
int tg_stream_wait_event(tg_context* ctx, void* stream, void* event);
/* Device index the context lives on. */
int tg_context_device(const tg_context* ctx);

/* Device memory pool of a context (stream-ordered allocations of every op).
 * tg_pool_reserve grows the pool to hold at least `bytes` (allocate + free),
 * so later allocations never map new memory inside a timed region;
 * tg_pool_stats reports reserved bytes and the used high-water mark. */
int tg_pool_reserve(tg_context* ctx, uint64_t bytes);
int tg_pool_stats(tg_context* ctx, uint64_t* reserved, uint64_t* used_high);

/* Page-locked host memory (end-to-end H2D/D2H staging). */
int tg_host_alloc_pinned(void** ptr, size_t bytes);
int tg_host_free_pinned(void* ptr);

/* ---- kernel timing -------------------------------------------------------
 * When enabled, every kernel launch of the context is bracketed by CUDA
 * events on its stream and attributed to an op class together with its
 * ALGORITHMIC bytes (inputs read once + outputs written once + key bytes,
 * SURVEY 8(d)). tg_profile_read synchronizes, accumulates per class and
 * clears: ms[i], launches[i], bytes[i] for i < TG_OP_COUNT. */
enum {
    TG_OP_NTT_FWD = 0,
    TG_OP_NTT_INV,
    TG_OP_ADDSUB,
    TG_OP_MUL,
    TG_OP_SCALAR,
    TG_OP_AUTOMORPHISM,
    TG_OP_RESCALE,
    TG_OP_TENSOR,
    TG_OP_MUL_PLAIN,
    TG_OP_MODUP,
    TG_OP_KEY_INNER,
    TG_OP_MOD_DOWN,
    TG_OP_REDUCE,
    TG_OP_LINCOMB,
    TG_OP_ENCODE,
    TG_OP_KS_FUSED, /* fused key-switch core: digits' NTT chunk phase + key inner product + iNTT chunk phase */
    TG_OP_COUNT
};
int tg_profile_enable(tg_context* ctx, int on);
int tg_profile_read(tg_context* ctx, double* ms, uint64_t* launches, double* bytes);
/* As tg_profile_read, plus the algorithmic FP64 operation count per class
 * where the op models it (the fused key-switch core: 8 per NTT butterfly, 7
 * per key-inner-product term; 0 elsewhere); any output may be NULL. */
int tg_profile_read_ops(tg_context* ctx, double* ms, uint64_t* launches, double* bytes, double* fp64_ops);
const char* tg_profile_op_name(int op);

/* ---- ring layer --------------------------------------------------------- */
/* Reduces arbitrary words mod their row modulus, in place: the fix-up after
 * an NCCL integer sum of per-rank partial ciphertexts (exact while
 * ranks * max q < 2^64). */
int tg_poly_reduce(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys,
                   void* stream);
/* Poly::ntt_forward / NttTables::forward (ring.hpp:64-80, :234-239), in place.
 * Negacyclic CT, natural -> bit-reversed evaluation order. */
int tg_ntt_forward(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys,
                   void* stream);
/* Poly::ntt_inverse / NttTables::inverse (ring.hpp:82-101, :241-246), in place. */
int tg_ntt_inverse(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys,
                   void* stream);
/* Out-of-place variants: out receives the transform of in (in unchanged;
 * out may equal in). */
int tg_ntt_forward_oop(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, int nspecial,
                       uint32_t npolys, void* stream);
int tg_ntt_inverse_oop(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, int nspecial,
                       uint32_t npolys, void* stream);
/* Poly::add_inplace / sub_inplace / negate_inplace (ring.hpp:250-276).
 * out may alias a or b. For neg, b is ignored. op: 0 add, 1 sub, 2 neg. */
int tg_poly_addsub(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int op,
                   int level, int nspecial, uint32_t npolys, void* stream);
/* tg_poly_addsub (op 0/1) over level-dropped views: operand poly p starts at
 * p * stride words (stride >= (level+1+nspecial) * N); out is packed. */
int tg_poly_addsub_strided(tg_context* ctx, uint64_t* out, const uint64_t* a, uint64_t a_stride,
                           const uint64_t* b, uint64_t b_stride, int op, int level, int nspecial,
                           uint32_t npolys, void* stream);
/* Poly::mul_pointwise_inplace (ring.hpp:278-288): out = a*b mod q (eval form). */
int tg_poly_mul(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int level,
                int nspecial, uint32_t npolys, void* stream);
/* Poly::mul_acc_pointwise (ring.hpp:290-304): out += a*b mod q. */
int tg_poly_mul_acc(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b,
                    int level, int nspecial, uint32_t npolys, void* stream);
/* Poly::mul_scalar_inplace (ring.hpp:307-315): scalar given per MODULUS INDEX
 * (nmod words, host memory); each is reduced mod its row modulus first. */
int tg_poly_mul_scalar(tg_context* ctx, uint64_t* out, const uint64_t* a,
                       const uint64_t* scalar_per_modulus, int level, int nspecial,
                       uint32_t npolys, void* stream);
/* Evaluator::add_scalar's residue update (ckks.hpp:296-313): adds
 * add_per_modulus[m] to every entry (eval form) or to index 0 (coeff form). */
int tg_poly_add_scalar(tg_context* ctx, uint64_t* out, const uint64_t* a,
                       const uint64_t* add_per_modulus, int form, int level, int nspecial,
                       uint32_t npolys, void* stream);
/* automorphism_apply (ring.hpp:410-436): X -> X^g, g odd; coeff form is a
 * signed scatter, eval form a slot gather. out must not alias in. */
int tg_automorphism(tg_context* ctx, uint64_t* out, const uint64_t* in, uint64_t exponent,
                    int form, int level, int nspecial, uint32_t npolys, void* stream);
/* Large-domain PFE eval_scores (pfe.hpp:73-114): out holds nrows
 * ciphertexts (2 parts x level+1 rows), row r = sum_c X^{exps[r*ncols+c]} tv_c.
 * tvs: ncols device pointers to test-vector ciphertexts (parts back to back);
 * exps: device array [nrows][ncols] of exponents in [0, 2N). */
#define TG_PFE_MAX_COLS 64
int tg_pfe_eval(tg_context* ctx, uint64_t* out, const uint64_t* const* tvs, uint32_t ncols,
                const uint32_t* exps, uint32_t nrows, int level, void* stream);
/* merge_embed / ring_split data movement (rlwe.hpp:702-790), ring-agnostic:
 * out[row][k*stride + i] = in_dev[i][row][k] (NULL or i >= count -> 0) over
 * rows_total rows of n_small; in_dev is a DEVICE array of count pointers.
 * tg_deinterleave is the inverse gather of one residue class (parity). */
int tg_interleave(uint64_t* out, const uint64_t* const* in_dev, uint32_t count, uint32_t stride,
                  uint32_t n_small, uint64_t rows_total, void* stream);
int tg_deinterleave(uint64_t* out, const uint64_t* in, uint32_t parity, uint32_t stride, uint32_t n_small,
                    uint64_t rows_total, void* stream);
/* Poly::mul_monomial (ring.hpp:343-361): out = X^e * in, coeff form.
 * out must not alias in. */
int tg_mul_monomial(tg_context* ctx, uint64_t* out, const uint64_t* in, uint64_t e, int level,
                    int nspecial, uint32_t npolys, void* stream);
/* raise_level (ring.hpp:523-545): level-0 coeff polys (one row each) lifted
 * to (new_level, nspecial) rows as centered integers mod q0. */
int tg_raise_level(tg_context* ctx, uint64_t* out, const uint64_t* in, int new_level, int nspecial,
                   uint32_t npolys, void* stream);
/* rescale_round (ring.hpp:493-518): coeff form, level -> level-1 rows.
 * out (level rows) must not alias in (level+1 rows). */
int tg_rescale(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
               void* stream);
/* Evaluator::add(rescale(in), addend) in one pass (ckks.hpp:315-324 then
 * :195-210), for rings whose rows 0..level are all below the FP64 bound:
 * out (out_level+1 rows per poly, packed) = rescale_round(in)[0..out_level]
 * + addend, coeff form; addend poly p starts at p * addend_stride words and
 * has at least out_level+1 rows; out_level <= level-1. TG_E_ARG (no work)
 * when a row is not FP64-eligible: the caller then runs the two ops. */
int tg_rescale_add(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
                   const uint64_t* addend, uint64_t addend_stride, int out_level, void* stream);
/* rescale_round on eval-form rows (level+1 rows in, level rows out):
 * == NTT(tg_rescale(iNTT(in))) residue for residue, with one inverse row and
 * `level` forward rows per poly instead of level+1 and level. */
int tg_rescale_eval(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
                    void* stream);

/* ---- fused residue expressions ------------------------------------------ */
#define TG_LINCOMB_MAX_TERMS 32
#define TG_LINCOMB_MAX_ROWS 32
/* out = [rescale_round]( sum_t coeffs[t][r] * term_t  (+ add_per_row[r]) ) mod q_r
 * over `nparts` parts of `level`+1 rows (no specials). Term t part p row r
 * is read at terms[t] + p*part_strides[t] + r*N (level-dropped views allowed).
 * coeffs: nterms x (level+1) host words (one integer per row modulus).
 * add_per_row (host, may be NULL) is added to part 0 only: to every
 * coefficient if add_all (eval form) else to coefficient 0 (coeff form).
 * With rescale, out has `level` rows (rescale_round, ring.hpp:493-518) and
 * the input must be coefficient form. One pass replaces the ladder /
 * combination chains of eval_chebyshev (ckks.hpp:538-578): add_inplace,
 * mul_scalar, sub_inplace, add_scalar, rescale. out must not alias a term. */
int tg_lincomb(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* terms,
               const uint64_t* part_strides, const uint64_t* coeffs, const uint64_t* add_per_row,
               int add_all, int level, uint32_t nparts, int rescale, void* stream);
/* tg_lincomb over a batch of ciphertexts stored part-major (parts
 * [0, add_polys) are the batch's part-0 polys): the constant goes to each
 * of the first add_polys parts. */
int tg_lincomb_batch(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* terms,
                     const uint64_t* part_strides, const uint64_t* coeffs, const uint64_t* add_per_row,
                     int add_all, int level, uint32_t nparts, uint32_t add_polys, int rescale, void* stream);

/* nouts (2..4) rescaled combinations of the SAME nterms (1..4) terms in one
 * pass: outs[o] = rescale_round( sum_t coeffs[o][t][r] * term_t (+
 * add_per_row[o][r] at coefficient 0 of the first add_polys parts) ), `level`
 * rows each (the combination steps of eval_chebyshev, ckks.hpp:556-578, for
 * the base blocks of one BSGS polynomial, which share their baby steps).
 * coeffs: nouts x nterms x (level+1) host words, add_per_row: nouts x
 * (level+1) or NULL. Coefficient form, every row 0..level FP64-eligible
 * (TG_E_ARG otherwise). Identical residues to nouts tg_lincomb_batch calls. */
int tg_lincomb_multi(tg_context* ctx, uint32_t nouts, uint64_t* const* outs, uint32_t nterms,
                     const uint64_t* const* terms, const uint64_t* part_strides, const uint64_t* coeffs,
                     const uint64_t* add_per_row, int level, uint32_t nparts, uint32_t add_polys,
                     void* stream);

/* dst[i*words .. (i+1)*words) = srcs[i][0 .. words) for i < npolys (device
 * pointers in a host array): stacking single ciphertexts' parts into one
 * part-major batch block with one launch (stack_ciphertexts). words even. */
int tg_gather_polys(tg_context* ctx, uint64_t* dst, const uint64_t* const* srcs, uint32_t npolys,
                    uint64_t words, void* stream);

/* ---- CKKS products ------------------------------------------------------ */
/* Evaluator::mul tensor step (ckks.hpp:229-237), eval form inputs:
 * p0 = x0*y0, p1 = x0*y1 + x1*y0, p2 = x1*y1. Outputs must not alias inputs. */
int tg_tensor(tg_context* ctx, uint64_t* p0, uint64_t* p1, uint64_t* p2, const uint64_t* x0,
              const uint64_t* x1, const uint64_t* y0, const uint64_t* y1, int level,
              uint32_t npolys, void* stream);
/* (p0 and p1 both NULL: only p2 = x1 y1 is formed; x0, y0 unused.) */
/* Sum of two tensors, add(mul(x, y), mul(u, v)) (ckks.hpp:229-237 twice, then
 * Ciphertext::add_inplace rlwe.hpp:300-305), in one pass: p0 = x0 y0 + u0 v0,
 * p1 = x0 y1 + x1 y0 + u0 v1 + u1 v0, p2 = x1 y1 + u1 v1 (lazy
 * relinearisation of a pair of products). u*, v* all NULL: tg_tensor. */
int tg_tensor2(tg_context* ctx, uint64_t* p0, uint64_t* p1, uint64_t* p2, const uint64_t* x0,
               const uint64_t* x1, const uint64_t* y0, const uint64_t* y1, const uint64_t* u0,
               const uint64_t* u1, const uint64_t* v0, const uint64_t* v1, int level, uint32_t npolys,
               void* stream);
/* The tensor's c2 = x1 y1 (eval form, written to c2_eval) and its inverse NTT
 * into c2 (coefficient form), npolys polys of level+1 rows: on all-FP64
 * rings the product is formed inside the first inverse phase (c2 read once
 * from HBM less); identical residues to tg_tensor + tg_ntt_inverse_oop. */
int tg_tensor_c2_inverse(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                         const uint64_t* y1, int level, uint32_t npolys, int* raw, void* stream);
/* The same for c2 = x1 y1 + u1 v1 (u1, v1 NULL: one product). */
int tg_tensor2_c2_inverse(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                          const uint64_t* y1, const uint64_t* u1, const uint64_t* v1, int level,
                          uint32_t npolys, int* raw, void* stream);
/* op_strides (here and in the *_strided entry points below): NULL, or 4 host
 * words = the distance in words between consecutive polys of the x, y, u, v
 * operand parts (0 = tight, (level+1)*N): level-dropped views of a
 * higher-level ciphertext batch are read in place instead of being gathered. */
int tg_tensor2_c2_inverse_strided(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                                  const uint64_t* y1, const uint64_t* u1, const uint64_t* v1,
                                  const uint64_t* op_strides, int level, uint32_t npolys, int* raw, void* stream);
/* raw (in/out, may be NULL): non-NULL lets the call leave c2 as the inverse
 * transform's raw doubles without the N^-1 factor (|v| <= 0.6q) when the
 * fused key switch can consume them; *raw reports whether it did (pass it on
 * as tg_relinearize_tensor_batch's c2_raw). */
/* Evaluator::mul_plain residue step (ckks.hpp:257-265): every part row r
 * (modulus index m) times plain row m; plain holds >= level+1 rows. */
int tg_mul_plain(tg_context* ctx, uint64_t* out, const uint64_t* ct_part, const uint64_t* plain,
                 int level, uint32_t nparts, void* stream);
/* LinearTransformPlan::apply giant-bucket sum (ckks.hpp:455-476), eval form:
 * out = sum_t ct_t (x) plain_t over nparts parts of level+1 rows; each ct_t
 * holds nparts parts back to back, each plain_t >= level+1 rows. */
#define TG_PLAIN_SUM_MAX_TERMS 256
int tg_mul_plain_sum(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* cts,
                     const uint64_t* const* plains, int level, uint32_t nparts, void* stream);
/* As tg_mul_plain_sum with term t's parts part_strides[t] words apart
 * (>= (level+1) N; NULL: contiguous), so the part-major views of a ciphertext
 * batch (stack_ciphertexts) are read in place. */
int tg_mul_plain_sum_strided(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* cts,
                             const uint64_t* part_strides, const uint64_t* const* plains, int level,
                             uint32_t nparts, void* stream);

/* ---- slot encoder ------------------------------------------------------- */
/* Encoder::encode_slots (ckks.hpp:59-86) for `batch` slot vectors of n slots:
 * the reference's O(n^2) inverse DFT replayed per output in the same
 * sequential order and IEEE operations, round_half_away(w * scale) and
 * from_centered per row, so residues are bit-identical to the reference.
 * v: [batch][n] complex as (re, im) doubles; psi: [4n] complex table of the
 * reference encoder (ckks.hpp:28-34, host-computed); rot5: [n] powers of 5
 * mod 4n (ckks.hpp:35-40); all device pointers. out: [batch][level+1][N]
 * coeff-form rows (fully written). max_abs_bits (device u64, may be NULL)
 * receives max(|Re w|, |Im w|) as double bits via atomicMax (must be zeroed
 * by the caller), for check_encoding_bound (ckks.hpp:137-142). */
int tg_encode_slots(tg_context* ctx, uint64_t* out, const double* v, uint32_t batch, uint32_t n,
                    const double* psi, const uint32_t* rot5, double scale, int level,
                    uint64_t* max_abs_bits, void* stream);

/* ---- key switching ------------------------------------------------------ */
/* GadgetPlan (rlwe.hpp:28-206) for this ring: RNS digit groups of group_size
 * primes (base2_bits > 0: single-prime groups split into balanced signed
 * base-2^b sub-digits, rlwe.hpp:103-135)
 * and the ModDown constants of mod_down_p (rlwe.hpp:555-579). */
int tg_gadget_create(tg_gadget** out, tg_context* ctx, uint32_t group_size, uint32_t base2_bits);
void tg_gadget_destroy(tg_gadget* g);
/* GadgetPlan::digit_count (rlwe.hpp:54-61). */
uint32_t tg_gadget_digit_count(const tg_gadget* g, int level);

/* GadgetPlan::decompose = ModUp (rlwe.hpp:65-139): d (coeff, level, no
 * specials) -> digit_count(level) digit polys of level+1+K rows each, in EVAL
 * form, written back to back at `digits`. Uncorrected fast base conversion. */
int tg_modup(tg_gadget* g, uint64_t* digits, const uint64_t* d, int level, void* stream);
/* KeyContext::ks_inner (rlwe.hpp:501-540): acc_{0,1} = sum_i digit_i * key_{b,a}[i]
 * over key rows (key_row map rlwe.hpp:517-518), then iNTT and mod_down_p.
 * key: digits x 2 x (max_level+1+K) x N words, [digit][b|a][row][N].
 * out0/out1: coeff form, level+1 rows. */
int tg_ks_inner(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* digits,
                uint32_t ndigits, const uint64_t* key, uint32_t key_digits, int level,
                void* stream);
/* KeyContext::mod_down_p (rlwe.hpp:547-592): in (coeff, level+1+K rows) ->
 * out (coeff, level+1 rows), centered fast base conversion of the specials. */
int tg_mod_down(tg_gadget* g, uint64_t* out, const uint64_t* in, int level, void* stream);
/* KeyContext::switch_key_apply (rlwe.hpp:542-544) = ks_inner(decompose(d)). */
int tg_switch_key_apply(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                        const uint64_t* key, uint32_t key_digits, int level, void* stream);
/* Key switch with the epilogue add fused into ModDown: out_i = add_i +
 * switch_key_apply(d)_i (add_i may be NULL). This is relinearize's
 * (c0+d0, c1+d1) (rlwe.hpp:607-613) and apply_galois' (phi(c0)+d0, d1)
 * (rlwe.hpp:646-648) in one pass. d_eval (may be NULL) is the eval form of d:
 * when given, each digit's own-group rows (equal to d's rows, rlwe.hpp:78-100)
 * are copied from it instead of being forward-transformed. */
int tg_keyswitch_add(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                     const uint64_t* d_eval, const uint64_t* key, uint32_t key_digits, int level,
                     const uint64_t* add0, const uint64_t* add1, void* stream);
/* tg_keyswitch_add for `npolys` sources under ONE key (a batch of
 * ciphertexts relinearised together, e.g. the record blocks of a query):
 * d, d_eval, out0, out1, add0, add1 each hold npolys polys back to back.
 * Same per-source result as npolys tg_keyswitch_add calls; the key is read
 * once per batch and every launch covers the whole batch. */
/* ks_inner on given eval-form digits with the epilogue add (out_i = add_i +
 * ModDown(iNTT(sum_k digit_k * key_k))): the hoisted rotation of
 * Evaluator::apply_galois_many (ckks.hpp:338-367), whose digits are the
 * automorphism of ONE decomposition. add0/add1 may be NULL. */
int tg_ks_inner_add(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* digits, uint32_t ndigits,
                    const uint64_t* key, uint32_t key_digits, int level, const uint64_t* add0,
                    const uint64_t* add1, void* stream);
/* tg_keyswitch_add_batch with EVAL-form output and eval-form addends: the
 * accumulators never leave the evaluation domain except their K special rows
 * (ModDown's conversion is computed in coefficient form and transformed
 * forward). d is the coefficient form of the sources (d_eval optional).
 * out_i == NTT(tg_keyswitch_add_batch output with coefficient-form addends). */
int tg_keyswitch_add_eval(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                          const uint64_t* d_eval, const uint64_t* key, uint32_t key_digits, int level,
                          const uint64_t* add0, const uint64_t* add1, uint32_t npolys, void* stream);
/* relinearize (rlwe.hpp:601-620) of npolys part-major degree-2 ciphertexts
 * straight from the tensor product: c2 (coefficient form; c2_eval optional)
 * is key-switched, and c0/c1 in EVAL form are folded into the accumulators'
 * Q rows as P * c before ModDown, which returns c + ModDown(acc) in
 * coefficient form. out0/out1 == tg_keyswitch_add_batch with the coefficient
 * forms of c0/c1 as addends, residue for residue. */
int tg_relinearize_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                         const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits, int level,
                         const uint64_t* c0_eval, const uint64_t* c1_eval, uint32_t npolys, void* stream);
int tg_keyswitch_add_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                           const uint64_t* d_eval, const uint64_t* key, uint32_t key_digits, int level,
                           const uint64_t* add0, const uint64_t* add1, uint32_t npolys, void* stream);
/* mul + relinearize (ckks.hpp:229-237, rlwe.hpp:601-620) of npolys degree-1
 * products x * y with the tensor's c0 = x0 y0 and c1 = x0 y1 + x1 y0 formed
 * inside the fused key-switch core from the EVAL-form operand parts (x0, x1,
 * y0, y1: npolys polys of level+1 rows each) instead of through HBM; c2 (its
 * coefficient form and, optional, eval form) as for tg_relinearize_batch.
 * Identical residues to tg_tensor + tg_relinearize_batch. Rings without the
 * fused core take exactly that pair. */
int tg_relinearize_tensor_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                                const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits, int level,
                                const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                uint32_t npolys, int c2_raw, void* stream);
/* rescale(mul_relin(x, y)) and rescale_add(mul_relin(x, y), add)
 * (ckks.hpp:229-237, rlwe.hpp:601-620, ckks.hpp:315-324, :195-210): the
 * relinearised product's ModDown rows are rescaled (and added) in the same
 * pass, so the level+1-row product never reaches HBM. out: 2*npolys polys
 * packed (c0 of every product, then c1) of `level` rows, or out_level+1 rows
 * with an addend (poly p of the 2*npolys at add + p*add_stride words,
 * out_level <= level-1). Every q-chain row 0..level must be FP64-eligible
 * (TG_E_ARG otherwise). Identical residues to tg_relinearize_tensor_batch
 * followed by tg_rescale / tg_rescale_add, which small batches take. */
int tg_relinearize_tensor_rescale_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                        const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits,
                                        int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0,
                                        const uint64_t* y1, uint32_t npolys, int c2_raw, const uint64_t* add,
                                        uint64_t add_stride, int out_level, void* stream);
/* mul_relin followed by the Chebyshev ladder step of eval_chebyshev
 * (ckks.hpp:532-555: T_k = rescale(2 T_a T_b - mul_scalar(T_{b-a}, 1, ratio))
 * or rescale(add_scalar(2 T_a^2, -1))): out = rescale_round( 2 relinearize(x
 * (x) y) - sub_coef[r] * sub (+ add_const[r] at coefficient 0 of the part-0
 * polys) ), 2*npolys polys of `level` rows. sub: coefficient-form ciphertext
 * batch (poly p of the 2*npolys at sub + p*sub_stride words, >= level+1 rows)
 * with its per-row multipliers sub_coef (host, level+1 words), or both NULL;
 * add_const: host, level+1 words, or NULL. Large batches on all-FP64 rings
 * apply the step inside ModDown (the product never reaches HBM); identical
 * residues to tg_relinearize_tensor_batch + tg_lincomb_batch(rescale). */
int tg_relinearize_tensor_ladder_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                       const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits,
                                       int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0,
                                       const uint64_t* y1, uint32_t npolys, int c2_raw, const uint64_t* sub,
                                       uint64_t sub_stride, const uint64_t* sub_coef,
                                       const uint64_t* add_const, void* stream);
int tg_relinearize_tensor_ladder_batch_strided(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                               const uint64_t* c2_eval, const uint64_t* key,
                                               uint32_t key_digits, int level, const uint64_t* x0,
                                               const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                               const uint64_t* op_strides, uint32_t npolys, int c2_raw,
                                               const uint64_t* sub, uint64_t sub_stride, const uint64_t* sub_coef,
                                               const uint64_t* add_const, void* stream);
/* Lazy relinearisation of two products: rescale(relinearize(add(mul(x, y),
 * mul(u, v)))) [+ add] (ckks.hpp:229-237, rlwe.hpp:300-305, :601-620,
 * ckks.hpp:315-324) with ONE key switch: c2 = x1 y1 + u1 v1 (from
 * tg_tensor2_c2_inverse), c0 / c1 of both tensors formed inside the fused
 * key-switch core. u0, u1, v0, v1 (npolys polys of level+1 rows, eval form)
 * all NULL: tg_relinearize_tensor_rescale_batch. */
int tg_relinearize_tensor2_rescale_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                         const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits,
                                         int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0,
                                         const uint64_t* y1, const uint64_t* u0, const uint64_t* u1,
                                         const uint64_t* v0, const uint64_t* v1, uint32_t npolys, int c2_raw,
                                         const uint64_t* add, uint64_t add_stride, int out_level, void* stream);
int tg_relinearize_tensor2_rescale_batch_strided(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                                 const uint64_t* c2_eval, const uint64_t* key,
                                                 uint32_t key_digits, int level, const uint64_t* x0,
                                                 const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                                 const uint64_t* u0, const uint64_t* u1, const uint64_t* v0,
                                                 const uint64_t* v1, const uint64_t* op_strides, uint32_t npolys,
                                                 int c2_raw, const uint64_t* add, uint64_t add_stride,
                                                 int out_level, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TETRIS_B200_H */
