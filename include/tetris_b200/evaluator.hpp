// tetris_b200 CKKS layer: encoder (host), evaluation keys, Evaluator,
// Chebyshev evaluation, slot sum and the private threshold. Drop-in for the
// reference ckks.hpp:24-370, :515-615 and threshold.hpp:13-157.
//
// The Evaluator keeps the reference's per-ciphertext, by-value API; scale
// bookkeeping, rounding of host constants and every contract check follow
// the reference's expression order exactly, so outputs are bit-identical.
#pragma once

#include <complex>
#include <functional>
#include <map>
#include <set>

#include "tetris_b200/keys.hpp"

namespace tetris_b200 {

using cplx = std::complex<double>;

// Canonical-embedding encoder (ckks.hpp:24-148); O(n^2) special DFT on the
// host, parallelised over output indices (per-index summation order kept).
class Encoder {
public:
    Encoder(const RingParams& ring, u32 nslots);
    const RingParams& ring() const { return *ring_; }
    u32 slots() const { return n_; }
    std::vector<cplx> dft(const std::vector<cplx>& w) const;
    std::vector<cplx> dft_inv(const std::vector<cplx>& v) const;
    // on the device (tg_encode_slots), bit-identical to the reference's host DFT
    Poly encode_slots(const std::vector<cplx>& v, double scale, int level) const;
    // several slot vectors in one launch; the polys share one HBM block
    std::vector<Poly> encode_slots_many(const std::vector<std::vector<cplx>>& vs, double scale, int level) const;
    std::vector<cplx> decode_slots(const Poly& poly, double scale) const;
    Poly encode_coeffs(const std::vector<double>& v, double scale, int level) const;
    std::vector<double> decode_coeffs(const Poly& poly, double scale, std::size_t count) const;
    // host residues of encode_slots (no device needed)
    std::vector<u64> encode_slots_host(const std::vector<cplx>& v, double scale, int level) const;
    std::vector<cplx> decode_slots_host(const u64* rows01, int level, double scale) const;
    // the encoder's tables: psi[t] = exp(i pi t / 2n) (4n entries), rot5[j] = 5^j mod 4n
    const std::vector<cplx>& psi() const { return psi_; }
    const std::vector<u32>& rot5() const { return rot5_; }

private:
    const RingParams* ring_;
    u32 n_;
    std::vector<cplx> psi_;
    std::vector<u32> rot5_;
    // device copies of psi_ ([4n] complex) and rot5_ ([n] u32), uploaded once
    const DeviceBuffer& device_tables() const;
    mutable std::shared_ptr<DeviceBuffer> dtab_;
    std::shared_ptr<std::mutex> dtab_mu_ = std::make_shared<std::mutex>();
};

struct EvalKeys {
    SwitchingKey relin;
    std::map<u64, SwitchingKey> galois;
    const SwitchingKey& galois_key(u64 exponent) const;
    bool has(u64 exponent) const { return galois.count(exponent) != 0; }
};

u64 rotation_exponent(const RingParams& ring, u32 k);
u64 conjugation_exponent(const RingParams& ring);

class Evaluator {
public:
    explicit Evaluator(const KeyContext& ctx) : ctx_(&ctx) {}
    const KeyContext& key_context() const { return *ctx_; }
    const RingParams& ring() const { return ctx_->ring(); }

    static void check_scales_match(double a, double b);
    void align_levels(Ciphertext& a, Ciphertext& b) const;
    Ciphertext add(const Ciphertext& a, const Ciphertext& b) const;
    Ciphertext sub(const Ciphertext& a, const Ciphertext& b) const;
    Ciphertext mul(const Ciphertext& a, const Ciphertext& b) const;
    Ciphertext mul_relin(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys) const;
    // Eval-form pipeline (B200 extensions): outputs stay in evaluation form;
    // to_coeff() of each equals mul_relin / rescale residue for residue.
    Ciphertext mul_relin_eval(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys) const;
    Ciphertext rescale_eval(const Ciphertext& ct) const;
    Ciphertext mul_plain(const Ciphertext& ct, const Poly& plain_eval, double plain_scale) const;
    Ciphertext mul_scalar(const Ciphertext& ct, double c, double scalar_scale) const;
    static u64 scaled_residue(double value, u64 q);
    Ciphertext add_scalar(const Ciphertext& ct, double c) const;
    Ciphertext rescale(const Ciphertext& ct) const;
    // Extension: add(rescale(prod), y) with identical results (ckks.hpp:315-324
    // then :195-210), one pass when every row is FP64-eligible and both are
    // coefficient-form degree-1 batches of the same shape.
    Ciphertext rescale_add(const Ciphertext& prod, const Ciphertext& y) const;
    // Extension: rescale(mul_relin(a, b)) (add == nullptr) or
    // rescale_add(mul_relin(a, b), *add), identical results and metadata; the
    // product's ModDown rows are rescaled (and added) in the same pass when
    // every row is FP64-eligible (KeyContext::relinearize_tensor_rescale).
    Ciphertext mul_relin_rescale(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys,
                                 const Ciphertext* add = nullptr) const;
    // Extension (lazy relinearisation): rescale(relinearize(add(mul(a, b),
    // mul(c, d)))) (+ add(., *add)) -- the reference's mul (ckks.hpp:220-245),
    // add (:201-208), relinearize (rlwe.hpp:601-620) and rescale (:315-324) in
    // that order, identical residues and metadata, with ONE key switch for the
    // two products. mul(c, d)'s level must not be below mul(a, b)'s for the
    // fast path (the second tensor is formed at the first's level: the tensor
    // is row-wise, so dropping operands first equals add's drop afterwards).
    Ciphertext mul2_relin_rescale(const Ciphertext& a, const Ciphertext& b, const Ciphertext& c,
                                  const Ciphertext& d, const EvalKeys& keys, const Ciphertext* add = nullptr) const;
    Ciphertext rotate(const Ciphertext& ct, u32 k, const EvalKeys& keys) const;
    Ciphertext conjugate(const Ciphertext& ct, const EvalKeys& keys) const;
    // Extension: sum_j mul_plain(cts[j], plains[j], plain_scale) in one
    // device pass (128-bit lazy accumulation); identical to the reference's
    // mul_plain / add sequence in j order (config 2's pt x ct MAC).
    Ciphertext mul_plain_sum(const std::vector<Ciphertext>& cts, const std::vector<Poly>& plains_eval,
                             double plain_scale) const;
    // Hoisted automorphism batch (ckks.hpp:338-367).
    std::vector<Ciphertext> apply_galois_many(const Ciphertext& ct, const std::vector<u64>& exps,
                                              const EvalKeys& keys) const;

private:
    const KeyContext* ctx_;
};

// BSGS linear transform plan (ckks.hpp:373-507): the nonzero diagonals of an
// n x n slot matrix, encoded once (device encoder) and pre-rotated for the
// giant steps; apply() = hoisted baby rotations, one plaintext-product sum
// kernel per giant bucket, giant rotations, rescale. Bit-exact with the
// reference plan.
class LinearTransformPlan {
public:
    LinearTransformPlan(const Encoder& enc, const std::map<u32, std::vector<cplx>>& diagonals, double plain_scale,
                        int encode_level);
    static std::map<u32, std::vector<cplx>> diagonals_of(const std::vector<std::vector<cplx>>& m);
    const std::vector<u64>& required_rotations() const { return rotations_; }
    double plain_scale() const { return plain_scale_; }
    u32 baby_count() const { return n1_; }
    Ciphertext apply(const Evaluator& ev, const Ciphertext& ct, const EvalKeys& keys) const;

private:
    struct Term {
        u32 g, b;
        Poly plain;  // eval form at encode_level
    };
    u32 n_;
    u32 n1_;
    double plain_scale_;
    int encode_level_;
    std::vector<Term> terms_;
    std::set<u64> baby_, giant_;
    std::vector<u64> rotations_;
};

// Chebyshev ladder evaluation (ckks.hpp:515-579), bit-exact with the reference.
Ciphertext eval_chebyshev(const Evaluator& ev, const Ciphertext& x, const std::vector<double>& cheb_coeffs,
                          const EvalKeys& keys);
// Baby-step/giant-step Chebyshev evaluation (same level budget as the ladder,
// ~sqrt(d) + log(d) products). Bit-exact with oracle/bsgs_ref.py, i.e. the
// same algorithm composed of the reference's Evaluator primitives.
Ciphertext eval_chebyshev_bsgs(const Evaluator& ev, const Ciphertext& x, const std::vector<double>& cheb_coeffs,
                               const EvalKeys& keys);
// Chebyshev evaluation with intermediate products kept in evaluation form
// (opt-in: TG_EVAL_PIPELINE=1 or set_eval_pipeline(true); slower for the
// BSGS shapes measured, see chebyshev.cpp). Results are identical either way.
void set_eval_pipeline(bool on);
bool eval_pipeline_enabled();
// Lazy relinearisation in eval_chebyshev_bsgs (default on; TG_LAZY_RELIN=0 or
// set_lazy_relin(false) restores one key switch per product): a node whose
// remainder is itself a giant-step node, Q T_n + (Q' T_n' + R'), adds the two
// degree-2 products before ONE relinearisation (Evaluator::mul2_relin_rescale).
// oracle/bsgs_ref.py (lazy=) restates both orders over reference primitives.
void set_lazy_relin(bool on);
bool lazy_relin_enabled();
// Which Chebyshev evaluator the threshold stages use.
enum class PolyEval { ladder, bsgs };
std::vector<double> power_to_chebyshev(const std::vector<double>& pow_coeffs);
// log2(n) rotate-and-add (ckks.hpp:605-615).
Ciphertext inner_sum(const Evaluator& ev, const Ciphertext& ct, u32 n, const EvalKeys& keys);

// ---------------------------------------------------------------------------
// Threshold (threshold.hpp)
// ---------------------------------------------------------------------------
struct ThresholdParams {
    u32 alpha = 8;
    u32 beta = 12;
    std::vector<u32> degrees;
    double epsilon = 1.0;
};

struct ChainStage {
    u32 degree = 0;
    double gamma = 0, upper = 1;
    std::vector<double> cheb;
    double error = 0;
};

struct MinimaxChain {
    ThresholdParams params;
    std::vector<ChainStage> stages;
    double sign_error = 0;
    double achieved_beta = 0;
    bool meets_target() const { return achieved_beta >= double(params.beta); }
    std::vector<double> eval_coeffs(std::size_t i) const;
    double eval_step(double x) const;
    u32 levels_required() const;
};

// Remez minimax of sign on [-U,-gamma] u [gamma,U] (remez.hpp:101-231).
struct MinimaxResult {
    u32 degree = 0;
    long double gamma = 0, upper = 1;
    std::vector<long double> odd_coeffs;
    long double error = 0;
    std::vector<long double> nodes;
    u32 iterations = 0;
    long double eval(long double x) const;
};
MinimaxResult remez_minimax(long double gamma, long double upper, u32 degree, u32 max_iters = 64);
MinimaxChain build_chain(const ThresholdParams& params);

// `mode` picks the stage evaluator: the reference ladder (default, bit-exact
// with the unmodified reference) or BSGS (bit-exact with oracle/bsgs_ref.py).
Ciphertext eval_private_threshold(const Evaluator& ev, const Ciphertext& ct_scores, const Ciphertext& ct_t,
                                  const Ciphertext& ct_norm, const MinimaxChain& chain, const EvalKeys& keys,
                                  PolyEval mode = PolyEval::ladder);
Ciphertext eval_private_threshold_plain_norm(const Evaluator& ev, const Ciphertext& ct_scores, const Ciphertext& ct_t,
                                             double norm, const MinimaxChain& chain, const EvalKeys& keys,
                                             PolyEval mode = PolyEval::ladder);

// Independent ciphertexts through eval_private_threshold_plain_norm
// concurrently: one host thread + one CUDA stream per ciphertext (up to
// max_streams), the reference's per-ciphertext thread pool
// (protocol.hpp:297-311). Each output is bit-identical to the single call.
std::vector<Ciphertext> eval_private_threshold_plain_norm_many(const Evaluator& ev,
                                                               const std::vector<Ciphertext>& scores,
                                                               const Ciphertext& ct_t, double norm,
                                                               const MinimaxChain& chain, const EvalKeys& keys,
                                                               int max_streams = 8, PolyEval mode = PolyEval::ladder);

}  // namespace tetris_b200
