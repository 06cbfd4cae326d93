// tetris_b200 RLWE layer: gadget decomposition, keys, encryption, key
// switching, relinearisation and Galois automorphisms. Drop-in for the
// reference rlwe.hpp evaluation path (keygen/encrypt/decrypt included so a
// caller can switch wholesale). Key material is sampled on the host from the
// reference's RNG streams and resident in HBM in the layout the key-switch
// kernels read: [digit][b|a][max_level+1+K rows][N].
#pragma once

#include <map>
#include <utility>

#include "tetris_b200/core.hpp"

namespace tetris_b200 {

struct GadgetVector {
    u32 group_size = 1;
    u32 base2_bits = 0;  // base-2 refinement (rlwe.hpp:103-135); host-only, not on the device path
    u32 sub_digits(u64 q) const;
};

// Replaces GadgetPlan (rlwe.hpp:28-206). The device tables (src_scale,
// conv_w, ModDown constants) live in a tg_gadget.
class GadgetPlan {
public:
    GadgetPlan() = default;
    GadgetPlan(const RingParams& ring, GadgetVector cfg);
    ~GadgetPlan();
    GadgetPlan(const GadgetPlan&) = delete;
    GadgetPlan& operator=(const GadgetPlan&) = delete;

    const RingParams& ring() const { return *ring_; }
    const GadgetVector& config() const { return cfg_; }
    u32 group_count(int level) const { return (u32(level) + cfg_.group_size) / cfg_.group_size; }
    u32 digit_count(int level) const;
    // ModUp: digits in eval form, each level+1+K rows (rlwe.hpp:65-139).
    std::vector<Poly> decompose(const Poly& d) const;
    // w_digit * P mod q_t per digit (rlwe.hpp:142-165), host.
    std::vector<std::vector<u64>> key_scalars() const;
    tg_gadget* dev() const;

private:
    const RingParams* ring_ = nullptr;
    GadgetVector cfg_;
    mutable std::once_flag once_;
    mutable std::shared_ptr<DeviceState> devstate_;  // keeps the context alive past the ring
    mutable tg_gadget* dev_ = nullptr;
};

class SecretKey {
public:
    SecretKey() = default;
    SecretKey(const RingParams& ring, const NoiseParams& noise, Rng& rng);
    SecretKey(const RingParams& ring, std::vector<i64> coeffs, u64 id);

    const RingParams& ring() const { return *ring_; }
    u32 hamming_weight() const { return hamming_weight_; }
    u64 id() const { return id_; }
    const std::vector<i64>& coeffs() const { return coeffs_; }
    // eval-form rows for (level, nspecial), extracted from the full key
    Poly shaped(int level, int nspecial) const;

private:
    const RingParams* ring_ = nullptr;
    u32 hamming_weight_ = 0;
    u64 id_ = 0;
    std::vector<i64> coeffs_;
    Poly eval_full_;
};

struct PublicKey {
    Poly b, a;
    u64 sk_id = 0;
};

enum class Domain { coeffs, slots };

// Replaces reference Ciphertext (rlwe.hpp:275-317).
struct Ciphertext {
    std::vector<Poly> parts;
    double scale = 1.0;
    Domain domain = Domain::coeffs;
    u64 sk_id = 0;
    double noise_bound = 0.0;
    // Extension (not in the reference): `batch` ciphertexts of one shape and
    // scale evaluated together, stored part-major: part k of ciphertext i is
    // parts[k * batch + i]. Every op treats a batch exactly as `batch`
    // independent ciphertexts (same residues); launches and key reads are
    // shared. See stack_ciphertexts / unstack_ciphertext.
    u32 batch = 1;

    const RingParams& ring() const { return parts.at(0).ring(); }
    int level() const { return parts.at(0).level(); }
    Form form() const { return parts.at(0).form(); }
    int degree() const { return int(parts.size() / batch) - 1; }
    void to_coeff();
    void to_eval();
    void drop_to_level(int new_level);
    void add_inplace(const Ciphertext& o);
    void sub_inplace(const Ciphertext& o);
    void negate_inplace();
};

// Batches: stack (copies into one part-major block; equal degree, level,
// form, domain, key and scale within 1e-4), unstack and slice (copies of
// ciphertexts [first, first + count) into their own block).
Ciphertext stack_ciphertexts(const std::vector<Ciphertext>& cts);
std::vector<Ciphertext> unstack_ciphertext(const Ciphertext& ct);
Ciphertext slice_ciphertext(const Ciphertext& ct, u32 first, u32 count);

// Switching key (rlwe.hpp:325-333). b[i]/a[i] are views into one HBM block.
struct SwitchingKey {
    GadgetVector gadget;
    u64 from_id = 0, to_id = 0;
    u64 a_seed = 0;
    std::vector<Poly> b, a;
    std::shared_ptr<DeviceBuffer> block;  // [digit][b|a][rows][N]
    const RingParams& ring() const { return b.at(0).ring(); }
    u32 digits() const { return u32(b.size()); }
    const u64* device_data() const { return block ? block->data() : nullptr; }
};

// Replaces KeyContext (rlwe.hpp:335-682).
class KeyContext {
public:
    KeyContext(const RingParams& ring, NoiseParams noise, GadgetVector gadget);

    const RingParams& ring() const { return *ring_; }
    const NoiseParams& noise() const { return noise_; }
    const GadgetPlan& plan() const { return *plan_; }

    std::pair<SecretKey, PublicKey> keygen(Rng& rng) const;
    PublicKey make_public(const SecretKey& sk, Rng& rng) const;
    Ciphertext encrypt(const SecretKey& sk, const Poly& m, double scale, Rng& rng,
                       Domain domain = Domain::coeffs) const;
    Ciphertext encrypt_pk(const PublicKey& pk, const Poly& m, double scale, Rng& rng,
                          Domain domain = Domain::coeffs) const;
    Poly decrypt(const SecretKey& sk, const Ciphertext& ct) const;
    Ciphertext zero_ciphertext(int level, double scale, u64 sk_id, Domain domain = Domain::coeffs) const;

    SwitchingKey switch_key_gen(const SecretKey& from, const SecretKey& to, Rng& rng) const;
    std::pair<Poly, Poly> ks_inner(const std::vector<Poly>& digits, const SwitchingKey& swk) const;
    std::pair<Poly, Poly> switch_key_apply(const Poly& d, const SwitchingKey& swk) const;
    Poly mod_down_p(const Poly& x) const;

    SwitchingKey relin_key_gen(const SecretKey& sk, Rng& rng) const;
    Ciphertext relinearize(const Ciphertext& ct, const SwitchingKey& rlk) const;
    // relinearize with EVAL-form output (B200 extension): the tensor's
    // eval-form c0/c1 are the ModDown addends as they are; only c2 and the
    // accumulators' special rows are inverse transformed. to_coeff() of the
    // result equals relinearize(ct, rlk) residue for residue.
    Ciphertext relinearize_eval(const Ciphertext& ct, const SwitchingKey& rlk) const;
    // relinearize(mul(x, y)) for EVAL-form, level-aligned degree-1 operands
    // (B200 extension, Evaluator::mul_relin): only c2 of the tensor goes
    // through HBM; c0 / c1 are formed inside the fused key-switch core
    // (tg_relinearize_tensor_batch). Residue for residue the same.
    Ciphertext relinearize_tensor(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk) const;
    // relinearize_tensor then rescale_round (+ add of `add`'s rows 0..out_level)
    // in the same ModDown pass (tg_relinearize_tensor_rescale_batch): parts of
    // level-1 (or out_level) rows; scale / noise_bound are the PRODUCT's, the
    // caller (Evaluator::mul_relin_rescale) applies rescale / add's metadata.
    // relinearize_tensor followed by the Chebyshev ladder step
    // (ckks.hpp:532-555) in the same ModDown pass
    // (tg_relinearize_tensor_ladder_batch): parts of level-1 rows holding
    // rescale(2 prod - sub_coef * sub (+ add_const at coefficient 0 of part
    // 0)); sub (coefficient form, level >= x's, uniformly strided parts) may
    // be null. Metadata is the PRODUCT's; the caller applies the step's.
    Ciphertext relinearize_tensor_ladder(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk,
                                         const Ciphertext* sub, const std::vector<u64>& sub_coef,
                                         const std::vector<u64>& add_const) const;
    // u, v (both or neither): a second product of the same level and batch,
    // added before the one relinearisation (tg_relinearize_tensor2_rescale_batch).
    Ciphertext relinearize_tensor_rescale(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk,
                                          const Ciphertext* add, int out_level, const Ciphertext* u = nullptr,
                                          const Ciphertext* v = nullptr) const;
    SwitchingKey galois_key_gen(const SecretKey& sk, u64 exponent, Rng& rng) const;
    Ciphertext apply_galois(const Ciphertext& ct, u64 exponent, const SwitchingKey& swk) const;
    // Hoisted automorphisms (Evaluator::apply_galois_many, ckks.hpp:338-367):
    // c1 decomposed once, the eval-form digits permuted per exponent; keys[i]
    // is the Galois key of exps[i] (ignored for exponent 1).
    std::vector<Ciphertext> apply_galois_hoisted(const Ciphertext& ct, const std::vector<u64>& exps,
                                                 const std::vector<const SwitchingKey*>& keys) const;
    double ks_noise_estimate() const;
    SecretKey square_secret(const SecretKey& sk) const;

private:
    const RingParams* ring_;
    NoiseParams noise_;
    std::shared_ptr<GadgetPlan> plan_;
};

}  // namespace tetris_b200
