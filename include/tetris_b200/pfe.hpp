// PFE, repacking and ring merge/split on the device (
// reference pfe.hpp, repack.hpp, rlwe.hpp:684-802). Same API, metadata and
// error messages; residues bit-identical (tests/test_gpu_pfe.py).
#pragma once

#include <map>
#include <string>

#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

// ---- large-domain PFE (pfe.hpp) ----
struct FunctionSpec {
    double lo = 0, hi = 0;
    std::vector<double> table;
    double out_min = 0, out_max = 0;
    double max_value() const;
    void validate(u32 ring_degree) const;
};

struct TestVector {
    Ciphertext ct;
    double lo = 0, hi = 0;
    double max_value = 0;
};

u32 encode_input(double x, double a, double b, u32 n);
TestVector build_test_vector(const KeyContext& ctx, const FunctionSpec& spec, const SecretKey& sk, double scale,
                             Rng& rng);
Ciphertext lookup(const TestVector& tv, u32 exponent);
// All rows in one device launch (tg_pfe_eval); op_trace as the reference's.
std::vector<Ciphertext> eval_scores(const std::vector<std::vector<double>>& rows, const std::vector<TestVector>& tvs,
                                    std::vector<std::string>* op_trace = nullptr);

// ---- ring repacking (repack.hpp) ----
struct RepackKeySet {
    std::vector<u64> exponents;
    std::map<u64, SwitchingKey> keys;
    u64 sk_id = 0;
    const SwitchingKey& key(u64 exponent) const;
};
struct RepackStats {
    u64 automorphisms = 0;
};
std::vector<u64> repack_exponents(const RingParams& ring);
RepackKeySet gen_repack_keys(const KeyContext& ctx, const SecretKey& sk, Rng& rng);
Ciphertext repack(const KeyContext& ctx, const std::vector<const Ciphertext*>& cts, const RepackKeySet& keys,
                  RepackStats* stats = nullptr);

// ---- ring split / merge (rlwe.hpp:684-802) ----
SecretKey embed_secret(const SecretKey& small_sk, const RingParams& big, u32 stride);
Ciphertext merge_embed(const std::vector<const Ciphertext*>& cts, const RingParams& big);
Ciphertext ring_merge(const KeyContext& big_ctx, const Ciphertext& ct0, const Ciphertext& ct1,
                      const SwitchingKey& swk);
Ciphertext ring_merge_many(const KeyContext& big_ctx, const std::vector<const Ciphertext*>& cts,
                           const SwitchingKey& swk);
std::pair<Ciphertext, Ciphertext> ring_split(const KeyContext& big_ctx, const RingParams& small, const Ciphertext& ct,
                                             const SwitchingKey& swk_to_embed, u64 small_sk_id);

}  // namespace tetris_b200
