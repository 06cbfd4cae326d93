// Half-BTS (reference bootstrap.hpp): ModRaise -> [trace map] -> CoeffsToSlots
// -> EvalMod, every ciphertext op on the device. SURVEY 8(f) rank 1.
#pragma once

#include <functional>
#include <memory>

#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

struct EvalModConfig {  // bootstrap.hpp:21-27
    u32 cheb_degree = 30;
    u32 double_angles = 3;
    u32 lattice_bound = 16;
    u32 arcsine_degree = 7;
    double arcsine_window = 0.65;
};

struct BootstrapParams {  // bootstrap.hpp:29-48
    u32 slots = 0;
    u32 sparse_log_gap = 0;
    u32 secret_hw = 32;
    u32 ephemeral_hw = 0;
    EvalModConfig evalmod;
    double delta_input = 0;
    double delta_evalmod = 0;
    u32 depth() const;
};

// Chebyshev interpolation at 4(d+1) Chebyshev nodes in long double
// (remez.hpp:12-26).
std::vector<double> chebyshev_fit(const std::function<long double(long double)>& f, u32 degree);

class BootstrapEvaluator {  // bootstrap.hpp:50-245
public:
    BootstrapEvaluator(const KeyContext& ctx, BootstrapParams params);
    const BootstrapParams& params() const { return params_; }
    const Encoder& encoder() const { return encoder_; }
    std::vector<u64> required_galois_exponents() const;
    std::vector<u64> trace_exponents() const;
    Ciphertext mod_raise(const Ciphertext& ct) const;
    Ciphertext trace_map(const Evaluator& ev, const Ciphertext& ct, u32 t, const EvalKeys& keys) const;
    std::pair<Ciphertext, Ciphertext> coeffs_to_slots(const Evaluator& ev, const Ciphertext& ct,
                                                      const EvalKeys& keys) const;
    Ciphertext eval_mod(const Evaluator& ev, const Ciphertext& ct, const EvalKeys& keys) const;
    Ciphertext slots_to_coeffs(const Evaluator& ev, const Ciphertext& ct_re, const Ciphertext& ct_im,
                               const EvalKeys& keys) const;
    std::pair<Ciphertext, Ciphertext> half_bts(const Evaluator& ev, const Ciphertext& ct, const EvalKeys& keys) const;
    int output_level() const { return ctx_->ring().max_level() - int(params_.depth()); }
    const std::vector<double>& cos_coeffs() const { return cheb_cos_; }
    const std::vector<double>& asin_coeffs() const { return cheb_asin_; }

private:
    const KeyContext* ctx_;
    BootstrapParams params_;
    Encoder encoder_;
    double q0_ = 0;
    std::unique_ptr<LinearTransformPlan> c2s_, s2c_;
    std::vector<double> cheb_cos_, cheb_asin_;
};

}  // namespace tetris_b200
