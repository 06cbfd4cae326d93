// Hoisted rotations and the BSGS linear transform (the
// building blocks of Half-BTS's CoeffToSlot/SlotToCoeff). Reference:
// Evaluator::apply_galois_many (ckks.hpp:338-367) and LinearTransformPlan
// (ckks.hpp:373-507). Same operation order and host constants, device
// arithmetic; bit-exact (tests/test_gpu_linear.py).
#include <cmath>

#include "internal.hpp"
#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

using detail::fresh_parts;

std::vector<Ciphertext> Evaluator::apply_galois_many(const Ciphertext& ct, const std::vector<u64>& exps,
                                                     const EvalKeys& keys) const {
    if (ct.degree() != 1) throw TetrisError("ckks", "hoisting expects degree-1 input");
    std::vector<const SwitchingKey*> ks;
    ks.reserve(exps.size());
    for (u64 g : exps) ks.push_back(g == 1 ? nullptr : &keys.galois_key(g));
    return ctx_->apply_galois_hoisted(ct, exps, ks);
}

Ciphertext Evaluator::mul_plain_sum(const std::vector<Ciphertext>& cts, const std::vector<Poly>& plains_eval,
                                    double plain_scale) const {
    if (cts.empty() || cts.size() != plains_eval.size()) throw TetrisError("ckks", "mul_plain_sum: size mismatch");
    if (cts.size() > TG_PLAIN_SUM_MAX_TERMS) throw TetrisError("ckks", "mul_plain_sum: too many terms");
    const RingParams& R = ring();
    std::vector<Ciphertext> ev(cts);
    const int lvl = ev[0].level();
    for (const auto& c : ev)
        if (c.level() != lvl) throw TetrisError("ckks", "mul_plain_sum expects ciphertexts at one level");
    double noise = 0;
    std::vector<Poly> keep;
    std::vector<const u64*> cp, pp;
    std::vector<u64> ps;  // words between each term's two parts
    for (std::size_t j = 0; j < ev.size(); ++j) {
        Ciphertext& c = ev[j];
        if (c.degree() != 1 || c.batch != 1) throw TetrisError("ckks", "mul_plain_sum expects single degree-1 ciphertexts");
        if (c.domain != ev[0].domain) throw TetrisError("rlwe", "domain tag mismatch");
        check_scales_match(c.scale, ev[0].scale);  // add's precondition on the products (same plain_scale)
        c.to_eval();
        if (plains_eval[j].level() < lvl || plains_eval[j].nspecial() != 0)
            throw TetrisError("ckks", "plaintext has fewer rows than the ciphertext");
        // parts on a uniform stride (a ciphertext, or the part-major views of
        // a batch from stack_ciphertexts) are read in place, others gathered
        const Poly &q0 = c.parts[0], &q1 = c.parts[1];
        const std::size_t S = q1.offset() > q0.offset() ? q1.offset() - q0.offset() : 0;
        if (q0.storage() == q1.storage() && S >= std::size_t(lvl + 1) * R.degree() && q0.level() == lvl &&
            q1.level() == lvl) {
            cp.push_back(c.parts[0].data());
            ps.push_back(u64(S));
        } else {
            cp.push_back(detail::group_data(c.parts, 0, 2, keep));
            ps.push_back(u64(lvl + 1) * R.degree());
        }
        pp.push_back(plains_eval[j].data());
        noise += c.noise_bound * plain_scale;
    }
    std::vector<Poly> out = fresh_parts(R, 2, lvl, Form::eval);
    check_tg(tg_mul_plain_sum_strided(R.dev(), const_cast<u64*>(out[0].data()), u32(ev.size()), cp.data(), ps.data(),
                                      pp.data(), lvl, 2, R.stream()));
    Ciphertext r;
    r.parts = std::move(out);
    r.scale = ev[0].scale * plain_scale;
    r.domain = ev[0].domain;
    r.sk_id = ev[0].sk_id;
    r.noise_bound = noise;
    return r;
}

LinearTransformPlan::LinearTransformPlan(const Encoder& enc, const std::map<u32, std::vector<cplx>>& diagonals,
                                         double plain_scale, int encode_level)
    : n_(enc.slots()), plain_scale_(plain_scale), encode_level_(encode_level) {
    if (diagonals.empty()) throw TetrisError("ckks", "empty linear transform");
    const double root = std::sqrt(double(diagonals.size()));
    u32 n1 = 1;
    while (double(n1 * 2) <= root * 1.42) n1 *= 2;
    n1_ = std::min(n1, n_);
    const RingParams& ring = enc.ring();
    std::vector<std::vector<cplx>> shifted_all;
    std::vector<std::pair<u32, u32>> gb;
    for (const auto& [d, diag] : diagonals) {
        if (diag.size() != n_) throw TetrisError("ckks", "diagonal length mismatch");
        const u32 g = d / n1_, b = d % n1_;
        std::vector<cplx> shifted(n_);
        const u32 shift = g * n1_;  // pre-rotate right by g*n1
        for (u32 i = 0; i < n_; ++i) shifted[(i + shift) % n_] = diag[i];
        shifted_all.push_back(std::move(shifted));
        gb.emplace_back(g, b);
    }
    // all diagonals in one encoder launch, then one batched forward NTT
    std::vector<Poly> pts = enc.encode_slots_many(shifted_all, plain_scale, encode_level);
    Ciphertext block;  // transform the block of plaintexts together
    block.parts = pts;
    block.to_eval();
    for (std::size_t i = 0; i < gb.size(); ++i) {
        const auto [g, b] = gb[i];
        terms_.push_back(Term{g, b, block.parts[i]});
        if (b != 0) baby_.insert(rotation_exponent(ring, b));
        if (g != 0) giant_.insert(rotation_exponent(ring, g * n1_));
    }
    for (u64 e : baby_) rotations_.push_back(e);
    for (u64 e : giant_) rotations_.push_back(e);
}

std::map<u32, std::vector<cplx>> LinearTransformPlan::diagonals_of(const std::vector<std::vector<cplx>>& m) {
    const u32 n = u32(m.size());
    std::map<u32, std::vector<cplx>> out;
    for (u32 d = 0; d < n; ++d) {
        std::vector<cplx> diag(n);
        bool nonzero = false;
        for (u32 i = 0; i < n; ++i) {
            diag[i] = m[i][(i + d) % n];
            if (std::abs(diag[i]) > 1e-300) nonzero = true;
        }
        if (nonzero) out.emplace(d, std::move(diag));
    }
    return out;
}

Ciphertext LinearTransformPlan::apply(const Evaluator& ev, const Ciphertext& ct, const EvalKeys& keys) const {
    if (ct.domain != Domain::slots) throw TetrisError("ckks", "linear transform expects slots domain");
    // hoisted baby rotations
    std::set<u32> baby_idx;
    for (const Term& t : terms_) baby_idx.insert(t.b);
    std::vector<u64> baby_exps;
    std::vector<u32> baby_ks;
    for (u32 b : baby_idx) {
        baby_exps.push_back(b == 0 ? 1 : rotation_exponent(ev.ring(), b));
        baby_ks.push_back(b);
    }
    std::vector<Ciphertext> rotated = ev.apply_galois_many(ct, baby_exps, keys);
    std::map<u32, const Ciphertext*> rot_of;
    for (std::size_t i = 0; i < baby_ks.size(); ++i) rot_of[baby_ks[i]] = &rotated[i];
    for (auto& r : rotated) r.to_eval();

    // one plaintext-product sum per giant bucket (u128 lazy accumulation on the device)
    std::map<u32, std::vector<const Term*>> by_g;
    for (const Term& t : terms_) by_g[t.g].push_back(&t);
    const Ciphertext& proto = *rot_of.begin()->second;
    const int lvl = proto.level();
    const RingParams& R = ev.ring();
    std::map<u32, Ciphertext> inner;
    for (auto& [g, ts] : by_g) {
        if (ts.size() > 256) throw TetrisError("ckks", "giant bucket exceeds lazy headroom");
        std::vector<Poly> keep;
        std::vector<const u64*> cts, pls;
        for (const Term* t : ts) {
            const Ciphertext& rot = *rot_of.at(t->b);
            cts.push_back(detail::group_data(rot.parts, 0, 2, keep));
            if (t->plain.level() < lvl) throw TetrisError("ckks", "plaintext has fewer rows than the ciphertext");
            pls.push_back(t->plain.data());
        }
        std::vector<Poly> sp = fresh_parts(R, 2, lvl, Form::eval);
        check_tg(tg_mul_plain_sum(R.dev(), const_cast<u64*>(sp[0].data()), u32(ts.size()), cts.data(), pls.data(),
                                  lvl, 2, R.stream()));
        Ciphertext sum;
        sum.parts = std::move(sp);
        sum.scale = proto.scale * plain_scale_;
        sum.domain = proto.domain;
        sum.sk_id = proto.sk_id;
        sum.noise_bound = proto.noise_bound * plain_scale_;
        inner.emplace(g, std::move(sum));
    }
    Ciphertext acc;
    bool first = true;
    for (auto& [g, sum] : inner) {
        Ciphertext term = g == 0 ? sum : ev.rotate(sum, g * n1_, keys);
        if (first) {
            acc = std::move(term);
            first = false;
        } else {
            acc.to_coeff();
            term.to_coeff();
            acc.add_inplace(term);
        }
    }
    return ev.rescale(acc);
}

}  // namespace tetris_b200
