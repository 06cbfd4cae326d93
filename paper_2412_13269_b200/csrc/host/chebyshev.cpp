// Chebyshev-series evaluation on the device:
//  * eval_chebyshev        — the reference's memoised T_k ladder
//                            (ckks.hpp:515-579), bit-exact with it;
//  * eval_chebyshev_bsgs   — baby-step/giant-step evaluation (BASELINE.json
//                            config 3), bit-exact with its oracle
//                            (oracle/bsgs_ref.py over the reference's own
//                            Evaluator primitives), same level budget,
//                            7/11/16 instead of 11/20/47 relinearised products
//                            for d = 15/27/63; with lazy relinearisation
//                            (default) one key switch fewer per node whose
//                            remainder is a giant-step node too.
// Every ladder step T_k = rescale(2 T_a T_b - v T_c | - 1) leaves its
// product's key switch in one pass (Ladder::fused_step: the linear step and
// the rescale inside ModDown, KeyContext::relinearize_tensor_ladder; rings
// with 60-bit rows and small launches relinearise, then one tg_lincomb pass);
// every combination step is ONE fused residue pass (tg_lincomb), and the base
// blocks of one BSGS polynomial share a multi-output pass (tg_lincomb_multi).
// Scales and noise bounds follow the reference's add_inplace / mul_scalar /
// sub_inplace / add_scalar / rescale sequence exactly.
// Eval-form pipeline (opt-in: TG_EVAL_PIPELINE=1 or set_eval_pipeline):
// products, combinations and rescales stay in evaluation form
// (relinearize_eval / tg_rescale_eval); the result is converted to
// coefficient form once at the end, residue for residue the same ciphertext.
// It saves two transformed rows per row of a product whose result is
// multiplied again, but every rescale then needs `level` forward rows, so
// for the BSGS shapes here it is slower (config 4: 121 vs 105 ms per step,
// DESIGN.md) and the coefficient-form pipeline is the default.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <deque>
#include <functional>
#include <map>
#include <optional>

#include "internal.hpp"
#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

using detail::fresh_parts;

namespace {

struct LinTerm {
    const Ciphertext* ct;
    std::vector<u64> coef;  // one integer per q row 0..level
};

// The kernel addresses part p of term t at ptr[t] + p * stride[t]: parts of
// a term must be uniformly strided (a single ciphertext always is; a batch
// is when its parts share one block, else it is gathered first).
bool uniform_parts(const std::vector<Poly>& parts) {
    if (parts.size() <= 2) return true;
    const u64 s = u64(parts[1].data() - parts[0].data());
    for (std::size_t p = 2; p < parts.size(); ++p)
        if (u64(parts[p].data() - parts[0].data()) != s * p) return false;
    return true;
}

std::atomic<int> g_eval_pipeline{-1};

bool eval_pipeline() {
    int v = g_eval_pipeline.load();
    if (v < 0) {
        const char* e = std::getenv("TG_EVAL_PIPELINE");
        v = (e && e[0] == '1') ? 1 : 0;
        g_eval_pipeline.store(v);
    }
    return v != 0;
}

std::atomic<int> g_lazy_relin{-1};

bool lazy_relin() {
    int v = g_lazy_relin.load();
    if (v < 0) {
        const char* e = std::getenv("TG_LAZY_RELIN");
        v = (e && e[0] == '0') ? 0 : 1;
        g_lazy_relin.store(v);
    }
    return v != 0;
}

bool multi_base() {
    static const bool off = [] {
        const char* e = std::getenv("TG_MULTI_BASE");
        return e && *e == '0';
    }();
    return !off;
}

std::vector<Poly> fused_lincomb(const RingParams& R, const std::vector<LinTerm>& terms,
                                const std::vector<u64>& add_per_row, int level, bool rescale) {
    const u32 nt = u32(terms.size());
    const u32 B = terms[0].ct->batch;
    const Form f = terms[0].ct->form();
    std::vector<const u64*> ptrs(nt);
    std::vector<u64> strides(nt);
    std::vector<u64> coeffs(std::size_t(nt) * (level + 1));
    std::vector<Poly> keep;
    for (u32 t = 0; t < nt; ++t) {
        const Ciphertext& c = *terms[t].ct;
        if (c.batch != B || c.parts.size() != 2 * B || c.form() != f || c.level() < level ||
            c.parts[0].nspecial() != 0)
            throw TetrisError("ckks", "fused combination expects degree-1 terms of one form");
        if (uniform_parts(c.parts)) {
            ptrs[t] = c.parts[0].data();
            strides[t] = u64(c.parts[1].data()) / 8 - u64(c.parts[0].data()) / 8;  // words (mod 2^64)
        } else {
            ptrs[t] = detail::group_data(c.parts, 0, c.parts.size(), keep);
            strides[t] = c.parts[0].words();
        }
        for (int r = 0; r <= level; ++r) coeffs[std::size_t(t) * (level + 1) + r] = terms[t].coef[r];
    }
    // eval form: a constant is added at every evaluation point; rescale runs
    // after the combination (tg_rescale_eval)
    const bool ev = f == Form::eval, fused_rs = rescale && !ev;
    std::vector<Poly> out = fresh_parts(R, int(2 * B), fused_rs ? level - 1 : level, f);
    check_tg(tg_lincomb_batch(R.dev(), const_cast<u64*>(out[0].data()), nt, ptrs.data(), strides.data(),
                              coeffs.data(), add_per_row.empty() ? nullptr : add_per_row.data(), ev ? 1 : 0, level,
                              2 * B, B, fused_rs ? 1 : 0, R.stream()));
    if (!rescale || !ev) return out;
    std::vector<Poly> rs = fresh_parts(R, int(2 * B), level - 1, Form::eval);
    check_tg(tg_rescale_eval(R.dev(), const_cast<u64*>(rs[0].data()), out[0].data(), level, 2 * B, R.stream()));
    return rs;
}

std::vector<u64> residues_of(const RingParams& R, i64 v, int level) {
    std::vector<u64> c(level + 1);
    for (int r = 0; r <= level; ++r) c[r] = from_centered(v, R.modulus(u32(r)));
    return c;
}

// The reference ladder T_k = 2 T_a T_b - T_{b-a}, a = floor(k/2) (ckks.hpp:532-555).
struct Ladder {
    const Evaluator& ev;
    const EvalKeys& keys;
    const RingParams& R;
    std::map<std::size_t, Ciphertext> T;
    const bool eval = eval_pipeline();
    Ladder(const Evaluator& e, const Ciphertext& x, const EvalKeys& k) : ev(e), keys(k), R(e.ring()) {
        Ciphertext x1 = x;
        if (eval) x1.to_eval();
        T.emplace(1, std::move(x1));
    }
    void to_form(Ciphertext& c) const { eval ? c.to_eval() : c.to_coeff(); }
    // the finished result in the reference's (coefficient) form
    Ciphertext finish(Ciphertext c) const {
        if (c.form() == Form::coeff) return c;
        const Ciphertext src = c;  // shared: transformed out of place, then cached
        detail::to_coeff_keep_eval(c);
        return c;
    }

    // The product and its ladder step in one ModDown pass
    // (KeyContext::relinearize_tensor_ladder): coefficient-form degree-1
    // operands of one batch and domain, FP64-eligible q rows.
    bool fused_ladder_ok(const Ciphertext& ta, const Ciphertext& tb) const {
        static const bool off = [] {
            const char* e = std::getenv("TG_RELIN_TENSOR");
            const char* f = std::getenv("TG_FUSED_LADDER");
            return (e && *e == '0') || (f && *f == '0');
        }();
        if (off || ta.domain != tb.domain || ta.degree() != 1 || tb.degree() != 1 || ta.batch != tb.batch) return false;
        const int lvl = std::min(ta.level(), tb.level());
        if (lvl < 1 || lvl + 1 > 32) return false;
        for (const Ciphertext* t : {&ta, &tb})
            for (const auto& p : t->parts)
                if (p.nspecial() != 0) return false;
        for (int r = 0; r <= lvl; ++r)
            if (R.modulus(u32(r)) >= 1351079888211148ull) return false;  // kFpMaxQ (tg_fp64.cuh)
        return true;
    }
    // mul_relin, add_inplace, [mul_scalar, sub_inplace | add_scalar], rescale
    // (ckks.hpp:532-555): the same checks and metadata in the same order
    Ciphertext fused_step(const Ciphertext& ta, const Ciphertext& tb, const Ciphertext* tc) {
        Ciphertext x = ta, y = tb;
        ev.align_levels(x, y);
        const int lvl = x.level();
        const double pscale = x.scale * y.scale;
        const double pnoise = (x.noise_bound * y.scale + y.noise_bound * x.scale) + ev.key_context().ks_noise_estimate();
        const double two_noise = pnoise + pnoise;
        const u64 ql = R.modulus(u32(lvl));
        std::vector<u64> coef, add;
        Ciphertext tc0;
        double noise;
        if (!tc) {
            add.resize(lvl + 1);
            for (int r = 0; r <= lvl; ++r) add[r] = Evaluator::scaled_residue(-1.0 * pscale, R.modulus(u32(r)));
            noise = two_noise / double(ql) + 1.0;
        } else {
            tc0 = *tc;
            tc0.to_coeff();
            const double ratio = pscale / tc0.scale;
            if (std::abs(1.0) * ratio >= 9.0e18)
                throw TetrisError("ckks", "scalar multiplier exceeds the integer range");
            const i64 v = round_half_away(1.0 * ratio);
            const double tc_scale = tc0.scale * ratio;
            Evaluator::check_scales_match(tc_scale, pscale);
            coef.resize(lvl + 1);
            for (int r = 0; r <= lvl; ++r) coef[r] = from_centered(v, R.modulus(u32(r)));
            noise = (two_noise + tc0.noise_bound) / double(ql) + 1.0;
        }
        x.to_eval();
        y.to_eval();
        Ciphertext res = ev.key_context().relinearize_tensor_ladder(x, y, keys.relin, tc ? &tc0 : nullptr, coef, add);
        res.noise_bound = noise;
        res.scale = pscale / double(ql);
        return res;
    }

    const Ciphertext& get(std::size_t k) {
        auto hit = T.find(k);
        if (hit != T.end()) return hit->second;
        const std::size_t a = k / 2, b = k - a;
        const Ciphertext& ta = get(a);
        const Ciphertext& tb = get(b);
        if (!eval && fused_ladder_ok(ta, tb)) return T.emplace(k, fused_step(ta, tb, a == b ? nullptr : &get(b - a))).first->second;
        Ciphertext prod = eval ? ev.mul_relin_eval(ta, tb, keys) : ev.mul_relin(ta, tb, keys);
        to_form(prod);
        const int lvl = prod.level();
        if (lvl == 0) throw TetrisError("ckks", "cannot rescale at level 0");
        const double two_noise = prod.noise_bound + prod.noise_bound;  // add_inplace(prod)
        const u64 ql = R.modulus(u32(lvl));
        Ciphertext res;
        if (a == b) {  // rescale(add_scalar(2 prod, -1))
            std::vector<u64> add(lvl + 1);
            for (int r = 0; r <= lvl; ++r) add[r] = Evaluator::scaled_residue(-1.0 * prod.scale, R.modulus(u32(r)));
            res.parts = fused_lincomb(R, {LinTerm{&prod, residues_of(R, 2, lvl)}}, add, lvl, true);
            res.noise_bound = two_noise / double(ql) + 1.0;
        } else {  // rescale(2 prod - mul_scalar(T_{b-a}, 1, ratio))
            Ciphertext tc0 = get(b - a);
            to_form(tc0);
            const double ratio = prod.scale / tc0.scale;
            if (std::abs(1.0) * ratio >= 9.0e18)
                throw TetrisError("ckks", "scalar multiplier exceeds the integer range");
            const i64 v = round_half_away(1.0 * ratio);
            const double tc_scale = tc0.scale * ratio;
            Evaluator::check_scales_match(tc_scale, prod.scale);
            std::vector<u64> negv(lvl + 1);
            for (int r = 0; r <= lvl; ++r) negv[r] = neg_mod(from_centered(v, R.modulus(u32(r))), R.modulus(u32(r)));
            res.parts = fused_lincomb(R, {LinTerm{&prod, residues_of(R, 2, lvl)}, LinTerm{&tc0, negv}}, {}, lvl, true);
            res.noise_bound = (two_noise + tc0.noise_bound) / double(ql) + 1.0;
        }
        res.batch = prod.batch;
        res.scale = prod.scale / double(ql);
        res.domain = prod.domain;
        res.sk_id = prod.sk_id;
        return T.emplace(k, std::move(res)).first->second;
    }
};

// The reference combination step (ckks.hpp:556-578) over ladder terms
// ks (coefficients cs[k]), at the common level min(x.level, T_k.level):
// rescale( sum_k mul_scalar(T_k, c_k, q_lvl) + add_scalar(c_0) ).
// target > 0 (BSGS blocks): the combination scale becomes
// q_lvl * target / scale(T_first), so the rescaled block lands on `target`.
// CombPlan: the checks, integer constants and metadata of one such step
// (everything but the residue pass).
struct CombPlan {
    int lvl = 0;
    std::vector<std::size_t> ks;
    std::vector<LinTerm> terms;
    std::vector<Ciphertext> conv;  // copies of terms in the ladder's form
    std::vector<u64> add;
    double acc_scale = 0, acc_noise = 0;
};

void plan_combine(CombPlan& P, Ladder& L, const Ciphertext& x, const std::vector<std::size_t>& ks,
                  const std::vector<double>& cs, double c0, double target) {
    const RingParams& R = L.R;
    int lvl = x.level();
    for (std::size_t k : ks) lvl = std::min(lvl, L.get(k).level());
    double comb_scale = double(R.modulus(u32(lvl)));
    if (target > 0.0) comb_scale = comb_scale * (target / L.get(ks[0]).scale);
    P.lvl = lvl;
    P.ks = ks;
    P.conv.reserve(ks.size());
    const Form f = L.eval ? Form::eval : Form::coeff;
    bool first = true;
    for (std::size_t k : ks) {
        const Ciphertext* tk = &L.get(k);
        if (tk->form() != f) {
            P.conv.push_back(*tk);
            L.to_form(P.conv.back());
            tk = &P.conv.back();
        }
        const double c = cs[k];
        if (std::abs(c) * comb_scale >= 9.0e18) throw TetrisError("ckks", "scalar multiplier exceeds the integer range");
        const double term_scale = tk->scale * comb_scale;
        if (first) {
            P.acc_scale = term_scale;
            P.acc_noise = tk->noise_bound;
            first = false;
        } else {
            Evaluator::check_scales_match(P.acc_scale, term_scale);
            P.acc_noise += tk->noise_bound;
        }
        P.terms.push_back(LinTerm{tk, residues_of(R, round_half_away(c * comb_scale), lvl)});
    }
    if (c0 != 0.0) {
        P.add.resize(lvl + 1);
        for (int r = 0; r <= lvl; ++r) P.add[r] = Evaluator::scaled_residue(c0 * P.acc_scale, R.modulus(u32(r)));
    }
    if (lvl == 0) throw TetrisError("ckks", "cannot rescale at level 0");
}

Ciphertext finish_combine(const CombPlan& P, const RingParams& R, const Ciphertext& x, std::vector<Poly> parts) {
    const u64 ql = R.modulus(u32(P.lvl));
    Ciphertext out;
    out.parts = std::move(parts);
    out.batch = x.batch;
    out.scale = P.acc_scale / double(ql);
    out.noise_bound = P.acc_noise / double(ql) + 1.0;
    out.domain = x.domain;
    out.sk_id = x.sk_id;
    return out;
}

Ciphertext run_combine(const CombPlan& P, Ladder& L, const Ciphertext& x) {
    const RingParams& R = L.R;
    const int lvl = P.lvl;
    const std::vector<LinTerm>& terms = P.terms;
    std::vector<Poly> parts;
    if (terms.size() <= TG_LINCOMB_MAX_TERMS) {
        parts = fused_lincomb(R, terms, P.add, lvl, true);
    } else {  // more terms than one pass holds: accumulate in chunks, rescale at the end
        Ciphertext partial;
        const std::vector<u64> one = residues_of(R, 1, lvl);
        const std::size_t step = TG_LINCOMB_MAX_TERMS - 1;
        for (std::size_t i = 0; i < terms.size(); i += step) {
            std::vector<LinTerm> chunk;
            if (i) chunk.push_back(LinTerm{&partial, one});
            for (std::size_t j = i; j < std::min(terms.size(), i + step); ++j) chunk.push_back(terms[j]);
            const bool last = i + step >= terms.size();
            Ciphertext next;
            next.batch = x.batch;
            next.parts = fused_lincomb(R, chunk, last ? P.add : std::vector<u64>{}, lvl, last);
            next.scale = P.acc_scale;
            partial = std::move(next);
        }
        parts = partial.parts;
    }
    return finish_combine(P, R, x, std::move(parts));
}

Ciphertext combine(Ladder& L, const Ciphertext& x, const std::vector<std::size_t>& ks, const std::vector<double>& cs,
                   double c0, double target = 0.0) {
    CombPlan P;
    plan_combine(P, L, x, ks, cs, c0, target);
    return run_combine(P, L, x);
}

// Several combination steps over the SAME terms at one level (the base blocks
// of one BSGS polynomial) in one residue pass: each term word is read once
// for all outputs (tg_lincomb_multi). Coefficient form, FP64-eligible rows,
// 1..4 uniformly strided terms; 2..4 plans per call.
bool multi_ok(const RingParams& R, const CombPlan& a, const CombPlan& b) {
    if (a.lvl != b.lvl || a.ks != b.ks || a.terms.size() > 4 || !a.conv.empty() || !b.conv.empty()) return false;
    for (int r = 0; r <= a.lvl; ++r)
        if (R.modulus(u32(r)) >= 1351079888211148ull) return false;  // kFpMaxQ (tg_fp64.cuh)
    for (const LinTerm& t : a.terms) {
        const Ciphertext& c = *t.ct;
        if (c.form() != Form::coeff || !uniform_parts(c.parts) || c.parts[0].nspecial() != 0) return false;
    }
    return true;
}

std::vector<Ciphertext> run_combine_multi(const std::vector<const CombPlan*>& plans, Ladder& L, const Ciphertext& x) {
    const RingParams& R = L.R;
    const CombPlan& P0 = *plans[0];
    const int lvl = P0.lvl;
    const u32 nt = u32(P0.terms.size()), no = u32(plans.size()), B = x.batch;
    const std::size_t rows = std::size_t(lvl) + 1;
    std::vector<const u64*> ptrs(nt);
    std::vector<u64> strides(nt), coeffs(std::size_t(no) * nt * rows), adds(std::size_t(no) * rows, 0);
    for (u32 t = 0; t < nt; ++t) {
        const Ciphertext& c = *P0.terms[t].ct;
        if (c.batch != B || c.parts.size() != 2 * B) throw TetrisError("ckks", "fused combination expects degree-1 terms");
        ptrs[t] = c.parts[0].data();
        strides[t] = u64(c.parts[1].data()) / 8 - u64(c.parts[0].data()) / 8;
    }
    bool any_add = false;
    std::vector<std::vector<Poly>> outs(no);
    std::vector<u64*> optr(no);
    for (u32 o = 0; o < no; ++o) {
        const CombPlan& P = *plans[o];
        for (u32 t = 0; t < nt; ++t)
            for (std::size_t r = 0; r < rows; ++r) coeffs[(std::size_t(o) * nt + t) * rows + r] = P.terms[t].coef[r];
        if (!P.add.empty()) {
            any_add = true;
            for (std::size_t r = 0; r < rows; ++r) adds[std::size_t(o) * rows + r] = P.add[r];
        }
        outs[o] = fresh_parts(R, int(2 * B), lvl - 1, Form::coeff);
        optr[o] = const_cast<u64*>(outs[o][0].data());
    }
    check_tg(tg_lincomb_multi(R.dev(), no, optr.data(), nt, ptrs.data(), strides.data(), coeffs.data(),
                              any_add ? adds.data() : nullptr, lvl, 2 * B, B, R.stream()));
    std::vector<Ciphertext> res;
    for (u32 o = 0; o < no; ++o) res.push_back(finish_combine(*plans[o], R, x, std::move(outs[o])));
    return res;
}

std::vector<double> trimmed(const std::vector<double>& c) {
    std::vector<double> v = c;
    while (v.size() > 1 && v.back() == 0.0) v.pop_back();
    return v;
}

}  // namespace

void set_eval_pipeline(bool on) { g_eval_pipeline.store(on ? 1 : 0); }
bool eval_pipeline_enabled() { return eval_pipeline(); }
void set_lazy_relin(bool on) { g_lazy_relin.store(on ? 1 : 0); }
bool lazy_relin_enabled() { return lazy_relin(); }

Ciphertext eval_chebyshev(const Evaluator& ev, const Ciphertext& x, const std::vector<double>& cheb_coeffs,
                          const EvalKeys& keys) {
    std::size_t d = cheb_coeffs.size() - 1;
    while (d > 0 && cheb_coeffs[d] == 0.0) --d;
    if (d == 0) {
        Ciphertext out = ev.mul_scalar(x, 0.0, 1.0);
        return ev.add_scalar(out, cheb_coeffs[0]);
    }
    if (x.level() < int(std::ceil(std::log2(double(d)))) + 1)
        throw TetrisError("ckks", "insufficient levels for polynomial evaluation");
    Ladder L(ev, x, keys);
    for (std::size_t k = d; k >= 1; k /= 2) L.get(k);  // warm the ladder top-down
    std::vector<std::size_t> ks;
    for (std::size_t k = 1; k <= d; ++k)
        if (cheb_coeffs[k] != 0.0) {
            L.get(k);
            ks.push_back(k);
        }
    return L.finish(combine(L, x, ks, cheb_coeffs, cheb_coeffs[0]));
}

Ciphertext eval_chebyshev_bsgs(const Evaluator& ev, const Ciphertext& x, const std::vector<double>& cheb_coeffs,
                               const EvalKeys& keys) {
    const std::vector<double> c = trimmed(cheb_coeffs);
    const std::size_t d = c.size() - 1;
    if (d == 0) {
        Ciphertext out = ev.mul_scalar(x, 0.0, 1.0);
        return ev.add_scalar(out, c[0]);
    }
    if (x.level() < int(std::ceil(std::log2(double(d)))) + 1)
        throw TetrisError("ckks", "insufficient levels for polynomial evaluation");
    const int lb = int(std::ceil(std::log2(double(d + 1)) / 2.0));
    const std::size_t b = std::size_t(1) << lb;
    Ladder L(ev, x, keys);
    const bool lazy = lazy_relin();

    auto base_terms = [&](const std::vector<double>& cs) {
        std::vector<std::size_t> ks;
        for (std::size_t k = 1; k < cs.size(); ++k)
            if (cs[k] != 0.0) ks.push_back(k);
        return ks;
    };
    // Chebyshev division at the largest giant n <= deg: cs = q * T_n + r
    auto split = [&](const std::vector<double>& cs, std::vector<double>& q, std::vector<double>& r) {
        const std::size_t m = cs.size() - 1;
        std::size_t n = b;
        while (2 * n <= m) n *= 2;
        q.assign(m - n + 1, 0.0);
        r.assign(cs.begin(), cs.begin() + n);
        q[0] = cs[n];
        for (std::size_t i = 1; i <= m - n; ++i) q[i] = 2.0 * cs[n + i];
        for (std::size_t i = 1; i <= m - n; ++i) r[n - i] = r[n - i] - cs[n + i];
        return n;
    };
    auto all_zero = [](const std::vector<double>& cs) {
        for (double v : cs)
            if (v != 0.0) return false;
        return true;
    };
    // output level of rec(cs) (levels do not depend on scales); -1: zero block
    std::function<int(std::vector<double>)> level_of = [&](std::vector<double> cs) -> int {
        cs = trimmed(cs);
        if (all_zero(cs)) return -1;
        if (cs.size() - 1 < b) {
            std::vector<std::size_t> ks = base_terms(cs);
            if (ks.empty()) ks = {1};
            int lvl = x.level();
            for (std::size_t k : ks) lvl = std::min(lvl, L.get(k).level());
            return lvl - 1;
        }
        std::vector<double> q, r;
        const std::size_t n = split(cs, q, r);
        const int lq = level_of(q), lr = level_of(r);
        if (lq < 0) return lr;
        const int lp = std::min(lq, L.get(n).level()) - 1;
        return lr < 0 ? lp : std::min(lp, lr);
    };

    // Two passes over the same recursion when base blocks are batched
    // (multi_base): the PLAN pass walks the tree without evaluating any
    // product and records every base block's combination step (its constants
    // depend only on the ladder's scales and levels); the blocks sharing
    // their terms and level are then evaluated together, one read of the baby
    // steps for up to four blocks (tg_lincomb_multi); the EXEC pass consumes
    // them in the same order.
    bool plan = false;
    std::deque<CombPlan> plans;
    std::vector<Ciphertext> ready;
    std::size_t next_ready = 0;
    const Ciphertext dummy;
    auto base = [&](const std::vector<double>& cs, double target) -> Ciphertext {
        if (!plan && next_ready < ready.size()) return ready[next_ready++];
        std::vector<std::size_t> ks = base_terms(cs);
        std::vector<double> z = cs;
        if (ks.empty()) {  // constant block: carried by 0 * T_1
            z = {cs[0], 0.0};
            ks = {1};
        }
        for (std::size_t k : ks) L.get(k);
        if (plan) {
            plans.emplace_back();
            plan_combine(plans.back(), L, x, ks, z, cs[0], target);
            return dummy;
        }
        return combine(L, x, ks, z, cs[0], target);
    };

    // the block evaluated at output scale `target`: blocks land exactly on the
    // scale their consumer needs (the output on scale(x), like the ladder's;
    // each quotient on target * q_lp / scale(T_n) so Q * T_n rescales onto
    // target), so deep chains keep matching scales (oracle/bsgs_ref.py)
    std::function<std::optional<Ciphertext>(std::vector<double>, double)> rec =
        [&](std::vector<double> cs, double target) -> std::optional<Ciphertext> {
        cs = trimmed(cs);
        if (all_zero(cs)) return std::nullopt;
        if (cs.size() - 1 < b) return base(cs, target);
        std::vector<double> q, r;
        const std::size_t n = split(cs, q, r);
        const int lq = level_of(q);
        std::optional<Ciphertext> Q;
        if (lq >= 0) {
            const Ciphertext& tn = L.get(n);
            const int lp = std::min(lq, tn.level());
            Q = rec(q, target * double(L.R.modulus(u32(lp))) / tn.scale);
            // lazy relinearisation: the remainder is a giant-step node too,
            // Q T_n + (Q2 T_n2 + R2): both tensors at one scale and level, one
            // key switch and one rescale for the pair (oracle/bsgs_ref.py)
            const std::vector<double> rt = trimmed(r);
            if (lazy && !L.eval && rt.size() - 1 >= b) {
                std::vector<double> q2, r2;
                const std::size_t n2 = split(rt, q2, r2);
                const int lq2 = level_of(q2);
                if (lq2 >= 0 && std::min(lq2, L.get(n2).level()) >= lp) {
                    const Ciphertext& tn2 = L.get(n2);
                    std::optional<Ciphertext> Q2 = rec(q2, target * double(L.R.modulus(u32(lp))) / tn2.scale);
                    std::optional<Ciphertext> R2 = rec(r2, target);
                    if (plan) return dummy;
                    return ev.mul2_relin_rescale(*Q, L.get(n), *Q2, tn2, keys, R2 ? &*R2 : nullptr);
                }
            }
        }
        std::optional<Ciphertext> Rr = rec(r, target);
        if (!Q) return Rr;
        if (plan) return dummy;
        if (!L.eval) {  // add(rescale(Q T_n), R) in one pass (Evaluator::rescale_add)
            if (!Rr) return ev.mul_relin_rescale(*Q, L.get(n), keys);
            return ev.mul_relin_rescale(*Q, L.get(n), keys, &*Rr);
        }
        Ciphertext P = ev.rescale_eval(ev.mul_relin_eval(*Q, L.get(n), keys));
        if (!Rr) return P;
        // Evaluator::add in eval form: level alignment drops rows in place
        Ciphertext y = *Rr;
        Evaluator::check_scales_match(P.scale, y.scale);
        const int lvl = std::min(P.level(), y.level());
        P.drop_to_level(lvl);
        y.drop_to_level(lvl);
        P.add_inplace(y);
        return P;
    };
    if (!L.eval && multi_base()) {
        plan = true;
        rec(c, x.scale);
        plan = false;
        // groups of up to four blocks over the same terms and level
        ready.resize(plans.size());
        std::vector<char> done(plans.size(), 0);
        for (std::size_t i = 0; i < plans.size(); ++i) {
            if (done[i]) continue;
            std::vector<std::size_t> grp = {i};
            for (std::size_t j = i + 1; j < plans.size() && grp.size() < 4; ++j)
                if (!done[j] && multi_ok(L.R, plans[i], plans[j])) grp.push_back(j);
            if (grp.size() == 1) {
                ready[i] = run_combine(plans[i], L, x);
                done[i] = 1;
                continue;
            }
            std::vector<const CombPlan*> ps;
            for (std::size_t j : grp) ps.push_back(&plans[j]);
            std::vector<Ciphertext> outs = run_combine_multi(ps, L, x);
            for (std::size_t k = 0; k < grp.size(); ++k) {
                ready[grp[k]] = std::move(outs[k]);
                done[grp[k]] = 1;
            }
        }
    }
    std::optional<Ciphertext> out = rec(c, x.scale);
    if (!out) return ev.add_scalar(ev.mul_scalar(x, 0.0, 1.0), 0.0);
    return L.finish(*out);
}

}  // namespace tetris_b200
