// PFE scoring, repacking and ring merge/split (reference pfe.hpp,
// repack.hpp, rlwe.hpp:684-802) over the device kernels. Control flow,
// metadata (scale, noise bound, key ids) and checks follow the reference.
#include <cmath>

#include "internal.hpp"
#include "tetris_b200/pfe.hpp"

namespace tetris_b200 {

using detail::fresh_parts;

// ---------------------------------------------------------------------------
// PFE
// ---------------------------------------------------------------------------
double FunctionSpec::max_value() const {
    double m = table.empty() ? 0 : table[0];
    for (double v : table) m = std::max(m, v);
    return m;
}

void FunctionSpec::validate(u32 ring_degree) const {
    if (!(lo < hi)) throw TetrisError("pfe", "empty function domain");
    if (table.size() != ring_degree) throw TetrisError("pfe", "table length must equal the ring degree");
    for (double v : table)
        if (!std::isfinite(v)) throw TetrisError("pfe", "non-finite table entry");
}

u32 encode_input(double x, double a, double b, u32 n) {
    if (!(x >= a && x < b)) throw TetrisError("pfe", "input outside the function domain");
    const double g = (x - a) / (b - a);
    i64 i = round_half_away(double(n) * g);
    if (i >= i64(n)) i = i64(n) - 1;  // rounding up to n would wrap to -f(grid 0)
    if (i < 0) i = 0;
    return u32(i);
}

TestVector build_test_vector(const KeyContext& ctx, const FunctionSpec& spec, const SecretKey& sk, double scale,
                             Rng& rng) {
    const RingParams& ring = ctx.ring();
    const u32 n = ring.degree();
    spec.validate(n);
    std::vector<i64> u(n);
    u[0] = round_half_away(spec.table[0] * scale);
    for (u32 i = 1; i < n; ++i) u[i] = -round_half_away(spec.table[n - i] * scale);
    Poly m = poly_from_i64(ring, u, 0);
    TestVector tv;
    tv.ct = ctx.encrypt(sk, m, scale, rng, Domain::coeffs);
    tv.lo = spec.lo;
    tv.hi = spec.hi;
    tv.max_value = spec.max_value();
    return tv;
}

Ciphertext lookup(const TestVector& tv, u32 exponent) {
    Ciphertext out = tv.ct;
    for (auto& p : out.parts) p = mul_monomial(p, exponent);
    return out;
}

std::vector<Ciphertext> eval_scores(const std::vector<std::vector<double>>& rows, const std::vector<TestVector>& tvs,
                                    std::vector<std::string>* op_trace) {
    if (tvs.empty()) throw TetrisError("pfe", "no scoring functions");
    const RingParams& ring = tvs[0].ct.ring();
    const u32 n = ring.degree();
    const u32 ncols = u32(tvs.size());
    std::vector<u32> exps;
    exps.reserve(rows.size() * ncols);
    for (std::size_t r = 0; r < rows.size(); ++r) {
        if (rows[r].size() != tvs.size())
            throw TetrisError("pfe", "row " + std::to_string(r) + " has " + std::to_string(rows[r].size()) +
                                         " attributes, expected " + std::to_string(tvs.size()));
        for (std::size_t c = 0; c < tvs.size(); ++c) {
            u32 idx;
            try {
                idx = encode_input(rows[r][c], tvs[c].lo, tvs[c].hi, n);
            } catch (const TetrisError&) {
                throw TetrisError("pfe", "attribute out of domain at row " + std::to_string(r) + ", column " +
                                             std::to_string(c));
            }
            if (op_trace) op_trace->push_back("rot " + std::to_string(c) + ":" + std::to_string(idx));
            if (c > 0 && op_trace) op_trace->push_back("add");
            exps.push_back(idx);
        }
    }
    if (rows.empty()) return {};
    // shapes: every test vector a degree-1 coefficient-form ciphertext of one level
    const Ciphertext& t0 = tvs[0].ct;
    double noise = 0;
    std::vector<Poly> keep;
    std::vector<const u64*> ptrs;
    for (const auto& tv : tvs) {
        if (tv.ct.parts.size() != 2 || tv.ct.batch != 1) throw TetrisError("rlwe", "ciphertext degree mismatch");
        for (const auto& p : tv.ct.parts) {
            if (p.form() != Form::coeff) throw TetrisError("ring", "mul_monomial expects coeff form");
            p.check_shape(t0.parts[0]);
        }
        if (tv.ct.domain != t0.domain) throw TetrisError("rlwe", "domain tag mismatch");
        ptrs.push_back(detail::group_data(tv.ct.parts, 0, 2, keep));
        noise += tv.ct.noise_bound;
    }
    const int lvl = t0.level();
    const u32 nrows = u32(rows.size());
    std::vector<Poly> out = fresh_parts(ring, int(2 * nrows), lvl, Form::coeff);
    DeviceBuffer d_exps(ring, (exps.size() + 1) / 2);
    check_tg(tg_memcpy_h2d(ring.dev(), d_exps.data(), exps.data(), exps.size() * 4, ring.stream()));
    check_tg(tg_pfe_eval(ring.dev(), const_cast<u64*>(out[0].data()), ptrs.data(), ncols,
                         reinterpret_cast<const u32*>(d_exps.data()), nrows, lvl, ring.stream()));
    std::vector<Ciphertext> cts(nrows);
    for (u32 r = 0; r < nrows; ++r) {
        cts[r].parts = {out[2 * r], out[2 * r + 1]};
        cts[r].scale = t0.scale;
        cts[r].domain = t0.domain;
        cts[r].sk_id = t0.sk_id;
        cts[r].noise_bound = noise;
    }
    return cts;
}

// ---------------------------------------------------------------------------
// Repacking
// ---------------------------------------------------------------------------
const SwitchingKey& RepackKeySet::key(u64 exponent) const {
    auto it = keys.find(exponent);
    if (it == keys.end()) throw TetrisError("repack", "missing repack key");
    return it->second;
}

std::vector<u64> repack_exponents(const RingParams& ring) {
    const u32 n = ring.degree();
    const u64 two_n = 2 * u64(n);
    std::vector<u64> exps{two_n - 1};
    for (u32 i = 1; i < ring.log_degree(); ++i) exps.push_back(pow_mod(5, 1ULL << (i - 1), two_n));
    return exps;
}

RepackKeySet gen_repack_keys(const KeyContext& ctx, const SecretKey& sk, Rng& rng) {
    RepackKeySet set;
    set.sk_id = sk.id();
    set.exponents = repack_exponents(ctx.ring());
    for (std::size_t i = 0; i < set.exponents.size(); ++i) {
        const u64 g = set.exponents[i];
        if (set.keys.count(g)) continue;
        Rng ri = rng.split(i);
        set.keys.emplace(g, ctx.galois_key_gen(sk, g, ri));
    }
    return set;
}

// The butterfly with every round as ONE ciphertext batch: slots [0, t) and
// [t, 2t) of the state are combined by batched monomial shifts, adds, subs
// and a batched automorphism + key switch (one key per round). Absent inputs
// are exact zero ciphertexts, which every step maps to zero, so the live
// slots carry the reference's residues; liveness and noise bounds are tracked
// on the host exactly as the reference's per-pair loop does.
Ciphertext repack(const KeyContext& ctx, const std::vector<const Ciphertext*>& cts, const RepackKeySet& keys,
                  RepackStats* stats) {
    const RingParams& ring = ctx.ring();
    const u32 n = ring.degree();
    if (cts.size() > n) throw TetrisError("repack", "more inputs than ring coefficients");
    const Ciphertext* first = nullptr;
    for (auto* c : cts)
        if (c) {
            first = c;
            break;
        }
    if (!first) throw TetrisError("repack", "all-zero repack batch");
    const int lvl = first->level();
    const double scale = first->scale;
    for (auto* c : cts) {
        if (!c) continue;
        if (c->level() != lvl) throw TetrisError("repack", "repack inputs at mixed levels");
        if (c->scale != scale) throw TetrisError("repack", "repack inputs at mixed scales");
        if (c->degree() != 1 || c->batch != 1)
            throw TetrisError("repack", "repack inputs must be single degree-1 ciphertexts");
        // the butterfly adds every live input into slot 0, where the reference
        // throws on the first domain mismatch (rlwe.hpp:302-309); inputs under
        // different secret keys have no meaningful repacking (the reference
        // key-switches them with one key set regardless) and are refused
        if (c->domain != first->domain) throw TetrisError("rlwe", "domain tag mismatch");
        if (c->sk_id != first->sk_id) throw TetrisError("repack", "repack inputs under different secret keys");
    }
    if (ring.log_degree() == 0) throw TetrisError("repack", "ring degree 1 has no repacking butterfly");
    std::vector<u64> n_inv(ring.moduli().size());
    for (std::size_t i = 0; i < n_inv.size(); ++i) n_inv[i] = inv_mod(n, ring.moduli()[i]);

    // state: n slots, part-major, zeros where absent
    const std::size_t w = std::size_t(lvl + 1) * n;
    std::vector<Poly> parts = fresh_parts(ring, int(2 * n), lvl, Form::coeff);
    check_tg(tg_memset0(ring.dev(), const_cast<u64*>(parts[0].data()), 2 * n * w * 8, ring.stream()));
    std::vector<bool> live(n, false);
    std::vector<double> noise(n, 0.0);
    for (std::size_t i = 0; i < cts.size(); ++i) {
        if (!cts[i]) continue;
        Ciphertext c = *cts[i];
        c.to_coeff();
        for (int part = 0; part < 2; ++part)
            check_tg(tg_memcpy_d2d(ring.dev(), const_cast<u64*>(parts[part * n + i].data()), c.parts[part].data(),
                                   w * 8, ring.stream()));
        live[i] = true;
        noise[i] = c.noise_bound;
    }
    Ciphertext state;
    state.parts = std::move(parts);
    state.batch = n;
    state.scale = scale;
    state.domain = first->domain;
    state.sk_id = first->sk_id;
    {  // x n^-1: the per-round doublings cancel (one launch for all slots)
        std::vector<Poly> scaled = fresh_parts(ring, int(2 * n), lvl, Form::coeff);
        check_tg(tg_poly_mul_scalar(ring.dev(), const_cast<u64*>(scaled[0].data()), state.parts[0].data(),
                                    n_inv.data(), lvl, 0, 2 * n, ring.stream()));
        state.parts = std::move(scaled);
    }
    const double ks_noise = ctx.ks_noise_estimate();
    for (u32 round = 0; round < ring.log_degree(); ++round) {
        const u32 t = n >> (round + 1);
        const u64 g = keys.exponents[round];
        const SwitchingKey& swk = keys.key(g);
        for (u32 j = 0; j < t; ++j) {  // the reference's bookkeeping
            const bool lj = live[j], lh = live[j + t];
            if (!lj && !lh) continue;
            const double dn = (lj ? noise[j] : 0.0) + (lh ? noise[j + t] : 0.0);
            noise[j] = dn + (dn + ks_noise);  // sum + rotated(diff)
            live[j] = true;
            if (stats) ++stats->automorphisms;
        }
        Ciphertext a = slice_ciphertext(state, 0, t);
        Ciphertext h = slice_ciphertext(state, t, t);
        std::vector<Poly> sh = fresh_parts(ring, int(2 * t), lvl, Form::coeff);
        check_tg(tg_mul_monomial(ring.dev(), const_cast<u64*>(sh[0].data()), h.parts[0].data(), t, lvl, 0, 2 * t,
                                 ring.stream()));
        h.parts = std::move(sh);
        Ciphertext sum = a, diff = a;
        sum.add_inplace(h);
        diff.sub_inplace(h);
        Ciphertext rotated = ctx.apply_galois(diff, g, swk);
        sum.add_inplace(rotated);
        state = std::move(sum);
    }
    state.batch = 1;  // one slot left
    state.noise_bound = noise[0];
    return state;
}

// ---------------------------------------------------------------------------
// Ring merge / split
// ---------------------------------------------------------------------------
SecretKey embed_secret(const SecretKey& small_sk, const RingParams& big, u32 stride) {
    const u32 n_small = small_sk.ring().degree();
    if (n_small * stride != big.degree()) throw TetrisError("rlwe", "embed_secret stride mismatch");
    std::vector<i64> c(big.degree(), 0);
    for (u32 i = 0; i < n_small; ++i) c[std::size_t(i) * stride] = small_sk.coeffs()[i];
    return SecretKey(big, std::move(c), splitmix64(small_sk.id() ^ (0x37ULL + stride)));
}

Ciphertext merge_embed(const std::vector<const Ciphertext*>& cts, const RingParams& big) {
    const std::size_t count = cts.size();
    const Ciphertext* first = nullptr;
    for (auto* c : cts)
        if (c) {
            first = c;
            break;
        }
    if (!first) throw TetrisError("rlwe", "merge_embed needs at least one ciphertext");
    const RingParams& small = first->ring();
    const u32 stride = big.degree() / small.degree();
    if (stride * small.degree() != big.degree() || count > stride)
        throw TetrisError("rlwe", "merge arity exceeds degree ratio");
    const int lvl = first->level();
    for (auto* c : cts)
        if (c && (c->level() != lvl || c->scale != first->scale))
            throw TetrisError("rlwe", "merge inputs must share level and scale");
    Ciphertext out;
    out.scale = first->scale;
    out.domain = Domain::coeffs;
    out.sk_id = 0;  // under the embedded secret until keyswitched
    std::vector<Ciphertext> src(count);
    std::vector<u64> ptrs(2 * count, 0);
    for (std::size_t i = 0; i < count; ++i) {
        if (!cts[i]) continue;
        src[i] = *cts[i];
        src[i].to_coeff();
        out.noise_bound += src[i].noise_bound;
        for (int part = 0; part < 2; ++part) ptrs[part * count + i] = u64(src[i].parts[part].data());
    }
    small.synchronize();  // the big ring's stream reads the small ring's buffers
    std::vector<Poly> parts = fresh_parts(big, 2, lvl, Form::coeff);
    DeviceBuffer d_ptrs(big, ptrs.size());
    check_tg(tg_memcpy_h2d(big.dev(), d_ptrs.data(), ptrs.data(), ptrs.size() * 8, big.stream()));
    for (int part = 0; part < 2; ++part)
        check_tg(tg_interleave(const_cast<u64*>(parts[part].data()),
                               reinterpret_cast<const u64* const*>(d_ptrs.data() + part * count), u32(count), stride,
                               small.degree(), u64(lvl + 1), big.stream()));
    big.synchronize();  // the small inputs may be released after return
    out.parts = std::move(parts);
    return out;
}

static Ciphertext merge_keyswitch(const KeyContext& big_ctx, Ciphertext emb, const SwitchingKey& swk) {
    auto [d0, d1] = big_ctx.switch_key_apply(emb.parts[1], swk);
    emb.parts[0].add_inplace(d0);
    emb.parts[1] = std::move(d1);
    emb.sk_id = swk.to_id;
    emb.noise_bound += big_ctx.ks_noise_estimate();
    return emb;
}

Ciphertext ring_merge(const KeyContext& big_ctx, const Ciphertext& ct0, const Ciphertext& ct1,
                      const SwitchingKey& swk) {
    if (ct0.level() != ct1.level()) throw TetrisError("rlwe", "ring_merge level mismatch");
    return merge_keyswitch(big_ctx, merge_embed({&ct0, &ct1}, big_ctx.ring()), swk);
}

Ciphertext ring_merge_many(const KeyContext& big_ctx, const std::vector<const Ciphertext*>& cts,
                           const SwitchingKey& swk) {
    return merge_keyswitch(big_ctx, merge_embed(cts, big_ctx.ring()), swk);
}

std::pair<Ciphertext, Ciphertext> ring_split(const KeyContext& big_ctx, const RingParams& small, const Ciphertext& ct,
                                             const SwitchingKey& swk_to_embed, u64 small_sk_id) {
    const RingParams& big = big_ctx.ring();
    if (small.degree() * 2 != big.degree()) throw TetrisError("rlwe", "ring_split expects a half-degree target");
    Ciphertext src = ct;
    src.to_coeff();
    auto [d0, d1] = big_ctx.switch_key_apply(src.parts[1], swk_to_embed);
    d0.add_inplace(src.parts[0]);  // (d0, d1) now under s_small(X^2): de-interleave
    const int lvl = src.level();
    big.synchronize();
    auto extract = [&](const Poly& p, u32 parity) {
        std::vector<Poly> o = fresh_parts(small, 1, lvl, Form::coeff);
        check_tg(tg_deinterleave(const_cast<u64*>(o[0].data()), p.data(), parity, 2, small.degree(), u64(lvl + 1),
                                 small.stream()));
        return o[0];
    };
    Ciphertext even, odd;
    even.parts = {extract(d0, 0), extract(d1, 0)};
    odd.parts = {extract(d0, 1), extract(d1, 1)};
    small.synchronize();
    for (Ciphertext* c : {&even, &odd}) {
        c->scale = ct.scale;
        c->domain = Domain::coeffs;
        c->sk_id = small_sk_id;
        c->noise_bound = ct.noise_bound + big_ctx.ks_noise_estimate();
    }
    return {std::move(even), std::move(odd)};
}

}  // namespace tetris_b200
