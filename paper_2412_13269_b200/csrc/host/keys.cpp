// RLWE layer: gadget plan, keys, encryption, key switching, relinearisation,
// Galois automorphisms (reference rlwe.hpp:16-682). Sampling happens on the
// host in the reference's exact draw order; every polynomial product, NTT and
// base conversion runs on the GPU.
#include <cmath>

#include "internal.hpp"

namespace tetris_b200 {

using detail::contiguous;
using detail::exclusively_owned;
using detail::fresh_parts;
using detail::new_block;
using detail::tg_form;

// ---------------------------------------------------------------------------
// GadgetVector / GadgetPlan (rlwe.hpp:16-206)
// ---------------------------------------------------------------------------
u32 GadgetVector::sub_digits(u64 q) const {
    if (base2_bits == 0) return 1;
    u32 bits = 0;
    while ((q >> bits) != 0) ++bits;
    return (bits + base2_bits - 1) / base2_bits;
}

GadgetPlan::GadgetPlan(const RingParams& ring, GadgetVector cfg) : ring_(&ring), cfg_(cfg) {
    if (cfg_.group_size == 0) throw TetrisError("rlwe", "gadget group size must be positive");
    if (cfg_.base2_bits != 0 && cfg_.group_size != 1)
        throw TetrisError("rlwe", "base2 refinement requires single-prime groups");
}

GadgetPlan::~GadgetPlan() {
    if (dev_) tg_gadget_destroy(dev_);
}

tg_gadget* GadgetPlan::dev() const {
    std::call_once(once_, [this] {
        tg_gadget* g = nullptr;
        devstate_ = ring_->device_state();
        check_tg(tg_gadget_create(&g, devstate_->ctx, cfg_.group_size, cfg_.base2_bits));
        dev_ = g;
    });
    if (!dev_) throw TetrisError("gpu", "gadget tables unavailable");
    return dev_;
}

u32 GadgetPlan::digit_count(int level) const {
    u32 n = 0;
    for (u32 j = 0; j < group_count(level); ++j)
        n += cfg_.base2_bits ? cfg_.sub_digits(ring_->modulus(j * cfg_.group_size)) : 1;
    return n;
}

std::vector<Poly> GadgetPlan::decompose(const Poly& d) const {
    if (d.form() != Form::coeff || d.nspecial() != 0)
        throw TetrisError("rlwe", "decompose expects coeff form without special rows");
    const int level = d.level(), k = int(ring_->special_count());
    const u32 nd = digit_count(level);
    std::vector<Poly> digits = fresh_parts(*ring_, int(nd), level, Form::eval, k);
    u64* base = const_cast<u64*>(digits[0].data());  // fresh block, exclusively ours
    check_tg(tg_modup(dev(), base, d.data(), level, ring_->stream()));
    return digits;
}

std::vector<std::vector<u64>> GadgetPlan::key_scalars() const {
    const u32 nq = ring_->q_count(), nmod = u32(ring_->moduli().size()), gs = cfg_.group_size;
    const u32 ngroups = (nq + gs - 1) / gs;
    std::vector<std::vector<u64>> out;
    for (u32 j = 0; j < ngroups; ++j) {
        const u32 first = j * gs, count = std::min(gs, nq - first);
        const u32 nsub = cfg_.base2_bits ? cfg_.sub_digits(ring_->modulus(first)) : 1;
        for (u32 s = 0; s < nsub; ++s) {
            std::vector<u64> row(nmod, 0);
            for (u32 t = first; t < first + count; ++t) {  // Dhat = 0 outside the group, P = 0 mod specials
                const u64 qt = ring_->modulus(t);
                u64 p_mod = 1;
                for (u32 sp = 0; sp < ring_->special_count(); ++sp)
                    p_mod = mul_mod(p_mod, ring_->modulus(nq + sp) % qt, qt);
                row[t] = mul_mod(pow_mod(2, u64(s) * cfg_.base2_bits, qt), p_mod, qt);
            }
            out.push_back(std::move(row));
        }
    }
    return out;
}

// ---------------------------------------------------------------------------
// Keys (rlwe.hpp:212-267)
// ---------------------------------------------------------------------------
SecretKey::SecretKey(const RingParams& ring, const NoiseParams& noise, Rng& rng)
    : ring_(&ring), hamming_weight_(noise.secret_hamming_weight) {
    id_ = splitmix64(rng.next());  // drawn before the ternary sample, as the reference's member init
    coeffs_ = sample_ternary_coeffs(ring.degree(), hamming_weight_, rng);
    eval_full_ = poly_from_i64(ring, coeffs_, ring.max_level(), int(ring.special_count()));
    eval_full_.ntt_forward();
}

SecretKey::SecretKey(const RingParams& ring, std::vector<i64> coeffs, u64 id)
    : ring_(&ring), id_(id), coeffs_(std::move(coeffs)) {
    hamming_weight_ = 0;
    for (i64 c : coeffs_) hamming_weight_ += c != 0;
    eval_full_ = poly_from_i64(ring, coeffs_, ring.max_level(), int(ring.special_count()));
    eval_full_.ntt_forward();
}

Poly SecretKey::shaped(int level, int nspecial) const {
    Poly out(*ring_, level, Form::eval, nspecial);
    const std::size_t n = ring_->degree();
    u64* dst = out.mutable_data();
    const u64* src = eval_full_.data();
    check_tg(tg_memcpy_d2d(ring_->dev(), dst, src, std::size_t(level + 1) * n * 8, ring_->stream()));
    if (nspecial)
        check_tg(tg_memcpy_d2d(ring_->dev(), dst + std::size_t(level + 1) * n,
                               src + std::size_t(ring_->max_level() + 1) * n, std::size_t(nspecial) * n * 8,
                               ring_->stream()));
    return out;
}

// ---------------------------------------------------------------------------
// Ciphertext (rlwe.hpp:287-317)
// ---------------------------------------------------------------------------
// Parts that share one block at a uniform stride S (a contiguous block, or
// one whose level was dropped: each part is then a row prefix of an S-word
// poly). Returns S in words, 0 if the parts are not laid out that way.
std::size_t detail::uniform_stride(const std::vector<Poly>& parts) {
    const Poly& p0 = parts[0];
    const std::size_t n = p0.ring().degree();
    std::size_t S = p0.words();
    if (parts.size() > 1) S = parts[1].offset() - p0.offset();
    if (S < p0.words() || S % n != 0) return 0;
    // a level-dropped view: the stride is a poly of some level of this ring
    if (S / n > std::size_t(p0.ring().q_count()) + std::size_t(p0.nspecial())) return 0;
    for (std::size_t i = 0; i < parts.size(); ++i) {
        const Poly& p = parts[i];
        if (p.storage() != p0.storage() || p.level() != p0.level() || p.nspecial() != p0.nspecial() ||
            p.form() != p0.form() || p.offset() != p0.offset() + i * S)
            return 0;
    }
    if (p0.offset() + parts.size() * S > p0.storage()->words()) return 0;
    return S;
}

// Transforms all parts in as few launches as possible. Parts on a uniform
// stride are transformed as full S-word polys (rows beyond a dropped level
// included: the NTT is row-wise, so the prefix rows are exactly the dropped
// poly's transform). A shared block's forward transform is memoised on the
// block, so ladder operands used several times (squares included) are
// transformed once.
static void transform_parts(Ciphertext& ct, Form target, bool keep_eval = false) {
    const Form from = target == Form::eval ? Form::coeff : Form::eval;
    bool any = false;
    for (auto& p : ct.parts) any |= p.form() == from;
    if (!any) return;
    const std::size_t np = ct.parts.size();
    const std::size_t S = detail::uniform_stride(ct.parts);
    if (S) {
        const Poly& p0 = ct.parts[0];
        const RingParams& ring = p0.ring();
        const int ns = p0.nspecial(), lvl = p0.level();
        const int full_level = int(S / ring.degree()) - 1 - ns;
        const bool own = p0.storage().use_count() == long(np);
        std::shared_ptr<DeviceBuffer> out_blk;
        std::size_t out_off = 0;
        if (!own && target == Form::eval)
            out_blk = p0.storage()->find_eval(p0.offset(), full_level, ns, int(np), ring.stream());
        if (!out_blk) {
            if (own) {  // transformed in place: drop memoised transforms of the old contents
                out_blk = p0.storage();
                out_off = p0.offset();
                out_blk->clear_eval_cache();
            } else {
                out_blk = detail::new_block(ring, S * np);
            }
            u64* dst = out_blk->data() + out_off;
            if (target == Form::eval)
                check_tg(tg_ntt_forward_oop(ring.dev(), dst, p0.data(), full_level, ns, u32(np), ring.stream()));
            else
                check_tg(tg_ntt_inverse_oop(ring.dev(), dst, p0.data(), full_level, ns, u32(np), ring.stream()));
            if (!own && target == Form::eval)
                p0.storage()->put_eval(p0.offset(), full_level, ns, int(np), ring.stream(), out_blk);
            if (keep_eval && !own && target == Form::coeff && out_off == 0 && p0.offset() == 0)
                out_blk->put_eval(0, full_level, ns, int(np), ring.stream(), p0.storage());
        }
        std::vector<Poly> v;
        v.reserve(np);
        for (std::size_t i = 0; i < np; ++i) v.push_back(Poly::view(ring, out_blk, out_off + S * i, lvl, target, ns));
        ct.parts = std::move(v);
        return;
    }
    for (auto& p : ct.parts)
        if (p.form() == from) target == Form::eval ? p.ntt_forward() : p.ntt_inverse();
}

void Ciphertext::to_coeff() { transform_parts(*this, Form::coeff); }
void detail::to_coeff_keep_eval(Ciphertext& ct) { transform_parts(ct, Form::coeff, true); }
void Ciphertext::to_eval() { transform_parts(*this, Form::eval); }

void Ciphertext::drop_to_level(int new_level) {
    for (auto& p : parts) p.drop_to_level(new_level);
}

static void addsub_ct(Ciphertext& x, const Ciphertext& o, int op) {
    if (x.parts.size() != o.parts.size() || x.batch != o.batch) throw TetrisError("rlwe", "ciphertext degree mismatch");
    if (x.domain != o.domain) throw TetrisError("rlwe", "domain tag mismatch");
    const std::size_t np = x.parts.size();
    for (std::size_t i = 0; i < np; ++i) x.parts[i].check_shape(o.parts[i]);
    if (contiguous(x.parts, 0, np) && contiguous(o.parts, 0, np)) {
        const Poly& p0 = x.parts[0];
        const RingParams& ring = p0.ring();
        const bool in_place = exclusively_owned(x.parts);
        if (in_place) p0.storage()->clear_eval_cache();  // the old contents' memoised eval form goes stale
        std::vector<Poly> dst =
            in_place ? x.parts : fresh_parts(ring, int(np), p0.level(), p0.form(), p0.nspecial());
        check_tg(tg_poly_addsub(ring.dev(), const_cast<u64*>(dst[0].data()), p0.data(), o.parts[0].data(), op,
                                p0.level(), p0.nspecial(), u32(np), ring.stream()));
        x.parts = std::move(dst);
        return;
    }
    const Poly& p0 = x.parts[0];
    const RingParams& ring = p0.ring();
    const int lvl = p0.level(), ns = p0.nspecial();
    // level-dropped views of one block each (aligned operands): one strided launch
    const std::size_t sx = detail::uniform_stride(x.parts), so = detail::uniform_stride(o.parts);
    if (sx && so && op != 2) {
        std::vector<Poly> dst = fresh_parts(ring, int(np), lvl, p0.form(), ns);
        check_tg(tg_poly_addsub_strided(ring.dev(), const_cast<u64*>(dst[0].data()), p0.data(), sx,
                                        o.parts[0].data(), so, op, lvl, ns, u32(np), ring.stream()));
        x.parts = std::move(dst);
        return;
    }
    x.parts = detail::map_parts2(x.parts, o.parts, [&](u64* d, const u64* a, const u64* b, u32 n) {
        check_tg(tg_poly_addsub(ring.dev(), d, a, b, op, lvl, ns, n, ring.stream()));
    });
}

void Ciphertext::add_inplace(const Ciphertext& o) {
    addsub_ct(*this, o, 0);
    noise_bound += o.noise_bound;
}

void Ciphertext::sub_inplace(const Ciphertext& o) {
    addsub_ct(*this, o, 1);
    noise_bound += o.noise_bound;
}

void Ciphertext::negate_inplace() {
    for (auto& p : parts) p.negate_inplace();
}

// ---------------------------------------------------------------------------
// KeyContext (rlwe.hpp:335-682)
// ---------------------------------------------------------------------------
KeyContext::KeyContext(const RingParams& ring, NoiseParams noise, GadgetVector gadget)
    : ring_(&ring), noise_(noise), plan_(std::make_shared<GadgetPlan>(ring, gadget)) {}

std::pair<SecretKey, PublicKey> KeyContext::keygen(Rng& rng) const {
    Rng r_s = rng.split(1), r_pk = rng.split(2);
    SecretKey sk(*ring_, noise_, r_s);
    PublicKey pk = make_public(sk, r_pk);
    return {std::move(sk), std::move(pk)};
}

PublicKey KeyContext::make_public(const SecretKey& sk, Rng& rng) const {
    const int lvl = ring_->max_level();
    Rng ra = rng.split(1), re = rng.split(2);
    Poly a = sample_uniform(*ring_, lvl, 0, ra);
    a.ntt_forward();
    Poly e = sample_gaussian(*ring_, noise_.gaussian_sigma, lvl, 0, re);
    e.ntt_forward();
    Poly as = a;
    as.mul_pointwise_inplace(sk.shaped(lvl, 0));
    e.sub_inplace(as);  // b = e - a*s
    return PublicKey{std::move(e), std::move(a), sk.id()};
}

Ciphertext KeyContext::encrypt(const SecretKey& sk, const Poly& m, double scale, Rng& rng, Domain domain) const {
    if (m.nspecial() != 0) throw TetrisError("rlwe", "message must not carry special rows");
    const int lvl = m.level();
    Rng ra = rng.split(1), re = rng.split(2);
    Poly a = sample_uniform(*ring_, lvl, 0, ra);  // c1 (coeff form, = iNTT(NTT(a)))
    Poly e = sample_gaussian(*ring_, noise_.gaussian_sigma, lvl, 0, re);
    // c0 = m + e - a*s   (exactly the reference's NTT(m+e) - a*s, then iNTT)
    std::vector<Poly> parts = fresh_parts(*ring_, 2, lvl, Form::coeff);
    const RingParams& R = *ring_;
    u64* c0 = const_cast<u64*>(parts[0].data());
    u64* c1 = const_cast<u64*>(parts[1].data());
    check_tg(tg_memcpy_d2d(R.dev(), c1, a.data(), a.words() * 8, R.stream()));
    Poly as = ntt_transform(a, Form::eval);
    as.mul_pointwise_inplace(sk.shaped(lvl, 0));
    as.ntt_inverse();
    Poly me = m.form() == Form::coeff ? m : ntt_transform(m, Form::coeff);
    check_tg(tg_poly_addsub(R.dev(), c0, me.data(), e.data(), 0, lvl, 0, 1, R.stream()));
    check_tg(tg_poly_addsub(R.dev(), c0, c0, as.data(), 1, lvl, 0, 1, R.stream()));
    Ciphertext ct;
    ct.parts = std::move(parts);
    ct.scale = scale;
    ct.domain = domain;
    ct.sk_id = sk.id();
    ct.noise_bound = 6.0 * noise_.gaussian_sigma;
    return ct;
}

Ciphertext KeyContext::encrypt_pk(const PublicKey& pk, const Poly& m, double scale, Rng& rng, Domain domain) const {
    const int lvl = m.level();
    Rng rv = rng.split(1), r0 = rng.split(2), r1 = rng.split(3);
    std::vector<i64> vc(ring_->degree());
    for (auto& x : vc) x = i64(rv.uniform(3)) - 1;
    Poly v = poly_from_i64(*ring_, vc, lvl);
    v.ntt_forward();
    Poly c0 = pk.b, c1 = pk.a;
    c0.drop_to_level(lvl);
    c1.drop_to_level(lvl);
    c0.mul_pointwise_inplace(v);
    c1.mul_pointwise_inplace(v);
    c0.ntt_inverse();
    c1.ntt_inverse();
    Poly e0 = sample_gaussian(*ring_, noise_.gaussian_sigma, lvl, 0, r0);
    Poly e1 = sample_gaussian(*ring_, noise_.gaussian_sigma, lvl, 0, r1);
    c0.add_inplace(e0);
    c0.add_inplace(m.form() == Form::coeff ? m : ntt_transform(m, Form::coeff));
    c1.add_inplace(e1);
    Ciphertext ct;
    ct.parts = {std::move(c0), std::move(c1)};
    ct.scale = scale;
    ct.domain = domain;
    ct.sk_id = pk.sk_id;
    ct.noise_bound = 6.0 * noise_.gaussian_sigma * (2.0 * std::sqrt(double(ring_->degree())) + 1.0);
    return ct;
}

Poly KeyContext::decrypt(const SecretKey& sk, const Ciphertext& ct) const {
    if (ct.sk_id != 0 && ct.sk_id != sk.id()) throw TetrisError("rlwe", "ciphertext bound to a different secret");
    if (ct.batch != 1) throw TetrisError("rlwe", "decrypt expects a single ciphertext (unstack the batch)");
    const int lvl = ct.level();
    Poly s = sk.shaped(lvl, 0);
    Poly acc = ct.parts[0].form() == Form::eval ? ct.parts[0] : ntt_transform(ct.parts[0], Form::eval);
    Poly spow = s;
    for (std::size_t k = 1; k < ct.parts.size(); ++k) {
        Poly pe = ct.parts[k].form() == Form::eval ? ct.parts[k] : ntt_transform(ct.parts[k], Form::eval);
        acc.mul_acc_pointwise(pe, spow);
        if (k + 1 < ct.parts.size()) spow.mul_pointwise_inplace(s);
    }
    acc.ntt_inverse();
    return acc;
}

Ciphertext KeyContext::zero_ciphertext(int level, double scale, u64 sk_id, Domain domain) const {
    Ciphertext ct;
    ct.parts = {Poly(*ring_, level, Form::coeff), Poly(*ring_, level, Form::coeff)};
    ct.scale = scale;
    ct.domain = domain;
    ct.sk_id = sk_id;
    ct.noise_bound = 0.0;
    return ct;
}

SwitchingKey KeyContext::switch_key_gen(const SecretKey& from, const SecretKey& to, Rng& rng) const {
    if (!from.ring().compatible(to.ring()) || !from.ring().compatible(*ring_))
        throw TetrisError("rlwe", "switching key requires matching rings");
    SwitchingKey swk;
    swk.gadget = plan_->config();
    swk.from_id = from.id();
    swk.to_id = to.id();
    swk.a_seed = splitmix64(rng.next());
    const auto scalars = plan_->key_scalars();
    const int lvl = ring_->max_level(), k = int(ring_->special_count());
    const Poly s_to = to.shaped(lvl, k);
    const Poly s_from = from.shaped(lvl, k);
    Rng ra(swk.a_seed);
    Rng re = rng.split(7);
    const std::size_t w = std::size_t(lvl + 1 + k) * ring_->degree();
    swk.block = new_block(*ring_, 2 * w * scalars.size());
    for (std::size_t i = 0; i < scalars.size(); ++i) {
        Rng rai = ra.split(i);
        Poly a = sample_uniform(*ring_, lvl, k, rai);
        a.ntt_forward();
        Rng rei = re.split(i);
        Poly e = sample_gaussian(*ring_, noise_.gaussian_sigma, lvl, k, rei);
        e.ntt_forward();
        Poly as = a;
        as.mul_pointwise_inplace(s_to);
        e.sub_inplace(as);
        Poly ws = s_from;
        ws.mul_scalar_inplace(scalars[i]);
        e.add_inplace(ws);  // b = e - a*s_to + w_i*P*s_from
        u64* bdst = swk.block->data() + 2 * w * i;
        check_tg(tg_memcpy_d2d(ring_->dev(), bdst, e.data(), w * 8, ring_->stream()));
        check_tg(tg_memcpy_d2d(ring_->dev(), bdst + w, a.data(), w * 8, ring_->stream()));
        swk.b.push_back(Poly::view(*ring_, swk.block, 2 * w * i, lvl, Form::eval, k));
        swk.a.push_back(Poly::view(*ring_, swk.block, 2 * w * i + w, lvl, Form::eval, k));
    }
    return swk;
}

static const u64* key_base(const SwitchingKey& swk) {
    if (!swk.block) throw TetrisError("rlwe", "switching key has no device block");
    return swk.block->data();
}

std::pair<Poly, Poly> KeyContext::ks_inner(const std::vector<Poly>& digits, const SwitchingKey& swk) const {
    if (digits.empty()) throw TetrisError("rlwe", "empty decomposition");
    if (digits.size() > swk.b.size()) throw TetrisError("rlwe", "switching key has too few digits");
    const int lvl = digits[0].level(), k = int(ring_->special_count());
    std::vector<Poly> src = digits;
    if (!contiguous(src, 0, src.size())) {  // gather into one block
        std::vector<Poly> g = fresh_parts(*ring_, int(src.size()), lvl, Form::eval, k);
        for (std::size_t i = 0; i < src.size(); ++i)
            check_tg(tg_memcpy_d2d(ring_->dev(), const_cast<u64*>(g[i].data()), src[i].data(), src[i].words() * 8,
                                   ring_->stream()));
        src = std::move(g);
    }
    std::vector<Poly> out = fresh_parts(*ring_, 2, lvl, Form::coeff);
    check_tg(tg_ks_inner(plan_->dev(), const_cast<u64*>(out[0].data()), const_cast<u64*>(out[1].data()),
                         src[0].data(), u32(src.size()), key_base(swk), swk.digits(), lvl, ring_->stream()));
    return {out[0], out[1]};
}

std::pair<Poly, Poly> KeyContext::switch_key_apply(const Poly& d, const SwitchingKey& swk) const {
    if (d.form() != Form::coeff || d.nspecial() != 0)
        throw TetrisError("rlwe", "decompose expects coeff form without special rows");
    const int lvl = d.level();
    std::vector<Poly> out = fresh_parts(*ring_, 2, lvl, Form::coeff);
    check_tg(tg_switch_key_apply(plan_->dev(), const_cast<u64*>(out[0].data()), const_cast<u64*>(out[1].data()),
                                 d.data(), key_base(swk), swk.digits(), lvl, ring_->stream()));
    return {out[0], out[1]};
}

Poly KeyContext::mod_down_p(const Poly& x) const {
    if (x.nspecial() == 0) throw TetrisError("rlwe", "mod_down_p expects special rows");
    if (x.form() != Form::coeff) throw TetrisError("rlwe", "mod_down_p expects coeff form");
    std::vector<Poly> out = fresh_parts(*ring_, 1, x.level(), Form::coeff);
    check_tg(tg_mod_down(plan_->dev(), const_cast<u64*>(out[0].data()), x.data(), x.level(), ring_->stream()));
    return out[0];
}

SwitchingKey KeyContext::relin_key_gen(const SecretKey& sk, Rng& rng) const {
    SecretKey s2 = square_secret(sk);
    return switch_key_gen(s2, sk, rng);
}

// relinearize (rlwe.hpp:601-620): c2 -> coeff, KS(c2), (c0+d0, c1+d1) in
// coeff form; the final adds are fused into ModDown (tg_keyswitch_add).
Ciphertext KeyContext::relinearize(const Ciphertext& ct, const SwitchingKey& rlk) const {
    if (ct.degree() != 2) throw TetrisError("rlwe", "relinearize expects a degree-2 ciphertext");
    if (rlk.to_id != ct.sk_id) throw TetrisError("rlwe", "relinearization key mismatch");
    const u32 B = ct.batch;
    const int lvl0 = ct.level();
    bool all_eval = true;
    for (const auto& p : ct.parts) all_eval &= p.form() == Form::eval && p.nspecial() == 0;
    if (all_eval) {
        // the tensor product's output: only c2 goes back to coefficient form
        // (ModUp's source); c0/c1 stay in eval form and are folded into the
        // key-switch accumulators (tg_relinearize_batch)
        std::vector<Poly> keep;
        const u64* a0 = detail::group_data(ct.parts, 0, B, keep);
        const u64* a1 = detail::group_data(ct.parts, B, B, keep);
        const u64* c2e = detail::group_data(ct.parts, 2 * B, B, keep);
        std::vector<Poly> c2 = fresh_parts(*ring_, int(B), lvl0, Form::coeff);
        check_tg(tg_ntt_inverse_oop(ring_->dev(), const_cast<u64*>(c2[0].data()), c2e, lvl0, 0, B, ring_->stream()));
        std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl0, Form::coeff);
        check_tg(tg_relinearize_batch(plan_->dev(), const_cast<u64*>(dst[0].data()), const_cast<u64*>(dst[B].data()),
                                      c2[0].data(), c2e, key_base(rlk), rlk.digits(), lvl0, a0, a1, B,
                                      ring_->stream()));
        Ciphertext out;
        out.batch = B;
        out.parts = std::move(dst);
        out.scale = ct.scale;
        out.domain = ct.domain;
        out.sk_id = ct.sk_id;
        out.noise_bound = ct.noise_bound + ks_noise_estimate();
        return out;
    }
    // keep the eval form of c2 (the tensor output): the digits' own-group rows
    // are its rows, so ModUp copies them instead of re-transforming
    const u64* c2_eval = nullptr;
    std::vector<Poly> keep;
    if (ct.parts[2 * B].form() == Form::eval && ct.parts[2 * B].nspecial() == 0 && contiguous(ct.parts, 2 * B, B)) {
        keep.push_back(ct.parts[2 * B]);  // holds the block
        c2_eval = ct.parts[2 * B].data();
    }
    Ciphertext src = ct;
    src.to_coeff();  // one batched iNTT when the parts share a block
    const int lvl = ct.level();
    const Poly& c2 = src.parts[2 * B];
    if (c2.form() != Form::coeff || c2.nspecial() != 0)
        throw TetrisError("rlwe", "decompose expects coeff form without special rows");
    const u64* d = detail::group_data(src.parts, 2 * B, B, keep);
    const u64* add0 = detail::group_data(src.parts, 0, B, keep);
    const u64* add1 = detail::group_data(src.parts, B, B, keep);
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl, Form::coeff);
    u64* out0 = const_cast<u64*>(dst[0].data());
    u64* out1 = const_cast<u64*>(dst[B].data());
    if (B == 1)
        check_tg(tg_keyswitch_add(plan_->dev(), out0, out1, d, c2_eval, key_base(rlk), rlk.digits(), lvl, add0, add1,
                                  ring_->stream()));
    else
        check_tg(tg_keyswitch_add_batch(plan_->dev(), out0, out1, d, c2_eval, key_base(rlk), rlk.digits(), lvl, add0,
                                        add1, B, ring_->stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = ct.scale;
    out.domain = ct.domain;
    out.sk_id = ct.sk_id;
    out.noise_bound = ct.noise_bound + ks_noise_estimate();
    return out;
}

Ciphertext KeyContext::relinearize_tensor(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk) const {
    if (rlk.to_id != x.sk_id) throw TetrisError("rlwe", "relinearization key mismatch");
    const u32 B = x.batch;
    const int lvl = x.level();
    std::vector<Poly> keep;
    const u64* x0 = detail::group_data(x.parts, 0, B, keep);
    const u64* x1 = detail::group_data(x.parts, B, B, keep);
    const u64* y0 = detail::group_data(y.parts, 0, B, keep);
    const u64* y1 = detail::group_data(y.parts, B, B, keep);
    std::vector<Poly> c2e = fresh_parts(*ring_, int(B), lvl, Form::eval);
    std::vector<Poly> c2 = fresh_parts(*ring_, int(B), lvl, Form::coeff);
    int raw = 1;  // c2 may stay the inverse transform's raw doubles (ModUp folds N^-1)
    check_tg(tg_tensor_c2_inverse(ring_->dev(), const_cast<u64*>(c2[0].data()), const_cast<u64*>(c2e[0].data()), x1,
                                  y1, lvl, B, &raw, ring_->stream()));
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl, Form::coeff);
    check_tg(tg_relinearize_tensor_batch(plan_->dev(), const_cast<u64*>(dst[0].data()),
                                         const_cast<u64*>(dst[B].data()), c2[0].data(), c2e[0].data(), key_base(rlk),
                                         rlk.digits(), lvl, x0, x1, y0, y1, B, raw, ring_->stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = x.scale * y.scale;  // Evaluator::mul (ckks.hpp:241-244), then relinearize
    out.domain = x.domain;
    out.sk_id = x.sk_id;
    out.noise_bound = (x.noise_bound * y.scale + y.noise_bound * x.scale) + ks_noise_estimate();
    return out;
}

Ciphertext KeyContext::relinearize_tensor_rescale(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk,
                                                  const Ciphertext* add, int out_level, const Ciphertext* u,
                                                  const Ciphertext* v) const {
    if (rlk.to_id != x.sk_id) throw TetrisError("rlwe", "relinearization key mismatch");
    const u32 B = x.batch;
    const int lvl = x.level();
    if ((u == nullptr) != (v == nullptr)) throw TetrisError("rlwe", "the second product needs both operands");
    if (u && (u->level() != lvl || v->level() != lvl || u->batch != B || v->batch != B))
        throw TetrisError("rlwe", "the second product must share the first's level and batch");
    std::vector<Poly> keep;
    u64 st[4] = {0, 0, 0, 0};  // poly strides of x, y, u, v (level-dropped batch views are read in place)
    const u64 *x0, *x1, *y0, *y1;
    detail::operand_groups(x, B, keep, x0, x1, st[0]);
    detail::operand_groups(y, B, keep, y0, y1, st[1]);
    const u64 *u0 = nullptr, *u1 = nullptr, *v0 = nullptr, *v1 = nullptr;
    if (u) {
        detail::operand_groups(*u, B, keep, u0, u1, st[2]);
        detail::operand_groups(*v, B, keep, v0, v1, st[3]);
    }
    const u64* ad = nullptr;
    std::size_t as = 0;
    if (add) {
        as = contiguous(add->parts, 0, 2 * B) ? add->parts[0].words() : detail::uniform_stride(add->parts);
        if (as == 0) throw TetrisError("ckks", "rescale_add addend parts without a uniform stride");
        ad = add->parts[0].data();
    }
    std::vector<Poly> c2e = fresh_parts(*ring_, int(B), lvl, Form::eval);
    std::vector<Poly> c2 = fresh_parts(*ring_, int(B), lvl, Form::coeff);
    int raw = 1;
    check_tg(tg_tensor2_c2_inverse_strided(ring_->dev(), const_cast<u64*>(c2[0].data()),
                                           const_cast<u64*>(c2e[0].data()), x1, y1, u1, v1, st, lvl, B, &raw,
                                           ring_->stream()));
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), add ? out_level : lvl - 1, Form::coeff);
    check_tg(tg_relinearize_tensor2_rescale_batch_strided(plan_->dev(), const_cast<u64*>(dst[0].data()), c2[0].data(),
                                                          c2e[0].data(), key_base(rlk), rlk.digits(), lvl, x0, x1, y0,
                                                          y1, u0, u1, v0, v1, st, B, raw, ad, as,
                                                          add ? out_level : 0, ring_->stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = x.scale * y.scale;  // the product's metadata; the caller rescales it
    out.domain = x.domain;
    out.sk_id = x.sk_id;
    out.noise_bound = (x.noise_bound * y.scale + y.noise_bound * x.scale) + ks_noise_estimate();
    return out;
}

Ciphertext KeyContext::relinearize_tensor_ladder(const Ciphertext& x, const Ciphertext& y, const SwitchingKey& rlk,
                                                 const Ciphertext* sub, const std::vector<u64>& sub_coef,
                                                 const std::vector<u64>& add_const) const {
    if (rlk.to_id != x.sk_id) throw TetrisError("rlwe", "relinearization key mismatch");
    const u32 B = x.batch;
    const int lvl = x.level();
    if (lvl < 1) throw TetrisError("ckks", "cannot rescale at level 0");
    std::vector<Poly> keep;
    u64 st[4] = {0, 0, 0, 0};
    const u64 *x0, *x1, *y0, *y1;
    detail::operand_groups(x, B, keep, x0, x1, st[0]);
    detail::operand_groups(y, B, keep, y0, y1, st[1]);
    const u64* sp = nullptr;
    std::size_t ss = 0;
    if (sub) {
        if (sub->form() != Form::coeff || sub->parts.size() != 2 * B || sub->level() < lvl ||
            sub_coef.size() != std::size_t(lvl) + 1)
            throw TetrisError("ckks", "ladder step: subtrahend shape");
        ss = contiguous(sub->parts, 0, 2 * B) ? sub->parts[0].words() : detail::uniform_stride(sub->parts);
        if (ss == 0) {  // parts of different blocks: gather them
            sp = detail::group_data(sub->parts, 0, 2 * B, keep);
            ss = sub->parts[0].words();
        } else {
            sp = sub->parts[0].data();
        }
    }
    if (!add_const.empty() && add_const.size() != std::size_t(lvl) + 1)
        throw TetrisError("ckks", "ladder step: constant per row");
    std::vector<Poly> c2e = fresh_parts(*ring_, int(B), lvl, Form::eval);
    std::vector<Poly> c2 = fresh_parts(*ring_, int(B), lvl, Form::coeff);
    int raw = 1;
    check_tg(tg_tensor2_c2_inverse_strided(ring_->dev(), const_cast<u64*>(c2[0].data()),
                                           const_cast<u64*>(c2e[0].data()), x1, y1, nullptr, nullptr, st, lvl, B, &raw,
                                           ring_->stream()));
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl - 1, Form::coeff);
    check_tg(tg_relinearize_tensor_ladder_batch_strided(plan_->dev(), const_cast<u64*>(dst[0].data()), c2[0].data(),
                                                        c2e[0].data(), key_base(rlk), rlk.digits(), lvl, x0, x1, y0,
                                                        y1, st, B, raw, sp, ss, sub ? sub_coef.data() : nullptr,
                                                        add_const.empty() ? nullptr : add_const.data(),
                                                        ring_->stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = x.scale * y.scale;  // the product's metadata; the caller applies the ladder step's
    out.domain = x.domain;
    out.sk_id = x.sk_id;
    out.noise_bound = (x.noise_bound * y.scale + y.noise_bound * x.scale) + ks_noise_estimate();
    return out;
}

Ciphertext KeyContext::relinearize_eval(const Ciphertext& ct, const SwitchingKey& rlk) const {
    if (ct.degree() != 2) throw TetrisError("rlwe", "relinearize expects a degree-2 ciphertext");
    if (rlk.to_id != ct.sk_id) throw TetrisError("rlwe", "relinearization key mismatch");
    const u32 B = ct.batch;
    Ciphertext src = ct;
    src.to_eval();
    const int lvl = ct.level();
    for (const auto& p : src.parts)
        if (p.nspecial() != 0) throw TetrisError("rlwe", "decompose expects a ciphertext without special rows");
    std::vector<Poly> keep;
    const u64* add0 = detail::group_data(src.parts, 0, B, keep);
    const u64* add1 = detail::group_data(src.parts, B, B, keep);
    const u64* c2_eval = detail::group_data(src.parts, 2 * B, B, keep);
    // c2 alone back to coefficient form (ModUp's source)
    std::vector<Poly> c2 = fresh_parts(*ring_, int(B), lvl, Form::coeff);
    check_tg(tg_ntt_inverse_oop(ring_->dev(), const_cast<u64*>(c2[0].data()), c2_eval, lvl, 0, B, ring_->stream()));
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl, Form::eval);
    check_tg(tg_keyswitch_add_eval(plan_->dev(), const_cast<u64*>(dst[0].data()), const_cast<u64*>(dst[B].data()),
                                   c2[0].data(), c2_eval, key_base(rlk), rlk.digits(), lvl, add0, add1, B,
                                   ring_->stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = ct.scale;
    out.domain = ct.domain;
    out.sk_id = ct.sk_id;
    out.noise_bound = ct.noise_bound + ks_noise_estimate();
    return out;
}

SwitchingKey KeyContext::galois_key_gen(const SecretKey& sk, u64 exponent, Rng& rng) const {
    const u32 n = ring_->degree();
    const u64 two_n = 2 * u64(n);
    const u64 g = exponent % two_n;
    if (g % 2 == 0) throw TetrisError("rlwe", "invalid automorphism exponent");
    std::vector<i64> c(n);
    const auto& s = sk.coeffs();
    for (u32 i = 0; i < n; ++i) {
        const u64 j = (u64(i) * g) % two_n;
        if (j < n) c[j] = s[i];
        else c[j - n] = -s[i];
    }
    SecretKey phi_s(*ring_, std::move(c), splitmix64(sk.id() ^ exponent));
    return switch_key_gen(phi_s, sk, rng);
}

// apply_galois (rlwe.hpp:637-654)
Ciphertext KeyContext::apply_galois(const Ciphertext& ct, u64 exponent, const SwitchingKey& swk) const {
    if (ct.degree() != 1) throw TetrisError("rlwe", "apply_galois expects degree-1 input");
    const u32 B = ct.batch;  // a batch: every ciphertext rotated under the same key
    Ciphertext src = ct;
    src.to_coeff();
    const int lvl = ct.level();
    const u64 g = exponent % (2 * u64(ring_->degree()));
    if (g % 2 == 0) throw TetrisError("ring", "automorphism exponent must be odd");
    std::vector<Poly> rot = fresh_parts(*ring_, int(2 * B), lvl, Form::coeff);
    if (contiguous(src.parts, 0, 2 * B)) {
        check_tg(tg_automorphism(ring_->dev(), const_cast<u64*>(rot[0].data()), src.parts[0].data(), g, TG_FORM_COEFF,
                                 lvl, 0, 2 * B, ring_->stream()));
    } else {
        for (u32 i = 0; i < 2 * B; ++i)
            check_tg(tg_automorphism(ring_->dev(), const_cast<u64*>(rot[i].data()), src.parts[i].data(), g,
                                     TG_FORM_COEFF, lvl, 0, 1, ring_->stream()));
    }
    // (phi(c0) + d0, d1): the add fused into ModDown
    Ciphertext out;
    std::vector<Poly> dst = fresh_parts(*ring_, int(2 * B), lvl, Form::coeff);
    if (B == 1)
        check_tg(tg_keyswitch_add(plan_->dev(), const_cast<u64*>(dst[0].data()), const_cast<u64*>(dst[1].data()),
                                  rot[1].data(), nullptr, key_base(swk), swk.digits(), lvl, rot[0].data(), nullptr,
                                  ring_->stream()));
    else
        check_tg(tg_keyswitch_add_batch(plan_->dev(), const_cast<u64*>(dst[0].data()), const_cast<u64*>(dst[B].data()),
                                        rot[B].data(), nullptr, key_base(swk), swk.digits(), lvl, rot[0].data(),
                                        nullptr, B, ring_->stream()));
    out.batch = B;
    out.parts = std::move(dst);
    out.scale = ct.scale;
    out.domain = ct.domain;
    out.sk_id = ct.sk_id;
    out.noise_bound = ct.noise_bound + ks_noise_estimate();
    return out;
}

std::vector<Ciphertext> KeyContext::apply_galois_hoisted(const Ciphertext& ct, const std::vector<u64>& exps,
                                                         const std::vector<const SwitchingKey*>& keys) const {
    if (ct.degree() != 1) throw TetrisError("ckks", "hoisting expects degree-1 input");
    if (ct.batch != 1) throw TetrisError("ckks", "hoisting on a batch is not supported (unstack it)");
    Ciphertext src = ct;
    src.to_coeff();
    const int lvl = src.level(), k = int(ring_->special_count());
    const u64 two_n = 2 * u64(ring_->degree());
    std::vector<Poly> digits = plan_->decompose(src.parts[1]);  // eval form, one block
    const u32 nd = u32(digits.size());
    std::vector<Ciphertext> out;
    out.reserve(exps.size());
    for (std::size_t e = 0; e < exps.size(); ++e) {
        const u64 g = exps[e];
        if (g == 1) {
            out.push_back(src);
            continue;
        }
        if ((g % two_n) % 2 == 0) throw TetrisError("ring", "automorphism exponent must be odd");
        const SwitchingKey& swk = *keys.at(e);
        std::vector<Poly> rd = fresh_parts(*ring_, int(nd), lvl, Form::eval, k);
        check_tg(tg_automorphism(ring_->dev(), const_cast<u64*>(rd[0].data()), digits[0].data(), g % two_n,
                                 TG_FORM_EVAL, lvl, k, nd, ring_->stream()));
        std::vector<Poly> c0g = fresh_parts(*ring_, 1, lvl, Form::coeff);
        check_tg(tg_automorphism(ring_->dev(), const_cast<u64*>(c0g[0].data()), src.parts[0].data(), g % two_n,
                                 TG_FORM_COEFF, lvl, 0, 1, ring_->stream()));
        std::vector<Poly> dst = fresh_parts(*ring_, 2, lvl, Form::coeff);
        // (phi(c0) + d0, d1): the add fused into ModDown
        check_tg(tg_ks_inner_add(plan_->dev(), const_cast<u64*>(dst[0].data()), const_cast<u64*>(dst[1].data()),
                                 rd[0].data(), nd, key_base(swk), swk.digits(), lvl, c0g[0].data(), nullptr,
                                 ring_->stream()));
        Ciphertext r;
        r.parts = std::move(dst);
        r.scale = ct.scale;
        r.domain = ct.domain;
        r.sk_id = ct.sk_id;
        r.noise_bound = ct.noise_bound + ks_noise_estimate();
        out.push_back(std::move(r));
    }
    return out;
}

double KeyContext::ks_noise_estimate() const {
    return 6.0 * noise_.gaussian_sigma * std::sqrt(double(ring_->degree())) *
           double(plan_->digit_count(ring_->max_level()));
}

SecretKey KeyContext::square_secret(const SecretKey& sk) const {
    const u32 n = ring_->degree();
    const auto& s = sk.coeffs();
    std::vector<u32> nz;
    for (u32 i = 0; i < n; ++i)
        if (s[i] != 0) nz.push_back(i);
    std::vector<i64> sq(n, 0);
    for (u32 i : nz)
        for (u32 j : nz) {
            const u32 k = i + j;
            const i64 v = s[i] * s[j];
            if (k < n) sq[k] += v;
            else sq[k - n] -= v;
        }
    return SecretKey(*ring_, std::move(sq), splitmix64(sk.id() ^ 0x5157ULL));
}

// ---------------------------------------------------------------------------
// Ciphertext batches (extension): part-major stacking of equal-shape cts
// ---------------------------------------------------------------------------
Ciphertext stack_ciphertexts(const std::vector<Ciphertext>& cts) {
    if (cts.empty()) throw TetrisError("ckks", "stack of no ciphertexts");
    const Ciphertext& c0 = cts[0];
    const u32 B = u32(cts.size());
    const std::size_t deg1 = c0.parts.size();
    double noise = 0;
    for (const auto& c : cts) {
        if (c.batch != 1 || c.parts.size() != deg1) throw TetrisError("ckks", "stack expects single ciphertexts of one degree");
        if (c.domain != c0.domain || c.sk_id != c0.sk_id) throw TetrisError("ckks", "stack: domain or key mismatch");
        if (std::abs(c.scale / c0.scale - 1.0) > 1e-4) throw TetrisError("ckks", "scaling factors diverged beyond tolerance");
        for (const auto& p : c.parts) p.check_shape(c0.parts[0]);
        noise = std::max(noise, c.noise_bound);
    }
    const Poly& p0 = c0.parts[0];
    const RingParams& ring = p0.ring();
    std::vector<Poly> out = fresh_parts(ring, int(deg1 * B), p0.level(), p0.form(), p0.nspecial());
    // one gather launch for the whole part-major block (was one copy per poly)
    std::vector<const u64*> srcs(deg1 * B);
    for (std::size_t k = 0; k < deg1; ++k)
        for (u32 i = 0; i < B; ++i) srcs[k * B + i] = cts[i].parts[k].data();
    check_tg(tg_gather_polys(ring.dev(), const_cast<u64*>(out[0].data()), srcs.data(), u32(srcs.size()), p0.words(),
                             ring.stream()));
    Ciphertext r;
    r.parts = std::move(out);
    r.batch = B;
    r.scale = c0.scale;
    r.domain = c0.domain;
    r.sk_id = c0.sk_id;
    r.noise_bound = noise;
    return r;
}

// Slices are copied into their own part-major block, so every downstream op
// sees the standard batch layout (one launch per op, no strided views).
Ciphertext slice_ciphertext(const Ciphertext& ct, u32 first, u32 count) {
    const u32 B = ct.batch;
    if (count == 0 || first + count > B) throw TetrisError("ckks", "batch slice out of range");
    const std::size_t deg1 = ct.parts.size() / B;
    const Poly& p0 = ct.parts[0];
    const RingParams& ring = p0.ring();
    std::vector<Poly> out = fresh_parts(ring, int(deg1 * count), p0.level(), p0.form(), p0.nspecial());
    for (std::size_t k = 0; k < deg1; ++k) {
        const std::size_t src = k * B + first;
        if (contiguous(ct.parts, src, count)) {
            check_tg(tg_memcpy_d2d(ring.dev(), const_cast<u64*>(out[k * count].data()), ct.parts[src].data(),
                                   out[0].words() * 8 * count, ring.stream()));
        } else {
            for (u32 i = 0; i < count; ++i)
                check_tg(tg_memcpy_d2d(ring.dev(), const_cast<u64*>(out[k * count + i].data()),
                                       ct.parts[src + i].data(), out[0].words() * 8, ring.stream()));
        }
    }
    Ciphertext r = ct;
    r.parts = std::move(out);
    r.batch = count;
    return r;
}

std::vector<Ciphertext> unstack_ciphertext(const Ciphertext& ct) {
    std::vector<Ciphertext> out;
    for (u32 i = 0; i < ct.batch; ++i) out.push_back(slice_ciphertext(ct, i, 1));
    return out;
}

}  // namespace tetris_b200
