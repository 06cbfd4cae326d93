// CKKS layer on the device: Encoder (host DFT), Evaluator, eval_chebyshev,
// inner_sum (reference ckks.hpp:24-615). Every ciphertext op runs on the GPU;
// host work is limited to scale bookkeeping and exact integer constants, in
// the reference's expression order.
#include <algorithm>
#include <cmath>
#include <thread>

#include <cstdlib>

#include "internal.hpp"
#include "tetris_b200/evaluator.hpp"

namespace tetris_b200 {

using detail::contiguous;
using detail::exclusively_owned;
using detail::fresh_parts;
using detail::tg_form;

// ---------------------------------------------------------------------------
// Encoder (ckks.hpp:24-148)
// ---------------------------------------------------------------------------
Encoder::Encoder(const RingParams& ring, u32 nslots) : ring_(&ring), n_(nslots) {
    if (n_ < 2 || (n_ & (n_ - 1)) != 0 || n_ > ring.degree() / 2)
        throw TetrisError("ckks", "slot count must be a power of two <= N/2");
    const u32 m = 4 * n_;
    psi_.resize(m);
    for (u32 t = 0; t < m; ++t) {
        const double ang = M_PI * double(t) / double(2 * n_);
        psi_[t] = cplx(std::cos(ang), std::sin(ang));
    }
    rot5_.resize(n_);
    u64 g = 1;
    for (u32 j = 0; j < n_; ++j) {
        rot5_[j] = u32(g);
        g = (g * 5) % m;
    }
}

// Runs body(lo, hi) over [0, n) on up to hardware_concurrency threads. Each
// output index is computed by exactly one thread with the sequential inner
// summation order, so the result does not depend on the thread count.
template <class F>
static void parallel_for(u32 n, F body) {
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    unsigned nt = std::min<unsigned>(hw, std::max<u32>(1, n / 256));
    if (nt <= 1) {
        body(0u, n);
        return;
    }
    std::vector<std::thread> th;
    const u32 per = (n + nt - 1) / nt;
    for (unsigned i = 0; i < nt; ++i) {
        const u32 lo = i * per, hi = std::min(n, lo + per);
        if (lo < hi) th.emplace_back(body, lo, hi);
    }
    for (auto& t : th) t.join();
}

std::vector<cplx> Encoder::dft(const std::vector<cplx>& w) const {
    std::vector<cplx> out(n_);
    const u64 mask = 4 * u64(n_);
    parallel_for(n_, [&](u32 lo, u32 hi) {
        for (u32 j = lo; j < hi; ++j) {
            cplx acc{0, 0};
            for (u32 t = 0; t < n_; ++t) acc += w[t] * psi_[u32((u64(t) * rot5_[j]) % mask)];
            out[j] = acc;
        }
    });
    return out;
}

std::vector<cplx> Encoder::dft_inv(const std::vector<cplx>& v) const {
    std::vector<cplx> out(n_);
    const u64 mask = 4 * u64(n_);
    parallel_for(n_, [&](u32 lo, u32 hi) {
        for (u32 t = lo; t < hi; ++t) {
            cplx acc{0, 0};
            for (u32 j = 0; j < n_; ++j) acc += v[j] * std::conj(psi_[u32((u64(t) * rot5_[j]) % mask)]);
            out[t] = acc / double(n_);
        }
    });
    return out;
}

std::vector<u64> Encoder::encode_slots_host(const std::vector<cplx>& v, double scale, int level) const {
    if (v.size() != n_) throw TetrisError("ckks", "slot vector length mismatch");
    const std::vector<cplx> w = dft_inv(v);
    const u32 N = ring_->degree(), stride = N / (2 * n_);
    double bound = 0;
    for (const cplx& c : w) bound = std::max({bound, std::abs(c.real()), std::abs(c.imag())});
    if (level == 0 && bound * scale * 2 >= double(ring_->modulus(0)))
        throw TetrisError("ckks", "plaintext overflows the level-0 modulus");
    std::vector<u64> res(std::size_t(level + 1) * N, 0);
    for (u32 t = 0; t < n_; ++t) {
        const i64 re = round_half_away(w[t].real() * scale);
        const i64 im = round_half_away(w[t].imag() * scale);
        for (int r = 0; r <= level; ++r) {
            const u64 q = ring_->modulus(r);
            res[std::size_t(r) * N + std::size_t(t) * stride] = from_centered(re, q);
            res[std::size_t(r) * N + std::size_t(n_ + t) * stride] = from_centered(im, q);
        }
    }
    return res;
}

const DeviceBuffer& Encoder::device_tables() const {
    std::lock_guard<std::mutex> g(*dtab_mu_);
    if (!dtab_) {
        static_assert(sizeof(cplx) == 16, "std::complex<double> layout");
        const std::size_t psi_words = 2 * psi_.size(), rot_words = (rot5_.size() + 1) / 2;
        auto buf = std::make_shared<DeviceBuffer>(*ring_, psi_words + rot_words);
        tg_context* c = ring_->dev();
        check_tg(tg_memcpy_h2d(c, buf->data(), psi_.data(), psi_words * 8, ring_->stream()));
        check_tg(tg_memcpy_h2d(c, buf->data() + psi_words, rot5_.data(), rot5_.size() * 4, ring_->stream()));
        ring_->synchronize();  // the tables are read from every stream afterwards
        dtab_ = std::move(buf);
    }
    return *dtab_;
}

std::vector<Poly> Encoder::encode_slots_many(const std::vector<std::vector<cplx>>& vs, double scale,
                                             int level) const {
    if (level < 0 || level > ring_->max_level()) throw TetrisError("ring", "poly level out of range");
    for (const auto& v : vs)
        if (v.size() != n_) throw TetrisError("ckks", "slot vector length mismatch");
    if (vs.empty()) return {};
    const DeviceBuffer& tab = device_tables();
    const std::size_t B = vs.size(), vw = 2 * std::size_t(n_);
    std::vector<double> h(B * vw + 1, 0.0);  // slot vectors + the bound word (zero)
    for (std::size_t b = 0; b < B; ++b) std::memcpy(h.data() + b * vw, vs[b].data(), vw * 8);
    DeviceBuffer in(*ring_, h.size());
    tg_context* c = ring_->dev();
    void* s = ring_->stream();
    check_tg(tg_memcpy_h2d(c, in.data(), h.data(), h.size() * 8, s));
    std::vector<Poly> out = detail::fresh_parts(*ring_, int(B), level, Form::coeff);
    u64* bound = level == 0 ? in.data() + B * vw : nullptr;
    check_tg(tg_encode_slots(c, const_cast<u64*>(out[0].data()), reinterpret_cast<const double*>(in.data()), u32(B),
                             n_, reinterpret_cast<const double*>(tab.data()),
                             reinterpret_cast<const u32*>(tab.data() + 2 * psi_.size()), scale, level, bound, s));
    if (bound) {  // check_encoding_bound (ckks.hpp:137-142)
        u64 bits = 0;
        check_tg(tg_memcpy_d2h(c, &bits, bound, 8, s));
        ring_->synchronize();
        double b;
        std::memcpy(&b, &bits, 8);
        if (b * scale * 2 >= double(ring_->modulus(0)))
            throw TetrisError("ckks", "plaintext overflows the level-0 modulus");
    }
    return out;
}

Poly Encoder::encode_slots(const std::vector<cplx>& v, double scale, int level) const {
    if (level < 0 || level > ring_->max_level()) throw TetrisError("ring", "poly level out of range");
    if (v.size() != n_) throw TetrisError("ckks", "slot vector length mismatch");
    return encode_slots_many({v}, scale, level)[0];
}

// Exact centered value from rows 0 and 1 (ckks.hpp:123-134).
static i128 centered_from_rows(const RingParams& ring, int level, u64 r0, u64 r1) {
    if (level == 0) return to_centered(r0, ring.modulus(0));
    const u64 q0 = ring.modulus(0), q1 = ring.modulus(1);
    const u64 d = sub_mod(r1 % q1, r0 % q1, q1);
    const u64 t = mul_mod(d, inv_mod(q0 % q1, q1), q1);
    i128 x = i128(r0) + i128(q0) * i128(t);
    const i128 q = i128(q0) * i128(q1);
    if (x > q / 2) x -= q;
    return x;
}

std::vector<cplx> Encoder::decode_slots_host(const u64* rows01, int level, double scale) const {
    const u32 N = ring_->degree(), stride = N / (2 * n_);
    const u64* row1 = level == 0 ? rows01 : rows01 + N;
    std::vector<cplx> w(n_);
    for (u32 t = 0; t < n_; ++t) {
        const std::size_t i0 = std::size_t(t) * stride, i1 = std::size_t(n_ + t) * stride;
        const double re = double(centered_from_rows(*ring_, level, rows01[i0], row1[i0])) / scale;
        const double im = double(centered_from_rows(*ring_, level, rows01[i1], row1[i1])) / scale;
        w[t] = cplx(re, im);
    }
    return dft(w);
}

static std::vector<u64> download_rows01(const Poly& p) {
    const u32 N = p.ring().degree();
    const int nrows = p.level() == 0 ? 1 : 2;
    std::vector<u64> h(std::size_t(nrows) * N);
    check_tg(tg_memcpy_d2h(p.ring().dev(), h.data(), p.data(), h.size() * 8, p.ring().stream()));
    p.ring().synchronize();
    return h;
}

// Reads rows 0/1 as stored (the reference does not convert forms either).
std::vector<cplx> Encoder::decode_slots(const Poly& poly, double scale) const {
    const std::vector<u64> h = download_rows01(poly);
    return decode_slots_host(h.data(), poly.level(), scale);
}

Poly Encoder::encode_coeffs(const std::vector<double>& v, double scale, int level) const {
    const u32 N = ring_->degree();
    if (v.size() > N) throw TetrisError("ckks", "coeff vector too long");
    const u32 stride = N / u32(v.size());
    std::vector<u64> res(std::size_t(level + 1) * N, 0);
    for (std::size_t t = 0; t < v.size(); ++t) {
        const i64 c = round_half_away(v[t] * scale);
        if (std::abs(double(c)) * 2 >= double(ring_->modulus(0)) && level == 0)
            throw TetrisError("ckks", "plaintext overflows the level-0 modulus");
        for (int r = 0; r <= level; ++r) res[std::size_t(r) * N + t * stride] = from_centered(c, ring_->modulus(r));
    }
    return Poly::from_host(*ring_, res, level, Form::coeff);
}

std::vector<double> Encoder::decode_coeffs(const Poly& poly, double scale, std::size_t count) const {
    const Poly& c = poly;
    const std::vector<u64> h = download_rows01(c);
    const u32 N = ring_->degree(), stride = N / u32(count);
    const u64* row1 = c.level() == 0 ? h.data() : h.data() + N;
    std::vector<double> v(count);
    for (std::size_t t = 0; t < count; ++t)
        v[t] = double(centered_from_rows(*ring_, c.level(), h[t * stride], row1[t * stride])) / scale;
    return v;
}

// ---------------------------------------------------------------------------
// EvalKeys / exponents (ckks.hpp:155-173)
// ---------------------------------------------------------------------------
const SwitchingKey& EvalKeys::galois_key(u64 exponent) const {
    auto it = galois.find(exponent);
    if (it == galois.end()) throw TetrisError("ckks", "missing rotation key for exponent " + std::to_string(exponent));
    return it->second;
}

u64 rotation_exponent(const RingParams& ring, u32 k) { return pow_mod(5, k, 2 * u64(ring.degree())); }
u64 conjugation_exponent(const RingParams& ring) { return 2 * u64(ring.degree()) - 1; }

// ---------------------------------------------------------------------------
// Evaluator (ckks.hpp:181-335)
// ---------------------------------------------------------------------------
void Evaluator::check_scales_match(double a, double b) {
    if (std::abs(a / b - 1.0) > 1e-4) throw TetrisError("ckks", "scaling factors diverged beyond tolerance");
}

void Evaluator::align_levels(Ciphertext& a, Ciphertext& b) const {
    const int lvl = std::min(a.level(), b.level());
    if (a.level() != lvl) {
        a.to_coeff();
        a.drop_to_level(lvl);
    }
    if (b.level() != lvl) {
        b.to_coeff();
        b.drop_to_level(lvl);
    }
}

Ciphertext Evaluator::add(const Ciphertext& a, const Ciphertext& b) const {
    Ciphertext x = a, y = b;
    align_levels(x, y);
    check_scales_match(x.scale, y.scale);
    if (x.form() != y.form()) {
        x.to_coeff();
        y.to_coeff();
    }
    x.add_inplace(y);
    return x;
}

Ciphertext Evaluator::sub(const Ciphertext& a, const Ciphertext& b) const {
    Ciphertext x = a, y = b;
    align_levels(x, y);
    check_scales_match(x.scale, y.scale);
    if (x.form() != y.form()) {
        x.to_coeff();
        y.to_coeff();
    }
    x.sub_inplace(y);
    return x;
}

// Tensor product (ckks.hpp:220-245): one fused kernel for the 4 products.
Ciphertext Evaluator::mul(const Ciphertext& a, const Ciphertext& b) const {
    if (a.domain != b.domain) throw TetrisError("ckks", "domain tag mismatch in mul");
    if (a.degree() != 1 || b.degree() != 1) throw TetrisError("ckks", "mul expects degree-1 operands");
    if (a.batch != b.batch) throw TetrisError("ckks", "batch size mismatch in mul");
    Ciphertext x = a, y = b;
    align_levels(x, y);
    if (x.level() == 0) throw TetrisError("ckks", "exhausted ciphertext: no level left to rescale");
    x.to_eval();
    y.to_eval();
    const RingParams& R = ring();
    const int lvl = x.level();
    const u32 B = x.batch;
    std::vector<Poly> keep;
    const u64* x0 = detail::group_data(x.parts, 0, B, keep);
    const u64* x1 = detail::group_data(x.parts, B, B, keep);
    const u64* y0 = detail::group_data(y.parts, 0, B, keep);
    const u64* y1 = detail::group_data(y.parts, B, B, keep);
    std::vector<Poly> p = fresh_parts(R, int(3 * B), lvl, Form::eval);
    check_tg(tg_tensor(R.dev(), const_cast<u64*>(p[0].data()), const_cast<u64*>(p[B].data()),
                       const_cast<u64*>(p[2 * B].data()), x0, x1, y0, y1, lvl, B, R.stream()));
    Ciphertext out;
    out.batch = B;
    out.parts = std::move(p);
    out.scale = x.scale * y.scale;
    out.domain = x.domain;
    out.sk_id = x.sk_id;
    out.noise_bound = x.noise_bound * y.scale + y.noise_bound * x.scale;
    return out;
}

// mul then relinearize (ckks.hpp:301-303); with the tensor's c0 / c1 formed
// inside the key-switch core (KeyContext::relinearize_tensor) -- the same
// checks in the same order as mul + relinearize, the same residues.
Ciphertext Evaluator::mul_relin(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys) const {
    static const bool off = [] {
        const char* e = std::getenv("TG_RELIN_TENSOR");
        return e && *e == '0';
    }();
    if (off) return ctx_->relinearize(mul(a, b), keys.relin);
    if (a.domain != b.domain) throw TetrisError("ckks", "domain tag mismatch in mul");
    if (a.degree() != 1 || b.degree() != 1) throw TetrisError("ckks", "mul expects degree-1 operands");
    if (a.batch != b.batch) throw TetrisError("ckks", "batch size mismatch in mul");
    Ciphertext x = a, y = b;
    align_levels(x, y);
    if (x.level() == 0) throw TetrisError("ckks", "exhausted ciphertext: no level left to rescale");
    x.to_eval();
    y.to_eval();
    return ctx_->relinearize_tensor(x, y, keys.relin);
}

Ciphertext Evaluator::mul_relin_rescale(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys,
                                        const Ciphertext* add) const {
    static const bool off = [] {
        const char* e = std::getenv("TG_RELIN_TENSOR");
        const char* f = std::getenv("TG_FUSED_RESCALE");
        return (e && *e == '0') || (f && *f == '0');
    }();
    auto two_ops = [&] { return add ? rescale_add(mul_relin(a, b, keys), *add) : rescale(mul_relin(a, b, keys)); };
    if (off) return two_ops();
    // mul's checks in mul's order
    if (a.domain != b.domain) throw TetrisError("ckks", "domain tag mismatch in mul");
    if (a.degree() != 1 || b.degree() != 1) throw TetrisError("ckks", "mul expects degree-1 operands");
    if (a.batch != b.batch) throw TetrisError("ckks", "batch size mismatch in mul");
    Ciphertext x = a, y = b;
    align_levels(x, y);
    if (x.level() == 0) throw TetrisError("ckks", "exhausted ciphertext: no level left to rescale");
    const RingParams& R = ring();
    const int lvl = x.level();
    for (int r = 0; r <= lvl; ++r)
        if (R.modulus(u32(r)) >= 1351079888211148ull) return two_ops();  // kFpMaxQ (tg_fp64.cuh)
    // rescale_add's one-pass conditions (otherwise add(rescale(prod), y))
    if (add) {
        if (add->form() != Form::coeff || add->degree() != 1 || add->batch != x.batch || add->domain != x.domain)
            return two_ops();
        for (const auto& p : add->parts)
            if (p.nspecial() != 0) return two_ops();
        if (!contiguous(add->parts, 0, add->parts.size()) && detail::uniform_stride(add->parts) == 0)
            return two_ops();
    }
    for (const auto& p : x.parts)
        if (p.nspecial() != 0) return two_ops();
    for (const auto& p : y.parts)
        if (p.nspecial() != 0) return two_ops();
    // the product's metadata (mul, relinearize), then rescale's (ckks.hpp:321-323)
    const u64 ql = R.modulus(u32(lvl));
    const double pscale = (x.scale * y.scale) / double(ql);
    const double pnoise = ((x.noise_bound * y.scale + y.noise_bound * x.scale) + ctx_->ks_noise_estimate()) / double(ql) + 1.0;
    int out_level = lvl - 1;
    if (add) {  // rescale_add: level alignment, scale check on the rescaled product first
        out_level = std::min(lvl - 1, add->level());
        check_scales_match(pscale, add->scale);
    }
    x.to_eval();
    y.to_eval();
    Ciphertext out = ctx_->relinearize_tensor_rescale(x, y, keys.relin, add, out_level);
    out.scale = pscale;
    out.noise_bound = add ? pnoise + add->noise_bound : pnoise;
    return out;
}

// rescale(relinearize(add(mul(a, b), mul(c, d)))) [+ add]: the reference's
// primitives in that order (ckks.hpp:220-245, :201-208, rlwe.hpp:601-620,
// ckks.hpp:315-324) with one key switch for both products.
Ciphertext Evaluator::mul2_relin_rescale(const Ciphertext& a, const Ciphertext& b, const Ciphertext& c,
                                         const Ciphertext& d, const EvalKeys& keys, const Ciphertext* add) const {
    // the reference's primitives one after the other (any ring, any levels)
    auto composed = [&] {
        Ciphertext t1 = mul(a, b);
        if (c.domain != d.domain) throw TetrisError("ckks", "domain tag mismatch in mul");
        if (c.degree() != 1 || d.degree() != 1) throw TetrisError("ckks", "mul expects degree-1 operands");
        if (c.batch != d.batch) throw TetrisError("ckks", "batch size mismatch in mul");
        Ciphertext x = c, y = d;
        align_levels(x, y);
        if (x.level() == 0) throw TetrisError("ckks", "exhausted ciphertext: no level left to rescale");
        Ciphertext sum;
        if (x.level() >= t1.level() && x.form() == Form::coeff && y.form() == Form::coeff) {
            // add() would drop mul(c, d) to t1's level (align_levels); every step of
            // the tensor is row-wise, so the operands are dropped first instead:
            // the same rows, without the dropped rows' products and transforms
            x.drop_to_level(t1.level());
            y.drop_to_level(t1.level());
            Ciphertext t2 = mul(x, y);
            check_scales_match(t1.scale, t2.scale);
            t1.add_inplace(t2);  // both in eval form; relinearize brings c2 back
            sum = std::move(t1);
        } else {
            sum = this->add(t1, mul(c, d));
        }
        Ciphertext r = ctx_->relinearize(sum, keys.relin);
        return add ? rescale_add(r, *add) : rescale(r);
    };
    static const bool off = [] {
        const char* e = std::getenv("TG_RELIN_TENSOR");
        const char* f = std::getenv("TG_FUSED_RESCALE");
        const char* g = std::getenv("TG_LAZY_FUSED");
        return (e && *e == '0') || (f && *f == '0') || (g && *g == '0');
    }();
    if (off) return composed();
    // one-pass conditions (mul_relin_rescale's, for both products): same
    // batch and domain, coefficient-form degree-1 operands without special
    // rows, the second product not below the first's level, FP64 q rows
    for (const Ciphertext* t : {&a, &b, &c, &d}) {
        if (t->degree() != 1 || t->batch != a.batch || t->domain != a.domain || t->form() != Form::coeff)
            return composed();
        for (const auto& p : t->parts)
            if (p.nspecial() != 0) return composed();
    }
    Ciphertext x = a, y = b, u = c, v = d;
    align_levels(x, y);
    align_levels(u, v);
    const int lvl = x.level();
    if (lvl == 0 || u.level() < lvl) return composed();
    const RingParams& R = ring();
    for (int r = 0; r <= lvl; ++r)
        if (R.modulus(u32(r)) >= 1351079888211148ull) return composed();  // kFpMaxQ (tg_fp64.cuh)
    if (add) {
        if (add->form() != Form::coeff || add->degree() != 1 || add->batch != x.batch || add->domain != x.domain)
            return composed();
        for (const auto& p : add->parts)
            if (p.nspecial() != 0) return composed();
        if (!contiguous(add->parts, 0, add->parts.size()) && detail::uniform_stride(add->parts) == 0)
            return composed();
    }
    // metadata of mul, mul, add, relinearize, rescale (, add) in that order
    const double s1 = x.scale * y.scale, s2 = u.scale * v.scale;
    const double n1 = x.noise_bound * y.scale + y.noise_bound * x.scale;
    const double n2 = u.noise_bound * v.scale + v.noise_bound * u.scale;
    check_scales_match(s1, s2);
    const u64 ql = R.modulus(u32(lvl));
    const double pscale = s1 / double(ql);
    const double pnoise = ((n1 + n2) + ctx_->ks_noise_estimate()) / double(ql) + 1.0;
    int out_level = lvl - 1;
    if (add) {
        out_level = std::min(lvl - 1, add->level());
        check_scales_match(pscale, add->scale);
    }
    u.drop_to_level(lvl);  // add()'s alignment, applied to the operands (row-wise tensor)
    v.drop_to_level(lvl);
    x.to_eval();
    y.to_eval();
    u.to_eval();
    v.to_eval();
    Ciphertext out = ctx_->relinearize_tensor_rescale(x, y, keys.relin, add, out_level, &u, &v);
    out.scale = pscale;
    out.noise_bound = add ? pnoise + add->noise_bound : pnoise;
    return out;
}

Ciphertext Evaluator::mul_relin_eval(const Ciphertext& a, const Ciphertext& b, const EvalKeys& keys) const {
    return ctx_->relinearize_eval(mul(a, b), keys.relin);
}

Ciphertext Evaluator::mul_plain(const Ciphertext& ct, const Poly& plain_eval, double plain_scale) const {
    Ciphertext out = ct;
    out.to_eval();
    const RingParams& R = ring();
    const int lvl = out.level();
    if (plain_eval.level() < lvl || plain_eval.nspecial() != 0)
        throw TetrisError("ckks", "plaintext has fewer rows than the ciphertext");
    const std::size_t np = out.parts.size();
    std::vector<Poly> dst = fresh_parts(R, int(np), lvl, Form::eval);
    if (contiguous(out.parts, 0, np)) {
        check_tg(tg_mul_plain(R.dev(), const_cast<u64*>(dst[0].data()), out.parts[0].data(), plain_eval.data(), lvl,
                              u32(np), R.stream()));
    } else {
        for (std::size_t i = 0; i < np; ++i)
            check_tg(tg_mul_plain(R.dev(), const_cast<u64*>(dst[i].data()), out.parts[i].data(), plain_eval.data(),
                                  lvl, 1, R.stream()));
    }
    out.parts = std::move(dst);
    out.scale = ct.scale * plain_scale;
    out.noise_bound = ct.noise_bound * plain_scale;
    return out;
}

// Applies a per-modulus Shoup scalar to every part, batched when contiguous.
static void scale_parts(Ciphertext& out, const std::vector<u64>& per_mod) {
    const std::size_t np = out.parts.size();
    const Poly& p0 = out.parts[0];
    const RingParams& R = p0.ring();
    (void)np;
    const int lvl = p0.level(), ns = p0.nspecial();
    out.parts = detail::map_parts(out.parts, lvl, p0.form(), [&](u64* d, const u64* s, u32 n) {
        check_tg(tg_poly_mul_scalar(R.dev(), d, s, per_mod.data(), lvl, ns, n, R.stream()));
    });
}

Ciphertext Evaluator::mul_scalar(const Ciphertext& ct, double c, double scalar_scale) const {
    if (std::abs(c) * scalar_scale >= 9.0e18) throw TetrisError("ckks", "scalar multiplier exceeds the integer range");
    const i64 v = round_half_away(c * scalar_scale);
    Ciphertext out = ct;
    std::vector<u64> per_mod(ring().moduli().size());
    for (std::size_t i = 0; i < per_mod.size(); ++i) per_mod[i] = from_centered(v, ring().moduli()[i]);
    scale_parts(out, per_mod);
    out.scale = ct.scale * scalar_scale;
    return out;
}

u64 Evaluator::scaled_residue(double value, u64 q) {
    if (std::abs(value) < 9.0e18) return from_centered(round_half_away(value), q);
    const long double r = std::fmod((long double)value, (long double)q);
    return from_centered((i64)llroundl(r), q);
}

Ciphertext Evaluator::add_scalar(const Ciphertext& ct, double c) const {
    Ciphertext out = ct;
    const Poly& p0 = ct.parts[0];
    const RingParams& R = ring();
    std::vector<u64> add(R.moduli().size(), 0);
    for (int r = 0; r < p0.rows(); ++r) add[p0.modulus_index(r)] = scaled_residue(c * ct.scale, p0.row_modulus(r));
    // keep all parts in one block (batched launches downstream); a batch
    // adds the constant to each ciphertext's part 0 (parts [0, batch))
    const std::size_t np = ct.parts.size(), B = ct.batch;
    std::vector<Poly> dst = fresh_parts(R, int(np), p0.level(), p0.form(), p0.nspecial());
    std::vector<Poly> keep;
    for (std::size_t i = 1; i < B; ++i)
        if (ct.parts[i].level() != p0.level() || ct.parts[i].form() != p0.form())
            throw TetrisError("ckks", "batch parts of different shapes");
    check_tg(tg_poly_add_scalar(R.dev(), const_cast<u64*>(dst[0].data()), detail::group_data(ct.parts, 0, B, keep),
                                add.data(), tg_form(p0.form()), p0.level(), p0.nspecial(), u32(B), R.stream()));
    if (B > 1) {
        if (contiguous(ct.parts, B, np - B)) {
            check_tg(tg_memcpy_d2d(R.dev(), const_cast<u64*>(dst[B].data()), ct.parts[B].data(),
                                   dst[B].words() * 8 * (np - B), R.stream()));
        } else {
            for (std::size_t i = B; i < np; ++i)
                check_tg(tg_memcpy_d2d(R.dev(), const_cast<u64*>(dst[i].data()), ct.parts[i].data(),
                                       dst[i].words() * 8, R.stream()));
        }
        out.parts = std::move(dst);
        return out;
    }
    for (std::size_t i = 1; i < np; ++i) {
        if (ct.parts[i].level() != p0.level() || ct.parts[i].form() != p0.form()) {  // irregular: keep as is
            out.parts[0] = dst[0];
            return out;
        }
        check_tg(tg_memcpy_d2d(R.dev(), const_cast<u64*>(dst[i].data()), ct.parts[i].data(), dst[i].words() * 8,
                               R.stream()));
    }
    out.parts = std::move(dst);
    return out;
}

Ciphertext Evaluator::rescale(const Ciphertext& ct) const {
    if (ct.level() == 0) throw TetrisError("ckks", "cannot rescale at level 0");
    Ciphertext out = ct;
    out.to_coeff();
    const u64 ql = ring().modulus(u32(ct.level()));
    const RingParams& R = ring();
    const int lvl = out.level();
    for (const auto& p : out.parts)
        if (p.nspecial() != 0) throw TetrisError("ring", "rescale with special rows");
    out.parts = detail::map_parts(out.parts, lvl - 1, Form::coeff, [&](u64* d, const u64* s, u32 n) {
        check_tg(tg_rescale(R.dev(), d, s, lvl, n, R.stream()));
    });
    out.scale = ct.scale / double(ql);
    out.noise_bound = ct.noise_bound / double(ql) + 1.0;
    return out;
}

Ciphertext Evaluator::rescale_add(const Ciphertext& prod, const Ciphertext& y) const {
    auto two_ops = [&] { return add(rescale(prod), y); };
    if (prod.level() == 0 || prod.form() != Form::coeff || y.form() != Form::coeff) return two_ops();
    if (prod.degree() != 1 || y.degree() != 1 || prod.batch != y.batch || prod.domain != y.domain) return two_ops();
    const RingParams& R = ring();
    const std::size_t np = prod.parts.size();
    if (y.parts.size() != np || !contiguous(prod.parts, 0, np)) return two_ops();
    for (std::size_t i = 0; i < np; ++i)
        if (prod.parts[i].nspecial() != 0 || y.parts[i].nspecial() != 0) return two_ops();
    for (int r = 0; r <= prod.level(); ++r)
        if (R.modulus(u32(r)) >= 1351079888211148ull) return two_ops();  // kFpMaxQ (tg_fp64.cuh)
    const std::size_t ys = contiguous(y.parts, 0, np) ? y.parts[0].words() : detail::uniform_stride(y.parts);
    if (ys == 0) return two_ops();
    const u64 ql = R.modulus(u32(prod.level()));
    // rescale's metadata (ckks.hpp:321-323), then add's (level alignment,
    // scale check on the rescaled operand first, noise sum)
    const double pscale = prod.scale / double(ql);
    const double pnoise = prod.noise_bound / double(ql) + 1.0;
    const int lvl = std::min(prod.level() - 1, y.level());
    check_scales_match(pscale, y.scale);
    std::vector<Poly> dst = fresh_parts(R, int(np), lvl, Form::coeff);
    check_tg(tg_rescale_add(R.dev(), const_cast<u64*>(dst[0].data()), prod.parts[0].data(), prod.level(), u32(np),
                            y.parts[0].data(), ys, lvl, R.stream()));
    Ciphertext out;
    out.batch = prod.batch;
    out.parts = std::move(dst);
    out.scale = pscale;
    out.domain = prod.domain;
    out.sk_id = prod.sk_id;
    out.noise_bound = pnoise + y.noise_bound;
    return out;
}

Ciphertext Evaluator::rescale_eval(const Ciphertext& ct) const {
    if (ct.level() == 0) throw TetrisError("ckks", "cannot rescale at level 0");
    Ciphertext out = ct;
    out.to_eval();
    const u64 ql = ring().modulus(u32(ct.level()));
    const RingParams& R = ring();
    const int lvl = out.level();
    for (const auto& p : out.parts)
        if (p.nspecial() != 0) throw TetrisError("ring", "rescale with special rows");
    out.parts = detail::map_parts(out.parts, lvl - 1, Form::eval, [&](u64* d, const u64* s, u32 n) {
        check_tg(tg_rescale_eval(R.dev(), d, s, lvl, n, R.stream()));
    });
    out.scale = ct.scale / double(ql);
    out.noise_bound = ct.noise_bound / double(ql) + 1.0;
    return out;
}

Ciphertext Evaluator::rotate(const Ciphertext& ct, u32 k, const EvalKeys& keys) const {
    if (k == 0) return ct;
    const u64 g = rotation_exponent(ring(), k);
    return ctx_->apply_galois(ct, g, keys.galois_key(g));
}

Ciphertext Evaluator::conjugate(const Ciphertext& ct, const EvalKeys& keys) const {
    const u64 g = conjugation_exponent(ring());
    return ctx_->apply_galois(ct, g, keys.galois_key(g));
}

// eval_chebyshev / eval_chebyshev_bsgs live in chebyshev.cpp

std::vector<double> power_to_chebyshev(const std::vector<double>& pow_coeffs) {
    const std::size_t d = pow_coeffs.size();
    std::vector<std::vector<double>> t(d, std::vector<double>(d, 0.0));
    t[0][0] = 1.0;
    if (d > 1) t[1][1] = 1.0;
    for (std::size_t k = 2; k < d; ++k)
        for (std::size_t i = 0; i < d; ++i) {
            double v = -t[k - 2][i];
            if (i > 0) v += 2.0 * t[k - 1][i - 1];
            t[k][i] = v;
        }
    std::vector<double> c(d, 0.0), rem = pow_coeffs;
    for (std::size_t k = d; k-- > 0;) {
        const double lead = t[k][k];
        c[k] = rem[k] / lead;
        for (std::size_t i = 0; i <= k; ++i) rem[i] -= c[k] * t[k][i];
    }
    return c;
}

Ciphertext inner_sum(const Evaluator& ev, const Ciphertext& ct, u32 n, const EvalKeys& keys) {
    if (ct.domain != Domain::slots) throw TetrisError("ckks", "inner_sum expects slots domain");
    if ((n & (n - 1)) != 0) throw TetrisError("ckks", "slot count must be a power of two");
    Ciphertext acc = ct;
    for (u32 k = 1; k < n; k <<= 1) {
        Ciphertext rot = ev.rotate(acc, k, keys);
        acc = ev.add(acc, rot);
    }
    return acc;
}

}  // namespace tetris_b200
