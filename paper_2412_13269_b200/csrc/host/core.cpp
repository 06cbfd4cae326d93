// Host side of the core layer: word arithmetic, RNG, primes, NTT tables,
// RingParams device binding, device Poly. Restates reference common.hpp /
// ring.hpp semantics (cited per function); arithmetic on polynomials is
// delegated to the CUDA kernels behind include/tetris_b200.h.
#include <algorithm>
#include <cmath>
#include <unordered_map>

#include "tetris_b200/core.hpp"

namespace tetris_b200 {

void check_tg(int rc) {
    if (rc == TG_OK) return;
    std::string msg = tg_last_error();
    std::string tag = "gpu";
    if (msg.size() > 2 && msg[0] == '[') {
        auto close = msg.find(']');
        if (close != std::string::npos) {
            tag = msg.substr(1, close - 1);
            msg = msg.substr(std::min(msg.size(), close + 2));
        }
    }
    throw TetrisError(tag, msg);
}

// ---------------------------------------------------------------------------
// common.hpp:52-97, 103-147
// ---------------------------------------------------------------------------
u64 pow_mod(u64 base, u64 exp, u64 q) {
    u64 acc = 1;
    base %= q;
    for (; exp; exp >>= 1) {
        if (exp & 1) acc = mul_mod(acc, base, q);
        base = mul_mod(base, base, q);
    }
    return acc;
}

u64 inv_mod(u64 a, u64 q) {
    if (a % q == 0) throw std::invalid_argument("inv_mod: zero has no inverse");
    return pow_mod(a % q, q - 2, q);
}

i64 round_half_away(double x) { return i64(std::llround(x)); }

bool is_prime_u64(u64 n) {
    static const u64 kBases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return false;
    for (u64 p : kBases)
        if (n % p == 0) return n == p;
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++s;
    }
    for (u64 a : kBases) {
        u64 x = pow_mod(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool composite = true;
        for (int i = 1; i < s && composite; ++i) {
            x = mul_mod(x, x, n);
            if (x == n - 1) composite = false;
        }
        if (composite) return false;
    }
    return true;
}

// Scan outward from 2^bits in steps of `modulus` (alternating below/above).
std::vector<u64> find_ntt_primes(int bits, std::size_t count, u64 modulus, std::vector<u64> exclude) {
    if (bits < 10 || bits > 62) throw std::invalid_argument("find_ntt_primes: bits out of range");
    std::vector<u64> found;
    const u64 center = u64(1) << bits;
    u64 below = center - center % modulus + 1;
    u64 above = below + modulus;
    auto used = [&](u64 p) {
        return std::find(exclude.begin(), exclude.end(), p) != exclude.end() ||
               std::find(found.begin(), found.end(), p) != found.end();
    };
    while (found.size() < count) {
        if (below > modulus && is_prime_u64(below) && !used(below)) found.push_back(below);
        if (found.size() >= count) break;
        if (is_prime_u64(above) && !used(above)) found.push_back(above);
        below -= modulus;
        above += modulus;
        if (above - center > (center >> 2)) throw std::runtime_error("find_ntt_primes: search exhausted");
    }
    return found;
}

u64 splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

Rng::Rng(u64 seed) : seed_(seed), eng_(splitmix64(seed)) {}

u64 Rng::uniform(u64 bound) {
    if (bound == 0) throw std::invalid_argument("Rng::uniform: zero bound");
    const u64 reject_below = (0 - bound) % bound;
    u64 x;
    do x = eng_();
    while (x < reject_below);
    return x % bound;
}

double Rng::normal() {
    if (spare_ok_) {
        spare_ok_ = false;
        return spare_;
    }
    auto unit = [](u64 x) { return (double(x >> 11) + 1.0) * 0x1p-53; };
    double u1 = unit(eng_());
    double u2 = unit(eng_());
    double rad = std::sqrt(-2.0 * std::log(u1));
    double th = 6.283185307179586476925 * u2;
    spare_ = rad * std::sin(th);
    spare_ok_ = true;
    return rad * std::cos(th);
}

Rng Rng::split(u64 label) const { return Rng(splitmix64(seed_ ^ splitmix64(label ^ 0xa5a5a5a55a5a5a5aULL))); }

// ---------------------------------------------------------------------------
// NttTables::init (ring.hpp:25-51)
// ---------------------------------------------------------------------------
static u32 reverse_bits(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
    return r;
}

void NttTables::init(u64 modulus, u32 degree, Rng& rng) {
    q = modulus;
    u32 logn = 0;
    while ((1u << logn) < degree) ++logn;
    const u64 two_n = 2 * u64(degree);
    if ((q - 1) % two_n != 0) throw TetrisError("ring", "modulus lacks a 2N-th root of unity");
    do {
        u64 x = rng.uniform(q - 2) + 2;
        psi = pow_mod(x, (q - 1) / two_n, q);
    } while (pow_mod(psi, degree, q) != q - 1);
    const u64 psi_inv = inv_mod(psi, q);
    w.assign(degree, 0);
    winv.assign(degree, 0);
    w_shoup.assign(degree, 0);
    winv_shoup.assign(degree, 0);
    for (u32 i = 0; i < degree; ++i) {
        const u32 e = reverse_bits(i, logn);
        w[i] = pow_mod(psi, e, q);
        winv[i] = pow_mod(psi_inv, e, q);
        w_shoup[i] = shoup_precompute(w[i], q);
        winv_shoup[i] = shoup_precompute(winv[i], q);
    }
    n_inv = inv_mod(degree, q);
    n_inv_shoup = shoup_precompute(n_inv, q);
}

// ---------------------------------------------------------------------------
// RingParams (ring.hpp:118-140)
// ---------------------------------------------------------------------------
static int g_default_device = 0;
void set_default_device(int device) { g_default_device = device; }
int default_device() { return g_default_device; }

RingParams::RingParams(u32 degree, std::vector<u64> moduli, u32 special_count)
    : degree_(degree), moduli_(std::move(moduli)), special_count_(special_count), device_(g_default_device) {
    if (degree_ < 16 || (degree_ & (degree_ - 1)) != 0) throw TetrisError("ring", "degree must be a power of two >= 16");
    if (moduli_.empty() || special_count_ >= moduli_.size())
        throw TetrisError("ring", "need at least one non-special prime");
    log_degree_ = 0;
    while ((1u << log_degree_) < degree_) ++log_degree_;
    for (std::size_t i = 0; i < moduli_.size(); ++i) {
        if (!is_prime_u64(moduli_[i]) || moduli_[i] >= (u64(1) << 62))
            throw TetrisError("ring", "moduli must be primes below 2^62");
        for (std::size_t j = 0; j < i; ++j)
            if (moduli_[j] == moduli_[i]) throw TetrisError("ring", "moduli must be distinct");
    }
    Rng root(0x7e7215a1d2c3ULL);  // the reference's table seed: tables are canonical per modulus
    tables_.resize(moduli_.size());
    for (std::size_t i = 0; i < moduli_.size(); ++i) {
        Rng r = root.split(i);
        tables_[i].init(moduli_[i], degree_, r);
    }
    build_eval_order_map();
}

// The forward transform leaves a(psi^(2*brv(j)+1)) in slot j (CT with
// psi^brv twiddles). The reference probes this map by transforming X
// (ring.hpp:165-186); tests check the closed form against that probe.
void RingParams::build_eval_order_map() {
    eval_exp_.assign(degree_, 0);
    slot_of_exp_.assign(2 * size_t(degree_), u32(-1));
    for (u32 j = 0; j < degree_; ++j) {
        const u32 e = 2 * reverse_bits(j, log_degree_) + 1;
        eval_exp_[j] = e;
        slot_of_exp_[e] = j;
    }
}

double RingParams::total_log2_q(int level) const {
    double s = 0;
    for (int i = 0; i <= level; ++i) s += std::log2(double(moduli_[i]));
    return s;
}

DeviceState::~DeviceState() {
    if (ctx) {
        for (void* s : workers) {
            tg_stream_sync(ctx, s);
            tg_stream_destroy(ctx, s);
        }
        tg_stream_sync(ctx, stream);
        tg_stream_destroy(ctx, stream);
        tg_context_destroy(ctx);
    }
}

void* DeviceState::worker_stream(std::size_t i) {
    std::lock_guard<std::mutex> g(mu);
    while (workers.size() <= i) {
        void* s = nullptr;
        check_tg(tg_stream_create(ctx, &s));
        workers.push_back(s);
    }
    return workers[i];
}

namespace {
thread_local const void* t_override_state = nullptr;
thread_local void* t_override_stream = nullptr;
}  // namespace

StreamScope::StreamScope(const RingParams& ring, void* stream)
    : prev_state_(t_override_state), prev_stream_(t_override_stream) {
    t_override_state = ring.device_state().get();
    t_override_stream = stream;
}

StreamScope::~StreamScope() {
    t_override_state = prev_state_;
    t_override_stream = prev_stream_;
}

const std::shared_ptr<DeviceState>& RingParams::device_state() const {
    std::call_once(dev_once_, [this] {
        const u32 nmod = u32(moduli_.size());
        std::vector<u64> tw(size_t(4) * nmod * degree_);
        std::vector<u64> ninv(2 * size_t(nmod));
        for (u32 i = 0; i < nmod; ++i) {
            const NttTables& t = tables_[i];
            u64* base = tw.data() + size_t(4) * i * degree_;
            std::copy(t.w.begin(), t.w.end(), base);
            std::copy(t.w_shoup.begin(), t.w_shoup.end(), base + degree_);
            std::copy(t.winv.begin(), t.winv.end(), base + 2 * size_t(degree_));
            std::copy(t.winv_shoup.begin(), t.winv_shoup.end(), base + 3 * size_t(degree_));
            ninv[2 * i] = t.n_inv;
            ninv[2 * i + 1] = t.n_inv_shoup;
        }
        auto st = std::make_shared<DeviceState>();
        check_tg(tg_context_create(&st->ctx, device_, degree_, moduli_.data(), nmod, special_count_, tw.data(),
                                   ninv.data(), eval_exp_.data(), slot_of_exp_.data()));
        check_tg(tg_stream_create(st->ctx, &st->stream));
        dev_ = std::move(st);
    });
    if (!dev_) throw TetrisError("gpu", "device context unavailable");
    return dev_;
}

tg_context* RingParams::dev() const { return device_state()->ctx; }

void* RingParams::stream() const {
    const auto& st = device_state();
    return t_override_state == st.get() ? t_override_stream : st->stream;
}

void RingParams::synchronize() const { check_tg(tg_stream_sync(dev(), stream())); }

RingParams::~RingParams() = default;

// ---------------------------------------------------------------------------
// Device storage and Poly
// ---------------------------------------------------------------------------
DeviceBuffer::DeviceBuffer(const RingParams& ring, std::size_t words)
    : dev_(ring.device_state()), stream_(ring.stream()), words_(words) {
    void* p = nullptr;
    check_tg(tg_alloc(dev_->ctx, &p, words * 8, stream_));
    ptr_ = static_cast<u64*>(p);
}

std::shared_ptr<DeviceBuffer> DeviceBuffer::find_eval(std::size_t off, int level, int nspecial, int nparts,
                                                      void* stream) const {
    std::lock_guard<std::mutex> g(cache_mu_);
    for (const auto& e : cache_)
        if (e.off == off && e.level == level && e.nspecial == nspecial && e.nparts == nparts && e.stream == stream)
            return e.buf;
    return nullptr;
}

void DeviceBuffer::put_eval(std::size_t off, int level, int nspecial, int nparts, void* stream,
                            std::shared_ptr<DeviceBuffer> buf) const {
    std::lock_guard<std::mutex> g(cache_mu_);
    if (cache_.size() >= 4) cache_.erase(cache_.begin());
    cache_.push_back(EvalCache{off, level, nspecial, nparts, stream, std::move(buf)});
}

void DeviceBuffer::clear_eval_cache() const {
    std::lock_guard<std::mutex> g(cache_mu_);
    cache_.clear();
}

// Freed on the destroying thread's current stream: ordered after that
// thread's uses; buffers crossing threads are handed over only after the
// producing stream was synchronized (see eval_private_threshold_many).
DeviceBuffer::~DeviceBuffer() {
    if (!ptr_) return;
    void* s = t_override_state == dev_.get() ? t_override_stream : dev_->stream;
    tg_free(dev_->ctx, ptr_, s);
}

Poly::Poly(const RingParams& ring, int level, Form form, int nspecial)
    : ring_(&ring), level_(level), nspecial_(nspecial), form_(form) {
    if (level < 0 || level > ring.max_level()) throw TetrisError("ring", "poly level out of range");
    if (nspecial != 0 && nspecial != int(ring.special_count()))
        throw TetrisError("ring", "special rows must be all-or-none");
    st_ = std::make_shared<DeviceBuffer>(ring, words());
    check_tg(tg_memset0(ring.dev(), st_->data(), words() * 8, ring.stream()));
}

Poly Poly::view(const RingParams& ring, std::shared_ptr<DeviceBuffer> st, std::size_t off, int level, Form form,
                int nspecial) {
    Poly p;
    p.ring_ = &ring;
    p.level_ = level;
    p.nspecial_ = nspecial;
    p.form_ = form;
    p.st_ = std::move(st);
    p.off_ = off;
    return p;
}

u64* Poly::mutable_data() {
    if (st_.use_count() > 1) {  // copy-on-write
        auto fresh = std::make_shared<DeviceBuffer>(*ring_, words());
        check_tg(tg_memcpy_d2d(ring_->dev(), fresh->data(), st_->data() + off_, words() * 8, ring_->stream()));
        st_ = std::move(fresh);
        off_ = 0;
    } else {
        st_->clear_eval_cache();  // written in place: a memoised transform of the old contents is stale
    }
    return st_->data() + off_;
}

std::vector<u64> Poly::to_host() const {
    std::vector<u64> out(words());
    to_host(out.data());
    return out;
}

void Poly::to_host(u64* dst) const {
    check_tg(tg_memcpy_d2h(ring_->dev(), dst, data(), words() * 8, ring_->stream()));
    ring_->synchronize();
}

Poly Poly::from_host(const RingParams& ring, const u64* src, int level, Form form, int nspecial) {
    if (level < 0 || level > ring.max_level()) throw TetrisError("ring", "poly level out of range");
    if (nspecial != 0 && nspecial != int(ring.special_count()))
        throw TetrisError("ring", "special rows must be all-or-none");
    const std::size_t words = std::size_t(level + 1 + nspecial) * ring.degree();
    auto st = std::make_shared<DeviceBuffer>(ring, words);
    check_tg(tg_memcpy_h2d(ring.dev(), st->data(), src, words * 8, ring.stream()));
    // the source may be a temporary: complete the copy before returning
    ring.synchronize();
    return view(ring, std::move(st), 0, level, form, nspecial);
}

Poly Poly::from_host(const RingParams& ring, const std::vector<u64>& src, int level, Form form, int nspecial) {
    const std::size_t words = std::size_t(level + 1 + nspecial) * ring.degree();
    if (src.size() != words) throw TetrisError("ring", "from_host: size mismatch");
    return from_host(ring, src.data(), level, form, nspecial);
}

void Poly::ntt_forward() {
    if (form_ != Form::coeff) throw TetrisError("ring", "ntt_forward expects coeff form");
    check_tg(tg_ntt_forward(ring_->dev(), mutable_data(), level_, nspecial_, 1, ring_->stream()));
    form_ = Form::eval;
}

void Poly::ntt_inverse() {
    if (form_ != Form::eval) throw TetrisError("ring", "ntt_inverse expects eval form");
    check_tg(tg_ntt_inverse(ring_->dev(), mutable_data(), level_, nspecial_, 1, ring_->stream()));
    form_ = Form::coeff;
}

void Poly::check_shape(const Poly& o) const {
    if (ring_ != o.ring_ || level_ != o.level_ || nspecial_ != o.nspecial_ || form_ != o.form_)
        throw TetrisError("ring", "poly shape mismatch");
}

void Poly::add_inplace(const Poly& o) {
    check_shape(o);
    const u64* b = o.data();
    u64* d = mutable_data();
    check_tg(tg_poly_addsub(ring_->dev(), d, d, b, 0, level_, nspecial_, 1, ring_->stream()));
}

void Poly::sub_inplace(const Poly& o) {
    check_shape(o);
    const u64* b = o.data();
    u64* d = mutable_data();
    check_tg(tg_poly_addsub(ring_->dev(), d, d, b, 1, level_, nspecial_, 1, ring_->stream()));
}

void Poly::negate_inplace() {
    u64* d = mutable_data();
    check_tg(tg_poly_addsub(ring_->dev(), d, d, d, 2, level_, nspecial_, 1, ring_->stream()));
}

void Poly::mul_pointwise_inplace(const Poly& o) {
    if (form_ != Form::eval || o.form_ != Form::eval) throw TetrisError("ring", "pointwise product expects eval form");
    check_shape(o);
    const u64* b = o.data();
    u64* d = mutable_data();
    check_tg(tg_poly_mul(ring_->dev(), d, d, b, level_, nspecial_, 1, ring_->stream()));
}

void Poly::mul_acc_pointwise(const Poly& x, const Poly& y) {
    if (form_ != Form::eval || x.form_ != Form::eval || y.form_ != Form::eval)
        throw TetrisError("ring", "mul_acc expects eval form");
    check_shape(x);
    check_shape(y);
    const u64 *a = x.data(), *b = y.data();
    u64* d = mutable_data();
    check_tg(tg_poly_mul_acc(ring_->dev(), d, a, b, level_, nspecial_, 1, ring_->stream()));
}

void Poly::mul_scalar_inplace(const std::vector<u64>& scalar_per_modulus) {
    if (scalar_per_modulus.size() < ring_->moduli().size()) throw TetrisError("ring", "scalar table too short");
    u64* d = mutable_data();
    check_tg(tg_poly_mul_scalar(ring_->dev(), d, d, scalar_per_modulus.data(), level_, nspecial_, 1, ring_->stream()));
}

void Poly::mul_small_scalar_inplace(u64 s) {
    std::vector<u64> per(ring_->moduli().size(), s);
    mul_scalar_inplace(per);
}

void Poly::drop_to_level(int new_level) {
    if (new_level > level_) throw TetrisError("ring", "drop_to_level cannot raise");
    if (nspecial_ != 0) throw TetrisError("ring", "drop_to_level with special rows");
    level_ = new_level;  // rows 0..new_level are a prefix of the view
}

void Poly::drop_special() { nspecial_ = 0; }

// ---------------------------------------------------------------------------
// Free operations (ring.hpp:380-518)
// ---------------------------------------------------------------------------
Poly poly_add(const Poly& a, const Poly& b) {
    Poly r = a;
    r.add_inplace(b);
    return r;
}
Poly poly_sub(const Poly& a, const Poly& b) {
    Poly r = a;
    r.sub_inplace(b);
    return r;
}
Poly ntt_transform(const Poly& p, Form target) {
    Poly r = p;
    if (target == Form::eval) r.ntt_forward();
    else r.ntt_inverse();
    return r;
}
Poly poly_mul(const Poly& a, const Poly& b) {
    Poly x = a, y = b;
    if (x.form() == Form::coeff) x.ntt_forward();
    if (y.form() == Form::coeff) y.ntt_forward();
    x.mul_pointwise_inplace(y);
    x.ntt_inverse();
    return x;
}

Poly automorphism_apply(const Poly& p, u64 exponent) {
    const RingParams& ring = p.ring();
    const u64 g = exponent % (2 * u64(ring.degree()));
    if (g % 2 == 0) throw TetrisError("ring", "automorphism exponent must be odd");
    auto st = std::make_shared<DeviceBuffer>(ring, p.words());
    check_tg(tg_automorphism(ring.dev(), st->data(), p.data(), g, p.form() == Form::eval ? TG_FORM_EVAL : TG_FORM_COEFF,
                             p.level(), p.nspecial(), 1, ring.stream()));
    return Poly::view(ring, std::move(st), 0, p.level(), p.form(), p.nspecial());
}

Poly mul_monomial(const Poly& p, u32 e) {
    if (p.form() != Form::coeff) throw TetrisError("ring", "mul_monomial expects coeff form");
    const RingParams& ring = p.ring();
    auto st = std::make_shared<DeviceBuffer>(ring, p.words());
    check_tg(tg_mul_monomial(ring.dev(), st->data(), p.data(), e % (2 * ring.degree()), p.level(), p.nspecial(), 1,
                             ring.stream()));
    return Poly::view(ring, std::move(st), 0, p.level(), Form::coeff, p.nspecial());
}

Poly raise_level(const Poly& p, int new_level, int nspecial) {
    if (p.level() != 0 || p.nspecial() != 0) throw TetrisError("ring", "raise_level expects a level-0 poly");
    if (p.form() != Form::coeff) throw TetrisError("ring", "raise_level expects coeff form");
    const RingParams& ring = p.ring();
    if (new_level < 0 || new_level > ring.max_level()) throw TetrisError("ring", "poly level out of range");
    auto st = std::make_shared<DeviceBuffer>(ring, std::size_t(new_level + 1 + nspecial) * ring.degree());
    check_tg(tg_raise_level(ring.dev(), st->data(), p.data(), new_level, nspecial, 1, ring.stream()));
    return Poly::view(ring, std::move(st), 0, new_level, Form::coeff, nspecial);
}

Poly rescale_round(const Poly& p) {
    if (p.level() < 1) throw TetrisError("ring", "cannot rescale at level 0");
    if (p.nspecial() != 0) throw TetrisError("ring", "rescale with special rows");
    if (p.form() != Form::coeff) throw TetrisError("ring", "rescale expects coeff form");
    const RingParams& ring = p.ring();
    auto st = std::make_shared<DeviceBuffer>(ring, std::size_t(p.level()) * ring.degree());
    check_tg(tg_rescale(ring.dev(), st->data(), p.data(), p.level(), 1, ring.stream()));
    return Poly::view(ring, std::move(st), 0, p.level() - 1, Form::coeff, 0);
}

// ---------------------------------------------------------------------------
// Samplers (ring.hpp:442-487): host draws, device residues
// ---------------------------------------------------------------------------
std::vector<u64> sample_uniform_host(const RingParams& ring, int level, int nspecial, Rng& rng) {
    const u32 n = ring.degree();
    const int rows = level + 1 + nspecial;
    std::vector<u64> v(std::size_t(rows) * n);
    for (int r = 0; r < rows; ++r) {
        const u32 m = r <= level ? u32(r) : ring.q_count() + u32(r - level - 1);
        const u64 q = ring.modulus(m);
        u64* row = v.data() + std::size_t(r) * n;
        for (u32 i = 0; i < n; ++i) row[i] = rng.uniform(q);
    }
    return v;
}

Poly sample_uniform(const RingParams& ring, int level, int nspecial, Rng& rng) {
    return Poly::from_host(ring, sample_uniform_host(ring, level, nspecial, rng), level, Form::coeff, nspecial);
}

Poly poly_from_i64(const RingParams& ring, const std::vector<i64>& coeffs, int level, int nspecial) {
    const u32 n = ring.degree();
    const int rows = level + 1 + nspecial;
    std::vector<u64> v(std::size_t(rows) * n, 0);
    const std::size_t cnt = std::min<std::size_t>(n, coeffs.size());
    for (int r = 0; r < rows; ++r) {
        const u32 m = r <= level ? u32(r) : ring.q_count() + u32(r - level - 1);
        const u64 q = ring.modulus(m);
        u64* row = v.data() + std::size_t(r) * n;
        for (std::size_t i = 0; i < cnt; ++i) row[i] = from_centered(coeffs[i], q);
    }
    return Poly::from_host(ring, v, level, Form::coeff, nspecial);
}

std::vector<i64> sample_gaussian_coeffs(u32 n, double sigma, Rng& rng) {
    if (sigma <= 0) throw TetrisError("ring", "sigma must be positive");
    const i64 tail = round_half_away(6.0 * sigma);
    std::vector<i64> c(n);
    for (u32 i = 0; i < n; ++i) c[i] = std::clamp(round_half_away(rng.normal() * sigma), -tail, tail);
    return c;
}

Poly sample_gaussian(const RingParams& ring, double sigma, int level, int nspecial, Rng& rng) {
    return poly_from_i64(ring, sample_gaussian_coeffs(ring.degree(), sigma, rng), level, nspecial);
}

std::vector<i64> sample_ternary_coeffs(u32 n, u32 h, Rng& rng) {
    if (h > n) throw TetrisError("ring", "hamming weight exceeds degree");
    std::vector<u32> perm(n);
    for (u32 i = 0; i < n; ++i) perm[i] = i;
    std::vector<i64> c(n, 0);
    for (u32 i = 0; i < h; ++i) {
        const u32 j = i + u32(rng.uniform(n - i));
        std::swap(perm[i], perm[j]);
        c[perm[i]] = rng.uniform(2) ? 1 : -1;
    }
    return c;
}

Poly sample_ternary_hw(const RingParams& ring, u32 h, int level, int nspecial, Rng& rng) {
    return poly_from_i64(ring, sample_ternary_coeffs(ring.degree(), h, rng), level, nspecial);
}

}  // namespace tetris_b200
