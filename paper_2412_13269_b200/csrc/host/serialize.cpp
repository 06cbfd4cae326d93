// TTRS wire formats (reference serialize.hpp). Poly bytes move with one
// device copy per poly; everything else is host metadata.
#include <bit>
#include <cstring>

#include "internal.hpp"
#include "tetris_b200/serialize.hpp"

namespace tetris_b200 {

namespace {

constexpr u32 kMagic = 0x54545253;  // "TTRS"
constexpr u16 kVersion = 1;

struct Writer {
    std::vector<uint8_t> buf;
    void raw(const void* p, std::size_t n) {
        const auto* b = static_cast<const uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);  // little-endian hosts
    }
    void u8(uint8_t v) { buf.push_back(v); }
    void u16v(u16 v) { raw(&v, 2); }
    void u32v(u32 v) { raw(&v, 4); }
    void u64v(u64 v) { raw(&v, 8); }
    void i64v(i64 v) { raw(&v, 8); }
    void f64(double v) { u64v(std::bit_cast<u64>(v)); }
};

struct Reader {
    const uint8_t* p;
    const uint8_t* end;
    explicit Reader(const std::vector<uint8_t>& v) : p(v.data()), end(v.data() + v.size()) {}
    const uint8_t* take(std::size_t n) {
        if (p + n > end) throw TetrisError("serialize", "truncated input");
        const uint8_t* r = p;
        p += n;
        return r;
    }
    template <class T>
    T get() {
        T v;
        std::memcpy(&v, take(sizeof(T)), sizeof(T));
        return v;
    }
    std::size_t left() const { return std::size_t(end - p); }
    // a count read from the input must fit the bytes that are left, each item
    // taking at least `min_item` bytes, before anything is allocated for it
    u32 count(std::size_t min_item) {
        const u32 n = u32v();
        if (min_item && std::size_t(n) > left() / min_item) throw TetrisError("serialize", "truncated input");
        return n;
    }
    uint8_t u8() { return *take(1); }
    u16 u16v() { return get<u16>(); }
    u32 u32v() { return get<u32>(); }
    u64 u64v() { return get<u64>(); }
    i64 i64v() { return get<i64>(); }
    double f64() { return std::bit_cast<double>(get<u64>()); }
};

void write_header(Writer& w, ObjectKind kind, const RingParams& ring) {
    w.u32v(kMagic);
    w.u16v(kVersion);
    w.u16v(u16(kind));
    w.u32v(ring.degree());
    w.u32v(u32(ring.moduli().size()));
    w.u32v(ring.special_count());
    for (u64 q : ring.moduli()) w.u64v(q);
}

ObjectKind read_header(Reader& r, const RingParams& ring) {
    if (r.u32v() != kMagic) throw TetrisError("serialize", "bad magic");
    if (r.u16v() != kVersion) throw TetrisError("serialize", "unsupported version");
    const ObjectKind kind = ObjectKind(r.u16v());
    if (r.u32v() != ring.degree()) throw TetrisError("serialize", "ring degree mismatch");
    const u32 nmod = r.u32v(), nspecial = r.u32v();
    if (nmod != ring.moduli().size() || nspecial != ring.special_count())
        throw TetrisError("serialize", "modulus chain mismatch");
    for (u32 i = 0; i < nmod; ++i)
        if (r.u64v() != ring.modulus(i)) throw TetrisError("serialize", "modulus value mismatch");
    return kind;
}

std::size_t header_size(const RingParams& ring) { return 20 + 8 * ring.moduli().size(); }

void write_poly(Writer& w, const Poly& p) {
    w.u32v(u32(p.level()));
    w.u32v(u32(p.nspecial()));
    w.u8(p.form() == Form::eval ? 1 : 0);
    const std::size_t at = w.buf.size(), bytes = p.words() * 8;
    w.buf.resize(at + bytes);
    p.to_host(reinterpret_cast<u64*>(w.buf.data() + at));  // rows back to back, as the reference writes them
}

Poly read_poly(Reader& r, const RingParams& ring) {
    const int level = int(r.u32v()), nspecial = int(r.u32v());
    const Form form = r.u8() ? Form::eval : Form::coeff;
    if (level < 0 || level > ring.max_level() || (nspecial != 0 && u32(nspecial) != ring.special_count()))
        throw TetrisError("serialize", "poly shape out of range");
    const std::size_t words = std::size_t(level + 1 + nspecial) * ring.degree();
    std::vector<u64> h(words);
    std::memcpy(h.data(), r.take(words * 8), words * 8);
    return Poly::from_host(ring, h, level, form, nspecial);
}

std::size_t poly_size(const RingParams& ring, int level, int nspecial) {
    return 9 + std::size_t(level + 1 + nspecial) * ring.degree() * 8;
}

void write_switching_key_body(Writer& w, const SwitchingKey& k) {
    w.u32v(k.gadget.group_size);
    w.u32v(k.gadget.base2_bits);
    w.u64v(k.from_id);
    w.u64v(k.to_id);
    w.u64v(k.a_seed);
    w.u32v(u32(k.b.size()));
    for (const Poly& p : k.b) write_poly(w, p);
}

SwitchingKey read_switching_key_body(Reader& r, const RingParams& ring) {
    SwitchingKey k;
    k.gadget.group_size = r.u32v();
    k.gadget.base2_bits = r.u32v();
    k.from_id = r.u64v();
    k.to_id = r.u64v();
    k.a_seed = r.u64v();
    const int lvl = ring.max_level(), ksp = int(ring.special_count());
    const u32 n = r.count(poly_size(ring, lvl, ksp));  // before the 2*w*n-word device block
    const std::size_t w = std::size_t(lvl + 1 + ksp) * ring.degree();
    k.block = detail::new_block(ring, 2 * w * n);  // the device layout [digit][b|a][rows][N]
    Rng ra(k.a_seed);
    for (u32 i = 0; i < n; ++i) {
        Poly b = read_poly(r, ring);
        if (b.level() != lvl || b.nspecial() != ksp || b.form() != Form::eval)
            throw TetrisError("serialize", "switching key part has the wrong shape");
        Rng ri = ra.split(i);  // regenerate the a-part from the stored seed
        Poly a = sample_uniform(ring, lvl, ksp, ri);
        a.ntt_forward();
        u64* dst = k.block->data() + 2 * w * i;
        check_tg(tg_memcpy_d2d(ring.dev(), dst, b.data(), w * 8, ring.stream()));
        check_tg(tg_memcpy_d2d(ring.dev(), dst + w, a.data(), w * 8, ring.stream()));
        k.b.push_back(Poly::view(ring, k.block, 2 * w * i, lvl, Form::eval, ksp));
        k.a.push_back(Poly::view(ring, k.block, 2 * w * i + w, lvl, Form::eval, ksp));
    }
    ring.synchronize();
    return k;
}

}  // namespace

std::vector<uint8_t> serialize_ciphertext(const Ciphertext& ct) {
    if (ct.batch != 1) throw TetrisError("serialize", "serialize a single ciphertext (unstack the batch)");
    Writer w;
    write_header(w, ObjectKind::ciphertext, ct.ring());
    w.u32v(u32(ct.parts.size()));
    w.f64(ct.scale);
    w.u8(ct.domain == Domain::slots ? 1 : 0);
    w.u64v(ct.sk_id);
    w.f64(ct.noise_bound);
    for (const Poly& p : ct.parts) write_poly(w, p);
    return std::move(w.buf);
}

Ciphertext deserialize_ciphertext(const std::vector<uint8_t>& buf, const RingParams& ring) {
    Reader r(buf);
    if (read_header(r, ring) != ObjectKind::ciphertext) throw TetrisError("serialize", "object kind mismatch");
    Ciphertext ct;
    const u32 parts = r.count(poly_size(ring, 0, 0));
    ct.scale = r.f64();
    ct.domain = r.u8() ? Domain::slots : Domain::coeffs;
    ct.sk_id = r.u64v();
    ct.noise_bound = r.f64();
    for (u32 i = 0; i < parts; ++i) ct.parts.push_back(read_poly(r, ring));
    return ct;
}

std::size_t ciphertext_size(const RingParams& ring, int level, u32 parts) {
    return header_size(ring) + 29 + parts * poly_size(ring, level, 0);
}

std::vector<uint8_t> serialize_switching_key(const SwitchingKey& k) {
    Writer w;
    write_header(w, ObjectKind::switching_key, k.ring());
    write_switching_key_body(w, k);
    return std::move(w.buf);
}

SwitchingKey deserialize_switching_key(const std::vector<uint8_t>& buf, const RingParams& ring) {
    Reader r(buf);
    if (read_header(r, ring) != ObjectKind::switching_key) throw TetrisError("serialize", "object kind mismatch");
    return read_switching_key_body(r, ring);
}

std::vector<uint8_t> serialize_chain(const MinimaxChain& c) {
    Writer w;
    w.u32v(kMagic);
    w.u16v(kVersion);
    w.u16v(u16(ObjectKind::chain));
    w.u32v(c.params.alpha);
    w.u32v(c.params.beta);
    w.f64(c.params.epsilon);
    w.u32v(u32(c.params.degrees.size()));
    for (u32 d : c.params.degrees) w.u32v(d);
    w.f64(c.sign_error);
    w.f64(c.achieved_beta);
    w.u32v(u32(c.stages.size()));
    for (const auto& st : c.stages) {
        w.u32v(st.degree);
        w.f64(st.gamma);
        w.f64(st.upper);
        w.f64(st.error);
        w.u32v(u32(st.cheb.size()));
        for (double x : st.cheb) w.f64(x);
    }
    return std::move(w.buf);
}

MinimaxChain deserialize_chain(const std::vector<uint8_t>& buf) {
    Reader r(buf);
    if (r.u32v() != kMagic) throw TetrisError("serialize", "bad magic");
    if (r.u16v() != kVersion) throw TetrisError("serialize", "unsupported version");
    if (ObjectKind(r.u16v()) != ObjectKind::chain) throw TetrisError("serialize", "object kind mismatch");
    MinimaxChain c;
    c.params.alpha = r.u32v();
    c.params.beta = r.u32v();
    c.params.epsilon = r.f64();
    const u32 nd = r.count(4);
    for (u32 i = 0; i < nd; ++i) c.params.degrees.push_back(r.u32v());
    c.sign_error = r.f64();
    c.achieved_beta = r.f64();
    const u32 ns = r.count(32);
    for (u32 i = 0; i < ns; ++i) {
        ChainStage st;
        st.degree = r.u32v();
        st.gamma = r.f64();
        st.upper = r.f64();
        st.error = r.f64();
        st.cheb.resize(r.count(8));
        for (auto& x : st.cheb) x = r.f64();
        c.stages.push_back(std::move(st));
    }
    return c;
}

std::vector<uint8_t> serialize_secret_key(const SecretKey& sk) {
    Writer w;
    write_header(w, ObjectKind::secret_key, sk.ring());
    w.u64v(sk.id());
    w.u32v(u32(sk.coeffs().size()));
    for (i64 c : sk.coeffs()) w.i64v(c);
    return std::move(w.buf);
}

SecretKey deserialize_secret_key(const std::vector<uint8_t>& buf, const RingParams& ring) {
    Reader r(buf);
    if (read_header(r, ring) != ObjectKind::secret_key) throw TetrisError("serialize", "object kind mismatch");
    const u64 id = r.u64v();
    std::vector<i64> c(r.count(8));
    for (auto& x : c) x = r.i64v();
    return SecretKey(ring, std::move(c), id);
}

}  // namespace tetris_b200
