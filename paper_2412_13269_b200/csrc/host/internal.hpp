// Host-internal helpers: ciphertext-part blocks (several polys of one shape
// back to back in one HBM allocation) so that per-part ops launch once.
#pragma once
#include <cstdlib>

#include "tetris_b200/keys.hpp"

namespace tetris_b200::detail {

inline std::shared_ptr<DeviceBuffer> new_block(const RingParams& ring, std::size_t words) {
    return std::make_shared<DeviceBuffer>(ring, words);
}

// `n` views of shape (level, form, nspecial) over a fresh block.
inline std::vector<Poly> fresh_parts(const RingParams& ring, int n, int level, Form form, int nspecial = 0) {
    const std::size_t w = std::size_t(level + 1 + nspecial) * ring.degree();
    auto blk = new_block(ring, w * std::size_t(n));
    std::vector<Poly> out;
    out.reserve(n);
    for (int i = 0; i < n; ++i) out.push_back(Poly::view(ring, blk, w * i, level, form, nspecial));
    return out;
}

// Parts that share one block at a uniform stride (keys.cpp): the stride in
// words, 0 if the parts are not laid out that way.
std::size_t uniform_stride(const std::vector<Poly>& parts);

// True if parts[first..first+n) have one shape and sit back to back in one block.
inline bool contiguous(const std::vector<Poly>& parts, std::size_t first, std::size_t n) {
    if (n == 0 || first + n > parts.size()) return false;
    const Poly& p0 = parts[first];
    for (std::size_t i = 1; i < n; ++i) {
        const Poly& p = parts[first + i];
        if (p.storage() != p0.storage() || p.level() != p0.level() || p.nspecial() != p0.nspecial() ||
            p.form() != p0.form() || p.offset() != p0.offset() + i * p0.words())
            return false;
    }
    return true;
}

// True if the parts are contiguous AND nothing outside them references the block.
inline bool exclusively_owned(const std::vector<Poly>& parts) {
    return contiguous(parts, 0, parts.size()) && parts[0].storage().use_count() == long(parts.size());
}

inline int tg_form(Form f) { return f == Form::eval ? TG_FORM_EVAL : TG_FORM_COEFF; }

// Device pointer to parts[first..first+n) back to back: the parts' own
// storage when they already are, else a gathered copy kept alive in `keep`.
inline const u64* group_data(const std::vector<Poly>& parts, std::size_t first, std::size_t n,
                             std::vector<Poly>& keep) {
    if (n == 1 || contiguous(parts, first, n)) return parts[first].data();
    const Poly& p0 = parts[first];
    const RingParams& ring = p0.ring();
    std::vector<Poly> g = fresh_parts(ring, int(n), p0.level(), p0.form(), p0.nspecial());
    std::vector<const u64*> srcs(n);
    for (std::size_t i = 0; i < n; ++i) {
        parts[first + i].check_shape(p0);
        srcs[i] = parts[first + i].data();
    }
    check_tg(tg_gather_polys(ring.dev(), const_cast<u64*>(g[0].data()), srcs.data(), u32(n), g[0].words(),
                             ring.stream()));  // one launch for the group
    keep.insert(keep.end(), g.begin(), g.end());
    return g[0].data();
}

// parts[first..first+n) as one group for a kernel that reads poly i at
// base + i * stride words: a contiguous group is tight (stride = words), the
// polys of a level-dropped batch view keep their block's stride and are read
// in place; anything else is gathered (tight copies kept alive in `keep`).
inline const u64* strided_group(const std::vector<Poly>& parts, std::size_t first, std::size_t n,
                                std::vector<Poly>& keep, u64& stride) {
    const Poly& p0 = parts[first];
    stride = p0.words();
    if (n == 1 || contiguous(parts, first, n)) return p0.data();
    bool uniform = parts[first + 1].storage() == p0.storage() && parts[first + 1].offset() > p0.offset();
    const std::size_t d = uniform ? parts[first + 1].offset() - p0.offset() : 0;
    for (std::size_t i = 0; i < n && uniform; ++i) {
        const Poly& p = parts[first + i];
        uniform = p.storage() == p0.storage() && p.level() == p0.level() && p.nspecial() == p0.nspecial() &&
                  p.form() == p0.form() && p.offset() == p0.offset() + i * d;
    }
    if (uniform && d >= p0.words()) {
        stride = d;
        return p0.data();
    }
    return group_data(parts, first, n, keep);
}

// Both part groups (c0 polys, c1 polys) of a degree-1 batch with ONE poly
// stride for the tensor entry points (op_strides); TG_OPERAND_STRIDES=0, or
// groups whose strides differ, fall back to tight gathered copies.
inline void operand_groups(const Ciphertext& c, u32 B, std::vector<Poly>& keep, const u64*& g0, const u64*& g1,
                           u64& stride) {
    static const bool off = [] {
        const char* e = std::getenv("TG_OPERAND_STRIDES");
        return e && *e == '0';
    }();
    u64 s0 = 0, s1 = 0;
    if (!off) {
        std::vector<Poly> k0;
        g0 = strided_group(c.parts, 0, B, k0, s0);
        g1 = strided_group(c.parts, B, B, k0, s1);
        if (s0 == s1 && k0.empty()) {
            stride = s0;
            return;
        }
    }
    g0 = group_data(c.parts, 0, B, keep);
    g1 = group_data(c.parts, B, B, keep);
    stride = c.parts[0].words();
}

// Applies a per-part kernel `fn(dst, src, npolys)` to all parts, writing one
// fresh contiguous block of shape (out_level, out_form): a single batched
// launch when the sources are contiguous, one launch per part otherwise.
// Keeping outputs contiguous keeps every downstream op batched.
// to_coeff() that leaves the eval-form source in the result's transform
// cache, so a later to_eval() of the result (the next product) is free.
void to_coeff_keep_eval(Ciphertext& ct);

template <class F>
std::vector<Poly> map_parts(const std::vector<Poly>& src, int out_level, Form out_form, F fn) {
    const Poly& p0 = src[0];
    const RingParams& ring = p0.ring();
    const std::size_t np = src.size();
    std::vector<Poly> dst = fresh_parts(ring, int(np), out_level, out_form, p0.nspecial());
    if (contiguous(src, 0, np)) {
        fn(const_cast<u64*>(dst[0].data()), p0.data(), u32(np));
    } else {
        for (std::size_t i = 0; i < np; ++i) fn(const_cast<u64*>(dst[i].data()), src[i].data(), 1u);
    }
    return dst;
}

// Binary variant: fn(dst, a, b, npolys).
template <class F>
std::vector<Poly> map_parts2(const std::vector<Poly>& a, const std::vector<Poly>& b, F fn) {
    const Poly& p0 = a[0];
    const RingParams& ring = p0.ring();
    const std::size_t np = a.size();
    std::vector<Poly> dst = fresh_parts(ring, int(np), p0.level(), p0.form(), p0.nspecial());
    if (contiguous(a, 0, np) && contiguous(b, 0, np)) {
        fn(const_cast<u64*>(dst[0].data()), p0.data(), b[0].data(), u32(np));
    } else {
        for (std::size_t i = 0; i < np; ++i) fn(const_cast<u64*>(dst[i].data()), a[i].data(), b[i].data(), 1u);
    }
    return dst;
}

}  // namespace tetris_b200::detail
