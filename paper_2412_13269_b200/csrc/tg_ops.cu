// Element-wise ring and CKKS residue kernels (HBM-bound, coalesced, one
// grid-stride pass per op). Each kernel cites the reference loop it replaces.
#include "tg_internal.cuh"
#include "tg_fp64.cuh"

namespace tg {
namespace {

constexpr u32 kThreads = 256;

inline u32 grid_for(size_t work) {
    // 148 SMs x 8 resident 256-thread blocks; grid-stride beyond that
    size_t b = (work + kThreads - 1) / kThreads;
    return u32(std::min<size_t>(b, size_t(148) * 8 * 4));
}

struct Shape {
    u32 rpp;  // rows per poly
    int level;
    u64 words;  // total words
};

__device__ __forceinline__ u32 row_mod(const DevRing& R, const Shape& S, u64 idx) {
    const u32 row = u32(idx >> R.logN);
    return mod_index(row % S.rpp, S.level, R.q_count);
}

// Poly::add_inplace / sub_inplace / negate_inplace (ring.hpp:250-276)
__global__ void k_addsub(DevRing R, Shape S, u64* out, const u64* a, const u64* b, int op) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 q = R.q[row_mod(R, S, i)];
        const u64 x = a[i];
        u64 r;
        if (op == 0) r = add_mod(x, b[i], q);
        else if (op == 1) r = sub_mod(x, b[i], q);
        else r = neg_mod(x, q);
        out[i] = r;
    }
}

// add/sub of level-dropped views: operand poly p starts at p * stride (words),
// the output is packed.
__global__ void k_addsub_strided(DevRing R, Shape S, u64* out, const u64* a, u64 sa, const u64* b, u64 sb, int op) {
    const u64 per = u64(S.rpp) * R.N;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i / per, w = i - p * per;
        const u64 q = R.q[row_mod(R, S, i)];
        const u64 x = a[p * sa + w], y = b[p * sb + w];
        out[i] = op == 0 ? add_mod(x, y, q) : sub_mod(x, y, q);
    }
}

// Poly::mul_pointwise_inplace (ring.hpp:278-288) and mul_acc_pointwise (:290-304)
__global__ void k_mul(DevRing R, Shape S, u64* out, const u64* a, const u64* b, int acc) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        const u64 q = R.q[m];
        u64 r;
        if (q < kFpMaxQ) {  // exact FP64 product (tg_fp64.cuh)
            const double qd = R.qd[4 * m];
            r = fp_canonical1(fp_mulmod_qi(u2d(a[i]), u2d(b[i]), qd, R.qd[4 * m + 1]), qd);
        } else {
            r = mul_mod(a[i], b[i], q, R.ratio[2 * m], R.ratio[2 * m + 1]);
        }
        if (acc) r = add_mod(out[i], r, q);
        out[i] = r;
    }
}

struct Scalars {
    u64 s[kMaxMod];
    u64 ss[kMaxMod];
};

// Poly::mul_scalar_inplace (ring.hpp:307-315): Shoup with per-modulus scalar
__global__ void k_mul_scalar(DevRing R, Shape S, u64* out, const u64* a, Scalars sc) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        out[i] = shoup(a[i], sc.s[m], sc.ss[m], R.q[m]);
    }
}

// Evaluator::add_scalar residue update (ckks.hpp:299-311)
__global__ void k_add_scalar(DevRing R, Shape S, u64* out, const u64* a, Scalars sc, int eval_form) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        u64 v = a[i];
        if (eval_form || (i & (R.N - 1)) == 0) v = add_mod(v, sc.s[m], R.q[m]);
        out[i] = v;
    }
}

// automorphism_apply, coefficient form (ring.hpp:417-427): signed scatter
__global__ void k_auto_coeff(DevRing R, Shape S, u64* out, const u64* in, u64 g) {
    const u64 two_n = 2 * u64(R.N);
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 row_off = i & ~u64(R.N - 1);
        const u64 c = i & (R.N - 1);
        const u64 j = (c * g) % two_n;
        const u64 v = in[i];
        if (j < R.N) out[row_off + j] = v;
        else out[row_off + j - R.N] = neg_mod(v, R.q[row_mod(R, S, i)]);
    }
}

// Poly::mul_monomial (ring.hpp:343-361): X^e * a, coefficient i -> i + e
// (mod 2N) with the negacyclic sign.
__global__ void k_mul_monomial(DevRing R, Shape S, u64* out, const u64* in, u64 e) {
    const u64 two_n = 2 * u64(R.N);
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 row_off = i & ~u64(R.N - 1);
        const u64 j = ((i & (R.N - 1)) + e) % two_n;
        const u64 v = in[i];
        if (j < R.N) out[row_off + j] = v;
        else out[row_off + j - R.N] = neg_mod(v, R.q[row_mod(R, S, i)]);
    }
}

// raise_level (ring.hpp:523-545): level-0 residues a (mod q0) lifted to every
// row of the new shape as the centered integer (a > q0/2 -> a - q0).
__global__ void k_raise_level(DevRing R, Shape S, u64* out, const u64* in) {
    const u64 q0 = R.q[0], half = q0 >> 1;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 poly = i / (u64(S.rpp) * R.N);
        const u64 a = in[poly * R.N + (i & (R.N - 1))];
        const u32 m = row_mod(R, S, i);
        if (m == 0) {
            out[i] = a;
            continue;
        }
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        const u64 v = reduce64(a, q, rl, rh);
        out[i] = a > half ? sub_mod(v, reduce64(q0, q, rl, rh), q) : v;
    }
}

// Large-domain PFE (pfe.hpp:73-114): row r of the output is
// sum_c X^{e[r][c]} * tv_c, a sum of negacyclic rotations of the test
// vectors (parts back to back, level+1 rows each). Gather form: coefficient j
// of X^e a is a[(j - e) mod 2N] if that index is < N, else -a[(j + N - e) mod 2N].
struct PfeTables {
    u32 ncols;
    const u64* tv[TG_PFE_MAX_COLS];
};

__global__ void k_pfe_eval(DevRing R, u64* __restrict__ out, const PfeTables T, const u32* __restrict__ exps,
                           u32 nrows, u32 rows) {
    const u64 N = R.N, two_n = 2 * N, per_ct = 2 * u64(rows) * N;
    const u64 total = per_ct * nrows;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 r = i / per_ct, w = i - r * per_ct;  // w: offset inside the ciphertext
        const u64 j = w & (N - 1), row_off = w - j;
        const u32 m = u32((w / N) % rows);
        const u64 q = R.q[m];
        u64 acc = 0;
        for (u32 c = 0; c < T.ncols; ++c) {
            const u64 e = exps[r * T.ncols + c];
            const u64 src = (j + two_n - e) % two_n;
            const u64 v = src < N ? T.tv[c][row_off + src] : neg_mod(T.tv[c][row_off + src - N], q);
            acc = add_mod(acc, v, q);
        }
        out[i] = acc;
    }
}

// merge_embed (rlwe.hpp:702-735): small-ring polys interleaved into one big
// ring poly, out[row][k * stride + i] = in_i[row][k]; absent inputs are zero.
// ring_split's extract (rlwe.hpp:780-790) is the inverse gather.
__global__ void k_interleave(u64* __restrict__ out, const u64* const* __restrict__ in, u32 count, u32 stride,
                             u32 n_small, u64 rows_total) {
    const u64 N = u64(n_small) * stride, total = rows_total * N;
    for (u64 x = blockIdx.x * u64(blockDim.x) + threadIdx.x; x < total; x += u64(gridDim.x) * blockDim.x) {
        const u64 row = x / N, c = x - row * N;
        const u32 i = u32(c % stride);
        const u64 k = c / stride;
        out[x] = (i < count && in[i]) ? in[i][row * n_small + k] : 0;
    }
}

__global__ void k_deinterleave(u64* __restrict__ out, const u64* __restrict__ in, u32 parity, u32 stride,
                               u32 n_small, u64 rows_total) {
    const u64 total = rows_total * n_small;
    for (u64 x = blockIdx.x * u64(blockDim.x) + threadIdx.x; x < total; x += u64(gridDim.x) * blockDim.x) {
        const u64 row = x / n_small, k = x - row * n_small;
        out[x] = in[row * u64(n_small) * stride + k * stride + parity];
    }
}

// automorphism_apply, evaluation form (ring.hpp:428-434): slot gather
__global__ void k_auto_eval(DevRing R, Shape S, u64* out, const u64* in, u64 g) {
    const u64 two_n = 2 * u64(R.N);
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u64 row_off = i & ~u64(R.N - 1);
        const u32 j = u32(i & (R.N - 1));
        const u32 src = R.slot_of_exp[u32((u64(R.eval_exp[j]) * g) % two_n)];
        out[i] = in[row_off + src];
    }
}

// rescale_round (ring.hpp:493-518): thread per coefficient, loop over targets
__global__ void k_rescale(DevRing R, u64* out, const u64* in, int level, u32 npolys) {
    const u32 N = R.N, lvl = u32(level);
    const u64 total = u64(npolys) * N;
    const u64 ql = R.q[lvl];
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i >> R.logN, c = i & (N - 1);
        const u64* src = in + p * (lvl + 1) * N;
        u64* dst = out + p * lvl * N;
        const u64 last = src[size_t(lvl) * N + c];
        const u64 hl = ql >> 1;
        // centred last residue as a signed FP64 integer (FP64 rows below)
        const double x = last > hl ? __dsub_rn(u2d(last), u2d(ql)) : u2d(last);
        for (u32 r = 0; r < lvl; ++r) {
            const u64 q = R.q[r];
            if (q < kFpMaxQ && ql < kFpMaxQ) {  // (v - x) * ql^-1, |v - x| < 1.1q: one exact FP64 product
                const double qd = R.qd[4 * r];
                const double* rsd = R.rsd + (size_t(lvl) * R.q_count + r) * 2;
                dst[size_t(r) * N + c] =
                    fp_canonical1(fp_mulmod(__dsub_rn(u2d(src[size_t(r) * N + c]), x), rsd[0], rsd[1], qd), qd);
                continue;
            }
            const u64* e = R.rs + (size_t(lvl) * R.q_count + r) * 4;
            u64 t = last < q ? last : reduce64(last, q, R.ratio[2 * r], R.ratio[2 * r + 1]);
            if (last > e[3]) t = sub_mod(t, e[0], q);  // centered remainder
            dst[size_t(r) * N + c] = shoup(sub_mod(src[size_t(r) * N + c], t, q), e[1], e[2], q);
        }
    }
}

// rescale_round when every row and q_l take the FP64 path: two coefficients
// per thread (16-byte accesses) and four rows' words loaded before any is
// used, so each thread keeps several loads in flight (k_rescale waits on one
// load per row).
__global__ void __launch_bounds__(256) k_rescale_fp(DevRing R, u64* out, const u64* in, int level, u32 npolys,
                                                    const u64* __restrict__ add = nullptr, u64 astride = 0,
                                                    u32 orows = 0) {
    // add: Evaluator::add of the rescaled rows 0..orows-1 with `add` (poly p at
    // p * astride words), out packed at orows rows per poly
    const u32 N = R.N, lvl = u32(level), half = N / 2;
    const u32 nout = add ? orows : lvl;
    const u64 total = u64(npolys) * half;
    const u64 ql = R.q[lvl], hl = ql >> 1;
    const double qld = u2d(ql);
    const double* rsd = R.rsd + size_t(lvl) * R.q_count * 2;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i / half, c = (i - p * half) * 2;
        const u64* src = in + p * (lvl + 1) * N + c;
        u64* dst = out + p * nout * N + c;
        const u64* ad = add ? add + p * astride + c : nullptr;
        const ulonglong2 lv = *reinterpret_cast<const ulonglong2*>(src + size_t(lvl) * N);
        // centred last residues as signed FP64 integers
        const double x0 = lv.x > hl ? __dsub_rn(u2d(lv.x), qld) : u2d(lv.x);
        const double x1 = lv.y > hl ? __dsub_rn(u2d(lv.y), qld) : u2d(lv.y);
        auto one = [&](u32 r, ulonglong2 v) {  // (v - x) * ql^-1, |v - x| < 1.1q: one exact FP64 product each
            const double qd = R.qd[4 * r], w = rsd[2 * r], wq = rsd[2 * r + 1];
            const u64 q = R.q[r];
            u64 o0 = fp_canon_small(fp_mulmod(__dsub_rn(u2d(v.x), x0), w, wq, qd), q);
            u64 o1 = fp_canon_small(fp_mulmod(__dsub_rn(u2d(v.y), x1), w, wq, qd), q);
            if (ad) {
                const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(ad + size_t(r) * N);
                o0 = add_mod(o0, a.x, q);
                o1 = add_mod(o1, a.y, q);
            }
            *reinterpret_cast<ulonglong2*>(dst + size_t(r) * N) = make_ulonglong2(o0, o1);
        };
        u32 r = 0;
        for (; r + 4 <= nout; r += 4) {
            ulonglong2 v[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) v[k] = *reinterpret_cast<const ulonglong2*>(src + size_t(r + k) * N);
#pragma unroll
            for (int k = 0; k < 4; ++k) one(r + k, v[k]);
        }
        for (; r < nout; ++r) one(r, *reinterpret_cast<const ulonglong2*>(src + size_t(r) * N));
    }
}

// Eval-form rescale_round, step 1: from the inverse-transformed last row,
// t_r = centered(last) mod q_r into rows 0..level-1 of the scratch t (same
// layout as the input, level+1 rows per poly).
__global__ void k_rescale_eval_prep(DevRing R, u64* __restrict__ t, int level, u32 npolys) {
    const u32 N = R.N, lvl = u32(level);
    const u64 total = u64(npolys) * N;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i >> R.logN, c = i & (N - 1);
        u64* base = t + p * (lvl + 1) * N;
        const u64 last = base[size_t(lvl) * N + c];
        for (u32 r = 0; r < lvl; ++r) {
            const u64 q = R.q[r];
            const u64* e = R.rs + (size_t(lvl) * R.q_count + r) * 4;
            u64 v = last < q ? last : reduce64(last, q, R.ratio[2 * r], R.ratio[2 * r + 1]);
            if (last > e[3]) v = sub_mod(v, e[0], q);
            base[size_t(r) * N + c] = v;
        }
    }
}

// step 3: out_r = (x_r - NTT(t)_r) * q_l^-1 on eval-form rows
__global__ void k_rescale_eval_finish(DevRing R, u64* __restrict__ out, const u64* __restrict__ in,
                                      const u64* __restrict__ t, int level, u32 npolys) {
    const u32 N = R.N, lvl = u32(level);
    const u64 per = u64(lvl) * N, total = per * npolys;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i / per, w = i - p * per;
        const u32 r = u32(w >> R.logN);
        const u64 q = R.q[r];
        const u64* e = R.rs + (size_t(lvl) * R.q_count + r) * 4;
        const size_t src = p * (lvl + 1) * N + w;
        out[i] = shoup(sub_mod(in[src], t[src], q), e[1], e[2], q);
    }
}

// Evaluator::mul tensor (ckks.hpp:229-237)
__global__ void k_tensor(DevRing R, Shape S, u64* p0, u64* p1, u64* p2, const u64* x0, const u64* x1,
                         const u64* y0, const u64* y1) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        const u64 a0 = x0[i], a1 = x1[i], b0 = y0[i], b1 = y1[i];
        if (q < kFpMaxQ) {  // exact FP64 products (tg_fp64.cuh): |r| < 0.81q each
            const double qd = R.qd[4 * m], qi = R.qd[4 * m + 1];
            const double da0 = u2d(a0), da1 = u2d(a1), db0 = u2d(b0), db1 = u2d(b1);
            p0[i] = fp_canonical1(fp_mulmod_qi(da0, db0, qd, qi), qd);
            p1[i] = fp_canonical(__dadd_rn(fp_mulmod_qi(da0, db1, qd, qi), fp_mulmod_qi(da1, db0, qd, qi)), qd);
            p2[i] = fp_canonical1(fp_mulmod_qi(da1, db1, qd, qi), qd);
            continue;
        }
        p0[i] = mul_mod(a0, b0, q, rl, rh);
        // x0*y1 + x1*y0 as one 128-bit sum (< 2^125), one reduction
        U128 acc{0, 0};
        mac128(acc, a0, b1);
        mac128(acc, a1, b0);
        p1[i] = barrett128(acc.lo, acc.hi, q, rl, rh);
        p2[i] = mul_mod(a1, b1, q, rl, rh);
    }
}

// npolys polys from scattered sources into one contiguous block (stacking
// single ciphertexts into a part-major batch): one launch instead of one
// device-to-device copy per poly.
constexpr int kGatherMax = 64;
struct GatherSrc {
    const u64* p[kGatherMax];
};
__global__ void k_gather_polys(u64* __restrict__ dst, GatherSrc S, u64 words) {
    const u64* __restrict__ src = S.p[blockIdx.y];
    u64* out = dst + u64(blockIdx.y) * words;
    const u64 n2 = words / 2;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n2; i += u64(gridDim.x) * blockDim.x)
        reinterpret_cast<ulonglong2*>(out)[i] = reinterpret_cast<const ulonglong2*>(src)[i];
}

// Sum of two tensors (lazy relinearisation, Evaluator::mul2_relin_rescale:
// add(mul(x, y), mul(u, v)), ckks.hpp:229-237 twice then :201-208) in one
// pass; p0 / p1 null: only c2 = x1 y1 + u1 v1.
__global__ void k_tensor2(DevRing R, Shape S, u64* p0, u64* p1, u64* p2, const u64* x0, const u64* x1,
                          const u64* y0, const u64* y1, const u64* u0, const u64* u1, const u64* v0,
                          const u64* v1) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        const u64 a1 = x1[i], b1 = y1[i], c1 = u1[i], d1 = v1[i];
        if (q < kFpMaxQ) {  // exact FP64 products (|r| < 0.81q each), sums < 3.24q < 2^53
            const double qd = R.qd[4 * m], qi = R.qd[4 * m + 1];
            const double da1 = u2d(a1), db1 = u2d(b1), dc1 = u2d(c1), dd1 = u2d(d1);
            p2[i] = fp_canonical(__dadd_rn(fp_mulmod_qi(da1, db1, qd, qi), fp_mulmod_qi(dc1, dd1, qd, qi)), qd);
            if (!p0) continue;
            const double da0 = u2d(x0[i]), db0 = u2d(y0[i]), dc0 = u2d(u0[i]), dd0 = u2d(v0[i]);
            p0[i] = fp_canonical(__dadd_rn(fp_mulmod_qi(da0, db0, qd, qi), fp_mulmod_qi(dc0, dd0, qd, qi)), qd);
            const double s1 = __dadd_rn(__dadd_rn(fp_mulmod_qi(da0, db1, qd, qi), fp_mulmod_qi(da1, db0, qd, qi)),
                                        __dadd_rn(fp_mulmod_qi(dc0, dd1, qd, qi), fp_mulmod_qi(dc1, dd0, qd, qi)));
            p1[i] = fp_canonical(fp_reduce(s1, qd, qi), qd);
            continue;
        }
        U128 acc{0, 0};  // 128-bit lazy sums (< 2^126), one reduction each
        mac128(acc, a1, b1);
        mac128(acc, c1, d1);
        p2[i] = barrett128(acc.lo, acc.hi, q, rl, rh);
        if (!p0) continue;
        const u64 a0 = x0[i], b0 = y0[i], c0 = u0[i], d0 = v0[i];
        acc = U128{0, 0};
        mac128(acc, a0, b0);
        mac128(acc, c0, d0);
        p0[i] = barrett128(acc.lo, acc.hi, q, rl, rh);
        acc = U128{0, 0};
        mac128(acc, a0, b1);
        mac128(acc, a1, b0);
        mac128(acc, c0, d1);
        mac128(acc, c1, d0);
        p1[i] = barrett128(acc.lo, acc.hi, q, rl, rh);
    }
}

// c2 = x1 y1 only (relinearisation through the fused key switch forms c0 and
// c1 from the operands inside the key-switch core: tg_relinearize_tensor_batch)
__global__ void k_tensor_c2(DevRing R, Shape S, u64* p2, const u64* x1, const u64* y1) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        const u64 q = R.q[m];
        if (q < kFpMaxQ) {
            const double qd = R.qd[4 * m], qi = R.qd[4 * m + 1];
            p2[i] = fp_canonical1(fp_mulmod_qi(u2d(x1[i]), u2d(y1[i]), qd, qi), qd);
            continue;
        }
        p2[i] = mul_mod(x1[i], y1[i], q, R.ratio[2 * m], R.ratio[2 * m + 1]);
    }
}

// LinearTransformPlan::apply giant bucket (ckks.hpp:455-476):
// out[p][r][i] = sum_t ct_t[p][r][i] * plain_t[r][i] mod q_r, 128-bit lazy
// accumulation (reduced every 15 terms: products < 2^124), one Barrett per
// output. ct_t parts are back to back (level+1 rows each); plain_t has at
// least level+1 rows.
struct PlainSum {
    u32 nterms;
    const u64* ct[TG_PLAIN_SUM_MAX_TERMS];
    const u64* plain[TG_PLAIN_SUM_MAX_TERMS];
    u64 pstride[TG_PLAIN_SUM_MAX_TERMS];  // words between a term's parts (level+1 rows: contiguous)
};

__global__ void k_mul_plain_sum(DevRing R, u64* __restrict__ out, const PlainSum P, int level, u32 nparts) {
    const u32 N = R.N, rows = u32(level) + 1;
    const u64 per = u64(rows) * N, total = per * nparts;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 w = i % per, part = i / per;
        const u32 m = u32(w >> R.logN);
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        if (q < kFpMaxQ) {  // exact FP64 products, reduced every 4 terms (|sum| < q/2 + 1 + 4 * 0.81q < 2^53)
            const double qd = R.qd[4 * m], qi = R.qd[4 * m + 1];
            double s = 0.0;
            for (u32 t = 0; t < P.nterms; ++t) {
                s = __dadd_rn(s, fp_mulmod_qi(u2d(P.ct[t][part * P.pstride[t] + w]), u2d(P.plain[t][w]), qd, qi));
                if ((t & 3) == 3) s = fp_reduce(s, qd, qi);
            }
            out[i] = fp_canonical(fp_reduce(s, qd, qi), qd);
            continue;
        }
        U128 acc{0, 0};
        u32 pending = 0;
        for (u32 t = 0; t < P.nterms; ++t) {
            mac128(acc, P.ct[t][part * P.pstride[t] + w], P.plain[t][w]);
            if (++pending == 15 && t + 1 < P.nterms) {
                acc = U128{barrett128(acc.lo, acc.hi, q, rl, rh), 0};
                pending = 0;
            }
        }
        out[i] = barrett128(acc.lo, acc.hi, q, rl, rh);
    }
}

// Evaluator::mul_plain (ckks.hpp:257-265): part row r x plain row m (= r here)
__global__ void k_mul_plain(DevRing R, u64* out, const u64* ct, const u64* plain, int level, u32 nparts) {
    const u32 N = R.N, rows = u32(level) + 1;
    const u64 per = u64(rows) * N, total = per * nparts;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 w = i % per;
        const u32 m = u32(w >> R.logN);
        const u64 q = R.q[m];
        if (q < kFpMaxQ) {
            const double qd = R.qd[4 * m];
            out[i] = fp_canonical1(fp_mulmod_qi(u2d(ct[i]), u2d(plain[w]), qd, R.qd[4 * m + 1]), qd);
        } else {
            out[i] = mul_mod(ct[i], plain[w], q, R.ratio[2 * m], R.ratio[2 * m + 1]);
        }
    }
}

// Post-NCCL fix-up: arbitrary word -> canonical residue of its row modulus.
__global__ void k_reduce(DevRing R, Shape S, u64* data) {
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < S.words; i += u64(gridDim.x) * blockDim.x) {
        const u32 m = row_mod(R, S, i);
        data[i] = reduce64(data[i], R.q[m], R.ratio[2 * m], R.ratio[2 * m + 1]);
    }
}

}  // namespace
}  // namespace tg

using namespace tg;

static int check_shape(tg_context* ctx, int level, int nspecial) {
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    if (level < 0 || u32(level) >= ctx->ring.q_count) return fail(TG_E_ARG, "[ring] poly level out of range");
    if (nspecial != 0 && u32(nspecial) != ctx->ring.K) return fail(TG_E_ARG, "[ring] special rows must be all-or-none");
    return TG_OK;
}

static Shape shape_of(tg_context* ctx, int level, int nspecial, u32 npolys) {
    Shape S;
    S.rpp = u32(level + 1 + nspecial);
    S.level = level;
    S.words = u64(S.rpp) * npolys * ctx->ring.N;
    return S;
}

#define PROF(op, bytes) ProfScope prof_(ctx, op, double(bytes), as_stream(stream))

extern "C" int tg_poly_addsub(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int op, int level,
                              int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    TG_REQUIRE(op >= 0 && op <= 2, "[ring] addsub op must be 0 (add), 1 (sub) or 2 (neg)");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_ADDSUB, (op == 2 ? 16 : 24) * S.words);
    k_addsub<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, a, b, op);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_poly_mul(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int level,
                           int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_MUL, 24 * S.words);
    k_mul<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, a, b, 0);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_poly_mul_acc(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* b, int level,
                               int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_MUL, 32 * S.words);
    k_mul<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, a, b, 1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

static Scalars make_scalars(tg_context* ctx, const uint64_t* per_mod, bool shoup_pre) {
    Scalars sc{};
    for (u32 m = 0; m < ctx->ring.nmod; ++m) {
        u64 q = ctx->h_q[m];
        u64 s = per_mod[m] % q;
        sc.s[m] = s;
        sc.ss[m] = shoup_pre ? h_shoup(s, q) : 0;
    }
    return sc;
}

extern "C" int tg_poly_mul_scalar(tg_context* ctx, uint64_t* out, const uint64_t* a,
                                  const uint64_t* scalar_per_modulus, int level, int nspecial, uint32_t npolys,
                                  void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    TG_REQUIRE(scalar_per_modulus, "[ring] null scalar table");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_SCALAR, 16 * S.words);
    k_mul_scalar<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, a,
                                                                        make_scalars(ctx, scalar_per_modulus, true));
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_poly_add_scalar(tg_context* ctx, uint64_t* out, const uint64_t* a, const uint64_t* add_per_modulus,
                                  int form, int level, int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    TG_REQUIRE(add_per_modulus, "[ring] null scalar table");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_SCALAR, 16 * S.words);
    k_add_scalar<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(
        ctx->ring, S, out, a, make_scalars(ctx, add_per_modulus, false), form == TG_FORM_EVAL ? 1 : 0);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_automorphism(tg_context* ctx, uint64_t* out, const uint64_t* in, uint64_t exponent, int form,
                               int level, int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    const u64 two_n = 2 * u64(ctx->ring.N);
    const u64 g = exponent % two_n;
    TG_REQUIRE(g % 2 == 1, "[ring] automorphism exponent must be odd");
    TG_REQUIRE(out != in, "[ring] automorphism output must not alias its input");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_AUTOMORPHISM, 16 * S.words);
    if (form == TG_FORM_COEFF)
        k_auto_coeff<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, in, g);
    else
        k_auto_eval<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, in, g);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_rescale_add(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
                              const uint64_t* addend, uint64_t addend_stride, int out_level, void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    TG_REQUIRE(level >= 1, "[ring] cannot rescale at level 0");
    TG_REQUIRE(out_level >= 0 && out_level <= level - 1, "[ring] rescale_add output level out of range");
    TG_REQUIRE(addend && addend_stride >= u64(out_level + 1) * ctx->ring.N, "[ring] rescale_add addend shape");
    TG_REQUIRE(out != in, "[ring] rescale output must not alias its input");
    for (int r = 0; r <= level; ++r)
        if (ctx->h_q[r] >= kFpMaxQ) return fail(TG_E_ARG, "[ring] rescale_add needs FP64-eligible rows");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    PROF(TG_OP_RESCALE, 8.0 * npolys * ctx->ring.N * (level + 1 + 2.0 * (out_level + 1)));
    k_rescale_fp<<<grid_for(size_t(npolys) * ctx->ring.N / 2), 256, 0, as_stream(stream)>>>(
        ctx->ring, out, in, level, npolys, addend, addend_stride, u32(out_level + 1));
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_rescale(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
                          void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    TG_REQUIRE(level >= 1, "[ring] cannot rescale at level 0");
    TG_REQUIRE(out != in, "[ring] rescale output must not alias its input");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    PROF(TG_OP_RESCALE, 8.0 * npolys * ctx->ring.N * (2 * level + 1));
    bool all_fp = true;
    for (int r = 0; r <= level; ++r) all_fp &= ctx->h_q[r] < kFpMaxQ;
    if (all_fp) {
        k_rescale_fp<<<grid_for(size_t(npolys) * ctx->ring.N / 2), 256, 0, as_stream(stream)>>>(ctx->ring, out, in,
                                                                                                level, npolys);
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    k_rescale<<<grid_for(size_t(npolys) * ctx->ring.N), kThreads, 0, as_stream(stream)>>>(ctx->ring, out, in, level,
                                                                                          npolys);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

// rescale_round on EVAL-form input and output: only the dropped row is
// inverse transformed; its centered residues are forward transformed per
// remaining modulus (NTT(t mod q_r) is what rescale subtracts in eval form).
// NTT(tg_rescale(iNTT(in))) == tg_rescale_eval(in), residue for residue.
extern "C" int tg_rescale_eval(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, uint32_t npolys,
                               void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    TG_REQUIRE(level >= 1, "[ring] cannot rescale at level 0");
    TG_REQUIRE(out != in, "[ring] rescale output must not alias its input");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    const DevRing& R = ctx->ring;
    cudaStream_t s = as_stream(stream);
    void* scratch = nullptr;
    const size_t words = size_t(npolys) * (level + 1) * R.N;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, words * 8, ctx->pool, s));
    u64* t = static_cast<u64*>(scratch);
    int rc = ntt_inverse_oop(ctx, t, in, level, 0, npolys, s, u32(level), 1);
    if (rc == TG_OK) {
        PROF(TG_OP_RESCALE, 8.0 * npolys * R.N * (level + 1));
        k_rescale_eval_prep<<<grid_for(size_t(npolys) * R.N), kThreads, 0, s>>>(R, t, level, npolys);
        rc = cudaGetLastError() == cudaSuccess ? TG_OK : cuda_fail(cudaGetLastError(), "rescale prep");
    }
    if (rc == TG_OK) rc = ntt_forward_oop(ctx, t, t, level, 0, npolys, s, 0, 0, u32(level));
    if (rc == TG_OK) {
        PROF(TG_OP_RESCALE, 8.0 * npolys * R.N * 3.0 * level);
        k_rescale_eval_finish<<<grid_for(size_t(npolys) * level * R.N), kThreads, 0, s>>>(R, out, in, t, level,
                                                                                           npolys);
        rc = cudaGetLastError() == cudaSuccess ? TG_OK : cuda_fail(cudaGetLastError(), "rescale finish");
    }
    cudaFreeAsync(scratch, s);
    return rc;
}

extern "C" int tg_tensor(tg_context* ctx, uint64_t* p0, uint64_t* p1, uint64_t* p2, const uint64_t* x0,
                         const uint64_t* x1, const uint64_t* y0, const uint64_t* y1, int level, uint32_t npolys,
                         void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, 0, npolys);
    if (!p0 && !p1) {  // c2 only
        PROF(TG_OP_TENSOR, 24 * S.words);
        k_tensor_c2<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, p2, x1, y1);
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    PROF(TG_OP_TENSOR, 56 * S.words);
    k_tensor<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, p0, p1, p2, x0, x1, y0, y1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_gather_polys(tg_context* ctx, uint64_t* dst, const uint64_t* const* srcs, uint32_t npolys,
                               uint64_t words, void* stream) {
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    if (npolys == 0 || words == 0) return TG_OK;
    if (words % 2) return fail(TG_E_ARG, "[ring] gather: odd word count");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    for (uint32_t first = 0; first < npolys; first += kGatherMax) {
        const uint32_t n = std::min<uint32_t>(kGatherMax, npolys - first);
        GatherSrc S{};
        for (uint32_t i = 0; i < n; ++i) {
            if (!srcs[first + i]) return fail(TG_E_ARG, "[ring] gather: null source");
            S.p[i] = srcs[first + i];
        }
        const u32 bx = u32(std::min<u64>((words / 2 + kThreads - 1) / kThreads, 148u * 8u / std::max(1u, n / 4) + 1));
        k_gather_polys<<<dim3(bx, n), kThreads, 0, s>>>(dst + u64(first) * words, S, words);
        TG_LAUNCH_CHECK();
    }
    return TG_OK;
}

extern "C" int tg_tensor2(tg_context* ctx, uint64_t* p0, uint64_t* p1, uint64_t* p2, const uint64_t* x0,
                          const uint64_t* x1, const uint64_t* y0, const uint64_t* y1, const uint64_t* u0,
                          const uint64_t* u1, const uint64_t* v0, const uint64_t* v1, int level, uint32_t npolys,
                          void* stream) {
    if (!u0 && !u1 && !v0 && !v1) return tg_tensor(ctx, p0, p1, p2, x0, x1, y0, y1, level, npolys, stream);
    if (int rc = check_shape(ctx, level, 0)) return rc;
    if (npolys == 0) return TG_OK;
    if (!p2 || (p0 == nullptr) != (p1 == nullptr)) return fail(TG_E_ARG, "[ckks] tensor2: p2 and both or none of p0 / p1");
    if (!x1 || !y1 || !u1 || !v1 || (p0 && (!x0 || !y0 || !u0 || !v0)))
        return fail(TG_E_ARG, "[ckks] tensor2: missing operand part");
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, 0, npolys);
    PROF(TG_OP_TENSOR, (p0 ? 88 : 40) * S.words);
    k_tensor2<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, p0, p1, p2, x0, x1, y0, y1, u0, u1,
                                                                     v0, v1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_mul_plain(tg_context* ctx, uint64_t* out, const uint64_t* ct_part, const uint64_t* plain, int level,
                            uint32_t nparts, void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    if (nparts == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    size_t words = size_t(level + 1) * ctx->ring.N * nparts;
    PROF(TG_OP_MUL_PLAIN, 16.0 * words + 8.0 * words / nparts);
    k_mul_plain<<<grid_for(words), kThreads, 0, as_stream(stream)>>>(ctx->ring, out, ct_part, plain, level, nparts);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_poly_reduce(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys,
                              void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_REDUCE, 16 * S.words);
    k_reduce<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, data);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_mul_plain_sum(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* cts,
                                const uint64_t* const* plains, int level, uint32_t nparts, void* stream) {
    return tg_mul_plain_sum_strided(ctx, out, nterms, cts, nullptr, plains, level, nparts, stream);
}

extern "C" int tg_mul_plain_sum_strided(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* cts,
                                        const uint64_t* part_strides, const uint64_t* const* plains, int level,
                                        uint32_t nparts, void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    if (nterms == 0 || nterms > TG_PLAIN_SUM_MAX_TERMS) return fail(TG_E_ARG, "[ckks] plain sum: 1..256 terms");
    if (nparts == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    PlainSum P{};
    P.nterms = nterms;
    const u64 per = u64(level + 1) * ctx->ring.N;
    for (u32 t = 0; t < nterms; ++t) {
        P.ct[t] = cts[t];
        P.plain[t] = plains[t];
        P.pstride[t] = part_strides ? part_strides[t] : per;
        if (P.pstride[t] < per && nparts > 1) return fail(TG_E_ARG, "[ckks] plain sum: parts overlap");
    }
    const size_t words = size_t(level + 1) * ctx->ring.N * nparts;
    PROF(TG_OP_MUL_PLAIN, 8.0 * words * (nterms + 1) + 8.0 * words / nparts * nterms);
    k_mul_plain_sum<<<grid_for(words), kThreads, 0, as_stream(stream)>>>(ctx->ring, out, P, level, nparts);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_mul_monomial(tg_context* ctx, uint64_t* out, const uint64_t* in, uint64_t e, int level,
                               int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_AUTOMORPHISM, 16.0 * S.words);
    k_mul_monomial<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, in,
                                                                         e % (2 * u64(ctx->ring.N)));
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_raise_level(tg_context* ctx, uint64_t* out, const uint64_t* in, int new_level, int nspecial,
                              uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, new_level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, new_level, nspecial, npolys);
    PROF(TG_OP_SCALAR, 8.0 * S.words + 8.0 * ctx->ring.N * npolys);
    k_raise_level<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, in);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_pfe_eval(tg_context* ctx, uint64_t* out, const uint64_t* const* tvs, uint32_t ncols,
                           const uint32_t* exps, uint32_t nrows, int level, void* stream) {
    if (int rc = check_shape(ctx, level, 0)) return rc;
    if (ncols == 0 || ncols > TG_PFE_MAX_COLS) return fail(TG_E_ARG, "[pfe] 1..64 scoring functions");
    if (nrows == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    PfeTables T{};
    T.ncols = ncols;
    for (u32 c = 0; c < ncols; ++c) T.tv[c] = tvs[c];
    const u32 rows = u32(level) + 1;
    const size_t words = size_t(nrows) * 2 * rows * ctx->ring.N;
    PROF(TG_OP_AUTOMORPHISM, 8.0 * words + 16.0 * ncols * rows * ctx->ring.N);
    k_pfe_eval<<<grid_for(words), kThreads, 0, as_stream(stream)>>>(ctx->ring, out, T, exps, nrows, rows);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_interleave(uint64_t* out, const uint64_t* const* in_dev, uint32_t count, uint32_t stride,
                             uint32_t n_small, uint64_t rows_total, void* stream) {
    if (!out || !in_dev || stride == 0 || count > stride) return fail(TG_E_ARG, "[rlwe] interleave arguments");
    const size_t words = size_t(rows_total) * n_small * stride;
    if (words == 0) return TG_OK;
    k_interleave<<<grid_for(words), kThreads, 0, as_stream(stream)>>>(out, in_dev, count, stride, n_small, rows_total);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_deinterleave(uint64_t* out, const uint64_t* in, uint32_t parity, uint32_t stride, uint32_t n_small,
                               uint64_t rows_total, void* stream) {
    if (!out || !in || parity >= stride) return fail(TG_E_ARG, "[rlwe] deinterleave arguments");
    const size_t words = size_t(rows_total) * n_small;
    if (words == 0) return TG_OK;
    k_deinterleave<<<grid_for(words), kThreads, 0, as_stream(stream)>>>(out, in, parity, stride, n_small, rows_total);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_poly_addsub_strided(tg_context* ctx, uint64_t* out, const uint64_t* a, uint64_t a_stride,
                                      const uint64_t* b, uint64_t b_stride, int op, int level, int nspecial,
                                      uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (op != 0 && op != 1) return fail(TG_E_ARG, "[ring] strided addsub: op must be add or sub");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    Shape S = shape_of(ctx, level, nspecial, npolys);
    PROF(TG_OP_ADDSUB, 24 * S.words);
    k_addsub_strided<<<grid_for(S.words), kThreads, 0, as_stream(stream)>>>(ctx->ring, S, out, a, a_stride, b,
                                                                           b_stride, op);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
