// Fused linear combination (+ constant, + rescale) of ciphertext parts.
//
// The Chebyshev ladder (ckks.hpp:538-551) and its coefficient combination
// (ckks.hpp:558-578), and the threshold normalisation (threshold.hpp:152-155),
// are chains of Poly ops: doubling (add_inplace), mul_scalar (Shoup by a
// per-modulus integer), sub_inplace, add_scalar, rescale_round. Every link is
// exact arithmetic mod q, so the whole chain equals ONE residue expression
//     out = rescale( sum_t c_t * term_t  +  const )        (mod q)
// evaluated here in one pass: each input word read once, each output word
// written once, no intermediate polys. Results are bit-identical to the
// sequential reference ops (canonical residues of the same integers).
#include <cstring>

#include "tg_internal.cuh"
#include "tg_fp64.cuh"

namespace tg {
namespace {

constexpr u32 kThreads = 256;

inline u32 grid_for(size_t work) {
    size_t b = (work + kThreads - 1) / kThreads;
    return u32(std::min<size_t>(b, size_t(148) * 8 * 4));
}

struct LinComb {
    u32 nterms, nparts, rescale, add_all, add_polys, all_fp;
    int level;
    const u64* ptr[TG_LINCOMB_MAX_TERMS];
    u64 pstride[TG_LINCOMB_MAX_TERMS];
    u64 c[TG_LINCOMB_MAX_TERMS][TG_LINCOMB_MAX_ROWS];
    u64 cs[TG_LINCOMB_MAX_TERMS][TG_LINCOMB_MAX_ROWS];
    u64 add[TG_LINCOMB_MAX_ROWS];
};

// sum_t c_t * term_t[p][r][c] (+ const) mod q_r, canonical. Rows with
// q < kFpMaxQ (the host stored (c, c/q) as doubles in (c, cs)) use exact
// FP64 products (tg_fp64.cuh): canonical x < q gives |term| <= 0.575q, eight
// terms plus the constant stay below 2^53 between reductions.
__device__ __forceinline__ u64 lc_row(const DevRing& R, const LinComb& L, u32 p, u32 r, u32 c, bool add_here) {
    const u64 q = R.q[r], one = R.one_shoup[r];
    if (q < kFpMaxQ) {
        const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1];
        double acc = add_here ? u2d(L.add[r]) : 0.0;
        for (u32 t = 0; t < L.nterms; ++t) {
            const u64 x = L.ptr[t][p * L.pstride[t] + size_t(r) * R.N + c];
            acc = __dadd_rn(acc, fp_mulmod(u2d(x), __longlong_as_double(static_cast<long long>(L.c[t][r])),
                                           __longlong_as_double(static_cast<long long>(L.cs[t][r])), qd));
            if ((t & 7) == 7) acc = fp_reduce(acc, qd, qi);
        }
        return fp_canonical(fp_reduce(acc, qd, qi), qd);
    }
    u64 acc = add_here ? L.add[r] : 0;
    for (u32 t = 0; t < L.nterms; ++t) {
        const u64 x = L.ptr[t][p * L.pstride[t] + size_t(r) * R.N + c];
        acc += shoup_lazy(x, L.c[t][r], L.cs[t][r], q);
        if ((t & 7) == 7) acc = shoup_lazy(acc, 1, one, q);  // keep the lazy sum < 16q < 2^64
    }
    return shoup(acc, 1, one, q);
}

// FP64 row sum reduced to |v| <= q/2 + 1 (not canonicalised): the rescale
// below consumes it directly.
__device__ __forceinline__ double lc_row_fp(const DevRing& R, const LinComb& L, u32 p, u32 r, u32 c, bool add_here) {
    const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1];
    double acc = add_here ? u2d(L.add[r]) : 0.0;
    const size_t o = size_t(r) * R.N + c;
#pragma unroll 4
    for (u32 t = 0; t < L.nterms; ++t) {
        const u64 x = L.ptr[t][p * L.pstride[t] + o];
        acc = __dadd_rn(acc, fp_mulmod(u2d(x), __longlong_as_double(static_cast<long long>(L.c[t][r])),
                                       __longlong_as_double(static_cast<long long>(L.cs[t][r])), qd));
        if ((t & 7) == 7) acc = fp_reduce(acc, qd, qi);
    }
    return fp_reduce(acc, qd, qi);
}

// Two rows at once (r, r2 with r2 == r allowed): their term loads are
// independent and issued together, so each thread keeps twice the loads in
// flight (the kernel is latency-bound on HBM at one row per pass).
__device__ __forceinline__ void lc_row2(const DevRing& R, const LinComb& L, u32 p, u32 r, u32 r2, u32 c,
                                        bool add_here, u64& v, u64& v2) {
    const u64 q = R.q[r], q2 = R.q[r2];
    if (q < kFpMaxQ && q2 < kFpMaxQ) {
        const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1], qd2 = R.qd[4 * r2], qi2 = R.qd[4 * r2 + 1];
        double acc = add_here ? u2d(L.add[r]) : 0.0, acc2 = add_here ? u2d(L.add[r2]) : 0.0;
        const size_t o = size_t(r) * R.N + c, o2 = size_t(r2) * R.N + c;
#pragma unroll 4
        for (u32 t = 0; t < L.nterms; ++t) {
            const u64* base = L.ptr[t] + p * L.pstride[t];
            const u64 x = base[o], x2 = base[o2];
            acc = __dadd_rn(acc, fp_mulmod(u2d(x), __longlong_as_double(static_cast<long long>(L.c[t][r])),
                                           __longlong_as_double(static_cast<long long>(L.cs[t][r])), qd));
            acc2 = __dadd_rn(acc2, fp_mulmod(u2d(x2), __longlong_as_double(static_cast<long long>(L.c[t][r2])),
                                             __longlong_as_double(static_cast<long long>(L.cs[t][r2])), qd2));
            if ((t & 7) == 7) {
                acc = fp_reduce(acc, qd, qi);
                acc2 = fp_reduce(acc2, qd2, qi2);
            }
        }
        v = fp_canonical(fp_reduce(acc, qd, qi), qd);
        v2 = fp_canonical(fp_reduce(acc2, qd2, qi2), qd2);
        return;
    }
    v = lc_row(R, L, p, r, c, add_here);
    v2 = lc_row(R, L, p, r2, c, add_here);
}

__global__ void __launch_bounds__(kThreads) k_lincomb(DevRing R, LinComb L, u64* __restrict__ out) {
    const u32 N = R.N, lvl = u32(L.level);
    const u32 rout = L.rescale ? lvl : lvl + 1;
    const u64 total = u64(L.nparts) * N;
    for (u64 i = blockIdx.x * u64(kThreads) + threadIdx.x; i < total; i += u64(gridDim.x) * kThreads) {
        const u32 p = u32(i >> R.logN), c = u32(i & (N - 1));
        const bool add_here = p < L.add_polys && (L.add_all || c == 0);
        u64* dst = out + size_t(p) * rout * N;
        if (!L.rescale) {
            for (u32 r = 0; r <= lvl; r += 2) {
                const u32 r2 = min(r + 1, lvl);
                u64 v, v2;
                lc_row2(R, L, p, r, r2, c, add_here, v, v2);
                dst[size_t(r) * N + c] = v;
                if (r2 != r) dst[size_t(r2) * N + c] = v2;
            }
            continue;
        }
        // rescale_round (ring.hpp:493-518) of the combined poly
        if (L.all_fp) {
            // all rows FP64: the last row's centred residue x (|x| <= (ql-1)/2)
            // is t mod q_r as a signed integer (|x| < q_r), and
            // out_r = (v_r - x) * ql^-1 with |v_r - x| < 1.1 q_r: one exact
            // FP64 product per row (tg_fp64.cuh), no integer reductions
            const double ql = R.qd[4 * lvl], hl = double(R.q[lvl] >> 1);
            double x = lc_row_fp(R, L, p, lvl, c, add_here);
            if (x > hl) x = __dsub_rn(x, ql);
            if (x < -hl) x = __dadd_rn(x, ql);
            const double* rsd = R.rsd + size_t(lvl) * R.q_count * 2;
            for (u32 r = 0; r < lvl; r += 2) {
                const u32 r2 = min(r + 1, lvl - 1);
                const double v = lc_row_fp(R, L, p, r, c, add_here);
                const double v2 = r2 != r ? lc_row_fp(R, L, p, r2, c, add_here) : 0.0;
                const double qd = R.qd[4 * r];
                dst[size_t(r) * N + c] =
                    fp_canonical1(fp_mulmod(__dsub_rn(v, x), rsd[2 * r], rsd[2 * r + 1], qd), qd);
                if (r2 != r) {
                    const double qd2 = R.qd[4 * r2];
                    dst[size_t(r2) * N + c] =
                        fp_canonical1(fp_mulmod(__dsub_rn(v2, x), rsd[2 * r2], rsd[2 * r2 + 1], qd2), qd2);
                }
            }
            continue;
        }
        const u64 last = lc_row(R, L, p, lvl, c, add_here);
        for (u32 r = 0; r < lvl; r += 2) {
            const u32 r2 = min(r + 1, lvl - 1);
            u64 v[2];
            lc_row2(R, L, p, r, r2, c, add_here, v[0], v[1]);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const u32 rr = h ? r2 : r;
                if (h && r2 == r) break;
                const u64 q = R.q[rr];
                const u64* e = R.rs + (size_t(lvl) * R.q_count + rr) * 4;
                u64 t = last < q ? last : reduce64(last, q, R.ratio[2 * rr], R.ratio[2 * rr + 1]);
                if (last > e[3]) t = sub_mod(t, e[0], q);
                dst[size_t(rr) * N + c] = shoup(sub_mod(v[h], t, q), e[1], e[2], q);
            }
        }
    }
}

// All rows FP64 and at most NT terms (the ladder steps and most combination
// steps): per-term base pointers hoisted out of the row loop and the term
// loop unrolled at compile time, so a row costs NT loads and NT exact FP64
// products instead of re-deriving every address from the parameter block.
template <int NT>
__global__ void __launch_bounds__(kThreads) k_lincomb_fp(DevRing R, LinComb L, u64* __restrict__ out) {
    const u32 N = R.N, lvl = u32(L.level);
    const u32 rout = L.rescale ? lvl : lvl + 1;
    const u64 total = u64(L.nparts) * N;
    for (u64 i = blockIdx.x * u64(kThreads) + threadIdx.x; i < total; i += u64(gridDim.x) * kThreads) {
        const u32 p = u32(i >> R.logN), c = u32(i & (N - 1));
        const bool add_here = p < L.add_polys && (L.add_all || c == 0);
        const u64* base[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) base[t] = u32(t) < L.nterms ? L.ptr[t] + p * L.pstride[t] + c : nullptr;
        auto row = [&](u32 r) {
            const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1];
            u64 x[NT];
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (u32(t) < L.nterms) x[t] = base[t][size_t(r) * N];
            double acc = add_here ? u2d(L.add[r]) : 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (u32(t) < L.nterms)
                    acc = __dadd_rn(acc, fp_mulmod(u2d(x[t]), __longlong_as_double(static_cast<long long>(L.c[t][r])),
                                                   __longlong_as_double(static_cast<long long>(L.cs[t][r])), qd));
                if ((t & 7) == 7) acc = fp_reduce(acc, qd, qi);
            }
            return fp_reduce(acc, qd, qi);  // |.| <= q/2 + 1
        };
        u64* dst = out + size_t(p) * rout * N + c;
        if (!L.rescale) {
            for (u32 r = 0; r <= lvl; ++r) dst[size_t(r) * N] = fp_canonical(row(r), R.qd[4 * r]);
            continue;
        }
        // rescale_round (ring.hpp:493-518): centred last row, then
        // (v_r - x) * ql^-1 per row (see k_lincomb)
        const double ql = R.qd[4 * lvl], hl = double(R.q[lvl] >> 1);
        double x = row(lvl);
        if (x > hl) x = __dsub_rn(x, ql);
        if (x < -hl) x = __dadd_rn(x, ql);
        const double* rsd = R.rsd + size_t(lvl) * R.q_count * 2;
        for (u32 r = 0; r < lvl; ++r) {
            const double qd = R.qd[4 * r];
            dst[size_t(r) * N] = fp_canonical1(fp_mulmod(__dsub_rn(row(r), x), rsd[2 * r], rsd[2 * r + 1], qd), qd);
        }
    }
}

// k_lincomb_fp with two coefficients per thread (16-byte loads and stores)
// and the next row's words loaded while the current row is combined: four
// times the loads in flight per thread (the one-coefficient kernel waits on
// NT loads per row; the fused ladder steps have NT = 1..2).
// NT = the exact term count (dispatch in tg_lincomb_batch): every term loop
// is compile-time, no predicated terms.
template <int NT>
__global__ void __launch_bounds__(kThreads) k_lincomb_fp2(DevRing R, LinComb L, u64* __restrict__ out) {
    const u32 N = R.N, lvl = u32(L.level), half = N / 2;
    const u32 rout = L.rescale ? lvl : lvl + 1;
    const u64 total = u64(L.nparts) * half;
    for (u64 i = blockIdx.x * u64(kThreads) + threadIdx.x; i < total; i += u64(gridDim.x) * kThreads) {
        const u32 p = u32(i / half), c = u32(i - u64(p) * half) * 2;
        const bool addp = p < L.add_polys;
        const bool add0 = addp && (L.add_all || c == 0), add1 = addp && L.add_all;
        const u64* base[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) base[t] = u32(t) < u32(NT) ? L.ptr[t] + p * L.pstride[t] + c : nullptr;
        auto load = [&](u32 r, ulonglong2 (&x)[NT]) {
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (u32(t) < u32(NT)) x[t] = *reinterpret_cast<const ulonglong2*>(base[t] + size_t(r) * N);
        };
        // sum_t c_t x_t (+ const) for both coefficients, reduced to |.| <= q/2 + 1
        auto comb = [&](u32 r, const ulonglong2 (&x)[NT], double& o0, double& o1) {
            const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1];
            const double ad = u2d(L.add[r]);
            double a0 = add0 ? ad : 0.0, a1 = add1 ? ad : 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                if (u32(t) < u32(NT)) {
                    const double w = __longlong_as_double(static_cast<long long>(L.c[t][r]));
                    const double wq = __longlong_as_double(static_cast<long long>(L.cs[t][r]));
                    a0 = __dadd_rn(a0, fp_mulmod(u2d(x[t].x), w, wq, qd));
                    a1 = __dadd_rn(a1, fp_mulmod(u2d(x[t].y), w, wq, qd));
                }
                if ((t & 7) == 7) {
                    a0 = fp_reduce(a0, qd, qi);
                    a1 = fp_reduce(a1, qd, qi);
                }
            }
            o0 = fp_reduce(a0, qd, qi);
            o1 = fp_reduce(a1, qd, qi);
        };
        u64* dst = out + size_t(p) * rout * N + c;
        ulonglong2 xa[NT], xb[NT];
        if (!L.rescale) {
            load(0, xa);
            for (u32 r = 0; r <= lvl; ++r) {
                if (r < lvl) load(r + 1, (r & 1) ? xa : xb);
                double o0, o1;
                comb(r, (r & 1) ? xb : xa, o0, o1);
                const u64 q = R.q[r];
                *reinterpret_cast<ulonglong2*>(dst + size_t(r) * N) =
                    make_ulonglong2(fp_canon_small(o0, q), fp_canon_small(o1, q));
            }
            continue;
        }
        // rescale_round (ring.hpp:493-518): centred last row, then
        // (v_r - x) * ql^-1 per row (see k_lincomb)
        const double ql = R.qd[4 * lvl], hl = double(R.q[lvl] >> 1);
        double x0, x1;
        load(lvl, xa);
        load(0, xb);
        comb(lvl, xa, x0, x1);
        if (x0 > hl) x0 = __dsub_rn(x0, ql);
        if (x0 < -hl) x0 = __dadd_rn(x0, ql);
        if (x1 > hl) x1 = __dsub_rn(x1, ql);
        if (x1 < -hl) x1 = __dadd_rn(x1, ql);
        const double* rsd = R.rsd + size_t(lvl) * R.q_count * 2;
        for (u32 r = 0; r < lvl; ++r) {  // row r's words are in xb (r even) / xa (r odd)
            if (r + 1 < lvl) load(r + 1, (r & 1) ? xb : xa);
            double v0, v1;
            comb(r, (r & 1) ? xa : xb, v0, v1);
            const double qd = R.qd[4 * r], w = rsd[2 * r], wq = rsd[2 * r + 1];
            const u64 q = R.q[r];
            *reinterpret_cast<ulonglong2*>(dst + size_t(r) * N) =
                make_ulonglong2(fp_canon_small(fp_mulmod(__dsub_rn(v0, x0), w, wq, qd), q),
                                fp_canon_small(fp_mulmod(__dsub_rn(v1, x1), w, wq, qd), q));
        }
    }
}

// Several combinations of the SAME terms in one pass (the BSGS base blocks of
// one polynomial: q, r, q', r' are all sum_k c_k T_k over the same baby steps
// with different constants): every term word is read once for all NO outputs
// instead of once per output. Rescaled coefficient-form outputs only, every
// row FP64 (k_lincomb_fp2's arithmetic per output).
constexpr int kMultiTerms = 4, kMultiOuts = 4;
struct MultiLin {
    u32 nparts, add_polys;
    int level;
    const u64* ptr[kMultiTerms];
    u64 pstride[kMultiTerms];
    u64* out[kMultiOuts];
    double c[kMultiOuts][kMultiTerms][TG_LINCOMB_MAX_ROWS];
    double cs[kMultiOuts][kMultiTerms][TG_LINCOMB_MAX_ROWS];
    double add[kMultiOuts][TG_LINCOMB_MAX_ROWS];  // centred constant (coefficient 0 of the first add_polys parts)
};

template <int NT, int NO>
__global__ void __launch_bounds__(kThreads) k_lincomb_multi(DevRing R, MultiLin L) {
    const u32 N = R.N, lvl = u32(L.level), half = N / 2;
    const u64 total = u64(L.nparts) * half;
    for (u64 i = blockIdx.x * u64(kThreads) + threadIdx.x; i < total; i += u64(gridDim.x) * kThreads) {
        const u32 p = u32(i / half), c = u32(i - u64(p) * half) * 2;
        const bool add0 = p < L.add_polys && c == 0;
        const u64* base[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) base[t] = L.ptr[t] + p * L.pstride[t] + c;
        auto load = [&](u32 r, ulonglong2 (&x)[NT]) {
#pragma unroll
            for (int t = 0; t < NT; ++t) x[t] = *reinterpret_cast<const ulonglong2*>(base[t] + size_t(r) * N);
        };
        // output o's sum_t c_t x_t (+ const) for both coefficients, |.| <= q/2 + 1
        // (NT <= 4 terms of |.| <= 0.58q plus |const| <= q/2: < 2^53)
        auto comb = [&](u32 r, const double (&xd)[NT][2], int o, double& o0, double& o1) {
            const double qd = R.qd[4 * r], qi = R.qd[4 * r + 1];
            double a0 = add0 ? L.add[o][r] : 0.0, a1 = 0.0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const double w = L.c[o][t][r], wq = L.cs[o][t][r];
                a0 = __dadd_rn(a0, fp_mulmod(xd[t][0], w, wq, qd));
                a1 = __dadd_rn(a1, fp_mulmod(xd[t][1], w, wq, qd));
            }
            o0 = fp_reduce(a0, qd, qi);
            o1 = fp_reduce(a1, qd, qi);
        };
        auto to_d = [&](const ulonglong2 (&x)[NT], double (&xd)[NT][2]) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                xd[t][0] = u2d(x[t].x);
                xd[t][1] = u2d(x[t].y);
            }
        };
        // rescale_round (ring.hpp:493-518) per output: centred last row, then
        // (v_r - x) * ql^-1 per row
        const double ql = R.qd[4 * lvl], hl = double(R.q[lvl] >> 1);
        ulonglong2 xa[NT], xb[NT];
        double xd[NT][2];
        load(lvl, xa);
        load(0, xb);
        to_d(xa, xd);
        double x0[NO], x1[NO];
#pragma unroll
        for (int o = 0; o < NO; ++o) {
            comb(lvl, xd, o, x0[o], x1[o]);
            if (x0[o] > hl) x0[o] = __dsub_rn(x0[o], ql);
            if (x0[o] < -hl) x0[o] = __dadd_rn(x0[o], ql);
            if (x1[o] > hl) x1[o] = __dsub_rn(x1[o], ql);
            if (x1[o] < -hl) x1[o] = __dadd_rn(x1[o], ql);
        }
        const double* rsd = R.rsd + size_t(lvl) * R.q_count * 2;
        const size_t po = size_t(p) * lvl * N + c;
        for (u32 r = 0; r < lvl; ++r) {  // row r's words are in xb (r even) / xa (r odd)
            if (r + 1 < lvl) load(r + 1, (r & 1) ? xb : xa);
            to_d((r & 1) ? xa : xb, xd);
            const double qd = R.qd[4 * r], w = rsd[2 * r], wq = rsd[2 * r + 1];
            const u64 q = R.q[r];
#pragma unroll
            for (int o = 0; o < NO; ++o) {
                double v0, v1;
                comb(r, xd, o, v0, v1);
                *reinterpret_cast<ulonglong2*>(L.out[o] + po + size_t(r) * N) =
                    make_ulonglong2(fp_canon_small(fp_mulmod(__dsub_rn(v0, x0[o]), w, wq, qd), q),
                                    fp_canon_small(fp_mulmod(__dsub_rn(v1, x1[o]), w, wq, qd), q));
            }
        }
    }
}

template <int NT>
void launch_multi(const DevRing& R, const MultiLin& L, u32 nouts, u32 grid, cudaStream_t st) {
    switch (nouts) {
        case 2: k_lincomb_multi<NT, 2><<<grid, kThreads, 0, st>>>(R, L); break;
        case 3: k_lincomb_multi<NT, 3><<<grid, kThreads, 0, st>>>(R, L); break;
        default: k_lincomb_multi<NT, 4><<<grid, kThreads, 0, st>>>(R, L); break;
    }
}

}  // namespace
}  // namespace tg

using namespace tg;

extern "C" int tg_lincomb_multi(tg_context* ctx, uint32_t nouts, uint64_t* const* outs, uint32_t nterms,
                                const uint64_t* const* terms, const uint64_t* part_strides, const uint64_t* coeffs,
                                const uint64_t* add_per_row, int level, uint32_t nparts, uint32_t add_polys,
                                void* stream) {
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    const DevRing& R = ctx->ring;
    if (level < 1 || u32(level) >= R.q_count) return fail(TG_E_ARG, "[ring] lincomb_multi: level out of range");
    if (nterms == 0 || nterms > u32(kMultiTerms) || nouts < 2 || nouts > u32(kMultiOuts))
        return fail(TG_E_ARG, "[ring] lincomb_multi: 1..4 terms, 2..4 outputs");
    if (u32(level) + 1 > TG_LINCOMB_MAX_ROWS) return fail(TG_E_ARG, "[ring] lincomb: too many rows");
    for (int r = 0; r <= level; ++r)
        if (ctx->h_q[r] >= kFpMaxQ) return fail(TG_E_ARG, "[ring] lincomb_multi needs FP64 q-chain rows");
    if (nparts == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    MultiLin L{};
    L.nparts = nparts;
    L.add_polys = add_polys;
    L.level = level;
    for (u32 t = 0; t < nterms; ++t) {
        L.ptr[t] = terms[t];
        L.pstride[t] = part_strides[t];
    }
    const size_t rows = size_t(level) + 1;
    for (u32 o = 0; o < nouts; ++o) {
        L.out[o] = outs[o];
        for (u32 t = 0; t < nterms; ++t)
            for (int r = 0; r <= level; ++r) {
                const u64 q = ctx->h_q[r], v = coeffs[(size_t(o) * nterms + t) * rows + r] % q;
                L.c[o][t][r] = double(v);
                L.cs[o][t][r] = double(v) / double(q);
            }
        for (int r = 0; r <= level; ++r) {
            const u64 q = ctx->h_q[r], e = add_per_row ? add_per_row[size_t(o) * rows + r] % q : 0;
            L.add[o][r] = e > q / 2 ? -double(q - e) : double(e);
        }
    }
    ProfScope prof(ctx, TG_OP_LINCOMB, 8.0 * nparts * R.N * (double(rows) * nterms + double(nouts) * level),
                   as_stream(stream));
    cudaStream_t st = as_stream(stream);
    const u32 grid = grid_for(size_t(nparts) * R.N / 2);
    switch (nterms) {
        case 1: launch_multi<1>(R, L, nouts, grid, st); break;
        case 2: launch_multi<2>(R, L, nouts, grid, st); break;
        case 3: launch_multi<3>(R, L, nouts, grid, st); break;
        default: launch_multi<4>(R, L, nouts, grid, st); break;
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

extern "C" int tg_lincomb(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* terms,
                          const uint64_t* part_strides, const uint64_t* coeffs, const uint64_t* add_per_row,
                          int add_all, int level, uint32_t nparts, int rescale, void* stream) {
    return tg_lincomb_batch(ctx, out, nterms, terms, part_strides, coeffs, add_per_row, add_all, level, nparts, 1,
                            rescale, stream);
}

extern "C" int tg_lincomb_batch(tg_context* ctx, uint64_t* out, uint32_t nterms, const uint64_t* const* terms,
                                const uint64_t* part_strides, const uint64_t* coeffs, const uint64_t* add_per_row,
                                int add_all, int level, uint32_t nparts, uint32_t add_polys, int rescale,
                                void* stream) {
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    const DevRing& R = ctx->ring;
    if (level < 0 || u32(level) >= R.q_count) return fail(TG_E_ARG, "[ring] poly level out of range");
    if (rescale && level < 1) return fail(TG_E_ARG, "[ring] cannot rescale at level 0");
    if (nterms == 0 || nterms > TG_LINCOMB_MAX_TERMS) return fail(TG_E_ARG, "[ring] lincomb: 1..32 terms");
    if (u32(level) + 1 > TG_LINCOMB_MAX_ROWS) return fail(TG_E_ARG, "[ring] lincomb: too many rows");
    if (nparts == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    LinComb L{};
    L.nterms = nterms;
    L.nparts = nparts;
    L.rescale = rescale ? 1 : 0;
    L.add_all = add_all ? 1 : 0;
    L.add_polys = add_polys;
    L.level = level;
    for (u32 t = 0; t < nterms; ++t) {
        L.ptr[t] = terms[t];
        L.pstride[t] = part_strides[t];
        for (int r = 0; r <= level; ++r) {
            const u64 q = ctx->h_q[r];
            const u64 v = coeffs[size_t(t) * (level + 1) + r] % q;
            if (q < kFpMaxQ) {  // FP64 row: (v, fl(v/q)) as double bits (exact: v < 2^53)
                const double vd = double(v), vq = vd / double(q);
                std::memcpy(&L.c[t][r], &vd, 8);
                std::memcpy(&L.cs[t][r], &vq, 8);
            } else {
                L.c[t][r] = v;
                L.cs[t][r] = h_shoup(v, q);
            }
        }
    }
    for (int r = 0; r <= level; ++r) L.add[r] = add_per_row ? add_per_row[r] % ctx->h_q[r] : 0;
    L.all_fp = 1;
    for (int r = 0; r <= level; ++r) L.all_fp &= ctx->h_q[r] < kFpMaxQ ? 1u : 0u;
    const double rows = double(level + 1);
    ProfScope prof(ctx, TG_OP_LINCOMB, 8.0 * nparts * R.N * (rows * nterms + (rescale ? rows - 1 : rows)),
                   as_stream(stream));
    const u32 grid = grid_for(size_t(nparts) * R.N);
    cudaStream_t st = as_stream(stream);
    const u32 grid2 = grid_for(size_t(nparts) * R.N / 2);
    if (L.all_fp && nterms <= 8) {
        switch (nterms) {
#define TG_LC_CASE(n) \
    case n: k_lincomb_fp2<n><<<grid2, kThreads, 0, st>>>(R, L, out); break;
            TG_LC_CASE(1) TG_LC_CASE(2) TG_LC_CASE(3) TG_LC_CASE(4) TG_LC_CASE(5) TG_LC_CASE(6) TG_LC_CASE(7)
            TG_LC_CASE(8)
#undef TG_LC_CASE
        }
    }
    else k_lincomb<<<grid, kThreads, 0, st>>>(R, L, out);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
