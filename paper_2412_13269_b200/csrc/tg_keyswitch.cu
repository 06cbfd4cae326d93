// Hybrid key switching: ModUp (GadgetPlan::decompose), key inner product
// (KeyContext::ks_inner) and ModDown (KeyContext::mod_down_p).
//
// Bit-exactness notes:
//  * ModUp is the reference's UNCORRECTED fast base conversion
//    (rlwe.hpp:78-100): y_i = x_i * (D'/q_i)^-1 mod q_i, then every output
//    row t gets sum_i (y_i * (D'/q_i) mod q_t) mod q_t. No overflow correction.
//  * ModDown is the CENTERED conversion (rlwe.hpp:555-589).
//  * Key row for modulus index m is m itself (rlwe.hpp:517-518 with full rows).
// One thread owns one coefficient of one digit (ModUp) / one output poly
// (ModDown) and keeps the <=16 source residues in registers, so each source
// word is read once and each output word written once.
#include <algorithm>
#include <type_traits>

#include "tg_internal.cuh"
#include "tg_fp64.cuh"

namespace tg {
namespace {

constexpr u32 kThreads = 256;

inline u32 grid_for(size_t work) {
    size_t b = (work + kThreads - 1) / kThreads;
    return u32(std::min<size_t>(b, size_t(148) * 8 * 4));
}

// ModUp base conversion for all digits of one level. grid.y = digit,
// one thread per coefficient. The uncorrected conversion reproduces the
// digit's own-group rows exactly (rlwe.hpp:78-100: conv_w[i][t] = 0 for
// t != i inside the group and y_i * D'/q_i = x_i), so those rows are copied
// and only the other rows are computed, 4 at a time for ILP. Terms are
// accumulated lazily (Shoup outputs in [0,2q), sum < 2*active*q < 2^64,
// checked on the host) and reduced once per output.
#ifndef MODUP_THREADS
#define MODUP_THREADS 128
#endif
// ModUp target rows of an all-FP64 digit with A active sources known at
// compile time: no per-term predicates or branches in the row loop (ncu: the
// generic loop spent ~60 integer/branch instructions per row around ~90 FP64
// ones). Same terms, same bounds, same order as the generic FP64 path.
// RAW: the converted rows are written as centred doubles (the reduced sum,
// |v| <= q/2 + 1) for the digits' column-pair NTT phase (kTgRawDigits).
template <int A, int CPT, int GMAX, bool RAW, class Y>
__device__ __forceinline__ void modup_rows_fp(const Y (&yd)[GMAX][CPT], const ulonglong2* smw, const u64* sq,
                                              u32 nrest, u32 v_begin, u32 v_end, u32 first, u64* out, u32 N) {
    for (u32 v = v_begin; v < v_end; ++v) {
        const u64 q = sq[v];
        const double qd = u2d(q), qi = __longlong_as_double(static_cast<long long>(sq[nrest + v]));
        const ulonglong2* wr = smw + size_t(v) * A;
        const u32 r = v < first ? v : v + A;
        double acc[CPT];
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) acc[cc] = 0.0;
#pragma unroll
        for (int i = 0; i < A; ++i) {
            const ulonglong2 w = wr[i];
            const double wd = __longlong_as_double(static_cast<long long>(w.x));
            const double wq = __longlong_as_double(static_cast<long long>(w.y));
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
                double yv;  // hoisted doubles, or u64 sources converted per use (16-source groups)
                if constexpr (sizeof(Y) == 8 && std::is_same<Y, double>::value) yv = yd[i][cc];
                else yv = u2d(yd[i][cc]);
                acc[cc] = __dadd_rn(acc[cc], fp_mulmod(yv, wd, wq, qd));
                if ((i & 7) == 7 && i + 1 < A) acc[cc] = fp_reduce(acc[cc], qd, qi);
            }
        }
        u64 o[CPT];
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) {
            const double v = fp_reduce(acc[cc], qd, qi);
            o[cc] = RAW ? static_cast<u64>(__double_as_longlong(v)) : fp_canon_small(v, q);
        }
        if constexpr (CPT == 2) *reinterpret_cast<ulonglong2*>(out + size_t(r) * N) = make_ulonglong2(o[0], o[1]);
        else out[size_t(r) * N] = o[0];
    }
}

#ifndef MODUP_CPT16
#define MODUP_CPT16 2  // measured: 110 -> 108 ms (config 5)
#endif
#ifndef MODUP_CPT8
#define MODUP_CPT8 2  // coefficients per thread of the group-size <= 8 ModUp (measured)
#endif
constexpr u32 kMUThreads = MODUP_THREADS;

__global__ void __launch_bounds__(kMUThreads)
k_modup(DevRing R, GadgetDev G, u64* __restrict__ digits, const u64* __restrict__ d, int level,
        const u64* __restrict__ d_eval) {
    const u32 N = R.N, lvl = u32(level), K = R.K;
    const u32 j = blockIdx.y;
    const u32 gs = G.group_size;
    const u32 first = j * gs;
    const u32 active = min(gs, lvl + 1 - first);
    const u32 rows_out = lvl + 1 + K;
    const u64* src_tb = G.src + ((size_t(j) * gs + (active - 1)) * gs) * 2;
    const u64* conv_tb = G.conv + ((size_t(j) * gs + (active - 1)) * gs) * R.nmod * 2;
    u64* out = digits + size_t(j) * rows_out * N;
    const u32 c = blockIdx.x * kMUThreads + threadIdx.x;
    if (c >= N) return;
    u64 y[kMaxGroup];
#pragma unroll
    for (u32 i = 0; i < u32(kMaxGroup); ++i) {
        if (i < active) {
            const u32 s = first + i;
            const u64 x = d[size_t(s) * N + c];
            // own-group row: exact copy (already transformed when the caller
            // holds the eval form of d; the digit NTT then skips this row)
            out[size_t(s) * N + c] = d_eval ? d_eval[size_t(s) * N + c] : x;
            y[i] = shoup(x, src_tb[2 * i], src_tb[2 * i + 1], R.q[s]);
        }
    }
    const u32 nrest = rows_out - active;
    for (u32 v0 = 0; v0 < nrest; v0 += 4) {
        u64 acc[4] = {0, 0, 0, 0};
        u32 t[4], r[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const u32 v = min(v0 + k, nrest - 1);
            r[k] = v < first ? v : v + active;
            t[k] = mod_index(r[k], level, R.q_count);
        }
        if (G.lazy_modup) {
#pragma unroll
            for (u32 i = 0; i < u32(kMaxGroup); ++i) {
                if (i < active) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const u64* cw = conv_tb + (size_t(i) * R.nmod + t[k]) * 2;
                        acc[k] += shoup_lazy(y[i], cw[0], cw[1], R.q[t[k]]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = shoup(acc[k], 1, R.one_shoup[t[k]], R.q[t[k]]);
        } else {
            for (u32 i = 0; i < active; ++i)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const u64* cw = conv_tb + (size_t(i) * R.nmod + t[k]) * 2;
                    acc[k] = add_mod(acc[k], shoup(y[i], cw[0], cw[1], R.q[t[k]]), R.q[t[k]]);
                }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (v0 + k < nrest) out[size_t(r[k]) * N + c] = acc[k];
    }
}

// GadgetPlan::decompose with base-2^b refinement (rlwe.hpp:103-135): group j
// is the single prime q_j; its centered residue splits into nsub balanced
// signed sub-digits (carry chain, the last sub-digit unbalanced), each written
// as from_centered(digit, q_r) to every row of its digit poly.
__global__ void k_decompose_base2(DevRing R, u64* __restrict__ digits, const u64* __restrict__ d, int level,
                                  u32 src, u32 nsub, u32 b, u64 dig_words, u64 in_words) {
    const u32 N = R.N, rows = u32(level) + 1 + R.K;
    const u32 t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    digits += blockIdx.y * dig_words;  // source poly blockIdx.y of the batch
    d += blockIdx.y * in_words;
    const u64 q = R.q[src], x = d[size_t(src) * N + t];
    const long long c = x > q / 2 ? (long long)x - (long long)q : (long long)x;  // to_centered
    const u64 mag = c < 0 ? u64(-c) : u64(c);
    const long long sign = c < 0 ? -1 : 1;
    const u64 half_base = u64(1) << (b - 1), mask = (u64(1) << b) - 1;
    u64 carry = 0;
    for (u32 s = 0; s < nsub; ++s) {
        const u64 u = ((mag >> (s * b)) & mask) + carry;
        long long dv;
        if (s + 1 < nsub && u >= half_base) {
            dv = (long long)u - (long long)(u64(1) << b);
            carry = 1;
        } else {
            dv = (long long)u;
            carry = 0;
        }
        dv *= sign;
        u64* out = digits + size_t(s) * rows * N + t;
        for (u32 r = 0; r < rows; ++r) {
            const u64 qr = R.q[mod_index(r, level, R.q_count)];
            // |dv| <= 2^b < q_r: from_centered is one conditional add
            out[size_t(r) * N] = dv < 0 ? qr - u64(-dv) : u64(dv);
        }
    }
}

// acc{0,1}[r][c] = sum_i digit_i[r][c] * key[i][{b,a}][m(r)][c], 128-bit lazy
// accumulation with a reduction every 15 terms (products < 2^124).
__global__ void __launch_bounds__(kThreads)
k_key_inner(DevRing R, u64* __restrict__ acc0, u64* __restrict__ acc1, const u64* __restrict__ digits, u32 nd,
            const u64* __restrict__ key, int level) {
    const u32 N = R.N, K = R.K;
    const u32 rows = u32(level) + 1 + K;
    const u64 words = u64(rows) * N;
    const size_t key_rows = size_t(R.nmod);  // max_level + 1 + K
    for (u64 i = blockIdx.x * u64(kThreads) + threadIdx.x; i < words; i += u64(gridDim.x) * kThreads) {
        const u32 r = u32(i >> R.logN);
        const u32 c = u32(i & (N - 1));
        const u32 m = mod_index(r, level, R.q_count);
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        U128 s0{0, 0}, s1{0, 0};
        u32 pending = 0;
        for (u32 k = 0; k < nd; ++k) {
            const u64 dv = digits[size_t(k) * words + i];
            const u64* kb = key + (size_t(k) * 2) * key_rows * N;
            const u64* ka = kb + key_rows * N;
            mac128(s0, dv, kb[size_t(m) * N + c]);
            mac128(s1, dv, ka[size_t(m) * N + c]);
            if (++pending == 15 && k + 1 < nd) {
                s0 = U128{barrett128(s0.lo, s0.hi, q, rl, rh), 0};
                s1 = U128{barrett128(s1.lo, s1.hi, q, rl, rh), 0};
                pending = 0;
            }
        }
        acc0[i] = barrett128(s0.lo, s0.hi, q, rl, rh);
        acc1[i] = barrett128(s1.lo, s1.hi, q, rl, rh);
    }
}

// Batched key inner product: npolys sources share one key. A thread owns one
// word (row, coefficient) of the key rows, keeps its nd (b, a) key words in
// registers and loops over the sources, so every key word is read once per
// batch ("switching key read once per batch").
// acc layout: [2][npolys][rows][N] (all b-accumulators, then all a).
template <int NDMAX>
__global__ void __launch_bounds__(kThreads)
k_key_inner_b(DevRing R, u64* __restrict__ acc, const u64* __restrict__ digits, u32 nd, u32 npolys,
              const u64* __restrict__ key, int level, u32 polys_per_thread, const u64* __restrict__ add0 = nullptr,
              const u64* __restrict__ add1 = nullptr, const u64* __restrict__ pmod = nullptr) {
    const u32 N = R.N, K = R.K;
    const u32 rows = u32(level) + 1 + K;
    const u64 words = u64(rows) * N;
    const size_t key_rows = size_t(R.nmod);
    // work item = (word pair, chunk of polys_per_thread sources): small rings
    // with large batches still fill the GPU. Two words per thread (16-byte
    // loads) and the next source's digits prefetched while the current one
    // is reduced keep enough loads in flight to cover HBM latency.
    const u64 pairs = words / 2;
    const u32 chunks = (npolys + polys_per_thread - 1) / polys_per_thread;
    for (u64 it = blockIdx.x * u64(kThreads) + threadIdx.x; it < pairs * chunks; it += u64(gridDim.x) * kThreads) {
        const u64 i = (it % pairs) * 2;
        const u32 b0 = u32(it / pairs) * polys_per_thread, b1 = min(npolys, b0 + polys_per_thread);
        const u32 r = u32(i >> R.logN);
        const u32 c = u32(i & (N - 1));
        const u32 m = mod_index(r, level, R.q_count);
        const u64 q = R.q[m], rl = R.ratio[2 * m], rh = R.ratio[2 * m + 1];
        ulonglong2 kb[NDMAX], ka[NDMAX], dv[NDMAX];
#pragma unroll
        for (int k = 0; k < NDMAX; ++k) {
            if (u32(k) < nd) {
                const u64* base = key + (size_t(k) * 2) * key_rows * N + size_t(m) * N + c;
                kb[k] = *reinterpret_cast<const ulonglong2*>(base);
                ka[k] = *reinterpret_cast<const ulonglong2*>(base + key_rows * N);
                dv[k] = *reinterpret_cast<const ulonglong2*>(digits + (size_t(b0) * nd + k) * words + i);
            }
        }
        const bool fp = q < kFpMaxQ;  // q-chain rows: exact FP64 products (tg_fp64.cuh)
        const double qd = fp ? R.qd[4 * m] : 0.0, qi = fp ? R.qd[4 * m + 1] : 0.0;
        // eval-form addends (c0, c1 of a relinearisation) enter the Q rows as
        // P * c: ModDown((acc + P c)) = ModDown(acc) + c (mod q_r)
        const bool addq = add0 && r <= u32(level);
        const u64 qwords = u64(level + 1) * N;
        u64 pm = 0, pms = 0;
        double pmd = 0, pmq = 0;
        if (addq) {
            pm = pmod[4 * r];
            pms = pmod[4 * r + 1];
            pmd = __longlong_as_double(static_cast<long long>(pmod[4 * r + 2]));
            pmq = __longlong_as_double(static_cast<long long>(pmod[4 * r + 3]));
        }
        for (u32 b = b0; b < b1; ++b) {
            ulonglong2 dn[NDMAX];
            if (b + 1 < b1) {
#pragma unroll
                for (int k = 0; k < NDMAX; ++k)
                    if (u32(k) < nd)
                        dn[k] = *reinterpret_cast<const ulonglong2*>(digits + (size_t(b + 1) * nd + k) * words + i);
            }
            if (fp) {
                // |product| < 0.81q; reduced every 4 digits: |sum| < q/2 + 1 + 3.3q < 2^53
                double s0 = 0, s1 = 0, t0 = 0, t1 = 0;
#pragma unroll
                for (int k = 0; k < NDMAX; ++k) {
                    if (u32(k) < nd) {
                        const double dx = u2d(dv[k].x), dy = u2d(dv[k].y);
                        s0 = __dadd_rn(s0, fp_mulmod_qi(dx, u2d(kb[k].x), qd, qi));
                        s1 = __dadd_rn(s1, fp_mulmod_qi(dx, u2d(ka[k].x), qd, qi));
                        t0 = __dadd_rn(t0, fp_mulmod_qi(dy, u2d(kb[k].y), qd, qi));
                        t1 = __dadd_rn(t1, fp_mulmod_qi(dy, u2d(ka[k].y), qd, qi));
                        if ((k & 3) == 3) {
                            s0 = fp_reduce(s0, qd, qi);
                            s1 = fp_reduce(s1, qd, qi);
                            t0 = fp_reduce(t0, qd, qi);
                            t1 = fp_reduce(t1, qd, qi);
                        }
                    }
                }
                if (addq) {  // |P c| < 0.58q on top of |sum| < 3.3q
                    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(add0 + size_t(b) * qwords + i);
                    const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(add1 + size_t(b) * qwords + i);
                    s0 = __dadd_rn(s0, fp_mulmod(u2d(a0.x), pmd, pmq, qd));
                    t0 = __dadd_rn(t0, fp_mulmod(u2d(a0.y), pmd, pmq, qd));
                    s1 = __dadd_rn(s1, fp_mulmod(u2d(a1.x), pmd, pmq, qd));
                    t1 = __dadd_rn(t1, fp_mulmod(u2d(a1.y), pmd, pmq, qd));
                }
                *reinterpret_cast<ulonglong2*>(acc + size_t(b) * words + i) = make_ulonglong2(
                    fp_canon_small(fp_reduce(s0, qd, qi), q), fp_canon_small(fp_reduce(t0, qd, qi), q));
                *reinterpret_cast<ulonglong2*>(acc + (size_t(npolys) + b) * words + i) = make_ulonglong2(
                    fp_canon_small(fp_reduce(s1, qd, qi), q), fp_canon_small(fp_reduce(t1, qd, qi), q));
                if (b + 1 < b1) {
#pragma unroll
                    for (int k = 0; k < NDMAX; ++k) dv[k] = dn[k];
                }
                continue;
            }
            U128 s0{0, 0}, s1{0, 0}, t0{0, 0}, t1{0, 0};
#pragma unroll
            for (int k = 0; k < NDMAX; ++k) {  // nd <= NDMAX <= 15: products < 2^124, no mid reduction
                if (u32(k) < nd) {
                    mac128(s0, dv[k].x, kb[k].x);
                    mac128(s1, dv[k].x, ka[k].x);
                    mac128(t0, dv[k].y, kb[k].y);
                    mac128(t1, dv[k].y, ka[k].y);
                }
            }
            if (addq) {  // products < 2^124 each, at most 16 terms: no overflow
                const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(add0 + size_t(b) * qwords + i);
                const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(add1 + size_t(b) * qwords + i);
                mac128(s0, a0.x, pm);
                mac128(t0, a0.y, pm);
                mac128(s1, a1.x, pm);
                mac128(t1, a1.y, pm);
            }
            (void)pms;
            *reinterpret_cast<ulonglong2*>(acc + size_t(b) * words + i) =
                make_ulonglong2(barrett128(s0.lo, s0.hi, q, rl, rh), barrett128(t0.lo, t0.hi, q, rl, rh));
            *reinterpret_cast<ulonglong2*>(acc + (size_t(npolys) + b) * words + i) =
                make_ulonglong2(barrett128(s1.lo, s1.hi, q, rl, rh), barrett128(t1.lo, t1.hi, q, rl, rh));
            if (b + 1 < b1) {
#pragma unroll
                for (int k = 0; k < NDMAX; ++k) dv[k] = dn[k];
            }
        }
    }
}

// ModDown of npolys polys (each level+1+K rows, coeff) -> level+1 rows,
// optionally added to `addend` (out = addend + ModDown(in); the relinearise
// / Galois epilogue, rlwe.hpp:612-613, :647). Centered y_s = |y_s| * sign
// multiplies |y_s| by +-(P/p_s) mod q (host-negated tables), so no per-term
// reduction of from_centered(y_s, q) is needed; terms are summed lazily
// (< 2Kq) and (x + 2Kq - sum) * P^-1 is one Shoup product.
__global__ void __launch_bounds__(256)
k_mod_down(DevRing R, GadgetDev G, u64* __restrict__ out, const u64* __restrict__ in, int level, u32 npolys,
           const u64* __restrict__ addend) {
    const u32 N = R.N, K = R.K, nq = R.q_count, lvl = u32(level);
    const u32 rin = lvl + 1 + K, rout = lvl + 1;
    const u64* c_s = G.md;                            // [K][2]
    const u64* w_sr = G.md + 2 * K;                   // [K][nq][4]
    const u64* pinv = w_sr + size_t(K) * nq * 4;      // [nq][2]
    const u64 total = u64(npolys) * N;
    for (u64 idx = blockIdx.x * u64(blockDim.x) + threadIdx.x; idx < total; idx += u64(gridDim.x) * blockDim.x) {
        const u64 p = idx >> R.logN;
        const u32 c = u32(idx & (N - 1));
        const u64* src = in + p * rin * N;
        u64* dst = out + p * rout * N;
        const u64* add = addend ? addend + p * rout * N : nullptr;
        u64 mag[kMaxSpecial];
        u32 sel[kMaxSpecial];
#pragma unroll
        for (u32 s = 0; s < u32(kMaxSpecial); ++s) {
            if (s < K) {
                const u64 ps = R.q[nq + s];
                const u64 v = shoup(src[size_t(lvl + 1 + s) * N + c], c_s[2 * s], c_s[2 * s + 1], ps);
                const bool neg = v > ps / 2;  // to_centered (common.hpp:84-86)
                mag[s] = neg ? ps - v : v;
                sel[s] = neg ? 2 : 0;
            }
        }
        for (u32 r0 = 0; r0 < rout; r0 += 4) {
            u64 acc[4] = {0, 0, 0, 0};
#pragma unroll
            for (u32 s = 0; s < u32(kMaxSpecial); ++s) {
                if (s < K) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const u32 r = min(r0 + k, rout - 1);
                        const u64* w = w_sr + (size_t(s) * nq + r) * 4 + sel[s];
                        if (G.lazy_moddown) acc[k] += shoup_lazy(mag[s], w[0], w[1], R.q[r]);
                        else acc[k] = add_mod(acc[k], shoup(mag[s], w[0], w[1], R.q[r]), R.q[r]);
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const u32 r = r0 + k;
                if (r >= rout) break;
                const u64 q = R.q[r];
                const u64 x = src[size_t(r) * N + c];
                const u64 val = G.lazy_moddown ? x + 2 * K * q - acc[k] : sub_mod(x, acc[k], q);
                u64 o = shoup(val, pinv[2 * r], pinv[2 * r + 1], q);
                if (add) o = add_mod(o, add[size_t(r) * N + c], q);
                dst[size_t(r) * N + c] = o;
            }
        }
    }
}

// ---- register-blocked variants (lazy sums) --------------------------------
// Same arithmetic as k_modup / k_mod_down, restructured so that the per-row
// constants are staged once per block in shared memory (one uniform LDS.128
// per (row, source) pair, shared by the CPT consecutive coefficients a thread
// owns), the source residues stay in registers sized by a compile-time bound
// (GMAX / KMAX), and every global access is a 16-byte vector.

// RAWIN: d holds raw inverse-NTT doubles (|v| <= 0.6q, no N^-1) -- the
// sources are formed on the FP64 pipe with N^-1 folded into their constants
// (G.srcn); the own-group rows then come from d_eval (required).
template <int GMAX, int CPT, bool RAW = false, bool RAWIN = false>
__global__ void __launch_bounds__(kMUThreads)
k_modup_v(DevRing R, GadgetDev G, u64* __restrict__ digits, const u64* __restrict__ d, int level,
          const u64* __restrict__ d_eval, u32 rows_per_group, u32 nd) {
    const u32 N = R.N, lvl = u32(level), K = R.K;
    // blockIdx.y = source poly * nd + digit: the whole batch in one launch
    const u32 j = blockIdx.y % nd, bsrc = blockIdx.y / nd, gs = G.group_size, first = j * gs;
    {
        const size_t in_words = size_t(lvl + 1) * N;
        d += bsrc * in_words;
        if (d_eval) d_eval += bsrc * in_words;
        digits += size_t(bsrc) * nd * (lvl + 1 + K) * N;
    }
    const u32 active = min(gs, lvl + 1 - first);
    const u32 rows_out = lvl + 1 + K, nrest = rows_out - active;
    const u64* src_tb = G.src + ((size_t(j) * gs + (active - 1)) * gs) * 2;
    const u64* conv_tb = G.conv + ((size_t(j) * gs + (active - 1)) * gs) * R.nmod * 2;
    // FP64 rows: every source q_i and the target q_t below 1.2 * 2^50
    // (the q-chain): y_i * w mod q_t by fp_mulmod; 0 <= y_i < 1.2 * 2^50
    // gives |term| <= 0.575 q_t (tg_fp64.cuh), summed exactly in doubles
    // (reduced every 8 terms: |sum| <= 4.6 q_t < 2^53). Other rows (60-bit
    // special primes) take the 64-bit Shoup path.
    bool src_fp = true;
    for (u32 i = 0; i < active; ++i) src_fp &= R.q[first + i] < kFpMaxQ;
    extern __shared__ ulonglong2 smw[];                                  // [nrest][active] (w, w') | (w, w/q) doubles
    u64* sq = reinterpret_cast<u64*>(smw + size_t(nrest) * active);      // [nrest] q, [nrest] one_shoup | 1/q
    for (u32 e = threadIdx.x; e < nrest * active; e += kMUThreads) {
        const u32 v = e / active, i = e - v * active;
        const u32 r = v < first ? v : v + active;
        const u32 t = mod_index(r, level, R.q_count);
        const u64* cw = conv_tb + (size_t(i) * R.nmod + t) * 2;
        if (src_fp && R.q[t] < kFpMaxQ) {
            const double wd = u2d(cw[0]);
            smw[e] = make_ulonglong2(static_cast<u64>(__double_as_longlong(wd)),
                                     static_cast<u64>(__double_as_longlong(__ddiv_rn(wd, u2d(R.q[t])))));
        } else {
            smw[e] = make_ulonglong2(cw[0], cw[1]);
        }
    }
    int tgt_fp = 1;  // every target row of this digit on the FP64 path
    for (u32 v = threadIdx.x; v < nrest; v += kMUThreads) {
        const u32 t = mod_index(v < first ? v : v + active, level, R.q_count);
        sq[v] = R.q[t];
        sq[nrest + v] = src_fp && R.q[t] < kFpMaxQ
                            ? static_cast<u64>(__double_as_longlong(__ddiv_rn(1.0, u2d(R.q[t]))))
                            : R.one_shoup[t];
        tgt_fp &= (src_fp && R.q[t] < kFpMaxQ) ? 1 : 0;
    }
    const bool all_fp = __syncthreads_and(tgt_fp) != 0;
    const u32 c0 = (blockIdx.x * kMUThreads + threadIdx.x) * CPT;
    if (c0 >= N) return;
    u64* out = digits + size_t(j) * rows_out * N + c0;
    u64 y[GMAX][CPT];
    // blockIdx.z = group of output rows (more threads in flight); the
    // sources are re-read per group, the own-group copy is group 0's
    const u32 v_begin = blockIdx.z * rows_per_group, v_end = min(nrest, v_begin + rows_per_group);
    const bool copy = blockIdx.z == 0;
#pragma unroll
    for (int i = 0; i < GMAX; ++i) {
        if (u32(i) < active) {
            const u32 s = first + i;
            const u64 q = R.q[s], w = src_tb[2 * i], ws = src_tb[2 * i + 1];
            u64 x[CPT];
            if constexpr (CPT == 2) {
                const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(d + size_t(s) * N + c0);
                x[0] = t.x;
                x[1] = t.y;
                // own-group row: exact copy (eval form when the caller has it;
                // the digit NTT then skips the row)
                if (copy)
                    *reinterpret_cast<ulonglong2*>(out + size_t(s) * N) =
                        d_eval ? *reinterpret_cast<const ulonglong2*>(d_eval + size_t(s) * N + c0) : t;
            } else {
                x[0] = d[size_t(s) * N + c0];
                if (copy) out[size_t(s) * N] = d_eval ? d_eval[size_t(s) * N + c0] : x[0];
            }
            if constexpr (RAWIN) {
                const u64* sn = G.srcn + ((size_t(j) * gs + (active - 1)) * gs + i) * 2;
                const double wd = __longlong_as_double(static_cast<long long>(sn[0]));
                const double wq = __longlong_as_double(static_cast<long long>(sn[1]));
                const double qd = u2d(q);
#pragma unroll
                for (int cc = 0; cc < CPT; ++cc) {
                    double v = fp_mulmod(__longlong_as_double(static_cast<long long>(x[cc])), wd, wq, qd);
                    if (v < 0) v = __dadd_rn(v, qd);
                    y[i][cc] = d2u(v);
                }
            } else {
#pragma unroll
                for (int cc = 0; cc < CPT; ++cc) y[i][cc] = shoup(x[cc], w, ws, q);
            }
        }
    }
    // sources as exact doubles once (FP64 targets), not per target row; the
    // 16-source variant converts per use (registers: measured slower hoisted)
    constexpr bool kHoist = GMAX <= 8;
    double yd[kHoist ? GMAX : 1][CPT];
    if constexpr (kHoist) {
#pragma unroll
        for (int i = 0; i < GMAX; ++i)
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) yd[i][cc] = (src_fp && u32(i) < active) ? u2d(y[i][cc]) : 0.0;
    }
    if (all_fp) {  // block-uniform: the source count as a compile-time constant
        u64* o = out;
        const u32 vb = v_begin, ve = v_end;
        switch (active) {
#define TG_MU_CASE(A)                                                                                 \
    case A:                                                                                           \
        if constexpr (A <= GMAX) {                                                                    \
            if constexpr (kHoist) modup_rows_fp<A, CPT, GMAX, RAW>(yd, smw, sq, nrest, vb, ve, first, o, N); \
            else modup_rows_fp<A, CPT, GMAX, RAW>(y, smw, sq, nrest, vb, ve, first, o, N);                 \
        }                                                                                             \
        return;
            TG_MU_CASE(1) TG_MU_CASE(2) TG_MU_CASE(3) TG_MU_CASE(4)
            TG_MU_CASE(5) TG_MU_CASE(6) TG_MU_CASE(7) TG_MU_CASE(8)
            TG_MU_CASE(9) TG_MU_CASE(10) TG_MU_CASE(11) TG_MU_CASE(12)
            TG_MU_CASE(13) TG_MU_CASE(14) TG_MU_CASE(15) TG_MU_CASE(16)
#undef TG_MU_CASE
            default: break;
        }
    }
    for (u32 v = v_begin; v < v_end; ++v) {
        const u64 q = sq[v];
        const ulonglong2* wr = smw + size_t(v) * active;
        const u32 r = v < first ? v : v + active;
        if (src_fp && q < kFpMaxQ) {
            const double qd = u2d(q), qi = __longlong_as_double(static_cast<long long>(sq[nrest + v]));
            double acc[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) acc[cc] = 0.0;
#pragma unroll
            for (int i = 0; i < GMAX; ++i) {
                if (u32(i) < active) {
                    const ulonglong2 w = wr[i];
                    const double wd = __longlong_as_double(static_cast<long long>(w.x));
                    const double wq = __longlong_as_double(static_cast<long long>(w.y));
#pragma unroll
                    for (int cc = 0; cc < CPT; ++cc) {
                        const double yv = kHoist ? yd[kHoist ? i : 0][cc] : u2d(y[i][cc]);
                        acc[cc] = __dadd_rn(acc[cc], fp_mulmod(yv, wd, wq, qd));
                        if ((i & 7) == 7 && u32(i + 1) < active) acc[cc] = fp_reduce(acc[cc], qd, qi);
                    }
                }
            }
            u64 o[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) o[cc] = fp_canon_small(fp_reduce(acc[cc], qd, qi), q);
            if constexpr (CPT == 2) *reinterpret_cast<ulonglong2*>(out + size_t(r) * N) = make_ulonglong2(o[0], o[1]);
            else out[size_t(r) * N] = o[0];
            continue;
        }
        u64 acc[CPT];
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) acc[cc] = 0;
#pragma unroll
        for (int i = 0; i < GMAX; ++i) {
            if (u32(i) < active) {
                const ulonglong2 w = wr[i];
#pragma unroll
                for (int cc = 0; cc < CPT; ++cc) acc[cc] += shoup_lazy(y[i][cc], w.x, w.y, q);
            }
        }
        const u64 one = sq[nrest + v];
        if constexpr (CPT == 2) {
            *reinterpret_cast<ulonglong2*>(out + size_t(r) * N) =
                make_ulonglong2(shoup(acc[0], 1, one, q), shoup(acc[1], 1, one, q));
        } else {
            out[size_t(r) * N] = shoup(acc[0], 1, one, q);
        }
    }
}

// CONV: the Q rows of `in` are not read (taken as 0): out = -conv * P^-1, the
// eval-form ModDown's coefficient part (tg_keyswitch_add_eval).
template <int KMAX, int CPT, bool CONV = false>
__global__ void __launch_bounds__(256)
k_mod_down_v(DevRing R, GadgetDev G, u64* __restrict__ out, const u64* __restrict__ in, int level, u32 npolys,
             const u64* __restrict__ addend, u32 rows_per_group) {
    const u32 N = R.N, K = R.K, nq = R.q_count, lvl = u32(level);
    const u32 rin = lvl + 1 + K, rout = lvl + 1;
    const u64* c_s = G.md;                        // [K][2]
    const u64* w_sr = G.md + 2 * K;               // [K][nq][4]: +w, +w', -w, -w'
    const u64* pinv = w_sr + size_t(K) * nq * 4;  // [nq][2]
    extern __shared__ ulonglong2 smd[];           // [rout][K] (+w, +w'), then [rout] (pinv, pinv'), [rout] q
    ulonglong2* sp = smd + size_t(rout) * K;
    u64* sq = reinterpret_cast<u64*>(sp + rout);
    for (u32 e = threadIdx.x; e < rout * K; e += blockDim.x) {
        const u32 r = e / K, s = e - r * K;
        const u64* w = w_sr + (size_t(s) * nq + r) * 4;
        smd[e] = make_ulonglong2(w[0], w[1]);
    }
    for (u32 r = threadIdx.x; r < rout; r += blockDim.x) {
        sp[r] = make_ulonglong2(pinv[2 * r], pinv[2 * r + 1]);
        sq[r] = R.q[r];
    }
    __syncthreads();
    const u32 per_poly = N / CPT;
    const u64 total = u64(npolys) * per_poly;
    for (u64 idx = blockIdx.x * u64(blockDim.x) + threadIdx.x; idx < total; idx += u64(gridDim.x) * blockDim.x) {
        const u32 p = u32(idx / per_poly);
        const u32 c0 = u32(idx - u64(p) * per_poly) * CPT;
        const u64* src = in + size_t(p) * rin * N + c0;
        u64* dst = out + size_t(p) * rout * N + c0;
        const u64* add = addend ? addend + size_t(p) * rout * N + c0 : nullptr;
        u64 mag[KMAX][CPT];
        bool neg[KMAX][CPT];
#pragma unroll
        for (int s = 0; s < KMAX; ++s) {
            if (u32(s) < K) {
                const u64 ps = R.q[nq + s], cw = c_s[2 * s], cws = c_s[2 * s + 1];
                u64 x[CPT];
                if constexpr (CPT == 2) {
                    const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(src + size_t(lvl + 1 + s) * N);
                    x[0] = t.x;
                    x[1] = t.y;
                } else {
                    x[0] = src[size_t(lvl + 1 + s) * N];
                }
#pragma unroll
                for (int cc = 0; cc < CPT; ++cc) {
                    const u64 v = shoup(x[cc], cw, cws, ps);
                    neg[s][cc] = v > ps / 2;  // to_centered (common.hpp:84-86)
                    mag[s][cc] = neg[s][cc] ? ps - v : v;
                }
            }
        }
        const u32 r_end = min(rout, (blockIdx.y + 1) * rows_per_group);  // blockIdx.y = group of output rows
        // row r's input (and addend) words are loaded one row ahead
        u64 xn[CPT], anx[CPT];
        auto load_row = [&](u32 r) {
            if constexpr (CONV) {
#pragma unroll
                for (int cc = 0; cc < CPT; ++cc) xn[cc] = anx[cc] = 0;
            } else if constexpr (CPT == 2) {
                const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(src + size_t(r) * N);
                xn[0] = t.x;
                xn[1] = t.y;
                if (add) {
                    const ulonglong2 u = *reinterpret_cast<const ulonglong2*>(add + size_t(r) * N);
                    anx[0] = u.x;
                    anx[1] = u.y;
                }
            } else {
                xn[0] = src[size_t(r) * N];
                if (add) anx[0] = add[size_t(r) * N];
            }
        };
        if (blockIdx.y * rows_per_group < r_end) load_row(blockIdx.y * rows_per_group);
        for (u32 r = blockIdx.y * rows_per_group; r < r_end; ++r) {
            u64 x[CPT], a[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
                x[cc] = xn[cc];
                a[cc] = anx[cc];
            }
            if (r + 1 < r_end) load_row(r + 1);
            const u64 q = sq[r];
            const ulonglong2* wr = smd + size_t(r) * K;
            u64 ap[CPT], an[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) ap[cc] = an[cc] = 0;
#pragma unroll
            for (int s = 0; s < KMAX; ++s) {
                if (u32(s) < K) {
                    const ulonglong2 w = wr[s];
#pragma unroll
                    for (int cc = 0; cc < CPT; ++cc) {
                        const u64 t = shoup_lazy(mag[s][cc], w.x, w.y, q);
                        ap[cc] += neg[s][cc] ? 0 : t;
                        an[cc] += neg[s][cc] ? t : 0;
                    }
                }
            }
            const ulonglong2 pv = sp[r];
            const u64 bias = 2 * u64(K) * q;
            u64 o[CPT];
#pragma unroll
            for (int cc = 0; cc < CPT; ++cc) {
                // (x - conv) * P^-1 with conv = ap - an (mod q)
                o[cc] = shoup(x[cc] + an[cc] + bias - ap[cc], pv.x, pv.y, q);
                if (add) o[cc] = add_mod(o[cc], a[cc], q);
            }
            if constexpr (CPT == 2) *reinterpret_cast<ulonglong2*>(dst + size_t(r) * N) = make_ulonglong2(o[0], o[1]);
            else dst[size_t(r) * N] = o[0];
        }
    }
}

// The Chebyshev ladder step on the relinearised product, before its rescale
// (ckks.hpp:532-555: rescale(2 prod - mul_scalar(T_c, 1, ratio)) or
// rescale(add_scalar(2 prod, -1))): row r of the ModDown value v becomes
// 2 v - m_r S_r (+ e_r at coefficient 0 of the part-0 polys). m_r, e_r are
// canonical residues mod q_r; S is a coefficient-form ciphertext batch (poly
// p at sub + p * stride). on = 0: plain rescale.
constexpr int kLadderRows = 32;
struct LadderPre {
    int on = 0;
    const u64* sub = nullptr;  // null: no subtrahend (the a == b step)
    u64 stride = 0;
    int has_e = 0;
    double m[kLadderRows], mq[kLadderRows];
    double e[kLadderRows];     // centred doubles of e_r
};

// FP64 ModDown (every special and q-chain prime below kFpMaxQ, tg_fp64.cuh):
// y_s = centered([x_s (P/p_s)^-1]_{p_s}) exactly as doubles, then
// out_r = x_r P^-1 + sum_s y_s (-(P/p_s) P^-1 mod q_r)  (mod q_r), which is
// (x_r - conv_r) P^-1 with the same canonical residue as mod_down_p
// (rlwe.hpp:579-589). Bounds: every product has |b| <= max(q, p/2) and
// b wq >= -0.6 * 2^50, so |term| <= 0.58 q; sums are reduced every 8 terms
// (|sum| <= 8 * 0.58 q + q/2 < 2^53).
// Host tables (G.mdf): [K][4] (p_s, fl(c_s/p_s), c_s, floor(p_s/2)) with
// c_s = (P/p_s)^-1 mod p_s; [nq][K][2] (w, fl(w/q_r)) with
// w = -(P/p_s) P^-1 mod q_r; [nq][4] (P^-1 mod q_r, fl(./q_r), q_r, fl(1/q_r)).
// KMAX = K exactly (dispatch in mod_down): every per-special loop is
// compile-time, no predicated terms.
// RAW: `in` holds the raw doubles of an inverse NTT without its N^-1 factor
// (|v| <= 0.6q, kw_inv_cols2<..., true>); the input constants carry N^-1
// (G.mdfn), so the canonical outputs are the same.
// RESCALE (relinearisation followed by rescale / rescale_add, ckks.hpp:315-324):
// every thread owns all rows of its coefficients; the last row is reduced
// first, centred exactly as rescale_round does (ring.hpp:493-518), and rows
// 0..nout-1 leave as (v_r - x_l) q_l^-1 mod q_r (+ radd's row: Evaluator::add
// of the rescaled product and y, k_rescale_fp's arithmetic) -- the ModDown
// output never goes through HBM. addend must be null. pre (LadderPre): the
// ladder step's linear part applied to every row before the rescale.
template <int KMAX, bool RAW = false, bool RESCALE = false>
__global__ void __launch_bounds__(256)
k_mod_down_fp(DevRing R, GadgetDev G, u64* __restrict__ out, const u64* __restrict__ in, int level, u32 npolys,
              const u64* __restrict__ addend, u32 rows_per_group, const u64* __restrict__ radd = nullptr,
              u64 astride = 0, u32 nout = 0, const LadderPre pre = LadderPre{}) {
    constexpr u32 K = KMAX;
    const u32 N = R.N, nq = R.q_count, lvl = u32(level);
    const u32 rin = lvl + 1 + K, rout = lvl + 1;
    const double* tab = RAW ? G.mdfn : G.mdf;
    const double* ys_t = tab;                           // [K][4]
    const double* w_rs = tab + 4 * K;                   // [nq][K][2]
    const double* p_r = w_rs + size_t(nq) * K * 2;      // [nq][4]
    auto in_d = [](u64 x) { return RAW ? __longlong_as_double(static_cast<long long>(x)) : u2d(x); };
    extern __shared__ double2 smf[];  // [rout][K] (w, wq), then [rout][2] (pinv, pinvq | q, qi), then [rout] q (u64)
    double2* sp = smf + size_t(rout) * K;
    u64* sq64 = reinterpret_cast<u64*>(sp + 2 * rout);
    for (u32 e = threadIdx.x; e < rout * K; e += blockDim.x) smf[e] = make_double2(w_rs[2 * e], w_rs[2 * e + 1]);
    for (u32 e = threadIdx.x; e < 2 * rout; e += blockDim.x) sp[e] = make_double2(p_r[2 * e], p_r[2 * e + 1]);
    for (u32 e = threadIdx.x; e < rout; e += blockDim.x) sq64[e] = R.q[e];
    __syncthreads();
    const u32 per_poly = N / 2;
    const u64 total = u64(npolys) * per_poly;
    for (u64 idx = blockIdx.x * u64(blockDim.x) + threadIdx.x; idx < total; idx += u64(gridDim.x) * blockDim.x) {
        const u32 p = u32(idx / per_poly);
        const u32 c0 = u32(idx - u64(p) * per_poly) * 2;
        const u64* src = in + size_t(p) * rin * N + c0;
        u64* dst = out + size_t(p) * rout * N + c0;
        const u64* add = addend ? addend + size_t(p) * rout * N + c0 : nullptr;
        double y[KMAX][2];
#pragma unroll
        for (int s = 0; s < KMAX; ++s) {
            if (u32(s) < K) {
                const double ps = ys_t[4 * s], cq = ys_t[4 * s + 1], cw = ys_t[4 * s + 2], half = ys_t[4 * s + 3];
                const ulonglong2 t = *reinterpret_cast<const ulonglong2*>(src + size_t(lvl + 1 + s) * N);
                const u64 xs[2] = {t.x, t.y};
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    double v = fp_mulmod(in_d(xs[cc]), cw, cq, ps);  // |v| <= 0.58 p
                    if (v < 0) v = __dadd_rn(v, ps);                 // canonical [0, p)
                    if (v > half) v = __dsub_rn(v, ps);              // to_centered (common.hpp:84-86)
                    y[s][cc] = v;
                }
            }
        }
        if constexpr (RESCALE) {
            // the reduced ModDown value of row r (|v| <= q/2 + 1) for both coefficients
            auto rowval = [&](u32 r, const ulonglong2 xv, double (&v)[2]) {
                const u64 x[2] = {xv.x, xv.y};
                const double2 pv = sp[2 * r], qv = sp[2 * r + 1];
                const double q = qv.x, qi = qv.y;
                const double2* wr = smf + size_t(r) * K;
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {
                    double acc = fp_mulmod(in_d(x[cc]), pv.x, pv.y, q);
#pragma unroll
                    for (int s = 0; s < KMAX; ++s) {
                        if (u32(s) < K) {
                            const double2 w = wr[s];
                            acc = __dadd_rn(acc, fp_mulmod(y[s][cc], w.x, w.y, q));
                            if ((s & 7) == 6 && u32(s + 1) < K) acc = fp_reduce(acc, q, qi);
                        }
                    }
                    v[cc] = fp_reduce(acc, q, qi);
                }
                if (pre.on) {  // 2 v - m_r S_r (+ e_r): |.| <= q + 2 + 0.58q + q/2 < 2^53
                    double t0 = __dadd_rn(v[0], v[0]), t1 = __dadd_rn(v[1], v[1]);
                    if (pre.sub) {
                        const ulonglong2 sv =
                            *reinterpret_cast<const ulonglong2*>(pre.sub + size_t(p) * pre.stride + size_t(r) * N + c0);
                        const double m = pre.m[r], mq = pre.mq[r];
                        t0 = __dsub_rn(t0, fp_mulmod(u2d(sv.x), m, mq, q));
                        t1 = __dsub_rn(t1, fp_mulmod(u2d(sv.y), m, mq, q));
                    }
                    if (pre.has_e && c0 == 0 && 2 * p < npolys) t0 = __dadd_rn(t0, pre.e[r]);
                    v[0] = fp_reduce(t0, q, qi);
                    v[1] = fp_reduce(t1, q, qi);
                }
            };
            const u64 ql = sq64[lvl], hl = ql >> 1;
            const double qld = u2d(ql);
            double xl[2];
            {
                double v[2];
                rowval(lvl, *reinterpret_cast<const ulonglong2*>(src + size_t(lvl) * N), v);
#pragma unroll
                for (int cc = 0; cc < 2; ++cc) {  // canonical, then centred as rescale_round does
                    const u64 cv = fp_canon_small(v[cc], ql);
                    xl[cc] = cv > hl ? __dsub_rn(u2d(cv), qld) : u2d(cv);
                }
            }
            const double* rsd = R.rsd + size_t(lvl) * nq * 2;
            u64* dr = out + size_t(p) * nout * N + c0;
            const u64* ar = radd ? radd + size_t(p) * astride + c0 : nullptr;
            ulonglong2 xn = *reinterpret_cast<const ulonglong2*>(src);
            for (u32 r = 0; r < nout; ++r) {
                const ulonglong2 xc = xn;
                if (r + 1 < nout) xn = *reinterpret_cast<const ulonglong2*>(src + size_t(r + 1) * N);
                double v[2];
                rowval(r, xc, v);
                const double q = sp[2 * r + 1].x, w = rsd[2 * r], wq = rsd[2 * r + 1];
                const u64 qu = sq64[r];
                u64 o[2];
#pragma unroll
                for (int cc = 0; cc < 2; ++cc)  // |v - x_l| <= q_r/2 + 1 + q_l/2 < 2^51: exact product
                    o[cc] = fp_canon_small(fp_mulmod(__dsub_rn(v[cc], xl[cc]), w, wq, q), qu);
                if (ar) {
                    const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(ar + size_t(r) * N);
                    o[0] = add_mod(o[0], a.x, qu);
                    o[1] = add_mod(o[1], a.y, qu);
                }
                *reinterpret_cast<ulonglong2*>(dr + size_t(r) * N) = make_ulonglong2(o[0], o[1]);
            }
            continue;
        }
        const u32 r_end = min(rout, (blockIdx.y + 1) * rows_per_group);
        // two rows in flight ahead of the one being reduced (ncu: the row
        // loads' long-scoreboard stalls dominated with one row of lookahead);
        // rows alternate between two register slots, unrolled by two so the
        // slots stay static registers
        const u32 r_begin = blockIdx.y * rows_per_group;
        auto load_row = [&](u32 r, ulonglong2& xv, ulonglong2& av) {
            if (r >= r_end) return;
            xv = *reinterpret_cast<const ulonglong2*>(src + size_t(r) * N);
            if (add) av = *reinterpret_cast<const ulonglong2*>(add + size_t(r) * N);
        };
        auto reduce_row = [&](u32 r, const ulonglong2 xv, const ulonglong2 av) {
            const u64 x[2] = {xv.x, xv.y}, a[2] = {av.x, av.y};
            const double2 pv = sp[2 * r], qv = sp[2 * r + 1];
            const double q = qv.x, qi = qv.y;
            const double2* wr = smf + size_t(r) * K;
            double acc[2];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) acc[cc] = fp_mulmod(in_d(x[cc]), pv.x, pv.y, q);
#pragma unroll
            for (int s = 0; s < KMAX; ++s) {
                if (u32(s) < K) {
                    const double2 w = wr[s];
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        acc[cc] = __dadd_rn(acc[cc], fp_mulmod(y[s][cc], w.x, w.y, q));
                        if ((s & 7) == 6 && u32(s + 1) < K) acc[cc] = fp_reduce(acc[cc], q, qi);
                    }
                }
            }
            const u64 qu = sq64[r];
            u64 o[2];
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                o[cc] = fp_canon_small(fp_reduce(acc[cc], q, qi), qu);  // |.| <= q/2 + 1
                if (add) o[cc] = add_mod(o[cc], a[cc], qu);
            }
            *reinterpret_cast<ulonglong2*>(dst + size_t(r) * N) = make_ulonglong2(o[0], o[1]);
        };
        ulonglong2 x0{}, a0{}, x1{}, a1{};
        load_row(r_begin, x0, a0);
        load_row(r_begin + 1, x1, a1);
        for (u32 r = r_begin; r < r_end; r += 2) {
            const ulonglong2 cx0 = x0, ca0 = a0;
            load_row(r + 2, x0, a0);
            reduce_row(r, cx0, ca0);
            if (r + 1 < r_end) {
                const ulonglong2 cx1 = x1, ca1 = a1;
                load_row(r + 3, x1, a1);
                reduce_row(r + 1, cx1, ca1);
            }
        }
    }
}

// Output-row groups so that about 1024 threads per SM are in flight.
inline u32 row_groups(u64 threads, u32 rows, int sms) {
    const u64 want = u64(sms) * 1024;
    u64 g = (want + threads - 1) / threads;
    return u32(g < 1 ? 1 : g > rows ? rows : g);
}

template <int GMAX, int CPT>
void launch_modup_v(const DevRing& R, const GadgetDev& G, int sms, u64* digits, const u64* d, int level, u32 nd,
                    const u64* d_eval, cudaStream_t s, u32 npolys = 1, bool raw = false, bool raw_in = false) {
    // worst-case table over the digits (the last digit may be partial)
    const u32 gs = G.group_size, rows_out = u32(level) + 1 + R.K;
    const size_t smem = size_t(rows_out) * gs * 16 + size_t(rows_out) * 16;
    const u32 bx = (R.N / CPT + kMUThreads - 1) / kMUThreads;
    const u32 groups = row_groups(u64(bx) * nd * npolys * kMUThreads, rows_out, sms);
    const u32 rpg = (rows_out + groups - 1) / groups;
    const dim3 grid(bx, nd * npolys, (rows_out + rpg - 1) / rpg);
    if (raw_in && raw)
        k_modup_v<GMAX, CPT, true, true><<<grid, kMUThreads, smem, s>>>(R, G, digits, d, level, d_eval, rpg, nd);
    else if (raw_in)
        k_modup_v<GMAX, CPT, false, true><<<grid, kMUThreads, smem, s>>>(R, G, digits, d, level, d_eval, rpg, nd);
    else if (raw) k_modup_v<GMAX, CPT, true><<<grid, kMUThreads, smem, s>>>(R, G, digits, d, level, d_eval, rpg, nd);
    else k_modup_v<GMAX, CPT><<<grid, kMUThreads, smem, s>>>(R, G, digits, d, level, d_eval, rpg, nd);
}

template <int KMAX, int CPT, bool CONV = false>
void launch_mod_down_v(const DevRing& R, const GadgetDev& G, int sms, u64* out, const u64* in, int level,
                       u32 npolys, const u64* addend, cudaStream_t s) {
    const u32 rout = u32(level) + 1;
    const size_t smem = size_t(rout) * R.K * 16 + size_t(rout) * 24;
    const u64 work = u64(npolys) * R.N / CPT;
    const u32 blocks = u32(std::min<u64>((work + 255) / 256, u64(sms) * 8));
    const u32 groups = row_groups(u64(blocks) * 256, rout, sms);
    const u32 rpg = (rout + groups - 1) / groups;
    k_mod_down_v<KMAX, CPT, CONV><<<dim3(blocks, (rout + rpg - 1) / rpg), 256, smem, s>>>(R, G, out, in, level,
                                                                                        npolys, addend, rpg);
}

// Eval-form ModDown epilogue: out_r = acc_r * P^-1 + negconv_r (+ add_r), all
// eval form; acc holds level+1+K rows per poly (Q rows read), negconv and add
// level+1 rows per poly. negconv = NTT(-conv * P^-1) from k_mod_down_v<CONV>.
__global__ void k_mod_down_finish(DevRing R, GadgetDev G, u64* __restrict__ out, const u64* __restrict__ acc,
                                  const u64* __restrict__ negconv, const u64* __restrict__ add, int level,
                                  u32 npolys) {
    const u32 N = R.N, K = R.K, nq = R.q_count, rout = u32(level) + 1, rin = rout + K;
    const u64* pinv = G.md + 2 * K + size_t(K) * nq * 4;  // [nq][2]
    const u64 per = u64(rout) * N, total = per * npolys;
    for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
        const u64 p = i / per, w = i - p * per;
        const u32 r = u32(w >> R.logN);
        const u64 q = R.q[r];
        u64 o = add_mod(shoup(acc[p * rin * N + w], pinv[2 * r], pinv[2 * r + 1], q), negconv[i], q);
        if (add) o = add_mod(o, add[i], q);
        out[i] = o;
    }
}

#include "tg_baseconv_tc.cuh"

}  // namespace

// ModUp of npolys coeff-form sources (level+1 rows each, back to back) into
// digits [npolys][nd][level+1+K][N], then one batched forward NTT of all
// digits (own-group rows skipped when the eval form d_eval is supplied).
inline bool raw_digits_on() {
    static const bool on = [] {
        const char* e = getenv("TG_RAW_DIGITS");
        return !(e && *e == '0');
    }();
    return on;
}

// TG_FUSED_RESCALE=0: relinearise-then-rescale as two passes (A/B switch)
inline bool fused_rescale_on() {
    static const bool on = [] {
        const char* e = getenv("TG_FUSED_RESCALE");
        return !(e && *e == '0');
    }();
    return on;
}

int modup(tg_gadget* g, u64* digits, const u64* d, int level, cudaStream_t s, const u64* d_eval = nullptr,
          u32 npolys = 1, bool cols_only = false, bool raw_in = false) {
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const u32 nd = tg_gadget_digit_count(g, level);
    const size_t in_words = size_t(level + 1) * R.N, dig_words = size_t(nd) * (level + 1 + R.K) * R.N;
    dim3 grid((R.N + kMUThreads - 1) / kMUThreads, nd);
    if (raw_in && !(d_eval && g->g.srcn && !g->g.base2_bits && g->g.lazy_modup && g->g.group_size <= 16))
        return fail(TG_E_ARG, "[rlwe] raw ModUp sources need the FP64 gadget tables and the eval form");
    // converted rows as centred doubles straight into the column-pair phase
    // (own rows skipped there: eval form given); N = 2^16, every row FP64
    const bool raw = cols_only && d_eval && !g->g.base2_bits && R.logN == 16 && ntt_inverse_cols_raw_ok(ctx) &&
                     g->g.lazy_modup && g->g.group_size <= 16 && raw_digits_on();
    {
        ProfScope prof(ctx, TG_OP_MODUP,
                       8.0 * R.N * npolys * (double(level + 1) + double(nd) * (level + 1 + R.K)), s);
        const GadgetDev& G = g->g;
        if (G.base2_bits) {  // sub-digits per prime, no own-group rows to reuse
            const size_t per_digit = size_t(level + 1 + R.K) * R.N;
            size_t off = 0;
            for (u32 j = 0; j <= u32(level); ++j) {  // one launch per prime for the whole batch
                k_decompose_base2<<<dim3((R.N + 127) / 128, npolys), 128, 0, s>>>(
                    R, digits + off * per_digit, d, level, j, g->nsub[j], G.base2_bits, dig_words, in_words);
                off += g->nsub[j];
            }
            d_eval = nullptr;
        } else if (G.tc_kb_mu && tc_modup_fits(R.K, level, G.group_size, nd) &&
                   (G.tc_mode == 2 || (G.tc_kb_mu <= 64 && level >= 16 && u64(nd) * npolys * R.N >= (u64(148) << 11)))) {
            // int8 tensor cores (tg_baseconv_tc.cuh); auto: where measured faster than k_modup_v
            // (digit groups <= 8, high levels, large batches: config 4 level 21 batch 8 229 -> 185 us)
            switch (G.tc_kb_mu) {
                case 32: launch_modup_tc<32>(R, G, ctx->sms, digits, d, level, nd, d_eval, npolys, s, raw, raw_in); break;
                case 64: launch_modup_tc<64>(R, G, ctx->sms, digits, d, level, nd, d_eval, npolys, s, raw, raw_in); break;
                case 96: launch_modup_tc<96>(R, G, ctx->sms, digits, d, level, nd, d_eval, npolys, s, raw, raw_in); break;
                default: launch_modup_tc<128>(R, G, ctx->sms, digits, d, level, nd, d_eval, npolys, s, raw, raw_in); break;
            }
        } else if (G.lazy_modup && G.group_size <= 4)
            launch_modup_v<4, 2>(R, G, ctx->sms, digits, d, level, nd, d_eval, s, npolys, raw, raw_in);
        else if (G.lazy_modup && G.group_size <= 8)
            launch_modup_v<8, MODUP_CPT8>(R, G, ctx->sms, digits, d, level, nd, d_eval, s, npolys, raw, raw_in);
        else if (G.lazy_modup && G.group_size <= 16)
            launch_modup_v<16, MODUP_CPT16>(R, G, ctx->sms, digits, d, level, nd, d_eval, s, npolys, raw, raw_in);
        else
            for (u32 b = 0; b < npolys; ++b)
                k_modup<<<grid, kMUThreads, 0, s>>>(R, G, digits + b * dig_words, d + b * in_words, level,
                                                    d_eval ? d_eval + b * in_words : nullptr);
    }
    TG_LAUNCH_CHECK();
    const u32 skip = d_eval ? (g->g.group_size | (npolys > 1 ? nd << 16 : 0u) | (raw ? kTgRawDigits : 0u)) : 0u;
    if (cols_only) return ntt_forward_cols(ctx, digits, level, int(R.K), nd * npolys, s, skip);
    return ntt_forward_oop(ctx, digits, digits, level, int(R.K), nd * npolys, s, skip);
}

// ModDown followed by rescale_round (+ add): out holds npolys polys of nout
// rows (nout = level without an addend, out_level + 1 with one); poly p's
// addend at radd + p * astride (k_mod_down_fp's RESCALE).
struct RescaleSpec {
    const u64* radd;
    u64 astride;
    u32 nout;
    const LadderPre* pre = nullptr;  // the ladder step before the rescale
};

template <int KMAX, bool RAW = false>
void launch_mod_down_fp(const DevRing& R, const GadgetDev& G, int sms, u64* out, const u64* in, int level,
                        u32 npolys, const u64* addend, cudaStream_t s, const RescaleSpec* rs = nullptr) {
    const u32 rout = u32(level) + 1;
    const size_t smem = size_t(rout) * R.K * 16 + size_t(rout) * 40;
    const u64 work = u64(npolys) * R.N / 2;
    const u32 blocks = u32(std::min<u64>((work + 255) / 256, u64(sms) * 8));
    if (rs) {  // every thread owns all rows of its coefficients
        k_mod_down_fp<KMAX, RAW, true><<<blocks, 256, smem, s>>>(R, G, out, in, level, npolys, nullptr, rout,
                                                                 rs->radd, rs->astride, rs->nout,
                                                                 rs->pre ? *rs->pre : LadderPre{});
        return;
    }
    const u32 groups = row_groups(u64(blocks) * 256, rout, sms);
    const u32 rpg = (rout + groups - 1) / groups;
    k_mod_down_fp<KMAX, RAW><<<dim3(blocks, (rout + rpg - 1) / rpg), 256, smem, s>>>(R, G, out, in, level, npolys,
                                                                                    addend, rpg);
}

int mod_down(tg_gadget* g, u64* out, const u64* in, int level, u32 npolys, cudaStream_t s,
             const u64* addend = nullptr, bool raw = false, const RescaleSpec* rs = nullptr) {
    const DevRing& R = g->ctx->ring;
    ProfScope prof(g->ctx, TG_OP_MOD_DOWN,
                   8.0 * R.N * npolys *
                       (rs ? (level + 1.0 + R.K + rs->nout * (rs->radd ? 2.0 : 1.0) +
                              ((rs->pre && rs->pre->sub) ? level + 1.0 : 0.0))
                           : (2.0 * (level + 1) + R.K + (addend ? level + 1 : 0))),
                   s);
    const GadgetDev& G = g->g;
    const int sms = g->ctx->sms;
    if (raw && !(G.fp_moddown && G.mdfn)) return fail(TG_E_ARG, "[rlwe] raw ModDown input needs the FP64 ModDown");
    if (rs && (addend || !G.fp_moddown || R.K > 16))
        return fail(TG_E_ARG, "[rlwe] ModDown + rescale needs the FP64 ModDown and no ModDown addend");
    bool done = false;
    // int8 tensor-core base conversion (tg_baseconv_tc.cuh); auto: batched, high
    // levels (measured: config 5 ModDown 77.3 -> 56.5 ms per query; small or
    // low-level launches stay on the FP64 kernel)
    if (!rs && G.tc_kb_md && tc_mod_down_fits(level) && (G.tc_mode == 2 || (npolys >= 4 && level >= 16))) {
        done = true;
#define TG_MDTC(kb)                                                                                     \
    case kb:                                                                                            \
        done = raw ? launch_mod_down_tc<kb, true>(R, G, sms, out, in, level, npolys, addend, s)        \
                   : launch_mod_down_tc<kb, false>(R, G, sms, out, in, level, npolys, addend, s);      \
        break;
        switch (G.tc_kb_md) { TG_MDTC(32) TG_MDTC(64) TG_MDTC(96) TG_MDTC(128) default: done = false; }
#undef TG_MDTC
    }
    if (done) {
    } else if (G.fp_moddown) {
        done = true;
        switch (R.K) {
#define TG_MD_CASE(k)                                                                    \
    case k:                                                                              \
        if (raw) launch_mod_down_fp<k, true>(R, G, sms, out, in, level, npolys, addend, s, rs); \
        else launch_mod_down_fp<k>(R, G, sms, out, in, level, npolys, addend, s, rs);       \
        break;
            TG_MD_CASE(1) TG_MD_CASE(2) TG_MD_CASE(3) TG_MD_CASE(4) TG_MD_CASE(5) TG_MD_CASE(6) TG_MD_CASE(7)
            TG_MD_CASE(8) TG_MD_CASE(9) TG_MD_CASE(10) TG_MD_CASE(11) TG_MD_CASE(12) TG_MD_CASE(13)
            TG_MD_CASE(14) TG_MD_CASE(15) TG_MD_CASE(16)
#undef TG_MD_CASE
            default: done = false;
        }
    }
    if (done) {
    } else if (G.lazy_moddown && R.K <= 4) launch_mod_down_v<4, 2>(R, G, sms, out, in, level, npolys, addend, s);
    else if (G.lazy_moddown && R.K <= 8) launch_mod_down_v<8, 2>(R, G, sms, out, in, level, npolys, addend, s);
    else if (G.lazy_moddown && R.K <= 16) launch_mod_down_v<16, 1>(R, G, sms, out, in, level, npolys, addend, s);
    else k_mod_down<<<grid_for(size_t(npolys) * R.N), kThreads, 0, s>>>(R, G, out, in, level, npolys, addend);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

// acc buffer holds 2 polys (level+1+K rows each) back to back.
int ks_inner(tg_gadget* g, u64* out0, u64* out1, const u64* digits, u32 nd, const u64* key, int level, u64* acc,
             cudaStream_t s, const u64* add0 = nullptr, const u64* add1 = nullptr) {
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const size_t words = size_t(level + 1 + R.K) * R.N;
    {
    // digits + both key halves read once, two accumulators written
    ProfScope prof(ctx, TG_OP_KEY_INNER, 8.0 * words * (3.0 * nd + 2.0), s);
    k_key_inner<<<grid_for(words), kThreads, 0, s>>>(R, acc, acc + words, digits, nd, key, level);
    }
    TG_LAUNCH_CHECK();
    if (int rc = ntt_inverse_rows(ctx, acc, level, int(R.K), 2, s)) return rc;
    const size_t ow = size_t(level + 1) * R.N;
    if (out1 == out0 + ow && ((!add0 && !add1) || (add0 && add1 == add0 + ow)))
        return mod_down(g, out0, acc, level, 2, s, add0);
    if (int rc = mod_down(g, out0, acc, level, 1, s, add0)) return rc;
    return mod_down(g, out1, acc + words, level, 1, s, add1);
}

// Batched key inner product + iNTT + ModDown(+add) for npolys sources.
// acc: [2][npolys][level+1+K][N] scratch; out0/out1/add0/add1: npolys polys
// of level+1 rows back to back.
int ks_inner_batch(tg_gadget* g, u64* out0, u64* out1, const u64* digits, u32 nd, u32 npolys, const u64* key,
                   int level, u64* acc, cudaStream_t s, const u64* add0, const u64* add1, bool eval_add = false) {
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const size_t words = size_t(level + 1 + R.K) * R.N;
    {
        // digits once, key once per batch, two accumulators written
        ProfScope prof(ctx, TG_OP_KEY_INNER, 8.0 * words * (npolys * (nd + 2.0) + 2.0 * nd), s);
        // sources per thread: all of them when the words alone fill the GPU
        // (each key word read once per batch), fewer for small rings
        const u64 want = u64(ctx->sms) * 2048;
        u32 ppt = npolys;
        while (ppt > 1 && words / 2 * ((npolys + ppt - 1) / ppt) < want) ppt = (ppt + 1) / 2;
        const u32 blocks = grid_for(words / 2 * ((npolys + ppt - 1) / ppt));
        const u64* ea0 = eval_add ? add0 : nullptr;
        const u64* ea1 = eval_add ? add1 : nullptr;
        const u64* pmod = g->g.md + 2 * R.K + size_t(R.K) * R.q_count * 4 + size_t(R.q_count) * 2;
        if (nd <= 4)
            k_key_inner_b<4><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt, ea0, ea1, pmod);
        else if (nd <= 8)
            k_key_inner_b<8><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt, ea0, ea1, pmod);
        else if (nd <= 15)
            k_key_inner_b<15><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt, ea0, ea1, pmod);
        else return fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
    }
    TG_LAUNCH_CHECK();
    if (int rc = ntt_inverse_rows(ctx, acc, level, int(R.K), 2 * npolys, s)) return rc;
    const u64* m0 = eval_add ? nullptr : add0;
    const u64* m1 = eval_add ? nullptr : add1;
    const size_t qwords = size_t(level + 1) * R.N;
    // both halves in one launch when outputs (and addends) are back to back
    if (out1 == out0 + size_t(npolys) * qwords && (m0 ? m1 == m0 + size_t(npolys) * qwords : !m1))
        return mod_down(g, out0, acc, level, 2 * npolys, s, m0);
    if (int rc = mod_down(g, out0, acc, level, npolys, s, m0)) return rc;
    return mod_down(g, out1, acc + size_t(npolys) * words, level, npolys, s, m1);
}

// Batched key switch through the fused core (ks_fused_ok): ModUp base
// conversion + forward column phase of the digits, kw_ks_chunks (digits'
// forward chunk phase, key inner product, accumulators' inverse chunk
// phase), inverse column phase, ModDown(+add). scratch: npolys*(nd+2) polys
// of level+1+K rows (digits, then both accumulators).
int ks_fused_batch(tg_gadget* g, u64* out0, u64* out1, const u64* d, const u64* d_eval, u32 nd, u32 npolys,
                   const u64* key, int level, u64* scratch, cudaStream_t s, const u64* add0, const u64* add1,
                   bool eval_add, const u64* ty0 = nullptr, const u64* ty1 = nullptr, bool raw_in = false,
                   const RescaleSpec* rs = nullptr, Tensor2 t2 = Tensor2{}) {
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const size_t words = size_t(level + 1 + R.K) * R.N;
    u64* digits = scratch;
    u64* acc = scratch + size_t(npolys) * nd * words;
    if (int rc = modup(g, digits, d, level, s, d_eval, npolys, true, raw_in)) return rc;
    const u64* pmod = g->g.md + 2 * R.K + size_t(R.K) * R.q_count * 4 + size_t(R.q_count) * 2;
    const u32 own = (d_eval && !g->g.base2_bits) ? g->g.group_size : 0u;
    if (int rc = ks_fused_chunks(ctx, acc, digits, nd, npolys, key, level, own, eval_add ? add0 : nullptr,
                                 eval_add ? add1 : nullptr, pmod, s, eval_add ? ty0 : nullptr,
                                 eval_add ? ty1 : nullptr, eval_add ? t2 : Tensor2{}))
        return rc;
    // the accumulators' inverse column phase hands ModDown raw doubles
    // (its N^-1 folded into ModDown's constants) when both kernels allow it
    const bool raw = g->g.fp_moddown && g->g.mdfn && ntt_inverse_cols_raw_ok(ctx);
    if (int rc = ntt_inverse_cols(ctx, acc, level, int(R.K), 2 * npolys, s, raw)) return rc;
    if (rs) {  // out0/out1 back to back, nout rows per poly
        if (!eval_add) return fail(TG_E_ARG, "[rlwe] ModDown + rescale takes eval-form addends only");
        return mod_down(g, out0, acc, level, 2 * npolys, s, nullptr, raw, rs);
    }
    const u64* m0 = eval_add ? nullptr : add0;
    const u64* m1 = eval_add ? nullptr : add1;
    const size_t qwords = size_t(level + 1) * R.N;
    if (out1 == out0 + size_t(npolys) * qwords && (m0 ? m1 == m0 + size_t(npolys) * qwords : !m1))
        return mod_down(g, out0, acc, level, 2 * npolys, s, m0, raw);
    if (int rc = mod_down(g, out0, acc, level, npolys, s, m0, raw)) return rc;
    return mod_down(g, out1, acc + size_t(npolys) * words, level, npolys, s, m1, raw);
}

}  // namespace tg

using namespace tg;

static int check_ks(tg_gadget* g, int level) {
    if (!g || !g->ctx) return fail(TG_E_ARG, "[rlwe] null gadget");
    if (level < 0 || u32(level) >= g->ctx->ring.q_count) return fail(TG_E_ARG, "[rlwe] level out of range");
    if (g->ctx->ring.K == 0) return fail(TG_E_ARG, "[rlwe] key switching needs special primes");
    return TG_OK;
}

extern "C" int tg_modup(tg_gadget* g, uint64_t* digits, const uint64_t* d, int level, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    DeviceGuard guard(g->ctx->device);
    return modup(g, digits, d, level, as_stream(stream));
}

extern "C" int tg_mod_down(tg_gadget* g, uint64_t* out, const uint64_t* in, int level, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    DeviceGuard guard(g->ctx->device);
    return mod_down(g, out, in, level, 1, as_stream(stream));
}

extern "C" int tg_ks_inner(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* digits, uint32_t ndigits,
                           const uint64_t* key, uint32_t key_digits, int level, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    if (ndigits == 0) return fail(TG_E_ARG, "[rlwe] empty decomposition");
    if (ndigits > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    tg_context* ctx = g->ctx;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* acc = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&acc, 2 * words * 8, ctx->pool, s));
    int rc = ks_inner(g, out0, out1, digits, ndigits, key, level, static_cast<u64*>(acc), s);
    cudaFreeAsync(acc, s);
    return rc;
}

extern "C" int tg_switch_key_apply(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                                   const uint64_t* key, uint32_t key_digits, int level, void* stream) {
    return tg_keyswitch_add(g, out0, out1, d, nullptr, key, key_digits, level, nullptr, nullptr, stream);
}

extern "C" int tg_keyswitch_add(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                                const uint64_t* d_eval, const uint64_t* key,
                                uint32_t key_digits, int level, const uint64_t* add0, const uint64_t* add1,
                                void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    tg_context* ctx = g->ctx;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, (nd + 2) * words * 8, ctx->pool, s));
    u64* digits = static_cast<u64*>(scratch);
    int rc;
    if (ks_fused_ok(ctx)) {
        rc = ks_fused_batch(g, out0, out1, d, d_eval, nd, 1, key, level, digits, s, add0, add1, false);
    } else {
        rc = modup(g, digits, d, level, s, d_eval);
        if (rc == TG_OK)
            rc = ks_inner(g, out0, out1, digits, nd, key, level, digits + size_t(nd) * words, s, add0, add1);
    }
    cudaFreeAsync(scratch, s);
    return rc;
}

extern "C" int tg_keyswitch_add_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                                      const uint64_t* d_eval, const uint64_t* key, uint32_t key_digits, int level,
                                      const uint64_t* add0, const uint64_t* add1, uint32_t npolys, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    if (npolys == 0) return TG_OK;
    tg_context* ctx = g->ctx;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, size_t(npolys) * (nd + 2) * words * 8, ctx->pool, s));
    u64* digits = static_cast<u64*>(scratch);
    int rc;
    if (ks_fused_ok(ctx)) {
        rc = ks_fused_batch(g, out0, out1, d, d_eval, nd, npolys, key, level, digits, s, add0, add1, false);
    } else {
        rc = modup(g, digits, d, level, s, d_eval, npolys);
        if (rc == TG_OK)
            rc = ks_inner_batch(g, out0, out1, digits, nd, npolys, key, level, digits + size_t(npolys) * nd * words,
                                s, add0, add1);
    }
    cudaFreeAsync(scratch, s);
    return rc;
}

// relinearize of a batch (rlwe.hpp:601-620) from the tensor product's eval-
// form parts: c2 in coefficient form (ModUp source; its eval form, optional,
// supplies the digits' own-group rows), c0/c1 in eval form are folded into
// the accumulators' Q rows as P * c before the inverse transform, so
// ModDown(acc + P c) = c + ModDown(acc) needs no coefficient form of c0/c1.
extern "C" int tg_relinearize_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                                    const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits, int level,
                                    const uint64_t* c0_eval, const uint64_t* c1_eval, uint32_t npolys,
                                    void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    if (npolys == 0) return TG_OK;
    if (!c0_eval || !c1_eval) return fail(TG_E_ARG, "[rlwe] relinearize needs both eval-form parts");
    tg_context* ctx = g->ctx;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    if (nd > 15) return fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, size_t(npolys) * (nd + 2) * words * 8, ctx->pool, s));
    u64* digits = static_cast<u64*>(scratch);
    int rc;
    if (ks_fused_ok(ctx)) {
        rc = ks_fused_batch(g, out0, out1, c2, c2_eval, nd, npolys, key, level, digits, s, c0_eval, c1_eval, true);
    } else {
        rc = modup(g, digits, c2, level, s, c2_eval, npolys);
        if (rc == TG_OK)
            rc = ks_inner_batch(g, out0, out1, digits, nd, npolys, key, level, digits + size_t(npolys) * nd * words,
                                s, c0_eval, c1_eval, true);
    }
    cudaFreeAsync(scratch, s);
    return rc;
}

// Operand strides of the tensor entry points: op_strides = NULL or 4 host
// words (words between consecutive polys of the x, y, u, v parts; 0 = tight).
static int set_op_strides(Tensor2& t2, const uint64_t* op_strides, size_t tight, bool& strided) {
    strided = false;
    if (!op_strides) return TG_OK;
    u64* dst[4] = {&t2.sx, &t2.sy, &t2.su, &t2.sv};
    for (int i = 0; i < 4; ++i)
        if (op_strides[i] && op_strides[i] != tight) {
            if (op_strides[i] < tight) return fail(TG_E_ARG, "[ckks] operand stride below the poly size");
            *dst[i] = op_strides[i];
            strided = true;
        }
    return TG_OK;
}

// Tight copies of strided operand parts for the paths that need them (rings
// without the fused core): ops = {x0, x1, y0, y1, u0, u1, v0, v1}.
static int gather_ops(tg_context* ctx, const u64* (&ops)[8], Tensor2& t2, u32 npolys, size_t tight, void** tmp,
                      cudaStream_t s) {
    const u64 st[4] = {t2.sx, t2.sy, t2.su, t2.sv};
    TG_CUDA(cudaMallocFromPoolAsync(tmp, 8 * tight * npolys * 8, ctx->pool, s));
    for (int i = 0; i < 8; ++i)
        if (ops[i] && st[i / 2]) {
            u64* d = static_cast<u64*>(*tmp) + size_t(i) * tight * npolys;
            TG_CUDA(cudaMemcpy2DAsync(d, tight * 8, ops[i], st[i / 2] * 8, tight * 8, npolys, cudaMemcpyDeviceToDevice,
                                      s));
            ops[i] = d;
        }
    t2.sx = t2.sy = t2.su = t2.sv = 0;
    return TG_OK;
}

static bool tensor2_given(const Tensor2& t2, bool& bad) {
    const int n = (t2.u0 != nullptr) + (t2.u1 != nullptr) + (t2.v0 != nullptr) + (t2.v1 != nullptr);
    bad = n != 0 && n != 4;
    return n == 4;
}

static int relinearize_tensor_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                                    const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits, int level,
                                    const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                    const Tensor2& t2, uint32_t npolys, int c2_raw, void* stream);

extern "C" int tg_relinearize_tensor_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                                           const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits,
                                           int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0,
                                           const uint64_t* y1, uint32_t npolys, int c2_raw, void* stream) {
    return relinearize_tensor_batch(g, out0, out1, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1, Tensor2{},
                                    npolys, c2_raw, stream);
}

static int relinearize_tensor_batch(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* c2,
                                    const uint64_t* c2_eval, const uint64_t* key, uint32_t key_digits, int level,
                                    const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                    const Tensor2& t2, uint32_t npolys, int c2_raw, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    bool bad = false;
    const bool two = tensor2_given(t2, bad);
    if (bad) return fail(TG_E_ARG, "[rlwe] the second product needs all four operand parts");
    if (npolys == 0) return TG_OK;
    if (!x0 || !x1 || !y0 || !y1) return fail(TG_E_ARG, "[rlwe] relinearize needs both operands' eval parts");
    if (c2_raw && !(c2_eval && ks_fused_ok(g->ctx)))
        return fail(TG_E_ARG, "[rlwe] a raw c2 needs its eval form and the fused key switch");
    tg_context* ctx = g->ctx;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    if (nd > 15) return fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    if (!ks_fused_ok(ctx)) {  // the tensor's c0 / c1 through HBM, then the plain batched relinearisation
        const size_t tight = size_t(level + 1) * ctx->ring.N, qw = tight * npolys;
        Tensor2 tt = t2;
        const u64* ops[8] = {x0, x1, y0, y1, tt.u0, tt.u1, tt.v0, tt.v1};
        void* gt = nullptr;
        if (tt.sx || tt.sy || tt.su || tt.sv)
            if (int rc = gather_ops(ctx, ops, tt, npolys, tight, &gt, s)) return rc;
        void* cc = nullptr;
        TG_CUDA(cudaMallocFromPoolAsync(&cc, 3 * qw * 8, ctx->pool, s));
        u64* c0 = static_cast<u64*>(cc);  // (c2 recomputed into the third slot, unused)
        int rc = two ? tg_tensor2(ctx, c0, c0 + qw, c0 + 2 * qw, ops[0], ops[1], ops[2], ops[3], ops[4], ops[5], ops[6],
                                  ops[7], level, npolys, stream)
                     : tg_tensor(ctx, c0, c0 + qw, c0 + 2 * qw, ops[0], ops[1], ops[2], ops[3], level, npolys, stream);
        if (rc == TG_OK)
            rc = tg_relinearize_batch(g, out0, out1, c2, c2_eval, key, key_digits, level, c0, c0 + qw, npolys,
                                      stream);
        cudaFreeAsync(cc, s);
        if (gt) cudaFreeAsync(gt, s);
        return rc;
    }
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, size_t(npolys) * (nd + 2) * words * 8, ctx->pool, s));
    const int rc = ks_fused_batch(g, out0, out1, c2, c2_eval, nd, npolys, key, level, static_cast<u64*>(scratch), s,
                                  x0, x1, true, y0, y1, c2_raw != 0, nullptr, t2);
    cudaFreeAsync(scratch, s);
    return rc;
}

extern "C" int tg_relinearize_tensor_rescale_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                                   const uint64_t* c2_eval, const uint64_t* key,
                                                   uint32_t key_digits, int level, const uint64_t* x0,
                                                   const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                                   uint32_t npolys, int c2_raw, const uint64_t* add,
                                                   uint64_t add_stride, int out_level, void* stream) {
    return tg_relinearize_tensor2_rescale_batch(g, out, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1, nullptr,
                                                nullptr, nullptr, nullptr, npolys, c2_raw, add, add_stride,
                                                out_level, stream);
}

extern "C" int tg_relinearize_tensor2_rescale_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                                    const uint64_t* c2_eval, const uint64_t* key,
                                                    uint32_t key_digits, int level, const uint64_t* x0,
                                                    const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                                    const uint64_t* u0, const uint64_t* u1, const uint64_t* v0,
                                                    const uint64_t* v1, uint32_t npolys, int c2_raw,
                                                    const uint64_t* add, uint64_t add_stride, int out_level,
                                                    void* stream) {
    return tg_relinearize_tensor2_rescale_batch_strided(g, out, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1,
                                                        u0, u1, v0, v1, nullptr, npolys, c2_raw, add, add_stride,
                                                        out_level, stream);
}

extern "C" int tg_relinearize_tensor2_rescale_batch_strided(
    tg_gadget* g, uint64_t* out, const uint64_t* c2, const uint64_t* c2_eval, const uint64_t* key,
    uint32_t key_digits, int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
    const uint64_t* u0, const uint64_t* u1, const uint64_t* v0, const uint64_t* v1, const uint64_t* op_strides,
    uint32_t npolys, int c2_raw, const uint64_t* add, uint64_t add_stride, int out_level, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    Tensor2 t2;
    t2.u0 = u0, t2.u1 = u1, t2.v0 = v0, t2.v1 = v1;
    bool bad = false;
    tensor2_given(t2, bad);
    if (bad) return fail(TG_E_ARG, "[rlwe] the second product needs all four operand parts");
    bool strided = false;
    if (int rc = set_op_strides(t2, op_strides, size_t(level + 1) * g->ctx->ring.N, strided)) return rc;
    if (level < 1) return fail(TG_E_ARG, "[ring] cannot rescale at level 0");
    if (add && (out_level < 0 || out_level > level - 1)) return fail(TG_E_ARG, "[ring] rescale_add level out of range");
    if (npolys == 0) return TG_OK;
    if (!x0 || !x1 || !y0 || !y1) return fail(TG_E_ARG, "[rlwe] relinearize needs both operands' eval parts");
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    for (int r = 0; r <= level; ++r)
        if (ctx->h_q[r] >= kFpMaxQ) return fail(TG_E_ARG, "[ring] fused rescale needs FP64 q-chain rows");
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    if (nd > 15) return fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const u32 nout = add ? u32(out_level) + 1 : u32(level);
    // fused while the batch alone fills the GPU (every thread walks all rows)
    const bool fuse = ks_fused_ok(ctx) && g->g.fp_moddown && R.K <= 16 && fused_rescale_on() &&
                      u64(npolys) * R.N >= u64(ctx->sms) * 512;
    if (!fuse) {  // relinearise into scratch, then rescale(_add)
        if (c2_raw && !ks_fused_ok(ctx))
            return fail(TG_E_ARG, "[rlwe] a raw c2 needs its eval form and the fused key switch");
        const size_t qw = size_t(level + 1) * R.N * npolys;
        void* tmp = nullptr;
        TG_CUDA(cudaMallocFromPoolAsync(&tmp, 2 * qw * 8, ctx->pool, s));
        u64* t = static_cast<u64*>(tmp);
        int rc = relinearize_tensor_batch(g, t, t + qw, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1, t2,
                                          npolys, c2_raw, stream);
        if (rc == TG_OK)
            rc = add ? tg_rescale_add(ctx, out, t, level, 2 * npolys, add, add_stride, out_level, stream)
                     : tg_rescale(ctx, out, t, level, 2 * npolys, stream);
        cudaFreeAsync(tmp, s);
        return rc;
    }
    const size_t words = size_t(level + 1 + R.K) * R.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, size_t(npolys) * (nd + 2) * words * 8, ctx->pool, s));
    const RescaleSpec rs{add, add_stride, nout};
    const int rc = ks_fused_batch(g, out, out + size_t(npolys) * nout * R.N, c2, c2_eval, nd, npolys, key, level,
                                  static_cast<u64*>(scratch), s, x0, x1, true, y0, y1, c2_raw != 0, &rs, t2);
    cudaFreeAsync(scratch, s);
    return rc;
}

// mul_relin followed by the Chebyshev ladder step (ckks.hpp:532-555):
// out = rescale( 2 relinearize(x (x) y) - sub_coef_r * sub (+ add_const_r at
// coefficient 0 of the part-0 polys) ), `level` rows per poly. Large batches
// on all-FP64 rings take the whole step inside ModDown (k_mod_down_fp RESCALE
// with LadderPre); everything else relinearises, then tg_lincomb_batch.
extern "C" int tg_relinearize_tensor_ladder_batch(tg_gadget* g, uint64_t* out, const uint64_t* c2,
                                                  const uint64_t* c2_eval, const uint64_t* key,
                                                  uint32_t key_digits, int level, const uint64_t* x0,
                                                  const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
                                                  uint32_t npolys, int c2_raw, const uint64_t* sub,
                                                  uint64_t sub_stride, const uint64_t* sub_coef,
                                                  const uint64_t* add_const, void* stream) {
    return tg_relinearize_tensor_ladder_batch_strided(g, out, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1,
                                                      nullptr, npolys, c2_raw, sub, sub_stride, sub_coef, add_const,
                                                      stream);
}

extern "C" int tg_relinearize_tensor_ladder_batch_strided(
    tg_gadget* g, uint64_t* out, const uint64_t* c2, const uint64_t* c2_eval, const uint64_t* key,
    uint32_t key_digits, int level, const uint64_t* x0, const uint64_t* x1, const uint64_t* y0, const uint64_t* y1,
    const uint64_t* op_strides, uint32_t npolys, int c2_raw, const uint64_t* sub, uint64_t sub_stride,
    const uint64_t* sub_coef, const uint64_t* add_const, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    Tensor2 t2;
    {
        bool strided = false;
        if (int rc = set_op_strides(t2, op_strides, size_t(level + 1) * g->ctx->ring.N, strided)) return rc;
    }
    if (level < 1) return fail(TG_E_ARG, "[ring] cannot rescale at level 0");
    if (npolys == 0) return TG_OK;
    if (!x0 || !x1 || !y0 || !y1) return fail(TG_E_ARG, "[rlwe] relinearize needs both operands' eval parts");
    if ((sub == nullptr) != (sub_coef == nullptr)) return fail(TG_E_ARG, "[ckks] ladder step: subtrahend without its constants");
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    if (nd > 15) return fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    bool all_fp = true;
    for (int r = 0; r <= level; ++r) all_fp &= ctx->h_q[r] < kFpMaxQ;
    static const bool off = [] {
        const char* e = getenv("TG_FUSED_LADDER");
        return e && *e == '0';
    }();
    const bool fuse = !off && all_fp && ks_fused_ok(ctx) && g->g.fp_moddown && R.K <= 16 && fused_rescale_on() &&
                      level + 1 <= kLadderRows && u64(npolys) * R.N >= u64(ctx->sms) * 512;
    if (!fuse) {  // relinearise into scratch, then the ladder step as one lincomb pass
        if (c2_raw && !ks_fused_ok(ctx))
            return fail(TG_E_ARG, "[rlwe] a raw c2 needs its eval form and the fused key switch");
        const size_t pw = size_t(level + 1) * R.N, qw = pw * npolys;
        void* tmp = nullptr;
        TG_CUDA(cudaMallocFromPoolAsync(&tmp, 2 * qw * 8, ctx->pool, s));
        u64* t = static_cast<u64*>(tmp);
        int rc = relinearize_tensor_batch(g, t, t + qw, c2, c2_eval, key, key_digits, level, x0, x1, y0, y1, t2,
                                          npolys, c2_raw, stream);
        if (rc == TG_OK) {
            const uint64_t* terms[2] = {t, sub};
            const uint64_t strides[2] = {pw, sub_stride};
            std::vector<u64> coef(size_t(2) * (level + 1));
            for (int r = 0; r <= level; ++r) {
                coef[r] = 2 % ctx->h_q[r];
                if (sub) coef[size_t(level + 1) + r] = (ctx->h_q[r] - sub_coef[r] % ctx->h_q[r]) % ctx->h_q[r];
            }
            rc = tg_lincomb_batch(ctx, out, sub ? 2 : 1, terms, strides, coef.data(), add_const, 0, level,
                                  2 * npolys, npolys, 1, stream);
        }
        cudaFreeAsync(tmp, s);
        return rc;
    }
    LadderPre pre;
    pre.on = 1;
    pre.sub = sub;
    pre.stride = sub_stride;
    pre.has_e = add_const ? 1 : 0;
    for (int r = 0; r <= level; ++r) {
        const u64 q = ctx->h_q[r];
        const u64 m = sub ? sub_coef[r] % q : 0;
        pre.m[r] = double(m);
        pre.mq[r] = double(m) / double(q);
        const u64 e = add_const ? add_const[r] % q : 0;
        pre.e[r] = e > q / 2 ? -double(q - e) : double(e);
    }
    const size_t words = size_t(level + 1 + R.K) * R.N;
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, size_t(npolys) * (nd + 2) * words * 8, ctx->pool, s));
    const RescaleSpec rs{nullptr, 0, u32(level), &pre};
    const int rc = ks_fused_batch(g, out, out + size_t(npolys) * level * R.N, c2, c2_eval, nd, npolys, key, level,
                                  static_cast<u64*>(scratch), s, x0, x1, true, y0, y1, c2_raw != 0, &rs, t2);
    cudaFreeAsync(scratch, s);
    return rc;
}

extern "C" int tg_ks_inner_add(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* digits,
                               uint32_t ndigits, const uint64_t* key, uint32_t key_digits, int level,
                               const uint64_t* add0, const uint64_t* add1, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    if (ndigits == 0) return fail(TG_E_ARG, "[rlwe] empty decomposition");
    if (ndigits > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    tg_context* ctx = g->ctx;
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + ctx->ring.K) * ctx->ring.N;
    void* acc = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&acc, 2 * words * 8, ctx->pool, s));
    int rc = ks_inner(g, out0, out1, digits, ndigits, key, level, static_cast<u64*>(acc), s, add0, add1);
    cudaFreeAsync(acc, s);
    return rc;
}

// Key switch with the epilogue add, eval-form output (tg_keyswitch_add_eval).
// Same residues as tg_keyswitch_add_batch followed by a forward NTT of its
// output: acc stays in eval form; only its K special rows are inverse
// transformed (out of place), ModDown's conversion -conv * P^-1 is computed in
// coefficient form and forward transformed (level+1 rows), and the epilogue
// out = acc * P^-1 + NTT(-conv * P^-1) + add runs on eval-form rows.
extern "C" int tg_keyswitch_add_eval(tg_gadget* g, uint64_t* out0, uint64_t* out1, const uint64_t* d,
                                     const uint64_t* d_eval, const uint64_t* key, uint32_t key_digits, int level,
                                     const uint64_t* add0, const uint64_t* add1, uint32_t npolys, void* stream) {
    if (int rc = check_ks(g, level)) return rc;
    if (npolys == 0) return TG_OK;
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const u32 nd = tg_gadget_digit_count(g, level);
    if (nd > key_digits) return fail(TG_E_ARG, "[rlwe] switching key has too few digits");
    if (!g->g.lazy_moddown || R.K > 16) return fail(TG_E_ARG, "[rlwe] eval-form ModDown needs the lazy ModDown path");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = as_stream(stream);
    const size_t words = size_t(level + 1 + R.K) * R.N, qwords = size_t(level + 1) * R.N;
    // digits | acc (2 * npolys polys) | specials scratch (same shape as acc) | negconv (2 * npolys x level+1 rows)
    void* scratch = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&scratch, (size_t(npolys) * (nd + 4) * words + 2 * npolys * qwords) * 8,
                                    ctx->pool, s));
    u64* digits = static_cast<u64*>(scratch);
    u64* acc = digits + size_t(npolys) * nd * words;
    u64* spec = acc + 2 * size_t(npolys) * words;
    u64* negc = spec + 2 * size_t(npolys) * words;
    int rc = modup(g, digits, d, level, s, d_eval, npolys);
    if (rc == TG_OK) {
        ProfScope prof(ctx, TG_OP_KEY_INNER, 8.0 * words * (npolys * (nd + 2.0) + 2.0 * nd), s);
        const u64 want = u64(ctx->sms) * 2048;
        u32 ppt = npolys;
        while (ppt > 1 && words / 2 * ((npolys + ppt - 1) / ppt) < want) ppt = (ppt + 1) / 2;
        const u32 blocks = grid_for(words / 2 * ((npolys + ppt - 1) / ppt));
        if (nd <= 4) k_key_inner_b<4><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt);
        else if (nd <= 8) k_key_inner_b<8><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt);
        else if (nd <= 15) k_key_inner_b<15><<<blocks, kThreads, 0, s>>>(R, acc, digits, nd, npolys, key, level, ppt);
        else rc = fail(TG_E_ARG, "[rlwe] batched key switch supports at most 15 digits");
        if (rc == TG_OK) rc = cudaGetLastError() == cudaSuccess ? TG_OK : cuda_fail(cudaGetLastError(), "key inner");
    }
    // the K special rows of both accumulators back to coefficient form
    if (rc == TG_OK)
        rc = ntt_inverse_oop(ctx, spec, acc, level, int(R.K), 2 * npolys, s, u32(level) + 1, R.K);
    if (rc == TG_OK) {
        ProfScope prof(ctx, TG_OP_MOD_DOWN, 8.0 * R.N * 2 * npolys * (R.K + (level + 1.0)), s);
        const GadgetDev& G = g->g;
        if (R.K <= 4) launch_mod_down_v<4, 2, true>(R, G, ctx->sms, negc, spec, level, 2 * npolys, nullptr, s);
        else if (R.K <= 8) launch_mod_down_v<8, 2, true>(R, G, ctx->sms, negc, spec, level, 2 * npolys, nullptr, s);
        else launch_mod_down_v<16, 1, true>(R, G, ctx->sms, negc, spec, level, 2 * npolys, nullptr, s);
        rc = cudaGetLastError() == cudaSuccess ? TG_OK : cuda_fail(cudaGetLastError(), "mod_down conv");
    }
    if (rc == TG_OK) rc = ntt_forward_oop(ctx, negc, negc, level, 0, 2 * npolys, s);
    if (rc == TG_OK) {
        ProfScope prof(ctx, TG_OP_MOD_DOWN, 8.0 * qwords * npolys * 2 * 4, s);
        const size_t n_out = size_t(npolys) * qwords;
        k_mod_down_finish<<<grid_for(n_out), kThreads, 0, s>>>(R, g->g, out0, acc, negc, add0, level, npolys);
        k_mod_down_finish<<<grid_for(n_out), kThreads, 0, s>>>(R, g->g, out1, acc + size_t(npolys) * words,
                                                                negc + size_t(npolys) * qwords, add1, level, npolys);
        rc = cudaGetLastError() == cudaSuccess ? TG_OK : cuda_fail(cudaGetLastError(), "mod_down finish");
    }
    cudaFreeAsync(scratch, s);
    return rc;
}
