// Exact modular arithmetic on FP64 for moduli q < 1.2 * 2^50 (every q-chain
// prime of the configs). B200 has full-rate FP64 (64 DFMA/clk/SM, a pipe
// separate from the integer IMAD/ALU pipes that bound the 64-bit Shoup path),
// and residues < 2^52 are exact doubles. All values are integers held in
// doubles; every operation below is exact (proofs inline), so the canonical
// residues produced are identical to the integer path's.
#pragma once

#include "tg_internal.cuh"

namespace tg {

constexpr double kTwo52 = 4503599627370496.0;        // 2^52
constexpr double kRoundMagic = 6755399441055744.0;   // M = 1.5 * 2^52
constexpr u64 kFpMaxQ = 1351079888211148ull;          // 1.2 * 2^50: FP path bound (see below)

// u64 x < 2^52 -> exact double (bit trick: 2^52 + x has x as its mantissa).
__device__ __forceinline__ double u2d(u64 x) {
    return __dsub_rn(__longlong_as_double(static_cast<long long>(0x4330000000000000ull | x)), kTwo52);
}
// canonical u64 x in [0, q) -> the exact double of its centred representative
// in (-q/2, q/2] (the sign choice on the integer ALU, one FP64 add: 1.5 * 2^52
// + s has s as the low bits of its mantissa for |s| < 2^51).
__device__ __forceinline__ double c2d(u64 x, u64 q) {
    const long long s = static_cast<long long>(x > (q >> 1) ? x - q : x);
    return __dsub_rn(__longlong_as_double(0x4338000000000000ll + s), kRoundMagic);
}
// exact double integer v in [0, 2^52) -> u64
__device__ __forceinline__ u64 d2u(double v) {
    return static_cast<u64>(__double_as_longlong(__dadd_rn(v, kTwo52))) & 0x000FFFFFFFFFFFFFull;
}

// r == b*w (mod q) exactly, for integer doubles b with |b| < 2^53 and
// b*wq >= -2^51, 0 <= w < q < 1.2 * 2^50, wq = fl(w/q) (|wq - w/q| <= 2^-54).
//   h = fl(b w) (an integer: |b w| < 2^103), l = b w - h exactly (FMA
//       error-free product), |l| <= 2^50.
//   t = fl(b wq + M): one rounding of the exact product-sum. b wq >= -2^51
//       puts t in [2^52, 2^54), where doubles are integers (ulp 1 or 2), so
//       k = t - M is an integer (Sterbenz: exact) with
//       |b wq - k| <= 1/2 (t < 2^53) or <= 1 (t >= 2^53).
//   |b w/q - k| <= |b| 2^-54 + {1/2 | 1}, so |b w - k q| <= q (1 + 1/2) < 2^52
//       and fma(-k, q, h) = h - k q is an exact integer (|.| < 2^53),
//       as is r = (h - k q) + l = b w - k q.
// Bound: |r| <= q (1/2 + |b| 2^-54) when b wq < 2^51, else q (1 + |b| 2^-54).
// NTT use: the FP64 twiddle tables hold CENTRED twiddles w in (-q/2, q/2]
// (tg_context.cu), so |wq| < 1/2, fl(w/q) errs by <= 2^-55 and the window
// b wq in [-2^51, 2^51) holds for every |b| < 2^52; the same derivation gives
// |r| <= q/2 + |b| q 2^-55 <= q/2 + 0.0375 |b| (q < 1.2 * 2^50).
//  * Forward (CT, x' = x + r, y' = x - r): from |v| <= q/2 + 1 (centred
//    inputs, c2d) the bound after s stages is B_s with B_(s+1) = 1.0375 B_s +
//    q/2: B_5 = 3.296q < 2^52 (the sixth stage's multiplier input) and B_6 =
//    3.92q < 2^53, so six stages run without a reduction (radix-8 blocks:
//    fp_reduce after the second block, then after the last; N = 2^15/2^14
//    phases of 7 stages: after the third and fourth blocks).
//  * Inverse (GS, x' = x + y, y' = (x - y) w): inputs |v| <= 0.6q; the sum is
//    reduced after every ODD stage (and the last one): an unreduced stage
//    leaves |v| <= 1.2q, so the next multiplier input |x - y| <= 2.4q < 2^52
//    and its products are <= 0.59q; after the reducing stage |v| <= 0.6q again.
// The config primes are the 50-bit NTT primes nearest 2^50 (both sides), all
// below the bound.
__device__ __forceinline__ double fp_mulmod(double b, double w, double wq, double q) {
    const double h = __dmul_rn(b, w);
    const double l = __fma_rn(b, w, -h);
    const double k = __dsub_rn(__fma_rn(b, wq, kRoundMagic), kRoundMagic);
    return __dadd_rn(__fma_rn(-k, q, h), l);
}

// r == a*b (mod q) exactly for canonical a, b in [0, q), q < 1.2 * 2^50,
// qi = fl(1/q); no per-operand quotient table (both operands are data):
//   h = fl(a b) (an integer), l = a b - h exactly (FMA), |l| <= 2^48.
//   h qi = (a b / q)(1 + e), |e| <= 2^-52 + 2^-106, so |h qi - a b/q| <=
//       1.2 * 2^50 * 2^-51.99 < 0.31; h qi in [0, 2^51) puts t = fl(h qi + M)
//       in [1.5 * 2^52, 2^53) (ulp 1): k = t - M is exact, |k - a b/q| < 0.81.
//   h - k q = (a b - k q) - l, |.| < 0.81 q + 2^48 < 2^51: fma(-k, q, h) is
//       exact, and r = (h - k q) + l = a b - k q with |r| < 0.81 q.
__device__ __forceinline__ double fp_mulmod_qi(double a, double b, double q, double qi) {
    const double h = __dmul_rn(a, b);
    const double l = __fma_rn(a, b, -h);
    const double k = __dsub_rn(__fma_rn(h, qi, kRoundMagic), kRoundMagic);
    return __dadd_rn(__fma_rn(-k, q, h), l);
}

// |v| < q -> canonical u64 in [0, q)
__device__ __forceinline__ u64 fp_canonical1(double v, double q) {
    if (v < 0) v = __dadd_rn(v, q);
    return d2u(v);
}

// v - rint(v/q) q for integer |v| < 2^53: |result| <= q/2 + 1 (qi = fl(1/q)
// gives |v qi - v/q| <= 2^-52 |v/q| < 1/2), exact by the same FMA argument.
__device__ __forceinline__ double fp_reduce(double v, double q, double qi) {
    const double k = __dsub_rn(__fma_rn(v, qi, kRoundMagic), kRoundMagic);
    return __fma_rn(-k, q, v);
}

// integer v in (-q, q) -> canonical u64 in [0, q), one FP64 add: v + 1.5 * 2^52
// lies in [2^52, 2^53) (|v| < 2^51), where doubles are the integers, so its
// mantissa field is exactly 2^51 + v; the sign fix-up runs on the integer ALU
// (fp_canonical spends three compares and three adds on the FP64 pipe).
__device__ __forceinline__ u64 fp_canon_small(double v, u64 q) {
    const long long m = static_cast<long long>(
        static_cast<u64>(__double_as_longlong(__dadd_rn(v, kRoundMagic))) & 0x000FFFFFFFFFFFFFull);
    const long long x = m - (1ll << 51);
    return static_cast<u64>(x < 0 ? x + static_cast<long long>(q) : x);
}

// |v| < 2q integer -> canonical u64 in [0, q)
__device__ __forceinline__ u64 fp_canonical(double v, double q) {
    if (v < 0) v = __dadd_rn(v, q);
    if (v < 0) v = __dadd_rn(v, q);
    if (v >= q) v = __dsub_rn(v, q);
    return d2u(v);
}

}  // namespace tg
