// Exact modular arithmetic on FP64 for moduli q < 2^50.5 (every q-chain
// prime of the configs). B200 has full-rate FP64 (64 DFMA/clk/SM, a pipe
// separate from the integer IMAD/ALU pipes that bound the 64-bit Shoup path),
// and residues < 2^52 are exact doubles. All values are integers held in
// doubles; every operation below is exact (proofs inline), so the canonical
// residues produced are identical to the integer path's.
#pragma once

#include "tg_internal.cuh"

namespace tg {

constexpr double kTwo52 = 4503599627370496.0;        // 2^52
constexpr double kRoundMagic = 6755399441055744.0;   // 1.5 * 2^52
constexpr u64 kFpMaxQ = 1591222034138579ull;          // floor(2^50.5): FP path bound

// u64 x < 2^52 -> exact double (bit trick: 2^52 + x has x as its mantissa).
__device__ __forceinline__ double u2d(u64 x) {
    return __dsub_rn(__longlong_as_double(static_cast<long long>(0x4330000000000000ull | x)), kTwo52);
}
// exact double integer v in [0, 2^52) -> u64
__device__ __forceinline__ u64 d2u(double v) {
    return static_cast<u64>(__double_as_longlong(__dadd_rn(v, kTwo52))) & 0x000FFFFFFFFFFFFFull;
}

// r == b*w (mod q), |r| <= 1.5q, for integer doubles |b| < 2^53, 0 <= w < q,
// wq = fl(w/q), q < 2^50.5.
//   h = fl(b w), l = b w - h exactly (FMA error-free product; |b w| < 2^104).
//   k = rint(b * wq) via fma(b, wq, 1.5*2^52) - 1.5*2^52 (one rounding of the
//       exact product to an integer; |b wq| < 2^51 so the sum lies in
//       [2^52, 2^53) where ulp = 1). |b wq - b w/q| <= |b| 2^-53 <= 1, so
//       |b w/q - k| <= 1.5 and |b w - k q| <= 1.5 q.
//   fma(-k, q, h) = h - k q exactly: |h - k q| <= 1.5q + |l| <= 1.5q + 2^51 < 2^53.
//   (h - k q) + l = b w - k q exactly (|.| <= 1.5q < 2^53).
__device__ __forceinline__ double fp_mulmod(double b, double w, double wq, double q) {
    const double h = __dmul_rn(b, w);
    const double l = __fma_rn(b, w, -h);
    const double k = __dsub_rn(__fma_rn(b, wq, kRoundMagic), kRoundMagic);
    return __dadd_rn(__fma_rn(-k, q, h), l);
}

// v - rint(v/q) q for integer |v| < 2^53: |result| <= q/2 + 1 (qi = fl(1/q)
// gives |v qi - v/q| <= 2^-52 |v/q| < 1/2), exact by the same FMA argument.
__device__ __forceinline__ double fp_reduce(double v, double q, double qi) {
    const double k = __dsub_rn(__fma_rn(v, qi, kRoundMagic), kRoundMagic);
    return __fma_rn(-k, q, v);
}

// |v| < 2q integer -> canonical u64 in [0, q)
__device__ __forceinline__ u64 fp_canonical(double v, double q) {
    if (v < 0) v = __dadd_rn(v, q);
    if (v < 0) v = __dadd_rn(v, q);
    if (v >= q) v = __dsub_rn(v, q);
    return d2u(v);
}

}  // namespace tg
