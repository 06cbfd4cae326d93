// Fused key-switch core (included by tg_ntt.cu after tg_ntt_warp.cuh, inside
// the anonymous namespace). Used when every modulus of the ring takes the
// FP64 path (tg_fp64.cuh).
//
// KeyContext::ks_inner (rlwe.hpp:501-540) after ModUp is: forward NTT of every
// digit (rlwe.hpp:137), acc_{0,1} = sum_i digit_i * key_{b,a}[i] (eval form,
// rlwe.hpp:514-536), inverse NTT of both accumulators (rlwe.hpp:537-538).
// Both transforms are four-step (tg_ntt_warp.cuh): the forward's second phase
// and the inverse's first phase work on the same contiguous M-word chunks of
// one row, and the inner product is pointwise. So one kernel per (row r,
// chunk block) takes the digits straight from the forward column phase,
// finishes their transform, multiplies by the key chunk, accumulates, and
// runs the accumulators' first inverse phase: neither the eval-form digits
// nor the eval-form accumulators go through HBM, and the separate inner-
// product pass disappears. The inverse column phase (N^-1) follows as usual.
//
// Digits' own-group rows copied in eval form by ModUp (d_eval given; the
// NTT's skip rule) are read as they are. Relinearisation's eval-form c0/c1
// enter the Q rows as P * c (see tg_relinearize_batch). Every product is an
// exact FP64 modular product; canonical residues are identical to the
// unfused path's.
//
// Bounds (tg_fp64.cuh): transformed digits |v| <= q/2 + 1, own rows [0, q);
// fp_mulmod_qi with |a| <= q/2 + 1, b in [0, q): |term| < 0.81q; sums reduced
// every 4 digits: |sum| < q/2 + 1 + 4 * 0.81q (+ 0.58q for P * c) < 2^53.

#ifndef KS_KEY_PREFETCH
#define KS_KEY_PREFETCH 0
#endif

#ifndef KS_L2_PREFETCH
#define KS_L2_PREFETCH 0  // measured: 454 -> 487 us per batched level-21 key switch (slower)
#endif
// Bulk prefetch of a contiguous range into L2 (TMA unit, no registers, no
// completion to wait for): the block's key chunks and digit rows of the NEXT
// digit pair are requested while the current pair is transformed, so their
// loads (the kernel's top stall: the key words' conversions waited on long
// scoreboard, ncu source page) hit L2 instead of DRAM.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, u32 bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// L2 eviction-priority hints (createpolicy + ld.global.L2::cache_hint): the
// key chunks are re-read for every poly of the batch, the digit rows exactly
// once; without hints the ~120 MB key set (level 21, dnum 4) is evicted by the
// streaming digits and accumulators (ncu: DRAM reads ~2x the algorithmic
// bytes).
#ifndef KS_L2_HINTS
#define KS_L2_HINTS 1
#endif
__device__ __forceinline__ u64 l2_policy_last() {
    u64 p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ u64 l2_policy_first() {
    u64 p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ ulonglong2 ld_v2_hint(const ulonglong2* a, u64 pol) {
    ulonglong2 r;
    asm volatile("ld.global.L2::cache_hint.v2.u64 {%0, %1}, [%2], %3;\n" : "=l"(r.x), "=l"(r.y) : "l"(a), "l"(pol));
    return r;
}
__device__ __forceinline__ u64 ld_hint(const u64* a, u64 pol) {
    u64 r;
    asm volatile("ld.global.L2::cache_hint.u64 %0, [%1], %2;\n" : "=l"(r) : "l"(a), "l"(pol));
    return r;
}
template <int E>
__device__ __forceinline__ void ld_strided_hint(u64 (&v)[E], const u64* x, u32 lane, u64 pol) {
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = KS_L2_HINTS ? ld_hint(x + lane + 32 * j, pol) : x[lane + 32 * j];
}

template <int E>
constexpr size_t ks_chunk_smem() {  // two exchange columns per warp + forward and inverse chunk twiddles
    return size_t(8) * (16 * WGeo<E>::CS + 4 * WGeo<E>::TW_CHUNK);
}

template <int E>
__device__ __forceinline__ void ks_chunks_int_body(const DevRing& R, u64* acc, const u64* digits, u32 nd, u32 npolys,
                                                   u32 ppb, const u64* key, int level, u32 logN1);

// MIXED: rows r >= int_from (the integer special rows of a mixed ring) take
// the 64-bit integer body; every other row the FP64 body below (a separate
// instantiation, so the all-FP64 kernel's registers are unaffected).
// ty0/ty1 (tensor mode, tg_relinearize_tensor_batch): add0/add1 are the
// operand x's eval parts and ty0/ty1 y's; c0 = x0 y0, c1 = x0 y1 + x1 y0 are
// formed here (exact FP64 products, |c0| < 0.81q, |c1| < 1.62q) and folded
// as P * c like the eval-form addends. t2 (lazy relinearisation of two
// products, tg_relinearize_tensor2_rescale_batch): c0 += u0 v0, c1 += u0 v1 +
// u1 v0 (|c0| < 1.62q, |c1| < 3.24q, brought back to |.| <= q/2 + 1 by
// fp_reduce before the P product).
template <int E, bool MIXED = false>
__global__ void __launch_bounds__(256, 2)
kw_ks_chunks(DevRing R, u64* acc, const u64* digits, u32 nd, u32 npolys, u32 ppb, const u64* key, int level,
             u32 logN1, u32 own_gs, const u64* add0, const u64* add1, const u64* pmod, u32 int_from,
             const u64* ty0, const u64* ty1, const Tensor2 t2) {
    using Gm = WGeo<E>;
    if constexpr (MIXED) {
        if (blockIdx.y >= int_from) {
            ks_chunks_int_body<E>(R, acc, digits, nd, npolys, ppb, key, level, logN1);
            return;
        }
    }
    extern __shared__ u64 dyn[];
    u64* swf = dyn + 16 * Gm::CS;
    u64* swi = swf + 2 * Gm::TW_CHUNK;
    const u32 N = R.N, rows = u32(level) + 1 + R.K;
    const u32 r = blockIdx.y;
    const u32 b0 = blockIdx.z * ppb, b1 = min(npolys, b0 + ppb);
    if (b0 >= b1) return;
    const u32 m = mod_index(r, level, R.q_count);
    const double qd = R.qd[4 * m], qi = R.qd[4 * m + 1];
    const u64* tw = reinterpret_cast<const u64*>(R.twd + size_t(m) * 4 * N);
    stage_chunk_twiddles<E, true>(swf, nullptr, tw, tw + N, logN1, blockIdx.x);
    stage_chunk_twiddles<E, false>(swi, nullptr, tw + 2 * size_t(N), tw + 3 * size_t(N), logN1, blockIdx.x);
    __syncthreads();
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t off = size_t(blockIdx.x * 8 + warp) * Gm::M;
    u64* col = dyn + warp * 2 * Gm::CS;  // the warp's contiguous pair-exchange region
    constexpr u32 CS2 = 8 * Gm::CS;
    const size_t words = size_t(rows) * N, key_rows = R.nmod;
    const bool addq = add0 && r <= u32(level);
    double pmd = 0, pmq = 0;
    if (addq) {
        pmd = __longlong_as_double(static_cast<long long>(pmod[4 * r + 2]));
        pmq = __longlong_as_double(static_cast<long long>(pmod[4 * r + 3]));
    }
    // digit d's own-group row (already eval form, canonical)
    const u32 own = (own_gs && r <= u32(level)) ? r / own_gs : 0xFFFFFFFFu;
    const u32 vo = lane << Gm::LOGE;  // layout 0: this lane's E contiguous eval slots
    auto kptr = [&](u32 d, u32 part) {
        return reinterpret_cast<const ulonglong2*>(key + ((size_t(d) * 2 + part) * key_rows + m) * N + off + vo);
    };
#if KS_KEY_PREFETCH
    // key chunk of one digit (E words of each half), loaded ahead of its transform
    auto kload = [&](ulonglong2 (&kb)[E / 2], ulonglong2 (&ka)[E / 2], u32 d) {
        const ulonglong2* pb = kptr(d, 0);
        const ulonglong2* pa = kptr(d, 1);
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
            kb[j] = __ldg(pb + j);
            ka[j] = __ldg(pa + j);
        }
    };
    auto mack = [&](double (&a0)[E], double (&a1)[E], const double (&v)[E], const ulonglong2 (&kb)[E / 2],
                    const ulonglong2 (&ka)[E / 2]) {
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
            const ulonglong2 tb = kb[j], ta = ka[j];
            a0[2 * j] = __dadd_rn(a0[2 * j], fp_mulmod_qi(v[2 * j], u2d(tb.x), qd, qi));
            a0[2 * j + 1] = __dadd_rn(a0[2 * j + 1], fp_mulmod_qi(v[2 * j + 1], u2d(tb.y), qd, qi));
            a1[2 * j] = __dadd_rn(a1[2 * j], fp_mulmod_qi(v[2 * j], u2d(ta.x), qd, qi));
            a1[2 * j + 1] = __dadd_rn(a1[2 * j + 1], fp_mulmod_qi(v[2 * j + 1], u2d(ta.y), qd, qi));
        }
    };
#endif
    const u64 pol_key = l2_policy_last(), pol_dig = l2_policy_first();
    auto mac = [&](double (&a0)[E], double (&a1)[E], const double (&v)[E], u32 d) {
        const ulonglong2* kb = kptr(d, 0);
        const ulonglong2* ka = kptr(d, 1);
#pragma unroll
        for (int j = 0; j < E / 2; ++j) {
            const ulonglong2 tb = KS_L2_HINTS ? ld_v2_hint(kb + j, pol_key) : kb[j];
            const ulonglong2 ta = KS_L2_HINTS ? ld_v2_hint(ka + j, pol_key) : ka[j];
            a0[2 * j] = __dadd_rn(a0[2 * j], fp_mulmod_qi(v[2 * j], u2d(tb.x), qd, qi));
            a0[2 * j + 1] = __dadd_rn(a0[2 * j + 1], fp_mulmod_qi(v[2 * j + 1], u2d(tb.y), qd, qi));
            a1[2 * j] = __dadd_rn(a1[2 * j], fp_mulmod_qi(v[2 * j], u2d(ta.x), qd, qi));
            a1[2 * j + 1] = __dadd_rn(a1[2 * j + 1], fp_mulmod_qi(v[2 * j + 1], u2d(ta.y), qd, qi));
        }
    };
    for (u32 b = b0; b < b1; ++b) {
        double a[2][E];
#pragma unroll
        for (int j = 0; j < E; ++j) a[0][j] = a[1][j] = 0.0;
        // P * c first (the accumulators start from it): its loads are in
        // flight with the first digits' instead of exposed after the last
        if (addq) {  // + P * c on the Q rows (|.| <= q/2 + 2^-15 q; the digit sums reduce every 4 as before)
            const size_t qw = size_t(level + 1) * N, ro = size_t(r) * N + off + vo;
            const size_t po = size_t(b) * (t2.sx ? t2.sx : qw) + ro;  // operand polys may be strided views
            const ulonglong2* c0 = reinterpret_cast<const ulonglong2*>(add0 + po);
            const ulonglong2* c1 = reinterpret_cast<const ulonglong2*>(add1 + po);
            if (ty0) {  // tensor mode: c0 = x0 y0, c1 = x0 y1 + x1 y0 from the operands
                const size_t py = size_t(b) * (t2.sy ? t2.sy : qw) + ro;
                const ulonglong2* d0 = reinterpret_cast<const ulonglong2*>(ty0 + py);
                const ulonglong2* d1 = reinterpret_cast<const ulonglong2*>(ty1 + py);
#pragma unroll
                for (int j = 0; j < E / 2; ++j) {
                    const ulonglong2 x0 = c0[j], x1 = c1[j], y0 = d0[j], y1 = d1[j];
                    const double xa[2] = {u2d(x0.x), u2d(x0.y)}, xb[2] = {u2d(x1.x), u2d(x1.y)};
                    const double ya[2] = {u2d(y0.x), u2d(y0.y)}, yb[2] = {u2d(y1.x), u2d(y1.y)};
                    double s0[2], s1[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        s0[h] = fp_mulmod_qi(xa[h], ya[h], qd, qi);
                        s1[h] = __dadd_rn(fp_mulmod_qi(xa[h], yb[h], qd, qi), fp_mulmod_qi(xb[h], ya[h], qd, qi));
                    }
                    if (t2.u0) {  // + the second product's c0 / c1
                        const size_t pu = size_t(b) * (t2.su ? t2.su : qw) + ro;
                        const size_t pv = size_t(b) * (t2.sv ? t2.sv : qw) + ro;
                        const ulonglong2 u0 = reinterpret_cast<const ulonglong2*>(t2.u0 + pu)[j];
                        const ulonglong2 u1 = reinterpret_cast<const ulonglong2*>(t2.u1 + pu)[j];
                        const ulonglong2 v0 = reinterpret_cast<const ulonglong2*>(t2.v0 + pv)[j];
                        const ulonglong2 v1 = reinterpret_cast<const ulonglong2*>(t2.v1 + pv)[j];
                        const double ua[2] = {u2d(u0.x), u2d(u0.y)}, ub[2] = {u2d(u1.x), u2d(u1.y)};
                        const double va[2] = {u2d(v0.x), u2d(v0.y)}, vb[2] = {u2d(v1.x), u2d(v1.y)};
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            s0[h] = fp_reduce(__dadd_rn(s0[h], fp_mulmod_qi(ua[h], va[h], qd, qi)), qd, qi);
                            s1[h] = fp_reduce(__dadd_rn(s1[h], __dadd_rn(fp_mulmod_qi(ua[h], vb[h], qd, qi),
                                                                         fp_mulmod_qi(ub[h], va[h], qd, qi))),
                                              qd, qi);
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        a[0][2 * j + h] = __dadd_rn(a[0][2 * j + h], fp_mulmod(s0[h], pmd, pmq, qd));
                        a[1][2 * j + h] = __dadd_rn(a[1][2 * j + h], fp_mulmod(s1[h], pmd, pmq, qd));
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < E / 2; ++j) {
                    const ulonglong2 x0 = c0[j], x1 = c1[j];
                    a[0][2 * j] = __dadd_rn(a[0][2 * j], fp_mulmod(u2d(x0.x), pmd, pmq, qd));
                    a[0][2 * j + 1] = __dadd_rn(a[0][2 * j + 1], fp_mulmod(u2d(x0.y), pmd, pmq, qd));
                    a[1][2 * j] = __dadd_rn(a[1][2 * j], fp_mulmod(u2d(x1.x), pmd, pmq, qd));
                    a[1][2 * j + 1] = __dadd_rn(a[1][2 * j + 1], fp_mulmod(u2d(x1.y), pmd, pmq, qd));
                }
            }
        }
        const u64* dig = digits + size_t(b) * nd * words + size_t(r) * N + off;
        // the block's 8 chunks of a (digit, key half) are one contiguous 16 KB range
        constexpr u32 kBlockBytes = 8u * Gm::M * 8u;
        const size_t blk0 = size_t(blockIdx.x) * 8 * Gm::M;
        auto prefetch_pair = [&](u32 bb, u32 d0) {  // digits d0, d0 + 1 of poly bb
            if (!KS_L2_PREFETCH || threadIdx.x != 0) return;
            for (u32 dd = d0; dd < min(nd, d0 + 2); ++dd) {
                prefetch_l2_bulk(key + ((size_t(dd) * 2 + 0) * key_rows + m) * N + blk0, kBlockBytes);
                prefetch_l2_bulk(key + ((size_t(dd) * 2 + 1) * key_rows + m) * N + blk0, kBlockBytes);
                prefetch_l2_bulk(digits + size_t(bb) * nd * words + size_t(dd) * words + size_t(r) * N + blk0,
                                 kBlockBytes);
            }
        };
        if (b == b0) prefetch_pair(b, 0);
        for (u32 d = 0; d < nd; d += 2) {
            if (d + 2 < nd) prefetch_pair(b, d + 2);
            else if (b + 1 < b1) prefetch_pair(b + 1, 0);
            const bool pair = d + 1 < nd;
            double v[2][E];
            if (pair && own != d && own != d + 1) {  // two digits transformed together
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    u64 t[E];
                    ld_strided_hint<E>(t, dig + size_t(d + n) * words, lane, pol_dig);
#pragma unroll
                    for (int j = 0; j < E; ++j) v[n][j] = __longlong_as_double(static_cast<long long>(t[j]));
                }
#if KS_KEY_PREFETCH
                ulonglong2 kb[E / 2], ka[E / 2];
                kload(kb, ka, d);  // in flight during the transform
                wfwd_all_fp<2, E, true, true>(v, col, CS2, lane, swf, qd, qi, warp);
                mack(a[0], a[1], v[0], kb, ka);
#else
                wfwd_all_fp<2, E, true, true>(v, col, CS2, lane, swf, qd, qi, warp);
                mac(a[0], a[1], v[0], d);
#endif
                mac(a[0], a[1], v[1], d + 1);
            } else {
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    if (n == 1 && !pair) break;
                    const u32 dd = d + n;
                    double (&vn)[1][E] = reinterpret_cast<double(&)[1][E]>(v[n]);
                    u64 t[E];
                    if (dd == own) {
                        ld_vec<E>(t, dig + size_t(dd) * words, lane);
#pragma unroll
                        for (int j = 0; j < E; ++j) vn[0][j] = u2d(t[j]);
                    } else {
                        ld_strided_hint<E>(t, dig + size_t(dd) * words, lane, pol_dig);
#pragma unroll
                        for (int j = 0; j < E; ++j) vn[0][j] = __longlong_as_double(static_cast<long long>(t[j]));
                        wfwd_all_fp<1, E, true>(vn, col, CS2, lane, swf, qd, qi, warp);
                    }
                    mac(a[0], a[1], vn[0], dd);
                }
            }
            if ((d & 3) == 2 && d + 2 < nd) {
#pragma unroll
                for (int j = 0; j < E; ++j) {
                    a[0][j] = fp_reduce(a[0][j], qd, qi);
                    a[1][j] = fp_reduce(a[1][j], qd, qi);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < E; ++j) {
            a[0][j] = fp_reduce(a[0][j], qd, qi);
            a[1][j] = fp_reduce(a[1][j], qd, qi);
        }
        // inverse chunk phase of both accumulators (layout 0 in, layout 5 out),
        // doubles (|v| <= 1.5q, raw bits) to the inverse column phase
        winv_all_fp<2, E, true, true>(a, col, CS2, lane, swi, qd, qi, warp);
        u64* o0 = acc + (size_t(b) * rows + r) * N + off;
        u64* o1 = acc + (size_t(npolys + b) * rows + r) * N + off;
#pragma unroll
        for (int j = 0; j < E; ++j) {
            o0[lane + 32 * j] = static_cast<u64>(__double_as_longlong(a[0][j]));
            o1[lane + 32 * j] = static_cast<u64>(__double_as_longlong(a[1][j]));
        }
    }
}

// Integer rows of a mixed ring (the 60-bit special primes of config 1; every
// q-chain row takes kw_ks_chunks): the same fusion on the 64-bit Shoup path
// of the warp NTT -- the digits' forward chunk phase (wfwd_all, Harvey-lazy,
// then canonical), the key inner product as exact 128-bit sums (< nd 2^120)
// with one Barrett reduction (rlwe.hpp:514-536), the accumulators' inverse
// chunk phase (winv_all) -- in the data formats of kw_fwd_chunks' input and
// kw_inv_chunks' output, so the integer column phases on either side are
// unchanged. Blocks of these rows run in the same launch as the FP64 rows
// (kw_ks_chunks, int_from); special rows are never own-group rows and get no
// P * c addend.
template <int E>
__device__ __forceinline__ void ks_chunks_int_body(const DevRing& R, u64* acc, const u64* digits, u32 nd, u32 npolys,
                                                   u32 ppb, const u64* key, int level, u32 logN1) {
    using Gm = WGeo<E>;
    extern __shared__ u64 dyn[];
    u64* swf = dyn + 16 * Gm::CS;
    u64* swfs = swf + Gm::TW_CHUNK;
    u64* swi = swfs + Gm::TW_CHUNK;
    u64* swis = swi + Gm::TW_CHUNK;
    const u32 N = R.N, rows = u32(level) + 1 + R.K;
    const u32 r = blockIdx.y;
    const u32 b0 = blockIdx.z * ppb, b1 = min(npolys, b0 + ppb);
    if (b0 >= b1) return;
    const u32 m = mod_index(r, level, R.q_count);
    const u64 q = R.q[m], q2 = 2 * q, rlo = R.ratio[2 * m], rhi = R.ratio[2 * m + 1];
    const u64* tw = R.tw + size_t(m) * 4 * N;
    stage_chunk_twiddles<E, true>(swf, swfs, tw, tw + N, logN1, blockIdx.x);
    stage_chunk_twiddles<E, false>(swi, swis, tw + 2 * size_t(N), tw + 3 * size_t(N), logN1, blockIdx.x);
    __syncthreads();
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t off = size_t(blockIdx.x * 8 + warp) * Gm::M;
    u64* col = dyn + warp * Gm::CS;
    const size_t words = size_t(rows) * N, key_rows = R.nmod;
    const u32 vo = lane << Gm::LOGE;  // layout 0: this lane's E contiguous eval slots
    for (u32 b = b0; b < b1; ++b) {
        U128 a0[E], a1[E];
#pragma unroll
        for (int j = 0; j < E; ++j) a0[j] = a1[j] = U128{0, 0};
        const u64* dig = digits + size_t(b) * nd * words + size_t(r) * N + off;
        u64 nx[E];
        ld_strided<E>(nx, dig, lane);
        for (u32 d = 0; d < nd; ++d) {
            u64 v[E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = nx[j];
            if (d + 1 < nd) ld_strided<E>(nx, dig + size_t(d + 1) * words, lane);  // in flight during the stages
            wfwd_all<E, true, false>(v, col, lane, swf, swfs, q, warp);
            const u64* kb = key + ((size_t(d) * 2 + 0) * key_rows + m) * N + off + vo;
            const u64* ka = key + ((size_t(d) * 2 + 1) * key_rows + m) * N + off + vo;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                u64 t = v[j];
                if (t >= q2) t -= q2;
                if (t >= q) t -= q;
                mac128(a0[j], t, kb[j]);
                mac128(a1[j], t, ka[j]);
            }
        }
        u64 x0[E], x1[E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            x0[j] = barrett128(a0[j].lo, a0[j].hi, q, rlo, rhi);
            x1[j] = barrett128(a1[j].lo, a1[j].hi, q, rlo, rhi);
        }
        winv_all<E, true, false>(x0, col, lane, swi, swis, q, warp);
        winv_all<E, true, false>(x1, col, lane, swi, swis, q, warp);
        st_strided<E>(acc + (size_t(b) * rows + r) * N + off, x0, lane);
        st_strided<E>(acc + (size_t(npolys + b) * rows + r) * N + off, x1, lane);
    }
}
