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
#include "tg_internal.cuh"

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
constexpr u32 kMUThreads = 128;

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

}  // namespace

int modup(tg_gadget* g, u64* digits, const u64* d, int level, cudaStream_t s, const u64* d_eval = nullptr) {
    tg_context* ctx = g->ctx;
    const DevRing& R = ctx->ring;
    const u32 nd = tg_gadget_digit_count(g, level);
    dim3 grid((R.N + kMUThreads - 1) / kMUThreads, nd);
    {
        ProfScope prof(ctx, TG_OP_MODUP, 8.0 * R.N * (double(level + 1) + double(nd) * (level + 1 + R.K)), s);
        k_modup<<<grid, kMUThreads, 0, s>>>(R, g->g, digits, d, level, d_eval);
    }
    TG_LAUNCH_CHECK();
    return ntt_forward_oop(ctx, digits, digits, level, int(R.K), nd, s, d_eval ? g->g.group_size : 0);
}

int mod_down(tg_gadget* g, u64* out, const u64* in, int level, u32 npolys, cudaStream_t s,
             const u64* addend = nullptr) {
    const DevRing& R = g->ctx->ring;
    ProfScope prof(g->ctx, TG_OP_MOD_DOWN, 8.0 * R.N * npolys * (2.0 * (level + 1) + R.K + (addend ? level + 1 : 0)), s);
    k_mod_down<<<grid_for(size_t(npolys) * R.N), kThreads, 0, s>>>(R, g->g, out, in, level, npolys, addend);
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
    int rc = modup(g, digits, d, level, s, d_eval);
    if (rc == TG_OK) rc = ks_inner(g, out0, out1, digits, nd, key, level, digits + size_t(nd) * words, s, add0, add1);
    cudaFreeAsync(scratch, s);
    return rc;
}
