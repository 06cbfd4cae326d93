// Negacyclic NTT / iNTT over 64-bit primes, batched over rows.
//
// Same transform as NttTables::forward / inverse (ring.hpp:64-101): the
// forward CT transform maps natural order to the bit-reversed evaluation
// order using w[m+i] = psi^brv(m+i); the inverse GS transform uses
// winv[h+i] and ends with the N^-1 Shoup scaling. The twiddle tables are the
// reference's own (uploaded verbatim), so outputs are bit-identical.
//
// B200 mapping: N = N1 * N2 with N1 = 2^floor(logN/2). The first log N1
// forward stages only mix elements of one column {c + k*N2}; the remaining
// stages only mix elements of one contiguous chunk of N2. Each phase stages a
// 16 KiB tile in shared memory (one HBM read + one HBM write per phase; the
// intermediate of a batched launch stays in the 126 MB L2). Butterflies are
// Harvey-lazy: values live in [0,4q) (forward) / [0,2q) (inverse) and are
// made canonical only at the end of the last phase.
#include <cstdlib>
#include <utility>

#include <cuda.h>  // CUtensorMap (TMA descriptors; the encoder is fetched through cudaGetDriverEntryPoint)

#include "tg_internal.cuh"
#include "tg_fp64.cuh"

namespace tg {

namespace {

constexpr u32 kThreads = 256;
constexpr u32 kLogTile = 11;

// Row-skip rule of ModUp digit transforms: poly p = digit p, whose own-group
// rows (r <= level, r / group_size == p) were copied already in eval form.
// skip = group_size | (digits per source poly << 16): poly p is digit
// p % digits of source p / digits (digits = 0: one source, digit p).
__device__ __forceinline__ bool ntt_row_skipped(u32 row, u32 rpp, int level, u32 skip) {
    skip &= ~kTgRawDigits;
    if (!skip) return false;
    const u32 gs = skip & 0xFFFFu, nd = skip >> 16;
    const u32 r = row % rpp, p = row / rpp;
    return r <= u32(level) && r / gs == (nd ? p % nd : p);
}  // 2048 words = 16 KiB of shared memory per block

struct Plan {
    u32 logN1, logN2, logC, logCpb;
};

Plan make_plan(u32 logN) {
    Plan p;
    p.logN1 = logN / 2;
    p.logN2 = logN - p.logN1;
    // columns per phase-1 block, chunks per phase-2 block
    p.logC = std::min(p.logN2, kLogTile > p.logN1 ? kLogTile - p.logN1 : 0u);
    p.logCpb = std::min(p.logN1, kLogTile > p.logN2 ? kLogTile - p.logN2 : 0u);
    return p;
}

__global__ void __launch_bounds__(kThreads)
k_fwd_cols(DevRing R, u64* data, const u64* src, u32 row_base, u32 rows_per_poly, int level, u32 logN1, u32 logC,
           u32 skip_gs) {
    extern __shared__ u64 sm[];
    if (ntt_row_skipped(row_base + blockIdx.y, rows_per_poly, level, skip_gs)) return;
    const u32 N = R.N, C = 1u << logC, N2 = N >> logN1;
    const u32 row = row_base + blockIdx.y;
    const u32 mi = mod_index(row % rows_per_poly, level, R.q_count);
    const u64 q = R.q[mi], q2 = 2 * q;
    const u64* __restrict__ w = R.tw + size_t(mi) * 4 * N;
    const u64* __restrict__ ws = w + N;
    u64* x = data + size_t(row) * N + size_t(blockIdx.x) * C;
    const u64* xs = src + size_t(row) * N + size_t(blockIdx.x) * C;
    const u32 tile = 1u << (logN1 + logC);
    for (u32 e = threadIdx.x; e < tile; e += kThreads) sm[e] = xs[size_t(e >> logC) * N2 + (e & (C - 1))];
    __syncthreads();
    for (u32 s = 0; s < logN1; ++s) {
        const u32 logt = logN1 - 1 - s;
        for (u32 b = threadIdx.x; b < (tile >> 1); b += kThreads) {
            const u32 cc = b & (C - 1), bb = b >> logC;
            const u32 i = bb >> logt, j = bb & ((1u << logt) - 1);
            const u32 a0 = ((((i << 1) << logt) + j) << logC) + cc;
            const u32 a1 = a0 + (1u << (logt + logC));
            const u32 widx = (1u << s) + i;
            u64 u = sm[a0], v = sm[a1];
            if (u >= q2) u -= q2;
            v = shoup_lazy(v, w[widx], ws[widx], q);
            sm[a0] = u + v;
            sm[a1] = u - v + q2;
        }
        __syncthreads();
    }
    for (u32 e = threadIdx.x; e < tile; e += kThreads) x[size_t(e >> logC) * N2 + (e & (C - 1))] = sm[e];
}

__global__ void __launch_bounds__(kThreads)
k_fwd_chunks(DevRing R, u64* __restrict__ data, u32 row_base, u32 rows_per_poly, int level, u32 logN1, u32 logCpb,
             u32 skip_gs) {
    extern __shared__ u64 sm[];
    if (ntt_row_skipped(row_base + blockIdx.y, rows_per_poly, level, skip_gs)) return;
    const u32 N = R.N, logN = R.logN, logN2 = logN - logN1;
    const u32 row = row_base + blockIdx.y;
    const u32 mi = mod_index(row % rows_per_poly, level, R.q_count);
    const u64 q = R.q[mi], q2 = 2 * q;
    const u64* __restrict__ w = R.tw + size_t(mi) * 4 * N;
    const u64* __restrict__ ws = w + N;
    const u32 chunk0 = blockIdx.x << logCpb;
    const u32 tile = 1u << (logN2 + logCpb);
    u64* x = data + size_t(row) * N + (size_t(chunk0) << logN2);
    for (u32 e = threadIdx.x; e < tile; e += kThreads) sm[e] = x[e];
    __syncthreads();
    for (u32 s = logN1; s < logN; ++s) {
        const u32 logt = logN - 1 - s;
        for (u32 b = threadIdx.x; b < (tile >> 1); b += kThreads) {
            const u32 cl = b >> (logN2 - 1), bb = b & ((1u << (logN2 - 1)) - 1);
            const u32 il = bb >> logt, j = bb & ((1u << logt) - 1);
            const u32 a0 = (cl << logN2) + ((il << 1) << logt) + j;
            const u32 a1 = a0 + (1u << logt);
            const u32 widx = (1u << s) + ((chunk0 + cl) << (s - logN1)) + il;
            u64 u = sm[a0], v = sm[a1];
            if (u >= q2) u -= q2;
            v = shoup_lazy(v, w[widx], ws[widx], q);
            sm[a0] = u + v;
            sm[a1] = u - v + q2;
        }
        __syncthreads();
    }
    for (u32 e = threadIdx.x; e < tile; e += kThreads) {
        u64 v = sm[e];
        if (v >= q2) v -= q2;
        if (v >= q) v -= q;
        x[e] = v;
    }
}

__global__ void __launch_bounds__(kThreads)
k_inv_chunks(DevRing R, u64* data, const u64* src, u32 row_base, u32 rows_per_poly, int level, u32 logN1, u32 logCpb) {
    extern __shared__ u64 sm[];
    const u32 N = R.N, logN = R.logN, logN2 = logN - logN1;
    const u32 row = row_base + blockIdx.y;
    const u32 mi = mod_index(row % rows_per_poly, level, R.q_count);
    const u64 q = R.q[mi], q2 = 2 * q;
    const u64* __restrict__ w = R.tw + size_t(mi) * 4 * N + 2 * size_t(N);  // winv
    const u64* __restrict__ ws = w + N;
    const u32 chunk0 = blockIdx.x << logCpb;
    const u32 tile = 1u << (logN2 + logCpb);
    u64* x = data + size_t(row) * N + (size_t(chunk0) << logN2);
    const u64* xs = src + size_t(row) * N + (size_t(chunk0) << logN2);
    for (u32 e = threadIdx.x; e < tile; e += kThreads) sm[e] = xs[e];
    __syncthreads();
    // h = 2^lh from N/2 down to N1: t = N/(2h) < N2 (chunk-local)
    for (int lh = int(logN) - 1; lh >= int(logN1); --lh) {
        const u32 logt = logN - 1 - u32(lh);
        for (u32 b = threadIdx.x; b < (tile >> 1); b += kThreads) {
            const u32 cl = b >> (logN2 - 1), bb = b & ((1u << (logN2 - 1)) - 1);
            const u32 il = bb >> logt, j = bb & ((1u << logt) - 1);
            const u32 a0 = (cl << logN2) + ((il << 1) << logt) + j;
            const u32 a1 = a0 + (1u << logt);
            const u32 widx = (1u << lh) + ((chunk0 + cl) << (u32(lh) - logN1)) + il;
            u64 u = sm[a0], v = sm[a1];
            u64 s0 = u + v;
            if (s0 >= q2) s0 -= q2;
            sm[a0] = s0;
            sm[a1] = shoup_lazy(u - v + q2, w[widx], ws[widx], q);
        }
        __syncthreads();
    }
    for (u32 e = threadIdx.x; e < tile; e += kThreads) x[e] = sm[e];
}

__global__ void __launch_bounds__(kThreads)
k_inv_cols(DevRing R, u64* __restrict__ data, u32 row_base, u32 rows_per_poly, int level, u32 logN1, u32 logC) {
    extern __shared__ u64 sm[];
    const u32 N = R.N, C = 1u << logC, N2 = N >> logN1;
    const u32 row = row_base + blockIdx.y;
    const u32 mi = mod_index(row % rows_per_poly, level, R.q_count);
    const u64 q = R.q[mi], q2 = 2 * q;
    const u64* __restrict__ w = R.tw + size_t(mi) * 4 * N + 2 * size_t(N);
    const u64* __restrict__ ws = w + N;
    const u64 ninv = R.ninv[2 * mi], ninv_s = R.ninv[2 * mi + 1];
    u64* x = data + size_t(row) * N + size_t(blockIdx.x) * C;
    const u32 tile = 1u << (logN1 + logC);
    for (u32 e = threadIdx.x; e < tile; e += kThreads) sm[e] = x[size_t(e >> logC) * N2 + (e & (C - 1))];
    __syncthreads();
    // h = 2^lh from N1/2 down to 1: column stride t' = N1/(2h)
    for (int lh = int(logN1) - 1; lh >= 0; --lh) {
        const u32 logt = logN1 - 1 - u32(lh);
        for (u32 b = threadIdx.x; b < (tile >> 1); b += kThreads) {
            const u32 cc = b & (C - 1), bb = b >> logC;
            const u32 i = bb >> logt, j = bb & ((1u << logt) - 1);
            const u32 a0 = ((((i << 1) << logt) + j) << logC) + cc;
            const u32 a1 = a0 + (1u << (logt + logC));
            const u32 widx = (1u << lh) + i;
            u64 u = sm[a0], v = sm[a1];
            u64 s0 = u + v;
            if (s0 >= q2) s0 -= q2;
            sm[a0] = s0;
            sm[a1] = shoup_lazy(u - v + q2, w[widx], ws[widx], q);
        }
        __syncthreads();
    }
    for (u32 e = threadIdx.x; e < tile; e += kThreads)
        x[size_t(e >> logC) * N2 + (e & (C - 1))] = shoup(sm[e], ninv, ninv_s, q);
}

#include "tg_ntt_warp.cuh"
#include "tg_ks_fused.cuh"

template <int E1, int E2>
void launch_ks_fused(const DevRing& R, int sms, u64* acc, const u64* digits, u32 nd, u32 npolys, const u64* key,
                     int level, u32 own_gs, const u64* add0, const u64* add1, const u64* pmod, cudaStream_t s,
                     bool all_fp, const u64* ty0, const u64* ty1, const Tensor2& t2) {
    static const bool attr = [] {
        cudaFuncSetAttribute(kw_ks_chunks<E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ks_chunk_smem<E2>()));
        return true;
    }();
    (void)attr;
    const u32 M1 = 32 * E1, rows = u32(level) + 1 + R.K;
    // batch split so that the grid covers about two waves (2 blocks per SM)
    const u64 base = u64(M1 / 8) * rows;
    u32 z = u32(std::min<u64>(npolys, (u64(sms) * 4 + base - 1) / base));
    static const int zf = [] {  // experiments: TG_KS_Z forces the batch split
        const char* e = getenv("TG_KS_Z");
        return e ? atoi(e) : 0;
    }();
    if (zf > 0) z = std::min<u32>(npolys, u32(zf));
    if (z < 1) z = 1;
    const u32 ppb = (npolys + z - 1) / z;
    // rows on the FP64 path: all of them, or (mixed ring, ks_fused_ok) the
    // q-chain, with the integer special rows' blocks in the same launch
    const dim3 grid(M1 / 8, rows, (npolys + ppb - 1) / ppb);
    if (all_fp) {
        kw_ks_chunks<E2><<<grid, 256, ks_chunk_smem<E2>(), s>>>(R, acc, digits, nd, npolys, ppb, key, level,
                                                                 WGeo<E1>::LOGM, own_gs, add0, add1, pmod, rows,
                                                                 ty0, ty1, t2);
        return;
    }
    static const bool attr_m = [] {
        cudaFuncSetAttribute(kw_ks_chunks<E2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(ks_chunk_smem<E2>()));
        return true;
    }();
    (void)attr_m;
    kw_ks_chunks<E2, true><<<grid, 256, ks_chunk_smem<E2>(), s>>>(R, acc, digits, nd, npolys, ppb, key, level,
                                                                   WGeo<E1>::LOGM, own_gs, add0, add1, pmod,
                                                                   u32(level) + 1, ty0, ty1, t2);
}

// every modulus on the FP64 path and no integer-row knob: column-pair kernels
bool ntt_pair_ok(const tg_context* ctx) {
    static const bool off = [] {
        const char* e = getenv("TG_NTT_PAIR");
        return e && *e == '0';
    }();
    if (off || ctx->ring.int_every != 0) return false;
    for (u64 q : ctx->h_q)
        if (q >= kFpMaxQ) return false;
    return true;
}

}  // namespace

// Every q-chain modulus on the FP64 path (kw_ks_chunks); special rows either
// FP64 too or -- the mixed rings of config 1 -- on the 64-bit integer path
// (kw_ks_chunks_int; TG_KS_FUSED_MIXED=0 keeps those rings on the unfused
// pipeline). The integer-row knob must be off: each row's class is fixed.
bool ks_fused_ok(const tg_context* ctx) {
    static const bool off = [] {
        const char* e = getenv("TG_KS_FUSED");
        return e && *e == '0';
    }();
    static const bool mixed_off = [] {
        const char* e = getenv("TG_KS_FUSED_MIXED");
        return e && *e == '0';
    }();
    int e1 = 0, e2 = 0;
    if (off || !warp_plan(ctx->ring.logN, e1, e2) || ctx->ring.int_every != 0) return false;
    bool specials_fp = true;
    for (u32 i = 0; i < ctx->h_q.size(); ++i) {
        if (ctx->h_q[i] < kFpMaxQ) continue;
        if (i < ctx->ring.q_count) return false;
        specials_fp = false;
    }
    return specials_fp || !mixed_off;
}

int ntt_forward_cols(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s, u32 skip_gs) {
    const DevRing& R = ctx->ring;
    const u32 rpp = u32(level + 1 + nspecial);
    ProfScope prof(ctx, TG_OP_NTT_FWD, 8.0 * rpp * npolys * R.N, s);  // half a transform's bytes
    const bool pair = ntt_pair_ok(ctx);
    if (R.logN == 16) launch_fwd_cols_any<8, 8>(R, ctx->sms, data, data, rpp, npolys, level, s, skip_gs, 0, rpp, pair);
    else if (R.logN == 15) launch_fwd_cols_any<4, 8>(R, ctx->sms, data, data, rpp, npolys, level, s, skip_gs, 0, rpp, pair);
    else launch_fwd_cols_any<4, 4>(R, ctx->sms, data, data, rpp, npolys, level, s, skip_gs, 0, rpp, pair);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

// The raw-output inverse column phase exists for the column-pair kernel (N = 2^16, every row FP64).
bool ntt_inverse_cols_raw_ok(const tg_context* ctx) {
    static const bool off = [] {
        const char* e = getenv("TG_RAW_MODDOWN");
        return e && *e == '0';
    }();
    return !off && ctx->ring.logN == 16 && ntt_pair_ok(ctx);
}

int ntt_inverse_cols(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s, bool raw) {
    const DevRing& R = ctx->ring;
    const u32 rpp = u32(level + 1 + nspecial);
    ProfScope prof(ctx, TG_OP_NTT_INV, 8.0 * rpp * npolys * R.N, s);
    const bool pair = ntt_pair_ok(ctx);
    if (raw && !(R.logN == 16 && pair)) return fail(TG_E_ARG, "[ring] raw inverse column phase needs N = 2^16, all FP64");
    if (R.logN == 16) launch_inv_cols_any<8, 8>(R, ctx->sms, data, rpp, npolys, level, s, 0, rpp, pair, raw);
    else if (R.logN == 15) launch_inv_cols_any<4, 8>(R, ctx->sms, data, rpp, npolys, level, s, 0, rpp, pair);
    else launch_inv_cols_any<4, 4>(R, ctx->sms, data, rpp, npolys, level, s, 0, rpp, pair);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

int ks_fused_chunks(tg_context* ctx, u64* acc, const u64* digits, u32 nd, u32 npolys, const u64* key, int level,
                    u32 own_gs, const u64* add0, const u64* add1, const u64* pmod, cudaStream_t s, const u64* ty0,
                    const u64* ty1, Tensor2 t2) {
    if (t2.u0 && !(ty0 && ty1 && t2.u1 && t2.v0 && t2.v1))
        return fail(TG_E_ARG, "[rlwe] a second product needs the first pair and all four of its parts");
    const DevRing& R = ctx->ring;
    const double rows = double(level + 1 + R.K);
    // algorithmic FP64 work: the chunk-phase butterflies of every transformed
    // digit row (an own-group row is read as it is) and of both accumulators
    // (8 ops each: exact modmul 6 + add/sub 2), the key inner product (7 per
    // term: exact modmul + add), P * c on the Q rows when adding
    int e1 = 0, e2 = 0;
    warp_plan(R.logN, e1, e2);
    const double l2 = double(WGeo<8>::LOGM) - (e2 == 8 ? 0.0 : 1.0);  // log2 of the chunk length
    const double bfly = double(R.N) / 2 * l2 * 8, own_rows = own_gs ? double(level + 1) : 0.0;
    const double fp64_ops =
        npolys * ((rows * nd - own_rows) * bfly + rows * nd * 2.0 * R.N * 7 + rows * 2 * bfly +
                  (add0 ? 2.0 * (level + 1) * R.N * 7 : 0.0) + (ty0 ? 3.0 * (level + 1) * R.N * 6.5 : 0.0) +
                  (t2.u0 ? 3.0 * (level + 1) * R.N * 8.5 : 0.0));
    // algorithmic: digits (phase-1 form) read, key once per batch, P*c addends, accumulators written
    ProfScope prof(ctx, TG_OP_KS_FUSED,
                   8.0 * R.N * (rows * (npolys * (nd + 2.0) + 2.0 * nd) +
                                (add0 ? (t2.u0 ? 8.0 : ty0 ? 4.0 : 2.0) * npolys * (level + 1) : 0.0)),
                   s, 1, fp64_ops);
    bool all_fp = true;
    for (u64 q : ctx->h_q) all_fp &= q < kFpMaxQ;
    if (R.logN == 16)
        launch_ks_fused<8, 8>(R, ctx->sms, acc, digits, nd, npolys, key, level, own_gs, add0, add1, pmod, s, all_fp, ty0, ty1, t2);
    else if (R.logN == 15)
        launch_ks_fused<4, 8>(R, ctx->sms, acc, digits, nd, npolys, key, level, own_gs, add0, add1, pmod, s, all_fp, ty0, ty1, t2);
    else
        launch_ks_fused<4, 4>(R, ctx->sms, acc, digits, nd, npolys, key, level, own_gs, add0, add1, pmod, s, all_fp, ty0, ty1, t2);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

int ntt_forward_rows(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s) {
    return ntt_forward_oop(ctx, data, data, level, nspecial, npolys, s);
}

int ntt_inverse_rows(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s) {
    return ntt_inverse_oop(ctx, data, data, level, nspecial, npolys, s);
}

int ntt_forward_oop(tg_context* ctx, u64* data, const u64* src, int level, int nspecial, u32 npolys, cudaStream_t s,
                    u32 skip_gs, u32 row0, u32 nrows) {
    const DevRing& R = ctx->ring;
    const Plan p = make_plan(R.logN);
    const u32 rpp = u32(level + 1 + nspecial);
    if (nrows == 0) nrows = rpp - row0;
    const u32 total = rpp * npolys;
    const size_t sm1 = size_t(8) << (p.logN1 + p.logC), sm2 = size_t(8) << (p.logN2 + p.logCpb);
    ProfScope prof(ctx, TG_OP_NTT_FWD, 16.0 * nrows * npolys * R.N, s, 2);
    int e1 = 0, e2 = 0;
    const bool pair = ntt_pair_ok(ctx);
    if (warp_plan(R.logN, e1, e2) && npolys <= 65535) {
        if (e1 == 8) launch_fwd_w<8, 8>(R, ctx->sms, data, src, rpp, npolys, level, s, skip_gs, row0, nrows, pair);
        else if (e2 == 8) launch_fwd_w<4, 8>(R, ctx->sms, data, src, rpp, npolys, level, s, skip_gs, row0, nrows, pair);
        else launch_fwd_w<4, 4>(R, ctx->sms, data, src, rpp, npolys, level, s, skip_gs, row0, nrows, pair);
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    if (row0 != 0 || nrows != rpp) {  // generic path: one launch pair per poly's row range
        for (u32 q = 0; q < npolys; ++q) {
            const u32 base = q * rpp + row0;
            dim3 g1((R.N >> p.logN1) >> p.logC, nrows), g2((1u << p.logN1) >> p.logCpb, nrows);
            k_fwd_cols<<<g1, kThreads, sm1, s>>>(R, data, src, base, rpp, level, p.logN1, p.logC, skip_gs);
            k_fwd_chunks<<<g2, kThreads, sm2, s>>>(R, data, base, rpp, level, p.logN1, p.logCpb, skip_gs);
        }
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    for (u32 base = 0; base < total; base += 65535) {
        const u32 rows = std::min(65535u, total - base);
        dim3 g1((R.N >> p.logN1) >> p.logC, rows), g2((1u << p.logN1) >> p.logCpb, rows);
        k_fwd_cols<<<g1, kThreads, sm1, s>>>(R, data, src, base, rpp, level, p.logN1, p.logC, skip_gs);
        k_fwd_chunks<<<g2, kThreads, sm2, s>>>(R, data, base, rpp, level, p.logN1, p.logCpb, skip_gs);
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

int ntt_inverse_oop(tg_context* ctx, u64* data, const u64* src, int level, int nspecial, u32 npolys, cudaStream_t s,
                    u32 row0, u32 nrows) {
    const DevRing& R = ctx->ring;
    const Plan p = make_plan(R.logN);
    const u32 rpp = u32(level + 1 + nspecial);
    if (nrows == 0) nrows = rpp - row0;
    const u32 total = rpp * npolys;
    const size_t sm1 = size_t(8) << (p.logN1 + p.logC), sm2 = size_t(8) << (p.logN2 + p.logCpb);
    ProfScope prof(ctx, TG_OP_NTT_INV, 16.0 * nrows * npolys * R.N, s, 2);
    int e1 = 0, e2 = 0;
    const bool pair = ntt_pair_ok(ctx);
    if (warp_plan(R.logN, e1, e2) && npolys <= 65535) {
        if (e1 == 8) launch_inv_w<8, 8>(R, ctx->sms, data, src, rpp, npolys, level, s, row0, nrows, pair);
        else if (e2 == 8) launch_inv_w<4, 8>(R, ctx->sms, data, src, rpp, npolys, level, s, row0, nrows, pair);
        else launch_inv_w<4, 4>(R, ctx->sms, data, src, rpp, npolys, level, s, row0, nrows, pair);
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    if (row0 != 0 || nrows != rpp) {
        for (u32 q = 0; q < npolys; ++q) {
            const u32 base = q * rpp + row0;
            dim3 g1((R.N >> p.logN1) >> p.logC, nrows), g2((1u << p.logN1) >> p.logCpb, nrows);
            k_inv_chunks<<<g2, kThreads, sm2, s>>>(R, data, src, base, rpp, level, p.logN1, p.logCpb);
            k_inv_cols<<<g1, kThreads, sm1, s>>>(R, data, base, rpp, level, p.logN1, p.logC);
        }
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    for (u32 base = 0; base < total; base += 65535) {
        const u32 rows = std::min(65535u, total - base);
        dim3 g1((R.N >> p.logN1) >> p.logC, rows), g2((1u << p.logN1) >> p.logCpb, rows);
        k_inv_chunks<<<g2, kThreads, sm2, s>>>(R, data, src, base, rpp, level, p.logN1, p.logCpb);
        k_inv_cols<<<g1, kThreads, sm1, s>>>(R, data, base, rpp, level, p.logN1, p.logC);
    }
    TG_LAUNCH_CHECK();
    return TG_OK;
}

}  // namespace tg

using namespace tg;

extern "C" int tg_tensor_c2_inverse(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                                    const uint64_t* y1, int level, uint32_t npolys, int* raw, void* stream) {
    return tg_tensor2_c2_inverse(ctx, c2, c2_eval, x1, y1, nullptr, nullptr, level, npolys, raw, stream);
}

extern "C" int tg_tensor2_c2_inverse(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                                     const uint64_t* y1, const uint64_t* u1, const uint64_t* v1, int level,
                                     uint32_t npolys, int* raw, void* stream) {
    return tg_tensor2_c2_inverse_strided(ctx, c2, c2_eval, x1, y1, u1, v1, nullptr, level, npolys, raw, stream);
}

// Tight copies of npolys polys `stride` words apart (one 2-D copy).
static int gather_polys(u64* dst, const u64* src, u64 stride, u32 npolys, size_t words, cudaStream_t s) {
    TG_CUDA(cudaMemcpy2DAsync(dst, words * 8, src, stride * 8, words * 8, npolys, cudaMemcpyDeviceToDevice, s));
    return TG_OK;
}

extern "C" int tg_tensor2_c2_inverse_strided(tg_context* ctx, uint64_t* c2, uint64_t* c2_eval, const uint64_t* x1,
                                             const uint64_t* y1, const uint64_t* u1, const uint64_t* v1,
                                             const uint64_t* op_strides, int level, uint32_t npolys, int* raw,
                                             void* stream) {
    if (raw) *raw = 0;
    if ((u1 == nullptr) != (v1 == nullptr)) return fail(TG_E_ARG, "[ckks] the second product needs both operands");
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    if (level < 0 || u32(level) >= ctx->ring.q_count) return fail(TG_E_ARG, "[ring] poly level out of range");
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    const DevRing& R = ctx->ring;
    cudaStream_t s = as_stream(stream);
    int e1 = 0, e2 = 0;
    static const bool off = [] {
        const char* e = getenv("TG_C2_FUSED");
        return e && *e == '0';
    }();
    // the fused chunk phase needs every row on the FP64 path, a warp plan and
    // the unstaged chunk kernel; otherwise the two separate passes
    const size_t tight = size_t(level + 1) * R.N;
    u64 st[4] = {tight, tight, tight, tight};  // words between the polys of x1, y1, u1, v1
    bool strided = false;
    if (op_strides)
        for (int i = 0; i < 4; ++i)
            if (op_strides[i] && op_strides[i] != tight) {
                if (op_strides[i] < tight) return fail(TG_E_ARG, "[ckks] operand stride below the poly size");
                st[i] = op_strides[i];
                strided = true;
            }
    if (off || NTT_CHUNK_STAGE || !ntt_pair_ok(ctx) || !warp_plan(R.logN, e1, e2) || npolys > 65535) {
        // two separate passes over tight operands (strided views gathered first)
        const u64* ops[4] = {x1, y1, u1, v1};
        void* tmp = nullptr;
        if (strided) {
            TG_CUDA(cudaMallocFromPoolAsync(&tmp, 4 * tight * npolys * 8, ctx->pool, s));
            for (int i = 0; i < 4; ++i)
                if (ops[i] && st[i] != tight) {
                    u64* d = static_cast<u64*>(tmp) + size_t(i) * tight * npolys;
                    if (int rc = gather_polys(d, ops[i], st[i], npolys, tight, s)) return rc;
                    ops[i] = d;
                }
        }
        int rc = tg_tensor2(ctx, nullptr, nullptr, c2_eval, ops[0], ops[0], ops[1], ops[1], ops[2], ops[2], ops[3],
                            ops[3], level, npolys, stream);
        if (tmp) cudaFreeAsync(tmp, s);
        if (rc) return rc;
        return tg_ntt_inverse_oop(ctx, c2, c2_eval, level, 0, npolys, stream);
    }
    // raw output (the inverse column phase's doubles, no N^-1: ModUp folds it
    // into its source constants) when the caller accepts it and the key
    // switch will take the fused path
    static const bool raw_off = [] {
        const char* e = getenv("TG_RAW_C2");
        return e && *e == '0';
    }();
    const bool out_raw = raw && !raw_off && ntt_inverse_cols_raw_ok(ctx) && ks_fused_ok(ctx);
    {
        const size_t words = size_t(level + 1) * R.N * npolys;
        // + the tensor's 2 (4) reads, 1 write
        ProfScope prof(ctx, TG_OP_NTT_INV, 16.0 * words + (u1 ? 40.0 : 24.0) * words, s, 2);
        const bool pair = true;
        if (e1 == 8) launch_inv_tensor_w<8, 8>(R, ctx->sms, c2, c2_eval, x1, y1, npolys, level, s, pair, out_raw, u1, v1, st);
        else if (e2 == 8) launch_inv_tensor_w<4, 8>(R, ctx->sms, c2, c2_eval, x1, y1, npolys, level, s, pair, false, u1, v1, st);
        else launch_inv_tensor_w<4, 4>(R, ctx->sms, c2, c2_eval, x1, y1, npolys, level, s, pair, false, u1, v1, st);
    }
    if (raw) *raw = (out_raw && e1 == 8) ? 1 : 0;
    TG_LAUNCH_CHECK();
    return TG_OK;
}

static int check_shape(tg_context* ctx, int level, int nspecial) {
    if (!ctx) return fail(TG_E_ARG, "[ring] null context");
    if (level < 0 || u32(level) >= ctx->ring.q_count) return fail(TG_E_ARG, "[ring] poly level out of range");
    if (nspecial != 0 && u32(nspecial) != ctx->ring.K) return fail(TG_E_ARG, "[ring] special rows must be all-or-none");
    return TG_OK;
}

extern "C" int tg_ntt_forward(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    return ntt_forward_rows(ctx, data, level, nspecial, npolys, as_stream(stream));
}

extern "C" int tg_ntt_inverse(tg_context* ctx, uint64_t* data, int level, int nspecial, uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    return ntt_inverse_rows(ctx, data, level, nspecial, npolys, as_stream(stream));
}

extern "C" int tg_ntt_forward_oop(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, int nspecial,
                                  uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    return ntt_forward_oop(ctx, out, in, level, nspecial, npolys, as_stream(stream));
}

extern "C" int tg_ntt_inverse_oop(tg_context* ctx, uint64_t* out, const uint64_t* in, int level, int nspecial,
                                  uint32_t npolys, void* stream) {
    if (int rc = check_shape(ctx, level, nspecial)) return rc;
    if (npolys == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    return ntt_inverse_oop(ctx, out, in, level, nspecial, npolys, as_stream(stream));
}
