// Internal header of the B200 evaluator: device ring descriptor, 64-bit
// modular arithmetic and error plumbing shared by every kernel file.
//
// Arithmetic contract: every residue that leaves a kernel
// is canonical in [0, q); inside a kernel values may be lazy in [0, 2q) or
// [0, 4q) (q < 2^62, so 4q fits a word). Any exact modular algorithm yields the
// same canonical residue as the reference's u128 `%` (common.hpp:37-39) or
// Shoup (common.hpp:46-50), so results are bit-identical by construction.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <mutex>
#include <vector>

#include "tetris_b200.h"

#define TG_STR_(x) #x
#define TG_STR(x) TG_STR_(x)

namespace tg {

using u64 = uint64_t;
using u32 = uint32_t;
using i64 = int64_t;

constexpr int kMaxMod = 64;      // max moduli per ring (q-chain + specials)
constexpr int kMaxGroup = 16;    // max primes per gadget digit group
constexpr int kMaxSpecial = 16;  // max special primes K

// Everything a kernel needs to know about the ring; passed by value.
struct DevRing {
    u32 N, logN, nmod, q_count, K;
    const u64* q;            // [nmod]
    const u64* ratio;        // [nmod][2] floor(2^128 / q) as (lo, hi)
    const u64* tw;           // [nmod][4][N]: w | w_shoup | winv | winv_shoup
    const u64* ninv;         // [nmod][2]: n_inv, n_inv_shoup
    const u32* eval_exp;     // [N]
    const u32* slot_of_exp;  // [2N]
    const u64* rs;           // [q_count][q_count][4]: ql mod q_r, ql^-1, shoup, half(ql)
    const u64* one_shoup;    // [nmod]: floor(2^64 / q) (Shoup companion of 1: word -> [0,2q))
    // FP64 NTT path (q < 1.2 * 2^50): [nmod][4][N] doubles w | w/q | winv | winv/q,
    // and [nmod][4] doubles q | 1/q | n_inv | n_inv/q (see tg_fp64.cuh)
    const double* twd;
    const double* qd;
    const double* rsd;  // [q_count][q_count][2]: (ql mod q_r)^-1, fl(. / q_r) (FP64 rescale)
    u32 int_every;  // NTT: one FP64-eligible row in int_every takes the integer path (0: none)
};

// NTT skip word (own-group digit rows): group size (bits 0-15), digits per
// poly of a batch (16-30), and this flag: the transformed digit rows hold
// ModUp's centred doubles, not canonical words (column-pair phase only).
constexpr u32 kTgRawDigits = 0x80000000u;

// Row r of a poly at (level, nspecial) -> modulus index (ring.hpp:227-229).
__host__ __device__ __forceinline__ u32 mod_index(u32 r, int level, u32 q_count) {
    return r <= u32(level) ? r : q_count + (r - u32(level) - 1);
}

// ---------------------------------------------------------------------------
// Word arithmetic
// ---------------------------------------------------------------------------

__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
    u64 r = a + b;
    return r >= q ? r - q : r;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
__device__ __forceinline__ u64 neg_mod(u64 a, u64 q) { return a == 0 ? 0 : q - a; }

// Shoup product a*w mod q for ANY a < 2^64, result in [0, 2q).
__device__ __forceinline__ u64 shoup_lazy(u64 a, u64 w, u64 ws, u64 q) {
    u64 hi = __umul64hi(a, ws);
    return a * w - hi * q;
}
__device__ __forceinline__ u64 shoup(u64 a, u64 w, u64 ws, u64 q) {
    u64 r = shoup_lazy(a, w, ws, q);
    return r >= q ? r - q : r;
}

// Exact z mod q for any 128-bit z = hi:lo, with mu = floor(2^128/q) = rhi:rlo.
// est = floor(z*mu / 2^128) (computed exactly, mod 2^64) lies in
// {floor(z/q)-1, floor(z/q)}, so z - est*q < 2q fits a word.
__device__ __forceinline__ u64 barrett128(u64 lo, u64 hi, u64 q, u64 rlo, u64 rhi) {
    u64 t = __umul64hi(lo, rlo);
    u64 m1l = lo * rhi, m1h = __umul64hi(lo, rhi);
    u64 m2l = hi * rlo, m2h = __umul64hi(hi, rlo);
    u64 s = t + m1l;
    u64 c = s < t;
    u64 s2 = s + m2l;
    c += s2 < s;
    u64 est = hi * rhi + m1h + m2h + c;
    u64 r = lo - est * q;
    return r >= q ? r - q : r;
}
// Exact x mod q for a single word.
__device__ __forceinline__ u64 reduce64(u64 x, u64 q, u64 rlo, u64 rhi) {
    // floor(x * mu / 2^128) with hi = 0
    u64 t = __umul64hi(x, rlo);
    u64 m1l = x * rhi, m1h = __umul64hi(x, rhi);
    u64 s = t + m1l;
    u64 est = m1h + (s < t);
    u64 r = x - est * q;
    return r >= q ? r - q : r;
}
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, u64 q, u64 rlo, u64 rhi) {
    return barrett128(a * b, __umul64hi(a, b), q, rlo, rhi);
}

// 128-bit accumulator helpers.
struct U128 {
    u64 lo, hi;
};
__device__ __forceinline__ void mac128(U128& acc, u64 a, u64 b) {
    u64 lo = a * b, hi = __umul64hi(a, b);
    acc.lo += lo;
    acc.hi += hi + (acc.lo < lo);
}

// ---------------------------------------------------------------------------
// Host-side exact helpers (context setup; never from floating point)
// ---------------------------------------------------------------------------
using u128 = unsigned __int128;
inline u64 h_mul_mod(u64 a, u64 b, u64 q) { return u64((u128(a) * b) % q); }
inline u64 h_pow_mod(u64 b, u64 e, u64 q) {
    u64 r = 1 % q;
    b %= q;
    while (e) {
        if (e & 1) r = h_mul_mod(r, b, q);
        b = h_mul_mod(b, b, q);
        e >>= 1;
    }
    return r;
}
inline u64 h_inv_mod(u64 a, u64 q) { return h_pow_mod(a % q, q - 2, q); }
inline u64 h_shoup(u64 w, u64 q) { return u64((u128(w) << 64) / q); }
inline void h_ratio(u64 q, u64* lo, u64* hi) {
    u128 mu = (~u128(0)) / q;  // = floor(2^128 / q) for odd q > 1
    *lo = u64(mu);
    *hi = u64(mu >> 64);
}

// ---------------------------------------------------------------------------
// Errors
// ---------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define TG_CUDA(expr)                                              \
    do {                                                           \
        cudaError_t _e = (expr);                                   \
        if (_e != cudaSuccess) return ::tg::cuda_fail(_e, #expr);  \
    } while (0)
#define TG_LAUNCH_CHECK()                                                      \
    do {                                                                       \
        cudaError_t _e = cudaGetLastError();                                   \
        if (_e != cudaSuccess) return ::tg::cuda_fail(_e, "kernel launch");   \
    } while (0)
#define TG_REQUIRE(cond, msg)                         \
    do {                                              \
        if (!(cond)) return ::tg::fail(TG_E_ARG, msg); \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Host-side exact constants of one gadget size table (rlwe.hpp:178-201).
struct GadgetDev {
    u32 group_size, ngroups;
    u64* src;   // [ngroups][group_size(active-1)][group_size(i)][2]
    const u64* srcn;  // the same constants times N^-1 as FP64 (value, fl(./q)) bits: raw inverse-NTT sources
    u64* conv;  // [ngroups][group_size][group_size][nmod][2]
    u64* md;    // ModDown: [K][2] (P/p_s)^-1 mod p_s; [K][q_count][4] +-(P/p_s) mod q_r; [q_count][2] P^-1 mod q_r;
                // [q_count][4] P mod q_r (u64, Shoup, FP64 value, FP64 quotient)
    double* mdf;  // FP64 ModDown (all moduli < kFpMaxQ): see k_mod_down_fp
    double* mdfn; // the same with N^-1 folded into the input constants (raw inverse-NTT input, RAW = true)
    bool lazy_modup, lazy_moddown;  // lazy sums provably fit a word (checked on the host)
    bool fp_moddown;                // every modulus below the FP64 bound: ModDown on the FP64 pipe
    u32 base2_bits;                 // 0: RNS digits; else balanced base-2^b sub-digits (group_size 1)
    // Base conversions on the int8 tensor cores (tg_baseconv_tc.cuh; all-FP64
    // rings, RNS digits, N a multiple of 128). tc_kb_mu == 0: off.
    u32 tc_kb_mu, tc_kb_md;      // GEMM K bytes (8 per source, rounded up to 32)
    u32 tc_mode;                 // TG_TC_BASECONV: 1 auto (where measured faster), 2 always
    u32 tc_tall;                 // target blocks per ModUp combo (K + q_count + 1)
    size_t tc_mu_bstride;        // bytes per ModUp (group, active count) B operand
    size_t tc_mu_cstride;        // words per ModUp combo constant block
    const uint8_t* tc_mu_b;      // [ngroups * group_size][tc_tall][8][tc_kb_mu] core-matrix layout
    const u64* tc_mu_c;          // [combo]: [tc_tall][4] target (q, 1/q, 2^32 mod q, ./q), [group_size][2] source
    const uint8_t* tc_md_b;      // [q_count + 1][8][tc_kb_md]
    const u64* tc_md_c;          // [q_count + 1][8]: q, 1/q, 2^32 mod q, ./q, P^-1, ./q, P^-1 N^-1, ./q
};

}  // namespace tg

namespace tg {
struct ProfRecord {
    int op;
    int kernels;  // kernel launches in the scope
    double bytes;
    double fp64_ops;  // algorithmic FP64 operations (0: not modelled for this op)
    cudaEvent_t start, stop;
};
}  // namespace tg

struct tg_context {
    int device = 0;
    int sms = 148;  // multiprocessor count (grid sizing)
    tg::DevRing ring{};
    std::vector<tg::u64> h_q;
    std::vector<tg::u64> h_ratio;
    void* dev_block = nullptr;  // one allocation for all tables
    void* dev_fp = nullptr;     // FP64 NTT tables (twd, qd)
    cudaMemPool_t pool = nullptr;
    // kernel timing (tg_profile_*); launches may come from several host threads
    std::mutex prof_mu;
    bool prof_on = false;
    std::vector<tg::ProfRecord> prof_recs;
    std::vector<cudaEvent_t> prof_free;
};

namespace tg {
// Brackets the launches of its scope with CUDA events when profiling is on.
struct ProfScope {
    tg_context* ctx;
    ProfRecord rec{};
    bool on;
    ProfScope(tg_context* c, int op, double bytes, cudaStream_t s, int kernels = 1, double fp64_ops = 0)
        : ctx(c), on(c && c->prof_on) {
        if (!on) return;
        rec.op = op;
        rec.kernels = kernels;
        rec.bytes = bytes;
        rec.fp64_ops = fp64_ops;
        {
            std::lock_guard<std::mutex> g(ctx->prof_mu);
            rec.start = take_event();
            rec.stop = take_event();
        }
        stream = s;
        cudaEventRecord(rec.start, s);
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(rec.stop, stream);
        std::lock_guard<std::mutex> g(ctx->prof_mu);
        ctx->prof_recs.push_back(rec);
    }
    cudaEvent_t take_event() {
        if (!ctx->prof_free.empty()) {
            cudaEvent_t e = ctx->prof_free.back();
            ctx->prof_free.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
    cudaStream_t stream = nullptr;
};
}  // namespace tg

struct tg_gadget {
    tg_context* ctx = nullptr;
    tg::GadgetDev g{};
    std::vector<tg::u32> group_first, group_count;
    std::vector<tg::u32> nsub;  // base-2 sub-digits per prime (rlwe.hpp:20-25)
    void* dev_block = nullptr;
};

namespace tg {
// Launch helpers implemented in tg_ntt.cu (used by the keyswitch pipeline).
int ntt_forward_rows(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s);
int ntt_inverse_rows(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s);
// Row ranges: rows [row0, row0 + nrows) of every poly (nrows 0: to the end).
int ntt_forward_oop(tg_context* ctx, u64* dst, const u64* src, int level, int nspecial, u32 npolys, cudaStream_t s,
                    u32 skip_gs = 0, u32 row0 = 0, u32 nrows = 0);
int ntt_inverse_oop(tg_context* ctx, u64* dst, const u64* src, int level, int nspecial, u32 npolys, cudaStream_t s,
                    u32 row0 = 0, u32 nrows = 0);
// Fused key-switch core (tg_ks_fused.cuh): usable when every modulus takes
// the FP64 path and N has a warp plan (2^14..2^16). The digits hold the
// forward column phase's output (ntt_forward_cols); acc receives both
// accumulators after the inverse chunk phase (finish with ntt_inverse_cols).
bool ks_fused_ok(const tg_context* ctx);
int ntt_forward_cols(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s, u32 skip_gs);
int ntt_inverse_cols(tg_context* ctx, u64* data, int level, int nspecial, u32 npolys, cudaStream_t s,
                     bool raw = false);
bool ntt_inverse_cols_raw_ok(const tg_context* ctx);
// Second operand pair of a lazily relinearised sum of two products
// (Evaluator::mul2_relin_rescale): eval-form parts u0, u1, v0, v1 laid out
// like the first pair's; all null when there is one product.
// sx, sy, su, sv: words between consecutive polys of a part of x, y, u, v
// (0: tight, (level+1) * N) -- level-dropped views of a higher-level batch
// are read in place instead of being gathered first.
struct Tensor2 {
    const u64* u0 = nullptr;
    const u64* u1 = nullptr;
    const u64* v0 = nullptr;
    const u64* v1 = nullptr;
    u64 sx = 0, sy = 0, su = 0, sv = 0;
};
int ks_fused_chunks(tg_context* ctx, u64* acc, const u64* digits, u32 nd, u32 npolys, const u64* key, int level,
                    u32 own_gs, const u64* add0, const u64* add1, const u64* pmod, cudaStream_t s,
                    const u64* ty0 = nullptr, const u64* ty1 = nullptr, Tensor2 t2 = Tensor2{});
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};
}  // namespace tg
