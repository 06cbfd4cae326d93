// Context, memory and gadget setup for the C-ABI (include/tetris_b200.h).
//
// tg_context replaces the reference RingParams (ring.hpp:116-195) on the
// device: the host-built NTT tables are uploaded verbatim; the exact integer
// constants of rescale (ring.hpp:505-508), the gadget size tables
// (rlwe.hpp:178-201) and ModDown (rlwe.hpp:555-579) are derived here from the
// moduli with exact 128-bit host arithmetic.
#include <cstring>
#include <mutex>

#include <cstdlib>

#include "tg_internal.cuh"
#include "tg_fp64.cuh"

namespace tg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    g_last_error = std::string("[gpu] ") + where + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? TG_E_NOMEM : TG_E_CUDA;
}

}  // namespace tg

using namespace tg;

extern "C" const char* tg_last_error(void) { return g_last_error.c_str(); }

extern "C" int tg_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" const char* tg_build_info(void) {
    return "tetris_b200 sm_100a (CUDA " TG_STR(__CUDACC_VER_MAJOR__) "." TG_STR(__CUDACC_VER_MINOR__) ")";
}

extern "C" int tg_context_create(tg_context** out, int device, uint32_t degree, const uint64_t* moduli,
                                 uint32_t nmod, uint32_t special_count, const uint64_t* tables,
                                 const uint64_t* n_inv, const uint32_t* eval_exp,
                                 const uint32_t* slot_of_exp) {
    if (!out) return fail(TG_E_ARG, "[ring] null output handle");
    *out = nullptr;
    if (degree < 16 || (degree & (degree - 1)) != 0) return fail(TG_E_ARG, "[ring] degree must be a power of two >= 16");
    if (nmod == 0 || nmod > u32(kMaxMod) || special_count >= nmod)
        return fail(TG_E_ARG, "[ring] need at least one non-special prime (and at most 64 moduli)");
    if (special_count > u32(kMaxSpecial)) return fail(TG_E_ARG, "[ring] too many special primes");
    for (u32 i = 0; i < nmod; ++i)
        if (moduli[i] >= (1ULL << 62) || moduli[i] < 3) return fail(TG_E_ARG, "[ring] moduli must be odd primes below 2^62");
    int ndev = tg_device_count();
    if (ndev <= 0) return fail(TG_E_STATE, "[gpu] no CUDA device visible");
    if (device < 0 || device >= ndev) return fail(TG_E_ARG, "[gpu] device index out of range");
    DeviceGuard guard(device);

    auto* ctx = new tg_context();
    ctx->device = device;
    if (const char* e = std::getenv("TG_NTT_INT_EVERY")) ctx->ring.int_every = u32(std::strtoul(e, nullptr, 10));
    if (cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || ctx->sms <= 0)
        ctx->sms = 148;
    DevRing& R = ctx->ring;
    R.N = degree;
    R.logN = 0;
    while ((1u << R.logN) < degree) ++R.logN;
    R.nmod = nmod;
    R.K = special_count;
    R.q_count = nmod - special_count;
    ctx->h_q.assign(moduli, moduli + nmod);
    ctx->h_ratio.resize(2 * nmod);
    for (u32 i = 0; i < nmod; ++i) h_ratio(moduli[i], &ctx->h_ratio[2 * i], &ctx->h_ratio[2 * i + 1]);

    // rescale constants per (level, target row): ql mod q_r, (ql mod q_r)^-1, shoup, ql>>1
    const u32 qc = R.q_count;
    std::vector<u64> rs(size_t(qc) * qc * 4, 0);
    for (u32 l = 1; l < qc; ++l) {
        u64 ql = moduli[l];
        for (u32 r = 0; r < l; ++r) {
            u64 q = moduli[r];
            u64 qlq = ql % q;
            u64 inv = h_inv_mod(qlq, q);
            u64* e = &rs[(size_t(l) * qc + r) * 4];
            e[0] = qlq;
            e[1] = inv;
            e[2] = h_shoup(inv, q);
            e[3] = ql >> 1;
        }
    }

    // one device block: q | ratio | tw | ninv | rs | eval_exp | slot_of_exp
    size_t n_q = nmod, n_ratio = 2 * nmod, n_tw = size_t(4) * nmod * degree, n_ninv = 2 * nmod, n_rs = rs.size();
    size_t words = n_q + n_ratio + n_tw + n_ninv + n_rs + nmod;  // + one_shoup
    size_t bytes = words * 8 + size_t(3) * degree * 4;
    cudaError_t e = cudaMalloc(&ctx->dev_block, bytes);
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "cudaMalloc(tables)");
    }
    u64* p = static_cast<u64*>(ctx->dev_block);
    R.q = p;
    R.ratio = p + n_q;
    R.tw = p + n_q + n_ratio;
    R.ninv = p + n_q + n_ratio + n_tw;
    R.rs = p + n_q + n_ratio + n_tw + n_ninv;
    R.one_shoup = p + n_q + n_ratio + n_tw + n_ninv + n_rs;
    u32* p32 = reinterpret_cast<u32*>(p + words);
    R.eval_exp = p32;
    R.slot_of_exp = p32 + degree;
    std::vector<u64> host(words);
    std::memcpy(host.data(), moduli, n_q * 8);
    std::memcpy(host.data() + n_q, ctx->h_ratio.data(), n_ratio * 8);
    std::memcpy(host.data() + n_q + n_ratio, tables, n_tw * 8);
    std::memcpy(host.data() + n_q + n_ratio + n_tw, n_inv, n_ninv * 8);
    std::memcpy(host.data() + n_q + n_ratio + n_tw + n_ninv, rs.data(), n_rs * 8);
    for (u32 i = 0; i < nmod; ++i) host[n_q + n_ratio + n_tw + n_ninv + n_rs + i] = h_shoup(1, moduli[i]);
    e = cudaMemcpy(p, host.data(), words * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p32, eval_exp, size_t(degree) * 4, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(p32 + degree, slot_of_exp, size_t(2) * degree * 4, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(ctx->dev_block);
        delete ctx;
        return cuda_fail(e, "cudaMemcpy(tables)");
    }
    // FP64 NTT tables: w, fl(w/q), winv, fl(winv/q) per modulus (exact w as a
    // double when q < 1.2 * 2^50, the only moduli that take the FP64 path) and
    // q, fl(1/q), n_inv, fl(n_inv/q).
    {
        const size_t nt = size_t(4) * nmod * degree, nq4 = size_t(4) * nmod;
        const u32 qc = nmod - special_count;
        std::vector<double> fp(nt + nq4 + size_t(qc) * qc * 2);
        // rescale in FP64: (ql mod q_r)^-1 and fl(that / q_r) per (level, row)
        for (u32 l = 1; l < qc; ++l)
            for (u32 r = 0; r < l; ++r) {
                const u64 inv = h_inv_mod(moduli[l] % moduli[r], moduli[r]);
                fp[nt + nq4 + (size_t(l) * qc + r) * 2] = double(inv);
                fp[nt + nq4 + (size_t(l) * qc + r) * 2 + 1] = double(inv) / double(moduli[r]);
            }
        for (u32 i = 0; i < nmod; ++i) {
            const double qd = double(moduli[i]);
            const u64* t = tables + size_t(4) * i * degree;
            double* o = fp.data() + size_t(4) * i * degree;
            // centred twiddles w in (-q/2, q/2]: |fl(w/q)| < 1/2 widens the
            // FP64 modmul's input window to |b| < 2^52 (tg_fp64.cuh), which
            // is what lets six forward stages / two inverse stages run
            // between reductions; w - q is exact (both < 2^53)
            const auto centred = [&](u64 x) { return x > moduli[i] / 2 ? double(x) - qd : double(x); };
            for (u32 j = 0; j < degree; ++j) {
                o[j] = centred(t[j]);
                o[degree + j] = o[j] / qd;
                o[2 * size_t(degree) + j] = centred(t[2 * size_t(degree) + j]);
                o[3 * size_t(degree) + j] = o[2 * size_t(degree) + j] / qd;
            }
            double* s = fp.data() + nt + 4 * size_t(i);
            s[0] = qd;
            s[1] = 1.0 / qd;
            s[2] = double(n_inv[2 * i]);
            s[3] = double(n_inv[2 * i]) / qd;
        }
        e = cudaMalloc(&ctx->dev_fp, fp.size() * sizeof(double));
        if (e == cudaSuccess) e = cudaMemcpy(ctx->dev_fp, fp.data(), fp.size() * sizeof(double), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) {
            cudaFree(ctx->dev_block);
            if (ctx->dev_fp) cudaFree(ctx->dev_fp);
            delete ctx;
            return cuda_fail(e, "cudaMemcpy(fp tables)");
        }
        R.twd = static_cast<const double*>(ctx->dev_fp);
        R.qd = R.twd + nt;
        R.rsd = R.qd + nq4;
    }
    // stream-ordered pool of this context: freed blocks stay cached (no
    // release back to the driver), and a block freed on one stream is reused
    // by another only once the free is known complete (opportunistic reuse):
    // the allocator never inserts waits between streams, so concurrent
    // pipelines (one stream each) are not serialised by memory reuse.
    {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        cudaError_t e = cudaMemPoolCreate(&ctx->pool, &props);
        if (e != cudaSuccess) {
            cudaFree(ctx->dev_block);
            if (ctx->dev_fp) cudaFree(ctx->dev_fp);
            delete ctx;
            return cuda_fail(e, "cudaMemPoolCreate");
        }
        uint64_t threshold = UINT64_MAX;
        int no = 0;
        cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &threshold);
        cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    *out = ctx;
    return TG_OK;
}

extern "C" void tg_context_destroy(tg_context* ctx) {
    if (!ctx) return;
    DeviceGuard guard(ctx->device);
    cudaDeviceSynchronize();
    for (auto& r : ctx->prof_recs) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    for (auto e : ctx->prof_free) cudaEventDestroy(e);
    cudaFree(ctx->dev_block);
    if (ctx->dev_fp) cudaFree(ctx->dev_fp);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
}

extern "C" uint32_t tg_context_degree(const tg_context* ctx) { return ctx ? ctx->ring.N : 0; }

extern "C" int tg_alloc(tg_context* ctx, void** ptr, size_t bytes, void* stream) {
    if (!ctx || !ptr) return fail(TG_E_ARG, "[gpu] tg_alloc: null argument");
    DeviceGuard guard(ctx->device);
    *ptr = nullptr;
    if (bytes == 0) return TG_OK;
    TG_CUDA(cudaMallocFromPoolAsync(ptr, bytes, ctx->pool, as_stream(stream)));
    return TG_OK;
}

extern "C" int tg_free(tg_context* ctx, void* ptr, void* stream) {
    if (!ctx) return fail(TG_E_ARG, "[gpu] tg_free: null context");
    if (!ptr) return TG_OK;
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaFreeAsync(ptr, as_stream(stream)));
    return TG_OK;
}

extern "C" int tg_memcpy_h2d(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream) {
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_memcpy_d2h(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream) {
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_memcpy_d2d(tg_context* ctx, void* dst, const void* src, size_t bytes, void* stream) {
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_memset0(tg_context* ctx, void* dst, size_t bytes, void* stream) {
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaMemsetAsync(dst, 0, bytes, as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_stream_sync(tg_context* ctx, void* stream) {
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return TG_OK;
}

extern "C" int tg_host_alloc_pinned(void** ptr, size_t bytes) {
    if (!ptr) return fail(TG_E_ARG, "[gpu] null argument");
    TG_CUDA(cudaHostAlloc(ptr, bytes, cudaHostAllocDefault));
    return TG_OK;
}
extern "C" int tg_host_free_pinned(void* ptr) {
    if (ptr) TG_CUDA(cudaFreeHost(ptr));
    return TG_OK;
}

extern "C" int tg_profile_enable(tg_context* ctx, int on) {
    if (!ctx) return fail(TG_E_ARG, "[gpu] null context");
    ctx->prof_on = on != 0;
    return TG_OK;
}

extern "C" int tg_profile_read(tg_context* ctx, double* ms, uint64_t* launches, double* bytes) {
    return tg_profile_read_ops(ctx, ms, launches, bytes, nullptr);
}

extern "C" int tg_profile_read_ops(tg_context* ctx, double* ms, uint64_t* launches, double* bytes,
                                   double* fp64_ops) {
    if (!ctx) return fail(TG_E_ARG, "[gpu] null context");
    DeviceGuard guard(ctx->device);
    std::lock_guard<std::mutex> lock(ctx->prof_mu);
    for (int i = 0; i < TG_OP_COUNT; ++i) {
        if (ms) ms[i] = 0;
        if (launches) launches[i] = 0;
        if (bytes) bytes[i] = 0;
        if (fp64_ops) fp64_ops[i] = 0;
    }
    for (auto& r : ctx->prof_recs) {
        TG_CUDA(cudaEventSynchronize(r.stop));
        float t = 0;
        TG_CUDA(cudaEventElapsedTime(&t, r.start, r.stop));
        if (ms) ms[r.op] += t;
        if (launches) launches[r.op] += u64(r.kernels);
        if (bytes) bytes[r.op] += r.bytes;
        if (fp64_ops) fp64_ops[r.op] += r.fp64_ops;
        ctx->prof_free.push_back(r.start);
        ctx->prof_free.push_back(r.stop);
    }
    ctx->prof_recs.clear();
    return TG_OK;
}

extern "C" const char* tg_profile_op_name(int op) {
    static const char* names[TG_OP_COUNT] = {"ntt_fwd", "ntt_inv",  "addsub", "mul_pointwise", "mul_scalar",
                                             "automorphism", "rescale", "tensor", "mul_plain", "modup_baseconv",
                                             "key_inner", "mod_down", "reduce", "lincomb", "encode", "ks_fused"};
    return op >= 0 && op < TG_OP_COUNT ? names[op] : "?";
}

extern "C" int tg_stream_create(tg_context* ctx, void** stream) {
    if (!ctx || !stream) return fail(TG_E_ARG, "[gpu] tg_stream_create: null argument");
    DeviceGuard guard(ctx->device);
    cudaStream_t s = nullptr;
    TG_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
    return TG_OK;
}
extern "C" int tg_stream_destroy(tg_context* ctx, void* stream) {
    if (!ctx || !stream) return TG_OK;
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaStreamDestroy(as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_event_create(tg_context* ctx, void** event) {
    if (!ctx || !event) return fail(TG_E_ARG, "[gpu] tg_event_create: null argument");
    DeviceGuard guard(ctx->device);
    cudaEvent_t e = nullptr;
    TG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *event = e;
    return TG_OK;
}
extern "C" int tg_event_destroy(tg_context* ctx, void* event) {
    if (!ctx || !event) return TG_OK;
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return TG_OK;
}
extern "C" int tg_event_record(tg_context* ctx, void* event, void* stream) {
    if (!ctx || !event) return fail(TG_E_ARG, "[gpu] tg_event_record: null argument");
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), as_stream(stream)));
    return TG_OK;
}
extern "C" int tg_stream_wait_event(tg_context* ctx, void* stream, void* event) {
    if (!ctx || !event) return fail(TG_E_ARG, "[gpu] tg_stream_wait_event: null argument");
    DeviceGuard guard(ctx->device);
    TG_CUDA(cudaStreamWaitEvent(as_stream(stream), static_cast<cudaEvent_t>(event), 0));
    return TG_OK;
}
extern "C" int tg_context_device(const tg_context* ctx) { return ctx ? ctx->device : -1; }

// ---------------------------------------------------------------------------
// Gadget: GadgetPlan size tables (rlwe.hpp:31-45, :178-201) + ModDown constants
// ---------------------------------------------------------------------------

extern "C" int tg_gadget_create(tg_gadget** out, tg_context* ctx, uint32_t group_size, uint32_t base2_bits) {
    if (!out || !ctx) return fail(TG_E_ARG, "[rlwe] null argument");
    *out = nullptr;
    if (group_size == 0) return fail(TG_E_ARG, "[rlwe] gadget group size must be positive");
    if (base2_bits != 0 && group_size != 1)
        return fail(TG_E_ARG, "[rlwe] base2 refinement requires single-prime groups");
    if (base2_bits > 62) return fail(TG_E_ARG, "[rlwe] base2 digit width out of range");
    if (group_size > u32(kMaxGroup)) return fail(TG_E_ARG, "[rlwe] gadget group size exceeds 16");
    DeviceGuard guard(ctx->device);
    const DevRing& R = ctx->ring;
    const std::vector<u64>& mod = ctx->h_q;
    const u32 nq = R.q_count, nmod = R.nmod, K = R.K, gs = group_size;
    const u32 ng = (nq + gs - 1) / gs;
    auto* g = new tg_gadget();
    g->ctx = ctx;
    g->g.group_size = gs;
    g->g.ngroups = ng;
    g->g.base2_bits = base2_bits;
    if (base2_bits) {  // GadgetVector::sub_digits (rlwe.hpp:20-25)
        for (u32 j = 0; j < nq; ++j) {
            u32 bits = 0;
            while ((mod[j] >> bits) != 0) ++bits;
            g->nsub.push_back((bits + base2_bits - 1) / base2_bits);
        }
    }
    std::vector<u64> src(size_t(ng) * gs * gs * 2, 0);
    std::vector<u64> conv(size_t(ng) * gs * gs * nmod * 2, 0);
    for (u32 j = 0; j < ng; ++j) {
        u32 first = j * gs, count = std::min(gs, nq - first);
        g->group_first.push_back(first);
        g->group_count.push_back(count);
        for (u32 a = 1; a <= count; ++a) {
            for (u32 i = 0; i < a; ++i) {
                u64 q = mod[first + i];
                u64 rest = 1;  // (D'/q_i) mod q_i over the `a` active primes
                for (u32 t = 0; t < a; ++t)
                    if (t != i) rest = h_mul_mod(rest, mod[first + t] % q, q);
                u64 sc = h_inv_mod(rest, q);
                u64* se = &src[((size_t(j) * gs + (a - 1)) * gs + i) * 2];
                se[0] = sc;
                se[1] = h_shoup(sc, q);
                for (u32 t = 0; t < nmod; ++t) {
                    u64 qt = mod[t];
                    u64 w = 1;  // D'/q_i mod q_t
                    for (u32 u = 0; u < a; ++u)
                        if (u != i) w = h_mul_mod(w, mod[first + u] % qt, qt);
                    u64* ce = &conv[(((size_t(j) * gs + (a - 1)) * gs + i) * nmod + t) * 2];
                    ce[0] = w;
                    ce[1] = h_shoup(w, qt);
                }
            }
        }
    }
    // ModDown (rlwe.hpp:555-579). Layout: [K][2] (P/p_s)^-1 mod p_s + Shoup;
    // [K][nq][4] (P/p_s) mod q_r, Shoup, its negation q_r - w, Shoup (so a
    // centered y_s < 0 multiplies |y_s| by -w: no per-term reduction);
    // [nq][2] P^-1 mod q_r + Shoup.
    // [nq][4] P mod q_r, Shoup, and as FP64 (P mod q_r, fl((P mod q_r) / q_r))
    // bit patterns: eval-form addends folded into the key-switch accumulators
    // as P * c (tg_relinearize_batch).
    std::vector<u64> md(size_t(K) * 2 + size_t(K) * nq * 4 + size_t(nq) * 2 + size_t(nq) * 4, 0);
    for (u32 s = 0; s < K; ++s) {
        u64 ps = mod[nq + s];
        u64 rest = 1;
        for (u32 t = 0; t < K; ++t)
            if (t != s) rest = h_mul_mod(rest, mod[nq + t] % ps, ps);
        u64 c = h_inv_mod(rest, ps);
        md[2 * s] = c;
        md[2 * s + 1] = h_shoup(c, ps);
    }
    for (u32 s = 0; s < K; ++s)
        for (u32 r = 0; r < nq; ++r) {
            u64 q = mod[r];
            u64 ws = 1;
            for (u32 t = 0; t < K; ++t)
                if (t != s) ws = h_mul_mod(ws, mod[nq + t] % q, q);
            u64* e = &md[2 * K + (size_t(s) * nq + r) * 4];
            e[0] = ws;
            e[1] = h_shoup(ws, q);
            e[2] = ws ? q - ws : 0;
            e[3] = h_shoup(e[2], q);
        }
    for (u32 r = 0; r < nq; ++r) {
        u64 q = mod[r];
        u64 pinv = 1;
        for (u32 s = 0; s < K; ++s) pinv = h_mul_mod(pinv, mod[nq + s] % q, q);
        pinv = h_inv_mod(pinv, q);
        u64* e = &md[2 * K + size_t(K) * nq * 4 + size_t(r) * 2];
        e[0] = pinv;
        e[1] = h_shoup(pinv, q);
        u64 pm = 1;
        for (u32 t = 0; t < K; ++t) pm = h_mul_mod(pm, mod[nq + t] % q, q);
        u64* f = &md[2 * K + size_t(K) * nq * 4 + size_t(nq) * 2 + size_t(r) * 4];
        const double pd = double(pm), pq = double(pm) / double(q);
        f[0] = pm;
        f[1] = h_shoup(pm, q);
        std::memcpy(&f[2], &pd, 8);
        std::memcpy(&f[3], &pq, 8);
    }
    // lazy-sum safety: 2*K*q_max + q_max < 2^64 for ModDown, 2*group*q < 2^64 for ModUp
    {
        u128 qmax = 0, allmax = 0;
        for (u32 r = 0; r < nq; ++r) qmax = std::max<u128>(qmax, mod[r]);
        for (u32 r = 0; r < nmod; ++r) allmax = std::max<u128>(allmax, mod[r]);
        // x + (neg terms) + 2Kq - (pos terms) < (4K + 1) q (k_mod_down_v)
        g->g.lazy_moddown = (u128(4 * K + 2) * qmax) < (u128(1) << 64);
        g->g.lazy_modup = (u128(2 * gs) * allmax) < (u128(1) << 64);
    }
    // FP64 ModDown tables (k_mod_down_fp), used when every modulus is below
    // the FP64 bound: [K][4] (p_s, fl(c_s/p_s), c_s, floor(p_s/2));
    // [nq][K][2] (w, fl(w/q_r)), w = -(P/p_s) P^-1 mod q_r;
    // [nq][4] (P^-1 mod q_r, fl(./q_r), q_r, fl(1/q_r)).
    std::vector<double> mdf(size_t(K) * 4 + size_t(nq) * K * 2 + size_t(nq) * 4, 0.0), mdfn;
    g->g.fp_moddown = K > 0;
    for (u32 t = 0; t < nmod; ++t) g->g.fp_moddown &= mod[t] < kFpMaxQ;
    if (const char* e = getenv("TG_INT_MODDOWN"); e && *e == '1') g->g.fp_moddown = false;  // A/B experiments
    if (g->g.fp_moddown) {
        for (u32 s = 0; s < K; ++s) {
            const u64 ps = mod[nq + s], c = md[2 * s];
            mdf[4 * s] = double(ps);
            mdf[4 * s + 1] = double(c) / double(ps);
            mdf[4 * s + 2] = double(c);
            mdf[4 * s + 3] = double(ps / 2);
        }
        for (u32 r = 0; r < nq; ++r) {
            const u64 q = mod[r], pinv = md[2 * K + size_t(K) * nq * 4 + size_t(r) * 2];
            for (u32 s = 0; s < K; ++s) {
                const u64 ws = md[2 * K + (size_t(s) * nq + r) * 4];
                const u64 w = h_mul_mod(ws ? q - ws : 0, pinv, q);
                mdf[4 * K + (size_t(r) * K + s) * 2] = double(w);
                mdf[4 * K + (size_t(r) * K + s) * 2 + 1] = double(w) / double(q);
            }
            double* e = &mdf[4 * K + size_t(nq) * K * 2 + size_t(r) * 4];
            e[0] = double(pinv);
            e[1] = double(pinv) / double(q);
            e[2] = double(q);
            e[3] = 1.0 / double(q);
        }
        // N^-1 folded into the input constants: the fused key switch hands
        // ModDown the accumulators' inverse transform WITHOUT its final
        // N^-1 scaling (raw doubles, |v| <= 0.6q); every input enters ModDown
        // only through an exact product with one of these constants, so
        // c_s N^-1 and P^-1 N^-1 give the same canonical residues
        mdfn = mdf;
        const u64 n = ctx->ring.N;
        for (u32 s = 0; s < K; ++s) {
            const u64 ps = mod[nq + s], c = h_mul_mod(md[2 * s], h_inv_mod(n % ps, ps), ps);
            mdfn[4 * s + 1] = double(c) / double(ps);
            mdfn[4 * s + 2] = double(c);
        }
        for (u32 r = 0; r < nq; ++r) {
            const u64 q = mod[r], pinv = md[2 * K + size_t(K) * nq * 4 + size_t(r) * 2];
            const u64 pn = h_mul_mod(pinv, h_inv_mod(n % q, q), q);
            double* e = &mdfn[4 * K + size_t(nq) * K * 2 + size_t(r) * 4];
            e[0] = double(pn);
            e[1] = double(pn) / double(q);
        }
    }
    // int8 tensor-core base conversion operands (tg_baseconv_tc.cuh): B in
    // the K-major core-matrix layout (byte (row n, col k) of a target block at
    // (k / 16) * 128 + (n % 8) * 16 + k % 16), plus the epilogue constants
    std::vector<uint8_t> tcb;
    std::vector<u64> tcc;
    size_t tc_mu_b_off = 0, tc_md_b_off = 0, tc_mu_c_off = 0, tc_md_c_off = 0;
    {
        const char* env = getenv("TG_TC_BASECONV");
        const bool on = g->g.fp_moddown && !base2_bits && R.N % 128 == 0 && K <= u32(kMaxSpecial) &&
                        !(env && *env == '0');
        if (on) {
            auto bits = [](double v) {
                u64 b;
                std::memcpy(&b, &v, 8);
                return b;
            };
            const u32 kbm = (8 * gs + 31) / 32 * 32, kbd = (8 * K + 31) / 32 * 32, tall = K + nq + 1;
            g->g.tc_mode = (env && *env == '2') ? 2 : 1;
            g->g.tc_kb_mu = kbm;
            g->g.tc_kb_md = kbd;
            g->g.tc_tall = tall;
            g->g.tc_mu_bstride = size_t(tall) * 8 * kbm;
            g->g.tc_mu_cstride = size_t(tall) * 4 + size_t(gs) * 4;  // + sources, then sources x N^-1
            const size_t ncombo = size_t(ng) * gs;
            tc_mu_b_off = 0;
            tc_md_b_off = ncombo * g->g.tc_mu_bstride;
            tcb.assign(tc_md_b_off + size_t(nq + 1) * 8 * kbd, 0);
            tc_mu_c_off = 0;
            tc_md_c_off = ncombo * g->g.tc_mu_cstride;
            tcc.assign(tc_md_c_off + size_t(nq + 1) * 8, 0);
            // byte b of v at (target block, row b, column k)
            auto set = [&](size_t blk_off, u32 b, u32 k, u64 v) {
                tcb[blk_off + (k / 16) * 128 + b * 16 + k % 16] = uint8_t(v >> (8 * b));
            };
            auto tgt_consts = [&](u64* e, u64 q) {
                const u64 r32 = (u64(1) << 32) % q;
                e[0] = q;
                e[1] = bits(1.0 / double(q));
                e[2] = bits(double(r32));
                e[3] = bits(double(r32) / double(q));
            };
            for (u32 j = 0; j < ng; ++j) {
                const u32 first = j * gs, count = std::min(gs, nq - first);
                for (u32 a = 1; a <= count; ++a) {
                    const size_t combo = size_t(j) * gs + (a - 1);
                    u64* cc = &tcc[tc_mu_c_off + combo * g->g.tc_mu_cstride];
                    const u32 T = K + nq - a;  // targets at the top level: specials, then q rows outside the group
                    for (u32 v = 0; v < T; ++v) {
                        const u32 t = v < K ? nq + v : (v - K < first ? v - K : v - K + a);
                        const u64 qt = mod[t];
                        tgt_consts(cc + size_t(v) * 4, qt);
                        const size_t blk = tc_mu_b_off + combo * g->g.tc_mu_bstride + size_t(v) * 8 * kbm;
                        for (u32 i = 0; i < a; ++i) {
                            const u64 w = conv[(((size_t(j) * gs + (a - 1)) * gs + i) * nmod + t) * 2];
                            u64 wa = w % qt;  // w 2^(8 al) mod q_t
                            for (u32 al = 0; al < 7; ++al) {
                                for (u32 b = 0; b < 8; ++b) set(blk, b, 8 * i + al, wa);
                                wa = h_mul_mod(wa, 256, qt);
                            }
                        }
                    }
                    for (u32 i = 0; i < a; ++i) {
                        const u64 q = mod[first + i], sc = src[((size_t(j) * gs + (a - 1)) * gs + i) * 2];
                        cc[size_t(tall) * 4 + 2 * i] = bits(double(sc));
                        cc[size_t(tall) * 4 + 2 * i + 1] = bits(double(sc) / double(q));
                        const u64 scn = h_mul_mod(sc, h_inv_mod(ctx->ring.N % q, q), q);
                        cc[size_t(tall) * 4 + size_t(gs) * 2 + 2 * i] = bits(double(scn));
                        cc[size_t(tall) * 4 + size_t(gs) * 2 + 2 * i + 1] = bits(double(scn) / double(q));
                    }
                }
            }
            const u64 n = ctx->ring.N;
            for (u32 r = 0; r < nq; ++r) {
                const u64 q = mod[r], pinv = md[2 * K + size_t(K) * nq * 4 + size_t(r) * 2];
                u64* e = &tcc[tc_md_c_off + size_t(r) * 8];
                tgt_consts(e, q);
                const u64 pn = h_mul_mod(pinv, h_inv_mod(n % q, q), q);
                e[4] = bits(double(pinv));
                e[5] = bits(double(pinv) / double(q));
                e[6] = bits(double(pn));
                e[7] = bits(double(pn) / double(q));
                const size_t blk = tc_md_b_off + size_t(r) * 8 * kbd;
                for (u32 s = 0; s < K; ++s) {
                    const u64 ws = md[2 * K + (size_t(s) * nq + r) * 4];
                    const u64 w = h_mul_mod(ws ? q - ws : 0, pinv, q);  // -(P/p_s) P^-1 mod q_r
                    u64 wa = w;
                    for (u32 al = 0; al < 7; ++al) {
                        for (u32 b = 0; b < 8; ++b) set(blk, b, 8 * s + al, wa);
                        wa = h_mul_mod(wa, 256, q);
                    }
                    const u64 pw = h_mul_mod(mod[nq + s] % q, w, q);  // sign column: -p_s w mod q_r
                    const u64 neg = pw ? q - pw : 0;
                    for (u32 b = 0; b < 8; ++b) set(blk, b, 8 * s + 7, neg);
                }
            }
        }
    }
    const size_t tcb_words = tcb.empty() ? 0 : (tcb.size() + 15) / 16 * 2 + 1;  // + alignment slack
    // ModUp source constants times N^-1 as FP64 pairs (raw inverse-NTT sources;
    // every modulus below the FP64 bound)
    std::vector<u64> srcn;
    if (g->g.fp_moddown) {
        srcn.assign(src.size(), 0);
        for (u32 j = 0; j < ng; ++j) {
            const u32 first = j * gs, count = std::min(gs, nq - first);
            for (u32 a = 1; a <= count; ++a)
                for (u32 i = 0; i < a; ++i) {
                    const size_t e = ((size_t(j) * gs + (a - 1)) * gs + i) * 2;
                    const u64 q = mod[first + i], scn = h_mul_mod(src[e], h_inv_mod(ctx->ring.N % q, q), q);
                    const double v = double(scn), vq = double(scn) / double(q);
                    std::memcpy(&srcn[e], &v, 8);
                    std::memcpy(&srcn[e + 1], &vq, 8);
                }
        }
    }
    size_t words = src.size() + conv.size() + md.size() + mdf.size() + mdfn.size() + tcc.size() + tcb_words +
                   srcn.size();
    cudaError_t e = cudaMalloc(&g->dev_block, words * 8);
    if (e != cudaSuccess) {
        delete g;
        return cuda_fail(e, "cudaMalloc(gadget)");
    }
    u64* p = static_cast<u64*>(g->dev_block);
    g->g.src = p;
    g->g.conv = p + src.size();
    g->g.md = p + src.size() + conv.size();
    g->g.mdf = reinterpret_cast<double*>(g->g.md + md.size());
    g->g.mdfn = mdfn.empty() ? nullptr : g->g.mdf + mdf.size();
    {
        u64* tc_c = p + src.size() + conv.size() + md.size() + mdf.size() + mdfn.size();
        const size_t off = size_t(tc_c + tcc.size() - p);
        uint8_t* tc_b = reinterpret_cast<uint8_t*>(p + (off + 1) / 2 * 2);  // 16-byte aligned
        u64* srcn_p = p + words - srcn.size();
        g->g.srcn = srcn.empty() ? nullptr : srcn_p;
        if (!srcn.empty()) {
            cudaError_t es = cudaMemcpy(srcn_p, srcn.data(), srcn.size() * 8, cudaMemcpyHostToDevice);
            if (es != cudaSuccess) {
                cudaFree(g->dev_block);
                delete g;
                return cuda_fail(es, "cudaMemcpy(gadget srcn)");
            }
        }
        g->g.tc_mu_c = tcc.empty() ? nullptr : tc_c + tc_mu_c_off;
        g->g.tc_md_c = tcc.empty() ? nullptr : tc_c + tc_md_c_off;
        g->g.tc_mu_b = tcb.empty() ? nullptr : tc_b + tc_mu_b_off;
        g->g.tc_md_b = tcb.empty() ? nullptr : tc_b + tc_md_b_off;
        if (!tcc.empty()) {
            cudaError_t ec = cudaMemcpy(tc_c, tcc.data(), tcc.size() * 8, cudaMemcpyHostToDevice);
            if (ec == cudaSuccess) ec = cudaMemcpy(tc_b, tcb.data(), tcb.size(), cudaMemcpyHostToDevice);
            if (ec != cudaSuccess) {
                cudaFree(g->dev_block);
                delete g;
                return cuda_fail(ec, "cudaMemcpy(gadget tc tables)");
            }
        }
    }
    e = cudaMemcpy(g->g.src, src.data(), src.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(g->g.conv, conv.data(), conv.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !md.empty()) e = cudaMemcpy(g->g.md, md.data(), md.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !mdf.empty()) e = cudaMemcpy(g->g.mdf, mdf.data(), mdf.size() * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !mdfn.empty())
        e = cudaMemcpy(g->g.mdfn, mdfn.data(), mdfn.size() * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(g->dev_block);
        delete g;
        return cuda_fail(e, "cudaMemcpy(gadget)");
    }
    *out = g;
    return TG_OK;
}

extern "C" void tg_gadget_destroy(tg_gadget* g) {
    if (!g) return;
    DeviceGuard guard(g->ctx->device);
    cudaDeviceSynchronize();
    cudaFree(g->dev_block);
    delete g;
}

extern "C" uint32_t tg_gadget_digit_count(const tg_gadget* g, int level) {
    if (!g || level < 0) return 0;
    // group_count(level) = (level + group_size) / group_size (rlwe.hpp:50-61)
    const u32 groups = (u32(level) + g->g.group_size) / g->g.group_size;
    if (!g->g.base2_bits) return groups;
    u32 n = 0;
    for (u32 j = 0; j < groups && j < g->nsub.size(); ++j) n += g->nsub[j];
    return n;
}

extern "C" int tg_pool_reserve(tg_context* ctx, uint64_t bytes) {
    if (!ctx) return fail(TG_E_ARG, "[gpu] null context");
    if (bytes == 0) return TG_OK;
    DeviceGuard guard(ctx->device);
    void* p = nullptr;
    TG_CUDA(cudaMallocFromPoolAsync(&p, bytes, ctx->pool, nullptr));
    TG_CUDA(cudaFreeAsync(p, nullptr));
    TG_CUDA(cudaStreamSynchronize(nullptr));
    return TG_OK;
}

extern "C" int tg_pool_stats(tg_context* ctx, uint64_t* reserved, uint64_t* used_high) {
    if (!ctx) return fail(TG_E_ARG, "[gpu] null context");
    DeviceGuard guard(ctx->device);
    unsigned long long r = 0, u = 0;
    TG_CUDA(cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrReservedMemCurrent, &r));
    TG_CUDA(cudaMemPoolGetAttribute(ctx->pool, cudaMemPoolAttrUsedMemHigh, &u));
    if (reserved) *reserved = r;
    if (used_high) *used_high = u;
    return TG_OK;
}
