// Slot encoder on the device: Encoder::encode_slots (reference ckks.hpp:59-86).
//
// The reference packs n slots with an O(n^2) inverse DFT on the host
// (ckks.hpp:59-68): w_t = (sum_{j<n} v_j * conj(psi[t * 5^j mod 4n])) / n,
// then round_half_away(w_t * scale) and from_centered per row (ckks.hpp:76-84).
// The residues depend on every floating-point rounding, so the device replays
// the reference's exact IEEE operation sequence per output t: the j loop runs
// sequentially in the same order, complex products expand as the compiler
// expands std::complex<double> * (re = ac - bd, im = ad + bc, each product
// rounded; x86-64 -O2 emits no FMA), and every operation is an explicit
// __d*_rn intrinsic so nvcc cannot contract it into an FMA. psi is the host
// table (std::cos/std::sin), uploaded as-is. The result is bit-identical to
// the reference for any thread layout: parallelism is only across outputs t
// and across slot vectors.
//
// Cost: n^2 complex MACs (8 FP64 ops) per vector; one psi gather per (t, j) is
// shared by the kEncVB vectors a thread carries.
#include "tg_internal.cuh"

namespace tg {
namespace {

constexpr u32 kEncThreads = 256;
constexpr u32 kEncChunk = 512;

template <int VB>
__global__ void __launch_bounds__(kEncThreads) k_encode_slots(u64* __restrict__ out, const double2* __restrict__ v,
                                                              u32 batch, u32 n, const double2* __restrict__ psi,
                                                              const u32* __restrict__ rot5, double scale, int level,
                                                              unsigned long long* max_bits, DevRing R) {
    __shared__ double2 sv[VB][kEncChunk];
    __shared__ u32 sr[kEncChunk];
    const u32 t = blockIdx.x * kEncThreads + threadIdx.x;
    const u32 b0 = blockIdx.y * VB;
    const u32 mask = 4 * n - 1;  // 4n is a power of two: (u64(t) * r) % 4n == (t * r) & mask
    double2 acc[VB];
#pragma unroll
    for (int b = 0; b < VB; ++b) acc[b] = make_double2(0.0, 0.0);

    for (u32 j0 = 0; j0 < n; j0 += kEncChunk) {
        const u32 cnt = min(kEncChunk, n - j0);
        __syncthreads();
        for (u32 i = threadIdx.x; i < cnt; i += kEncThreads) {
            sr[i] = rot5[j0 + i];
#pragma unroll
            for (int b = 0; b < VB; ++b)
                sv[b][i] = (b0 + b < batch) ? v[std::size_t(b0 + b) * n + j0 + i] : make_double2(0.0, 0.0);
        }
        __syncthreads();
        if (t < n) {
#pragma unroll 4
            for (u32 j = 0; j < cnt; ++j) {
                const double2 p = __ldg(&psi[(t * sr[j]) & mask]);
                const double c = p.x, d = -p.y;  // std::conj(psi)
#pragma unroll
                for (int b = 0; b < VB; ++b) {
                    const double2 a = sv[b][j];
                    const double re = __dsub_rn(__dmul_rn(a.x, c), __dmul_rn(a.y, d));
                    const double im = __dadd_rn(__dmul_rn(a.x, d), __dmul_rn(a.y, c));
                    acc[b].x = __dadd_rn(acc[b].x, re);
                    acc[b].y = __dadd_rn(acc[b].y, im);
                }
            }
        }
    }
    if (t >= n) return;
    const u32 stride = R.N / (2 * n);
    const double dn = double(n);
#pragma unroll
    for (int b = 0; b < VB; ++b) {
        if (b0 + b >= batch) break;
        const double wr = __ddiv_rn(acc[b].x, dn), wi = __ddiv_rn(acc[b].y, dn);  // acc / double(n)
        if (max_bits) {
            atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(fabs(wr))));
            atomicMax(max_bits, static_cast<unsigned long long>(__double_as_longlong(fabs(wi))));
        }
        const long long re = llround(__dmul_rn(wr, scale));  // round_half_away (common.hpp:95-97)
        const long long im = llround(__dmul_rn(wi, scale));
        u64* o = out + std::size_t(b0 + b) * (level + 1) * R.N;
        for (int r = 0; r <= level; ++r) {
            const long long q = static_cast<long long>(R.q[r]);
            long long x = re % q, y = im % q;  // from_centered (common.hpp)
            o[std::size_t(r) * R.N + std::size_t(t) * stride] = u64(x < 0 ? x + q : x);
            o[std::size_t(r) * R.N + std::size_t(n + t) * stride] = u64(y < 0 ? y + q : y);
        }
    }
}

}  // namespace
}  // namespace tg

using namespace tg;

extern "C" int tg_encode_slots(tg_context* ctx, uint64_t* out, const double* v, uint32_t batch, uint32_t n,
                               const double* psi, const uint32_t* rot5, double scale, int level,
                               uint64_t* max_abs_bits, void* stream) {
    TG_REQUIRE(ctx && out && v && psi && rot5, "null argument");
    TG_REQUIRE(n >= 1 && (n & (n - 1)) == 0 && n <= ctx->ring.N / 2, "slot count must be a power of two <= N/2");
    TG_REQUIRE(level >= 0 && u32(level) < ctx->ring.q_count, "level out of range");
    if (batch == 0) return TG_OK;
    DeviceGuard dg(ctx->device);
    cudaStream_t s = as_stream(stream);
    const std::size_t words = std::size_t(batch) * (level + 1) * ctx->ring.N;
    if (ctx->ring.N / (2 * n) > 1) TG_CUDA(cudaMemsetAsync(out, 0, words * 8, s));
    ProfScope ps(ctx, TG_OP_ENCODE, double(words) * 8 + double(batch) * n * 16, s);
    constexpr int VB = 4;
    const dim3 grid((n + kEncThreads - 1) / kEncThreads, (batch + VB - 1) / VB);
    k_encode_slots<VB><<<grid, kEncThreads, 0, s>>>(out, reinterpret_cast<const double2*>(v), batch, n,
                                                    reinterpret_cast<const double2*>(psi), rot5, scale, level,
                                                    reinterpret_cast<unsigned long long*>(max_abs_bits),
                                                    ctx->ring);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
