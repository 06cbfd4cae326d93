// RNS base conversion on the int8 tensor cores (tcgen05.mma.kind::i8), for
// rings whose every modulus takes the FP64 path (q < 1.2 * 2^50: configs 3-5).
// Included by tg_keyswitch.cu inside its anonymous namespace.
//
// Both key-switch conversions are, per coefficient, a small matrix-vector
// product followed by a reduction per target modulus:
//   ModUp   (rlwe.hpp:78-100, UNCORRECTED): out_t = sum_i y_i W_it mod q_t,
//           y_i = x_i (D'/q_i)^-1 mod q_i, W_it = D'/q_i mod q_t;
//   ModDown (rlwe.hpp:555-589, CENTERED):   out_r = x_r P^-1 + sum_s y_s W_sr
//           mod q_r, y_s = centred(x_s (P/p_s)^-1 mod p_s),
//           W_sr = -(P/p_s) P^-1 mod q_r.
// On the FP64 pipe each term costs an exact modular product (~7 DP ops: the
// k_modup_v / k_mod_down_fp kernels run at the FP64 roofline). Here the sum
// over sources is ONE integer GEMM over a coefficient tile:
//   A [128 coefficients][8 * sources] bytes: y_i as a little-endian u64
//     (byte a of source i at column 8i + a; y_i < 2^50, so byte 7 is free:
//     ModDown puts the sign flag neg_s = [y_s < 0] there);
//   B [8 * targets][8 * sources] bytes: row 8t + b, column 8i + a holds byte b
//     of (W_it 2^(8a) mod q_t) for a < 7, and for ModDown's a = 7 byte b of
//     (-p_s W_st mod q_t) (the centred y_s = u_s - p_s neg_s);
//   D [128][8 * targets] s32 in TMEM: c_tb = sum_(i,a) A_(i,a) B_(8t+b,(i,a))
//     (< 112 * 255^2 + 16 * 255 < 2^23 for <= 16 sources, exact), and
//     V_t = sum_b c_tb 2^(8b) == sum_i y_i W_it (mod q_t).
// The epilogue (one thread per coefficient, from TMEM) rebuilds V_t as
// lo + 2^32 hi (lo < 2^47.01, hi < 2^39.01, exact doubles) and reduces it
// exactly on the FP64 pipe: fp_mulmod(hi, 2^32 mod q) (|.| <= q/2 + 2^-15 q)
// + lo, one fp_reduce, canonical -- ~12 DP ops per output instead of ~7 per
// TERM, and the same canonical residues as the reference's u128 arithmetic
// (every step is exact). Operands are K-major SWIZZLE_NONE core matrices
// (8 rows x 16 bytes, LBO = 128 B along K, SBO = 8 * KB between 8-row groups;
// tools/diag/tc_i8_probe.cu checks the convention on the device). B is built
// once per gadget on the host directly in that layout (targets ordered so
// that every level uses a prefix), so a CTA copies it with 16-byte loads.

namespace tc {

__device__ __forceinline__ u64 sdesc(u32 saddr, u32 lbo, u32 sbo) {
    return u64((saddr >> 4) & 0x3FFF) | (u64((lbo >> 4) & 0x3FFF) << 16) | (u64((sbo >> 4) & 0x3FFF) << 32) |
           (u64(1) << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}
// kind::i8 instruction descriptor: D s32, A/B u8, both K-major, M = 128.
__device__ __forceinline__ u32 idesc_u8(u32 n) { return (2u << 4) | ((n >> 3) << 17) | ((128u >> 4) << 24); }

__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mma_u8(u32 tmem, u64 ad, u64 bd, u32 idesc, u32 acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(u64* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bar_init(u64* bar, u32 count = 1) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void bar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void bar_arrive(u64* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// the waiting warp is suspended in try_wait (time hint) instead of spinning
// through issue slots the working warps need
__device__ __forceinline__ void bar_wait(u64* bar, u32 parity) {
    asm volatile(
        "{\n.reg .pred P1;\nTC_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra TC_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// warp-wide
__device__ __forceinline__ void tmem_alloc(u32* slot, u32 ncols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(slot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(u32 taddr, u32 ncols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
// 16 consecutive 32-bit columns of this thread's lane (two targets)
__device__ __forceinline__ void ld16(u32 taddr, u32 (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
// 8 consecutive 32-bit columns of this thread's lane (one target)
__device__ __forceinline__ void ld8(u32 taddr, u32 (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int Nw>
__device__ __forceinline__ void cp_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(Nw) : "memory"); }

__host__ __device__ constexpr u32 tmem_cols(u32 n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

// V = sum_b c_b 2^(8b) (mod q) as an exact double in (-q/2 - 1, q/2 + 1]
// (see the header): r32 = 2^32 mod q, r32q = fl(r32 / q). With c_b < 2^23:
// p0 = c0 + 2^8 c1, p1 = c2 + 2^8 c3, p2 = c4 + 2^8 c5 fit 32 bits, and
// lo = p0 + 2^16 p1 < 2^48.1, hi = p2 + 2^16 c6 < 2^39.1 are formed directly
// as the bit patterns 2^52 + lo, 2^52 + hi (one 32x32+64 multiply-add each
// onto the exponent word 0x433), so V = lo + 2^32 hi.
__device__ __forceinline__ double bits_plus(u32 lo, u32 x) {  // double with bit pattern (0x43300000:lo) + x * 2^16
    u64 r;
    asm("{\n.reg .u32 hw;\nmov.u32 hw, 0x43300000;\nmov.b64 %0, {%1, hw};\nmad.wide.u32 %0, %2, 65536, %0;\n}\n"
        : "=l"(r)
        : "r"(lo), "r"(x));
    return __longlong_as_double(static_cast<long long>(r));
}
__device__ __forceinline__ double recon(const u32* c, double q, double qi, double r32, double r32q) {
    const u32 p0 = c[0] + (c[1] << 8), p1 = c[2] + (c[3] << 8), p2 = c[4] + (c[5] << 8);
    const double lo = __dsub_rn(bits_plus(p0, p1), kTwo52);
    const double hi = __dsub_rn(bits_plus(p2, c[6]), kTwo52);
    return __dadd_rn(fp_mulmod(hi, r32, r32q, q), lo);
}
// integer v in (-q, q) as a double -> canonical u64 in [0, q): q added on the
// FP64 side when negative, then the integer read from the mantissa of
// v + 2^52 (exact for 0 <= v < 2^52)
// (q52 = 2^52 + q: the bit pattern 0x433 | q, no arithmetic)
__device__ __forceinline__ u64 canon_fp(double v, double q52) {
    const double w = __dadd_rn(v, v < 0 ? q52 : kTwo52);
    return static_cast<u64>(__double_as_longlong(w)) & 0x000FFFFFFFFFFFFFull;
}

// Issue the tile's MMAs (one elected thread): D[128][npad] = A[128][KB] B^T,
// N split into <= 256-column chunks.
template <int KB>
__device__ __forceinline__ void issue_tile(u32 tmem, const uint8_t* sa, const uint8_t* sb, u32 npad) {
    constexpr u32 SBO = 8 * KB;
    const u32 a0 = smem_u32(sa), b0 = smem_u32(sb);
    for (u32 nc = 0; nc < npad; nc += 256) {
        const u32 n = min(256u, npad - nc);
        const u32 id = idesc_u8(n);
#pragma unroll
        for (u32 k = 0; k < u32(KB) / 32; ++k)
            mma_u8(tmem + nc, sdesc(a0 + k * 256, 128, SBO), sdesc(b0 + (nc / 8) * SBO + k * 256, 128, SBO), id,
                   k > 0);
    }
}

}  // namespace tc

// Warp-specialised pipeline (one CTA per SM, no CTA-wide barrier in the
// loop), over a contiguous range of the launch's (unit, tile) items:
//   warps 0-7  producers: two threads per coefficient row of the tile (half
//              h = warp / 4 takes the 16-byte chunks kc == h (mod 2)); load
//              the sources (prefetched one item ahead), build the A tile in
//              stage i & 1, fence to the async proxy, arrive on a_full;
//   warp  8    MMA: waits a_full and tmem_empty, (re)loads B and the stage's
//              epilogue constants when the digit changes, issues the tile's
//              tcgen05.mma into TMEM stage i & 1, commits to a_empty and
//              tmem_full (+ an explicit arrive releasing the constants);
//   warps 9-20 epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 and the
//              target pairs g == (w - 9) / 4 (mod 3); waits tmem_full,
//              rebuilds and reduces its outputs, stores them, arrives on
//              tmem_empty.
// Two A tiles and two TMEM accumulators of 256 columns: the MMA of item i+1
// and the A tile of item i+2 overlap item i's epilogue.
constexpr u32 kTcProd = 8, kTcEpi = 12, kTcWarps = kTcProd + 1 + kTcEpi, kTcThreads = 32 * kTcWarps;
constexpr u32 kTcEpq = kTcEpi / 4;  // epilogue warps per TMEM lane quadrant

constexpr u32 kTcAStages = 4;  // A tiles in flight (producers run up to 4 items ahead)
struct TcBars {  // mbarriers (shared memory)
    u64 a_full[kTcAStages], a_empty[kTcAStages], t_full[2], t_empty[2], drain;
    u32 tmem;
};
__device__ __forceinline__ void tc_init_bars(TcBars* b) {
    for (u32 s = 0; s < kTcAStages; ++s) {
        tc::bar_init(&b->a_full[s], 32 * kTcProd);
        tc::bar_init(&b->a_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
        tc::bar_init(&b->t_full[s], 2);
        tc::bar_init(&b->t_empty[s], kTcEpi);
    }
    tc::bar_init(&b->drain, 1);
    tc::bar_init_fence();
}

// Shared-memory plan: [kTcAStages] A tiles | B (npad x KB) | TcBars | [2]
// per-stage epilogue constants (cons words) | [2] per-stage output row
// offsets (u32).
template <int KB>
struct TcPlan {
    static constexpr u32 A_BYTES = 128 * KB;
    u32 npad, cons;  // B rows; constant words per stage
    __host__ __device__ size_t b_off() const { return kTcAStages * size_t(A_BYTES); }
    __host__ __device__ size_t bars_off() const { return b_off() + size_t(npad) * KB; }
    __host__ __device__ size_t cons_off() const { return bars_off() + (sizeof(TcBars) + 15) / 16 * 16; }
    __host__ __device__ size_t rows_off() const { return cons_off() + 2 * size_t(cons) * 8; }
    __host__ __device__ size_t bytes() const { return rows_off() + 2 * size_t(npad / 8) * 4 + 16; }
};

template <int KB>
__device__ __forceinline__ void tc_store_a_row(uint8_t* at, u32 m, u32 kc, u64 y0, u64 y1) {
    *reinterpret_cast<ulonglong2*>(at + (m >> 3) * (8 * KB) + kc * 128 + (m & 7) * 16) = make_ulonglong2(y0, y1);
}

// ModUp: unit = j * npolys + bsrc (digit-major: B, which depends on the
// digit, changes only with the digit). Writes every digit's level+1+K rows:
// own-group rows copied (eval form when d_eval is given), the others
// converted.
template <int KB, bool RAW = false, bool RAWIN = false>
__global__ void __launch_bounds__(kTcThreads, 1)
k_modup_tc(DevRing R, GadgetDev G, u64* __restrict__ digits, const u64* __restrict__ d, int level,
           const u64* __restrict__ d_eval, u32 nd, u32 npolys, u32 per_cta, u32 npad_max) {
    constexpr u32 SL = KB / 8;  // source slots of an A row
    const u32 N = R.N, lvl = u32(level), K = R.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u32 gs = G.group_size, tiles = N / 128, total = nd * npolys * tiles;
    const size_t in_words = size_t(lvl + 1) * N, dig_words = size_t(lvl + 1 + K) * N;
    const TcPlan<KB> P{npad_max, npad_max / 2};  // 4 words per target
    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t* sa = tsm;
    uint8_t* sb = tsm + P.b_off();
    TcBars* bars = reinterpret_cast<TcBars*>(tsm + P.bars_off());
    u64* scons = reinterpret_cast<u64*>(tsm + P.cons_off());  // [2][npad/8][4]
    u32* srow = reinterpret_cast<u32*>(tsm + P.rows_off());   // [2][npad/8]
    const u32 i0 = blockIdx.x * per_cta, i_end = min(total, i0 + per_cta);
    if (i0 >= i_end) return;
    const u32 nitems = i_end - i0;
    if (tid == 0) tc_init_bars(bars);
    if (warp == kTcProd) tc::tmem_alloc(&bars->tmem, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const u32 tmem = bars->tmem;
    // item i (0-based in this CTA) -> (tile, source poly, digit), division-free
    const u32 tl0 = i0 % tiles, bs0 = (i0 / tiles) % npolys, j0 = i0 / tiles / npolys;
    auto advance = [&](u32& t_, u32& b_, u32& j_) {
        if (++t_ == tiles) {
            t_ = 0;
            if (++b_ == npolys) {
                b_ = 0;
                ++j_;
            }
        }
    };
    if (warp < kTcProd) {
        // ---------------- producers ----------------
        constexpr u32 HS = (SL + 3) / 4 * 2;  // source slots per half (chunks kc == h mod 2)
        const u32 m = tid & 127, h = tid >> 7;  // tile row, half
        auto slot = [&](u32 u) { return 2 * (2 * (u >> 1) + h) + (u & 1); };  // u-th slot of this half
        u32 tl = tl0, bs = bs0, j = j0;
        constexpr bool kPE = HS <= 4;  // own-group eval rows prefetched too (registers)
        u64 xs[HS], xe[kPE ? HS : 1];
        auto load = [&](u32 t_, u32 b_, u32 j_) {
            const u32 first = j_ * gs, A = min(gs, lvl + 1 - first);
            const size_t o = b_ * in_words + size_t(first) * N + t_ * 128 + m;
#pragma unroll
            for (u32 u = 0; u < HS; ++u)
                if (slot(u) < A) {
                    xs[u] = d[o + size_t(slot(u)) * N];
                    if (kPE && d_eval) xe[kPE ? u : 0] = d_eval[o + size_t(slot(u)) * N];
                }
        };
        load(tl, bs, j);
        for (u32 it = 0; it < nitems; ++it) {
            const u32 as = it % kTcAStages, ause = it / kTcAStages;
            const u32 first = j * gs, A = min(gs, lvl + 1 - first);
            // source constants (x N^-1 for raw inverse-NTT sources, RAWIN)
            const u64* sconst = G.tc_mu_c + size_t(j * gs + A - 1) * G.tc_mu_cstride + size_t(G.tc_tall) * 4 +
                                (RAWIN ? size_t(gs) * 2 : 0);
            const size_t off = (size_t(bs) * nd + j) * dig_words + tl * 128 + m;
            tc::bar_wait(&bars->a_empty[as], (ause & 1) ^ 1);
            uint8_t* at = sa + as * TcPlan<KB>::A_BYTES;
#pragma unroll
            for (u32 kk = 0; kk < HS / 2; ++kk) {
                const u32 kc = 2 * kk + h;
                if (kc >= KB / 16) break;
                u64 y[2];
#pragma unroll
                for (u32 s2 = 0; s2 < 2; ++s2) {
                    const u32 u = 2 * kk + s2, i = 2 * kc + s2;
                    y[s2] = 0;
                    if (i < A) {
                        const u32 s = first + i;
                        digits[off + size_t(s) * N] =  // own-group row
                            !d_eval ? xs[u]
                            : kPE   ? xe[kPE ? u : 0]
                                    : d_eval[size_t(bs) * in_words + size_t(s) * N + tl * 128 + m];
                        const double q = u2d(R.q[s]);
                        const double xv = RAWIN ? __longlong_as_double(static_cast<long long>(xs[u])) : u2d(xs[u]);
                        double v = fp_mulmod(xv, __longlong_as_double(static_cast<long long>(__ldg(sconst + 2 * i))),
                                             __longlong_as_double(static_cast<long long>(__ldg(sconst + 2 * i + 1))), q);
                        if (v < 0) v = __dadd_rn(v, q);
                        y[s2] = d2u(v);
                    }
                }
                tc_store_a_row<KB>(at, m, kc, y[0], y[1]);
            }
            tc::fence_async_smem();
            tc::bar_arrive(&bars->a_full[as]);
            advance(tl, bs, j);
            if (it + 1 < nitems) load(tl, bs, j);  // in flight while the next stage frees up
        }
    } else if (warp == kTcProd) {
        // ---------------- MMA issuer ----------------
        u32 tl = tl0, bs = bs0, j = j0, bj = ~0u, dph = 0;
        u32 held0 = ~0u, held1 = ~0u;  // digit whose constants each stage holds
        for (u32 it = 0; it < nitems; ++it) {
            const u32 st = it & 1, use = it >> 1;
            const u32 first = j * gs, A = min(gs, lvl + 1 - first), T = K + lvl + 1 - A, npad = (T + 1) / 2 * 16;
            const u32 combo = j * gs + A - 1;
            if (j != bj) {  // B of this digit: every issued MMA must have completed first
                if (it > 0) {
                    if (lane == 0) tc::commit(&bars->drain);
                    __syncwarp();
                    tc::bar_wait(&bars->drain, dph);
                    dph ^= 1;
                }
                const uint8_t* Bg = G.tc_mu_b + size_t(combo) * G.tc_mu_bstride;
                for (u32 e = lane; e < npad * KB / 16; e += 32) tc::cp16(sb + 16 * e, Bg + 16 * e);
                tc::cp_wait_all();
                tc::fence_async_smem();
                __syncwarp();
                bj = j;
            }
            tc::bar_wait(&bars->t_empty[st], (use & 1) ^ 1);  // the epilogue of item it-2 is done
            if ((st ? held1 : held0) != j) {  // this stage's epilogue constants and output rows
                const u64* Cg = G.tc_mu_c + size_t(combo) * G.tc_mu_cstride;
                u64* sc = scons + size_t(st) * P.cons * 1;
                for (u32 e = lane; e < npad / 8 * 4; e += 32) sc[e] = __ldg(Cg + e);
                u32* sr = srow + st * (npad_max / 8);
                for (u32 v = lane; v < T; v += 32)  // target order: the K specials, then the q rows outside the group
                    sr[v] = (v < K ? lvl + 1 + v : (v - K < first ? v - K : v - K + A)) * N * 8;  // bytes
                (st ? held1 : held0) = j;
                __syncwarp();  // every lane's constants before lane 0's releasing arrive
            }
            const u32 as = it % kTcAStages, ause = it / kTcAStages;
            tc::bar_wait(&bars->a_full[as], ause & 1);
            tc::fence_after();
            if (lane == 0) {
                tc::issue_tile<KB>(tmem + st * 256, sa + as * TcPlan<KB>::A_BYTES, sb, npad);
                tc::commit(&bars->a_empty[as]);
                tc::commit(&bars->t_full[st]);
                tc::bar_arrive(&bars->t_full[st]);  // releases the constants written above
            }
            __syncwarp();
            advance(tl, bs, j);
        }
    } else {
        // ---------------- epilogue ----------------
        const u32 ew = warp - kTcProd - 1, quad = warp & 3, sub = ew >> 2;  // sub < kTcEpq
        const u32 tbase = tmem + ((quad * 32) << 16);
        const u32 m = quad * 32 + lane;
        u32 tl = tl0, bs = bs0, j = j0;
        for (u32 it = 0; it < nitems; ++it) {
            const u32 st = it & 1, use = it >> 1;
            const u32 A = min(gs, lvl + 1 - j * gs), T = K + lvl + 1 - A, NG2 = (T + 1) / 2;
            u64* dig = digits + (size_t(bs) * nd + j) * dig_words + tl * 128 + m;
            const u64* sc = scons + size_t(st) * P.cons;
            const u32* sr = srow + st * (npad_max / 8);
            tc::bar_wait(&bars->t_full[st], use & 1);
            tc::fence_after();
            for (u32 g = sub; g < NG2; g += kTcEpq) {
                u32 r[16];
                tc::ld16(tbase + st * 256 + g * 16, r);
                tc::ld_wait();
#pragma unroll
                for (u32 k = 0; k < 2; ++k) {
                    const u32 v = 2 * g + k;
                    if (k && v >= T) break;
                    const ulonglong2 c01 = *reinterpret_cast<const ulonglong2*>(sc + 4 * v);
                    const double2 c23 = *reinterpret_cast<const double2*>(sc + 4 * v + 2);
                    const double q52 = __longlong_as_double(static_cast<long long>(0x4330000000000000ull | c01.x));
                    const double q = __dsub_rn(q52, kTwo52), qi = __longlong_as_double(static_cast<long long>(c01.y));
                    const double acc = tc::recon(r + 8 * k, q, qi, c23.x, c23.y);
                    const double red = fp_reduce(acc, q, qi);  // |.| <= q/2 + 1
                    *reinterpret_cast<u64*>(reinterpret_cast<char*>(dig) + sr[v]) =
                        RAW ? static_cast<u64>(__double_as_longlong(red)) : tc::canon_fp(red, q52);
                }
            }
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::bar_arrive(&bars->t_empty[st]);
            advance(tl, bs, j);
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == kTcProd) tc::tmem_dealloc(tmem, 512);
}

// ModDown of npolys polys (level+1+K rows each, back to back) into level+1
// rows each (+ addend); unit = poly. RAW: inputs are raw inverse-NTT doubles
// (|v| <= 0.6q) and the input constants carry N^-1 (k_mod_down_fp<K, true>).
// B and the constants do not depend on the unit: loaded once.
template <int KB, bool RAW>
__global__ void __launch_bounds__(kTcThreads, 1)
k_mod_down_tc(DevRing R, GadgetDev G, u64* __restrict__ out, const u64* __restrict__ in, int level,
              const u64* __restrict__ addend, u32 npolys, u32 per_cta) {
    constexpr u32 SL = KB / 8;
    constexpr u32 VT = 6;  // target pairs per epilogue warp (T <= 32: 16 pairs over 3 warps per quadrant)
    const u32 N = R.N, lvl = u32(level), K = R.K, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const u32 rin = lvl + 1 + K, T = lvl + 1, NG2 = (T + 1) / 2, npad = NG2 * 16;
    const u32 tiles = N / 128, total = npolys * tiles;
    auto in_d = [](u64 x) { return RAW ? __longlong_as_double(static_cast<long long>(x)) : u2d(x); };
    const TcPlan<KB> P{npad, npad};  // 8 words per target, one set
    extern __shared__ __align__(1024) uint8_t tsm[];
    uint8_t* sa = tsm;
    uint8_t* sb = tsm + P.b_off();
    TcBars* bars = reinterpret_cast<TcBars*>(tsm + P.bars_off());
    u64* sc = reinterpret_cast<u64*>(tsm + P.cons_off());  // [npad/8][8]
    u64* xsm = reinterpret_cast<u64*>(tsm + (P.bytes() + 15) / 16 * 16);  // epilogue input buffers
    const u32 i0 = blockIdx.x * per_cta, i_end = min(total, i0 + per_cta);
    if (i0 >= i_end) return;
    const u32 nitems = i_end - i0;
    for (u32 e = tid; e < npad * KB / 16; e += kTcThreads) tc::cp16(sb + 16 * e, G.tc_md_b + 16 * e);
    for (u32 e = tid; e < npad / 2; e += kTcThreads) tc::cp16(sc + 2 * e, G.tc_md_c + 2 * e);
    tc::cp_wait_all();
    tc::fence_async_smem();
    if (tid == 0) tc_init_bars(bars);
    if (warp == kTcProd) tc::tmem_alloc(&bars->tmem, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const u32 tmem = bars->tmem;
    const u32 tl0 = i0 % tiles, p0 = i0 / tiles;
    if (warp < kTcProd) {
        // ---------------- producers ----------------
        constexpr u32 HS = (SL + 3) / 4 * 2;
        const u32 m = tid & 127, h = tid >> 7;
        auto slot = [&](u32 u) { return 2 * (2 * (u >> 1) + h) + (u & 1); };
        const double* tab = RAW ? G.mdfn : G.mdf;
        u32 tl = tl0, p = p0;
        u64 xs[HS];
        auto load = [&](u32 t_, u32 p_) {
            const u64* src = in + (size_t(p_) * rin + lvl + 1) * N + t_ * 128 + m;
#pragma unroll
            for (u32 u = 0; u < HS; ++u)
                if (slot(u) < K) xs[u] = src[size_t(slot(u)) * N];
        };
        load(tl, p);
        for (u32 it = 0; it < nitems; ++it) {
            const u32 as = it % kTcAStages, ause = it / kTcAStages;
            tc::bar_wait(&bars->a_empty[as], (ause & 1) ^ 1);
            uint8_t* at = sa + as * TcPlan<KB>::A_BYTES;
#pragma unroll
            for (u32 kk = 0; kk < HS / 2; ++kk) {
                const u32 kc = 2 * kk + h;
                if (kc >= KB / 16) break;
                u64 y[2];
#pragma unroll
                for (u32 s2 = 0; s2 < 2; ++s2) {
                    const u32 s = 2 * kc + s2, u = 2 * kk + s2;
                    y[s2] = 0;
                    if (s < K) {
                        const double ps = __ldg(tab + 4 * s), cq = __ldg(tab + 4 * s + 1), cw = __ldg(tab + 4 * s + 2),
                                     half = __ldg(tab + 4 * s + 3);
                        double v = fp_mulmod(in_d(xs[u]), cw, cq, ps);  // |v| <= 0.58 p
                        if (v < 0) v = __dadd_rn(v, ps);
                        y[s2] = d2u(v) | (u64(v > half) << 56);  // sign of the centred value in byte 7
                    }
                }
                tc_store_a_row<KB>(at, m, kc, y[0], y[1]);
            }
            tc::fence_async_smem();
            tc::bar_arrive(&bars->a_full[as]);
            if (++tl == tiles) {
                tl = 0;
                ++p;
            }
            if (it + 1 < nitems) load(tl, p);
        }
    } else if (warp == kTcProd) {
        // ---------------- MMA issuer ----------------
        for (u32 it = 0; it < nitems; ++it) {
            const u32 st = it & 1, use = it >> 1;
            tc::bar_wait(&bars->t_empty[st], (use & 1) ^ 1);
            const u32 as = it % kTcAStages, ause = it / kTcAStages;
            tc::bar_wait(&bars->a_full[as], ause & 1);
            tc::fence_after();
            if (lane == 0) {
                tc::issue_tile<KB>(tmem + st * 256, sa + as * TcPlan<KB>::A_BYTES, sb, npad);
                tc::commit(&bars->a_empty[as]);
                tc::commit(&bars->t_full[st]);
                tc::bar_arrive(&bars->t_full[st]);
            }
            __syncwarp();
        }
    } else {
        // ---------------- epilogue ----------------
        const u32 ew = warp - kTcProd - 1, quad = warp & 3, sub = ew >> 2;  // sub < kTcEpq
        const u32 tbase = tmem + ((quad * 32) << 16);
        const u32 m = quad * 32 + lane;
        const u32 po = RAW ? 6 : 4;  // P^-1 (N^-1) constant pair in the target table
        // this warp's q-row inputs and addends (rows 2g, 2g + 1 of g = sub +
        // 3e; 32 coefficients each), double-buffered in shared memory: the
        // next item's rows load (cp.async) while this item's are reduced
        u64* xbuf = xsm + size_t(ew) * 2 * (4 * VT) * 32;  // [2][2 VT rows x (input, addend)][32]
        const bool has_add = addend != nullptr;
        auto fetch = [&](u32 t_, u32 p_, u32 b) {
            const size_t cbase = t_ * 128 + quad * 32 + 2 * (lane & 15);
            const u64* inp = in + size_t(p_) * rin * N + cbase;
            const u64* addp = has_add ? addend + size_t(p_) * T * N + cbase : nullptr;
            u64* dst = xbuf + size_t(b) * (4 * VT) * 32 + 2 * (lane & 15);
#pragma unroll
            for (u32 e = 0; e < VT; ++e) {
                const u32 g = sub + kTcEpq * e;
                if (g < NG2) {
                    const u32 row = min(2 * g + (lane >> 4), T - 1);  // half-warp per row of the pair
                    tc::cp16(dst + (4 * e + (lane >> 4)) * 32, inp + size_t(row) * N);
                    if (has_add) tc::cp16(dst + (4 * e + 2 + (lane >> 4)) * 32, addp + size_t(row) * N);
                }
            }
            tc::cp_commit();
        };
        u32 tl = tl0, p = p0;
        fetch(tl, p, 0);
        for (u32 it = 0; it < nitems; ++it) {
            const u32 st = it & 1, use = it >> 1;
            const u32 c = tl * 128 + m;
            u64* outp = out + size_t(p) * T * N + c;
            u32 ntl = tl + 1, np = p;
            if (ntl == tiles) {
                ntl = 0;
                ++np;
            }
            if (it + 1 < nitems) fetch(ntl, np, st ^ 1);
            else tc::cp_commit();  // (an empty group keeps the wait count uniform)
            tc::cp_wait_group<1>();
            __syncwarp();
            const u64* xb = xbuf + size_t(st) * (4 * VT) * 32 + lane;
            tc::bar_wait(&bars->t_full[st], use & 1);
            tc::fence_after();
#pragma unroll
            for (u32 e = 0; e < VT; ++e) {
                const u32 g = sub + kTcEpq * e;
                if (g >= NG2) break;
                u32 r[16];
                tc::ld16(tbase + st * 256 + g * 16, r);
                tc::ld_wait();
#pragma unroll
                for (u32 k = 0; k < 2; ++k) {
                    const u32 row = 2 * g + k;
                    if (k && row >= T) break;
                    const u64* cv = sc + 8 * row;
                    const ulonglong2 c01 = *reinterpret_cast<const ulonglong2*>(cv);
                    const double2 c23 = *reinterpret_cast<const double2*>(cv + 2);
                    const double2 cp = *reinterpret_cast<const double2*>(cv + po);
                    const double q52 = __longlong_as_double(static_cast<long long>(0x4330000000000000ull | c01.x));
                    const double q = __dsub_rn(q52, kTwo52), qi = __longlong_as_double(static_cast<long long>(c01.y));
                    const double conv = tc::recon(r + 8 * k, q, qi, c23.x, c23.y);
                    const double xt = fp_mulmod(in_d(xb[(4 * e + k) * 32]), cp.x, cp.y, q);
                    u64 o = tc::canon_fp(fp_reduce(__dadd_rn(xt, conv), q, qi), q52);  // |sum| < 1.1q + 2^47
                    if (has_add) o = add_mod(o, xb[(4 * e + 2 + k) * 32], c01.x);
                    outp[size_t(row) * N] = o;
                }
            }
            tc::fence_before();
            __syncwarp();  // (also: every lane is done with this buffer before it is refilled)
            if (lane == 0) tc::bar_arrive(&bars->t_empty[st]);
            tl = ntl;
            p = np;
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == kTcProd) tc::tmem_dealloc(tmem, 512);
}

// Items per CTA: one CTA per SM.
inline u32 tc_items_per_cta(u32 total, int sms) { return (total + u32(sms) - 1) / u32(sms); }
// One accumulator stage holds npad <= 256 columns; ModDown epilogue warps
// hold at most 4 target pairs each (T <= 32).
inline bool tc_modup_fits(u32 K, int level, u32 gs, u32 nd) {
    const u32 amin = std::min(gs, u32(level) + 1 - (nd - 1) * gs);
    return (K + u32(level) + 2 - amin) / 2 * 16 <= 256;
}
inline bool tc_mod_down_fits(int level) { return level + 1 <= 32; }

template <int KB>
void launch_modup_tc(const DevRing& R, const GadgetDev& G, int sms, u64* digits, const u64* d, int level, u32 nd,
                     const u64* d_eval, u32 npolys, cudaStream_t s, bool raw = false, bool raw_in = false) {
    const u32 gs = G.group_size, amin = std::min(gs, u32(level) + 1 - (nd - 1) * gs);
    const u32 npad_max = (R.K + u32(level) + 2 - amin) / 2 * 16;
    const TcPlan<KB> P{npad_max, npad_max / 2};
    static const bool attr = [] {  // thread-safe one-time init per instantiation
        cudaFuncSetAttribute(k_modup_tc<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k_modup_tc<KB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k_modup_tc<KB, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        cudaFuncSetAttribute(k_modup_tc<KB, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        return true;
    }();
    (void)attr;
    const u32 total = nd * npolys * (R.N / 128), per = tc_items_per_cta(total, sms);
    const u32 nb = (total + per - 1) / per;
    if (raw_in && raw)
        k_modup_tc<KB, true, true><<<nb, kTcThreads, P.bytes(), s>>>(R, G, digits, d, level, d_eval, nd, npolys, per,
                                                                     npad_max);
    else if (raw_in)
        k_modup_tc<KB, false, true><<<nb, kTcThreads, P.bytes(), s>>>(R, G, digits, d, level, d_eval, nd, npolys, per,
                                                                      npad_max);
    else if (raw)
        k_modup_tc<KB, true><<<(total + per - 1) / per, kTcThreads, P.bytes(), s>>>(R, G, digits, d, level, d_eval,
                                                                                    nd, npolys, per, npad_max);
    else
        k_modup_tc<KB><<<(total + per - 1) / per, kTcThreads, P.bytes(), s>>>(R, G, digits, d, level, d_eval, nd,
                                                                              npolys, per, npad_max);
}

// false: the plan does not fit shared memory (the caller falls back)
template <int KB, bool RAW>
bool launch_mod_down_tc(const DevRing& R, const GadgetDev& G, int sms, u64* out, const u64* in, int level,
                        u32 npolys, const u64* addend, cudaStream_t s) {
    const u32 T = u32(level) + 1, npad = (T + 1) / 2 * 16;
    const TcPlan<KB> P{npad, npad};
    const size_t smem = (P.bytes() + 15) / 16 * 16 + size_t(kTcEpi) * 2 * 24 * 32 * 8;  // + epilogue input buffers
    if (smem > size_t(227) * 1024) return false;
    static const bool attr = [] {
        cudaFuncSetAttribute(k_mod_down_tc<KB, RAW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        return true;
    }();
    (void)attr;
    const u32 total = npolys * (R.N / 128), per = tc_items_per_cta(total, sms);
    k_mod_down_tc<KB, RAW><<<(total + per - 1) / per, kTcThreads, smem, s>>>(R, G, out, in, level, addend, npolys,
                                                                           per);
    return true;
}
