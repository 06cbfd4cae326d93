// Column phase with column PAIRS (included by tg_ntt.cu after tg_ntt_warp.cuh,
// inside the anonymous namespace). Used when every row of a launch takes the
// FP64 path.
//
// kw_fwd_cols / kw_inv_cols give each warp one 256-point column of two polys
// (interleaved transforms), so every global and shared access is 8 bytes:
// the column tile needs 8 LDGSTS + 8 LDS + 8 STG per thread and poly, and the
// MIO queue throttles (ncu: mio_throttle second-largest stall). Here a warp
// owns two ADJACENT columns of one poly, stored as 16-byte pairs (layout
// below). Then
//   * the tile moves with 16-byte cp.async / stores (a row segment of 16
//     columns is 128 contiguous bytes), half the instructions;
//   * the warp reads and writes its two columns as one 16-byte access per
//     element, and every exchange moves (v0, v1) pairs: half the shared-memory
//     instructions, all conflict-free (swizzled tile);
//   * the two columns share every staged twiddle (the column phase's
//     twiddles do not depend on the column), as the two polys did.
// Same stages, same bounds, same outputs as the one-column kernels.

// Tile layout: M rows x 8 column pairs of 16 bytes, row-major, with the pair
// index XOR-swizzled per row: element k of warp w's pair sits in 16-byte unit
//   U(k, w) = 8k + (w ^ f(k)),  f(k) = (k ^ (k >> 3)) & 7.
// A row's 8 units stay one contiguous 128-byte block (the 16-byte cp.async
// fill of a row is contiguous on both sides: LDGSTS with scattered
// destinations costs one wavefront per lane, ncu), and for every
// lane -> element pattern of the radix-8 stage blocks (layouts 5, 3, 2, 0:
// k = l + 32j, 8j + l, 32(l/4) + 4j + l%4, 8l + j) the 8 lanes of a 16-byte
// access phase hit 8 distinct bank groups. E = 8 (N = 2^16) only.
__device__ __forceinline__ u32 pu(u32 k, u32 w) { return 8 * k + (w ^ ((k ^ (k >> 3)) & 7)); }

template <int E>
struct PGeo {
    static constexpr int M = WGeo<E>::M;
};

// pair exchange: both columns' values of element k move as one 16-byte word
template <int E>
__device__ __forceinline__ void wxchg_pair(double (&v)[2][E], double2* tile, u32 w, u32 lane, u32 lo_from,
                                           u32 lo_to) {
    constexpr int LOGE = WGeo<E>::LOGE;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) tile[pu(wins<LOGE>(lane, u32(j), lo_from), w)] = make_double2(v[0][j], v[1][j]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const double2 t = tile[pu(wins<LOGE>(lane, u32(j), lo_to), w)];
        v[0][j] = t.x;
        v[1][j] = t.y;
    }
}

template <int E>
__device__ __forceinline__ void wfwd_all_pair(double (&v)[2][E], double2* pr, u32 pw, u32 lane, const u64* sw,
                                              double q, double qi) {
    if constexpr (E == 8) {
        wfwd_fp<2, 8, false, 5, 7, 5, false>(v, lane, sw, q, qi, 0);
        wxchg_pair<8>(v, pr, pw, lane, 5, 2);
        wfwd_fp<2, 8, false, 2, 4, 2>(v, lane, sw, q, qi, 0);
        wxchg_pair<8>(v, pr, pw, lane, 2, 0);
        wfwd_fp<2, 8, false, 0, 1, 0>(v, lane, sw, q, qi, 0);
    } else {
        wfwd_fp<2, 4, false, 5, 6, 5, false>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 5, 3);
        wfwd_fp<2, 4, false, 3, 4, 3, false>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 3, 1);
        wfwd_fp<2, 4, false, 1, 2, 1>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 1, 0);
        wfwd_fp<2, 4, false, 0, 0, 0>(v, lane, sw, q, qi, 0);
    }
}

template <int E>
__device__ __forceinline__ void winv_all_pair(double (&v)[2][E], double2* pr, u32 pw, u32 lane, const u64* sw,
                                              double q, double qi) {
    if constexpr (E == 8) {
        winv_fp<2, 8, false, 0, 0, 2>(v, lane, sw, q, qi, 0);
        wxchg_pair<8>(v, pr, pw, lane, 0, 3);
        winv_fp<2, 8, false, 3, 3, 5>(v, lane, sw, q, qi, 0);
        wxchg_pair<8>(v, pr, pw, lane, 3, 5);
        winv_fp<2, 8, false, 5, 6, 7>(v, lane, sw, q, qi, 0);
    } else {
        winv_fp<2, 4, false, 0, 0, 1>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 0, 2);
        winv_fp<2, 4, false, 2, 2, 3>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 2, 4);
        winv_fp<2, 4, false, 4, 4, 5>(v, lane, sw, q, qi, 0);
        wxchg_pair<4>(v, pr, pw, lane, 4, 5);
        winv_fp<2, 4, false, 5, 6, 6>(v, lane, sw, q, qi, 0);
    }
}

// 16-column tile of the row at rb (row base + first column), M rows at
// stride N2: thread t moves column pair w = t%8 of rows m = t/8 + 32i. With
// m0 = t/8 < 32, f(m0 + 32i) = f(m0) ^ 4(i&1), so even and odd i have one
// base address each and compile-time offsets (512 units per 2i).
template <int OS, int OG>
__device__ __forceinline__ void cp_async16_imm(u32 sa, const u64* g) {
    asm volatile("cp.async.cg.shared.global [%0+%2], [%1+%3], 16;\n" ::"r"(sa), "l"(g), "n"(OS), "n"(OG) : "memory");
}
template <int N2, int... I>
__device__ __forceinline__ void issue_pair_elems(u32 sa0, u32 sa1, const u64* g, std::integer_sequence<int, I...>) {
    ((I & 1 ? cp_async16_imm<(I / 2) * 512 * 16, I * 32 * N2 * 8>(sa1, g)
            : cp_async16_imm<(I / 2) * 512 * 16, I * 32 * N2 * 8>(sa0, g)),
     ...);
}
template <int E, int N2>
__device__ __forceinline__ void issue_pair_tile(double2* tile, const u64* rb) {
    using Pg = PGeo<E>;
    const u32 t = threadIdx.x, w = t & 7, m0 = t >> 3;
    const u32 sa0 = static_cast<u32>(__cvta_generic_to_shared(tile + pu(m0, w)));
    const u32 sa1 = static_cast<u32>(__cvta_generic_to_shared(tile + pu(m0 + 32, w)));
    issue_pair_elems<N2>(sa0, sa1, rb + size_t(m0) * N2 + 2 * w, std::make_integer_sequence<int, Pg::M / 32>{});
    cp_async_commit();
}
template <int E, int N2>
__device__ __forceinline__ void store_pair_tile(const double2* tile, u64* rb) {
    using Pg = PGeo<E>;
    const u32 t = threadIdx.x, w = t & 7, m0 = t >> 3;
    const double2* s0 = tile + pu(m0, w);
    const double2* s1 = tile + pu(m0 + 32, w);
    ulonglong2* g = reinterpret_cast<ulonglong2*>(rb + size_t(m0) * N2 + 2 * w);
#pragma unroll
    for (int i = 0; i < Pg::M / 32; ++i) {
        const double2 v = (i & 1 ? s1 : s0)[(i / 2) * 512];
        g[size_t(i) * 32 * N2 / 2] = make_ulonglong2(static_cast<u64>(__double_as_longlong(v.x)),
                                                     static_cast<u64>(__double_as_longlong(v.y)));
    }
}

#ifndef NTT_PAIR_PREFETCH
#define NTT_PAIR_PREFETCH 1  // two tiles: the next poly's tile loads during the current transform
#endif
template <int E>
constexpr size_t pair_smem() {  // column-pair tile(s) + column twiddles
    return size_t(16) * 8 * PGeo<E>::M * (NTT_PAIR_PREFETCH ? 2 : 1) + size_t(8) * 2 * WGeo<E>::TW_COL;
}

// Phase 1 forward (all rows FP64): 16 columns x M1 rows per poly, stages
// 0 .. log M1 - 1; canonical u64 in, doubles (|v| <= q/2 + 1, raw bits) out.
template <int E, int E2>
__global__ void __launch_bounds__(256, NTT_MIN_BLOCKS)
kw_fwd_cols2(DevRing R, u64* data, const u64* src, u32 rpp, u32 npolys, u32 ppb, int level, u32 skip_gs,
             u32 row0) {
    using Pg = PGeo<E>;
    constexpr u32 N = 32 * E * 32 * E2, N2 = 32 * E2;  // == R.N (warp_plan)
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = next_poly(blockIdx.z * ppb, pend, r, rpp, level, skip_gs);
    if (p >= pend) return;
    extern __shared__ __align__(16) u64 dyn[];
    constexpr u32 NT = NTT_PAIR_PREFETCH ? 2 : 1;
    u64* sw = dyn + 16 * Pg::M * NT;  // after the M x 8 units of each tile
    const u32 mi = mod_index(r, level, R.q_count);
    const u64* w = reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N);
    const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
    const u64 qq = R.q[mi];
    const bool raw = (skip_gs & kTgRawDigits) != 0;
    const u32 c0 = blockIdx.x * 16;
    issue_pair_tile<E, N2>(reinterpret_cast<double2*>(dyn), src + size_t(p * rpp + r) * N + c0);
    stage_col_twiddles<E, true>(sw, nullptr, w, w + N);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (u32 cur = 0, first = 1; p < pend; first = 0) {
        const u32 pn = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        double2* tile = reinterpret_cast<double2*>(dyn) + cur * 8 * Pg::M;
        if constexpr (NT == 2) {
            if (pn < pend) {  // next poly's tile in flight during this transform
                issue_pair_tile<E, N2>(reinterpret_cast<double2*>(dyn) + (cur ^ 1) * 8 * Pg::M,
                                       src + size_t(pn * rpp + r) * N + c0);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
        } else {
            if (!first) issue_pair_tile<E, N2>(tile, src + size_t(p * rpp + r) * N + c0);
            cp_async_wait<0>();
        }
        (void)first;
        double2* pr = tile;
        __syncthreads();
        double v[2][E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const double2 t = pr[pu(lane + 32 * j, warp)];
            if (raw) {  // ModUp's centred doubles (|v| <= q/2 + 1, the bound c2d gives)
                v[0][j] = t.x;
                v[1][j] = t.y;
            } else {
                v[0][j] = c2d(static_cast<u64>(__double_as_longlong(t.x)), qq);
                v[1][j] = c2d(static_cast<u64>(__double_as_longlong(t.y)), qq);
            }
        }
        wfwd_all_pair<E>(v, pr, warp, lane, sw, qd, qi);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < E; ++j) pr[pu((lane << WGeo<E>::LOGE) | j, warp)] = make_double2(v[0][j], v[1][j]);
        __syncthreads();
        store_pair_tile<E, N2>(tile, data + size_t(p * rpp + r) * N + c0);
        __syncthreads();  // the tile is the next prefetch target
        p = pn;
        cur ^= (NT - 1);
    }
}

// Phase B inverse (all rows FP64): phase-A doubles in, N^-1 and canonical out
// (RAW: the raw doubles out, |v| <= 0.6q, for a consumer that folds N^-1 into
// its own constants: the key switch's ModDown, k_mod_down_fp<K, true>).
template <int E, int E2, bool RAW = false>
__global__ void __launch_bounds__(256, NTT_MIN_BLOCKS)
kw_inv_cols2(DevRing R, u64* data, u32 rpp, u32 npolys, u32 ppb, int level, u32 row0) {
    using Pg = PGeo<E>;
    constexpr u32 N = 32 * E * 32 * E2, N2 = 32 * E2;
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = blockIdx.z * ppb;
    if (p >= pend) return;
    extern __shared__ __align__(16) u64 dyn[];
    constexpr u32 NT = NTT_PAIR_PREFETCH ? 2 : 1;
    u64* sw = dyn + 16 * Pg::M * NT;
    const u32 mi = mod_index(r, level, R.q_count);
    const u64 q = R.q[mi];
    const u64* w = reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N + 2 * size_t(N));
    const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1], nd = R.qd[4 * mi + 2], ndq = R.qd[4 * mi + 3];
    const u32 c0 = blockIdx.x * 16;
    issue_pair_tile<E, N2>(reinterpret_cast<double2*>(dyn), data + size_t(p * rpp + r) * N + c0);
    stage_col_twiddles<E, false>(sw, nullptr, w, w + N);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (u32 cur = 0, first = 1; p < pend; first = 0, ++p, cur ^= (NT - 1)) {
        double2* tile = reinterpret_cast<double2*>(dyn) + cur * 8 * Pg::M;
        if constexpr (NT == 2) {
            if (p + 1 < pend) {
                issue_pair_tile<E, N2>(reinterpret_cast<double2*>(dyn) + (cur ^ 1) * 8 * Pg::M,
                                       data + size_t((p + 1) * rpp + r) * N + c0);
                cp_async_wait<1>();
            } else {
                cp_async_wait<0>();
            }
        } else {
            if (!first) issue_pair_tile<E, N2>(tile, data + size_t(p * rpp + r) * N + c0);
            cp_async_wait<0>();
        }
        (void)first;
        double2* pr = tile;
        __syncthreads();
        double v[2][E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const double2 t = pr[pu((lane << WGeo<E>::LOGE) | j, warp)];
            v[0][j] = t.x;
            v[1][j] = t.y;
        }
        winv_all_pair<E>(v, pr, warp, lane, sw, qd, qi);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if constexpr (RAW) {
                pr[pu(lane + 32 * j, warp)] = make_double2(v[0][j], v[1][j]);
            } else {
                const u64 a = fp_canon_small(fp_mulmod(v[0][j], nd, ndq, qd), q);
                const u64 b = fp_canon_small(fp_mulmod(v[1][j], nd, ndq, qd), q);
                pr[pu(lane + 32 * j, warp)] = make_double2(__longlong_as_double(static_cast<long long>(a)),
                                                       __longlong_as_double(static_cast<long long>(b)));
            }
        }
        __syncthreads();
        store_pair_tile<E, N2>(tile, data + size_t(p * rpp + r) * N + c0);
        __syncthreads();  // the tile is the next prefetch target
    }
}

// ---------------------------------------------------------------------------
// TMA fill of the forward column-pair tile (cp.async.bulk.tensor.2d): the
// row is viewed as a 2-D tensor [rows x 256][256] of u64 (column index
// innermost, row stride 2 KB); one thread issues ONE 16-column x 256-row box
// (32 KB) per tile into a 1024-byte-aligned buffer with the hardware 128-byte
// swizzle (16-byte unit w of tile row k lands in unit 8k + (w ^ (k & 7))),
// completion tracked by an mbarrier (expect_tx = 32 KB). Replaces the 8
// 16-byte cp.async per thread of issue_pair_tile; the tile is read once in
// the TMA layout (conflict-free: lanes l..l+7 read k = l + 32j, distinct
// k & 7), after which every exchange uses the pu() layout as before.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 pu_tma(u32 k, u32 w) { return 8 * k + (w ^ (k & 7)); }

__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
    const u32 a = static_cast<u32>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
    const u32 a = static_cast<u32>(__cvta_generic_to_shared(bar));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    const u32 a = static_cast<u32>(__cvta_generic_to_shared(bar));
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra LAB_WAIT;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_tile(void* smem_dst, const void* tmap, u64* bar, int c0, int row) {
    const u32 d = static_cast<u32>(__cvta_generic_to_shared(smem_dst));
    const u32 b = static_cast<u32>(__cvta_generic_to_shared(bar));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(d),
        "l"(tmap), "r"(c0), "r"(row), "r"(b)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <int E>
constexpr size_t pair_tma_smem() {  // two tiles + twiddles + 2 mbarriers
    return size_t(16) * 8 * PGeo<E>::M * 2 + size_t(8) * 2 * WGeo<E>::TW_COL + 16;
}

template <int E, int E2>
__global__ void __launch_bounds__(256, NTT_MIN_BLOCKS)
kw_fwd_cols2_tma(const __grid_constant__ CUtensorMap tmap, DevRing R, u64* data, u32 rpp, u32 npolys, u32 ppb,
                 int level, u32 skip_gs, u32 row0) {
    using Pg = PGeo<E>;
    constexpr u32 N = 32 * E * 32 * E2, N2 = 32 * E2, M = Pg::M;
    constexpr u32 TILE_BYTES = 16u * 8u * M;
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = next_poly(blockIdx.z * ppb, pend, r, rpp, level, skip_gs);
    if (p >= pend) return;
    extern __shared__ __align__(1024) u64 dyn_tma[];  // 128-byte swizzle atoms need a 1024-byte aligned tile
    double2* tiles = reinterpret_cast<double2*>(dyn_tma);
    u64* sw = reinterpret_cast<u64*>(tiles + 2 * 8 * M);
    u64* bars = sw + 2 * WGeo<E>::TW_COL;
    const u32 mi = mod_index(r, level, R.q_count);
    const u64* w = reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N);
    const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
    const u64 qq = R.q[mi];
    const bool raw = (skip_gs & kTgRawDigits) != 0;
    const u32 c0 = blockIdx.x * 16;
    if (threadIdx.x == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        mbar_expect_tx(bars, TILE_BYTES);
        tma_load_tile(tiles, &tmap, bars, int(c0), int((p * rpp + r) * M));
    }
    stage_col_twiddles<E, true>(sw, nullptr, w, w + N);
    __syncthreads();  // barrier init and twiddles visible to every thread
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    u32 phase[2] = {0, 0};
    for (u32 cur = 0; p < pend;) {
        const u32 pn = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        double2* tile = tiles + cur * 8 * M;
        if (threadIdx.x == 0 && pn < pend) {  // next poly's tile in flight during this transform
            fence_proxy_async();  // the other buffer's last generic-proxy accesses precede the async write
            mbar_expect_tx(bars + (cur ^ 1), TILE_BYTES);
            tma_load_tile(tiles + (cur ^ 1) * 8 * M, &tmap, bars + (cur ^ 1), int(c0), int((pn * rpp + r) * M));
        }
        mbar_wait(bars + cur, phase[cur]);
        phase[cur] ^= 1;
        double2* pr = tile;
        double v[2][E];
#pragma unroll
        for (int j = 0; j < E; ++j) {
            const double2 t = pr[pu_tma(lane + 32 * j, warp)];
            if (raw) {  // ModUp's centred doubles (|v| <= q/2 + 1, the bound c2d gives)
                v[0][j] = t.x;
                v[1][j] = t.y;
            } else {
                v[0][j] = c2d(static_cast<u64>(__double_as_longlong(t.x)), qq);
                v[1][j] = c2d(static_cast<u64>(__double_as_longlong(t.y)), qq);
            }
        }
        __syncthreads();  // every warp has read the TMA layout before the exchanges overwrite the tile
        wfwd_all_pair<E>(v, pr, warp, lane, sw, qd, qi);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < E; ++j) pr[pu((lane << WGeo<E>::LOGE) | j, warp)] = make_double2(v[0][j], v[1][j]);
        __syncthreads();
        store_pair_tile<E, N2>(tile, data + size_t(p * rpp + r) * N + c0);
        __syncthreads();  // the tile is the next TMA target
        p = pn;
        cur ^= 1;
    }
}
