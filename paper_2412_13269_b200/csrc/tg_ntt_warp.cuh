// Warp-level NTT for N = 2^14 .. 2^16 (included by tg_ntt.cu, inside the
// anonymous namespace).
//
// One warp owns one M-point sub-transform (M = 32*E, E = 4 or 8 residues per
// lane). Radix-E stages run in registers; between stage blocks the warp
// re-distributes its M residues through a private, padded shared-memory
// column (__syncwarp only). A block is 8 warps = 8 columns (phase 1) or 8
// consecutive chunks (phase 2). Every twiddle the block needs is staged in
// shared memory at kernel start with coalesced loads that overlap the data
// load, so no stage waits on an L2 round trip.
//
// Layout `lo`: lane l, register j hold element k = ins(l, j, lo), i.e. the
// register index supplies bits [lo, lo+LOGE) of k.
//
// Twiddle index algebra (reference tables, ring.hpp:64-101):
//   forward, phase-2 chunk r, local stage s: w[2^(logN1+s) + r*2^s + i]
//   inverse, phase-A chunk r, u = LOGM-1-p:  winv[2^(logN1+u) + r*2^u + i]
//   both column phases: table[2^u + i]  (u = stage, i = group)
// so a block of 8 consecutive chunks needs, per u, one contiguous run of
// 8*2^u entries starting at 2^(logN1+u) + 8*bx*2^u, and a column block needs
// table[1 .. M1).

constexpr u64 kSmallQ = u64(1) << 55;  // lazy-bound threshold of the SQ path

#ifndef NTT_MIN_BLOCKS
#define NTT_MIN_BLOCKS 3
#endif
#ifndef NTT_COLS_PAIR
#define NTT_COLS_PAIR 1  // FP64 column phase: polys in interleaved pairs (1) or one at a time, next prefetched (0)
#endif
#ifndef NTT_CHUNK_STAGE
#define NTT_CHUNK_STAGE 0
#endif
#ifndef NTT_CHUNK_MIN_BLOCKS
#define NTT_CHUNK_MIN_BLOCKS 2  // registers for two interleaved transforms (measured best)
#endif

template <int E>
struct WGeo {
    static constexpr int LOGE = E == 8 ? 3 : 2;
    static constexpr int M = 32 * E;
    static constexpr int LOGM = 5 + LOGE;
    static constexpr int CS = M + M / 8 + 2;  // padded column stride (words)
    static constexpr int TW_CHUNK = 8 * (M - 1);  // staged twiddles of 8 chunks
    static constexpr int TW_COL = M;              // staged twiddles of a column block
};

__device__ __forceinline__ u32 wpad(u32 k) { return k + (k >> 3); }

template <int LOGE>
__device__ __forceinline__ u32 wins(u32 lane, u32 j, u32 lo) {
    return ((lane >> lo) << (lo + LOGE)) | (j << lo) | (lane & ((1u << lo) - 1));
}

// Small-modulus variants (SQ, q < 2^55, i.e. every q-chain prime here):
// no Harvey corrections inside a phase. Forward: values grow by < 2q per
// stage, < 33q after both phases (< 2^64). Inverse: with B_p = 2q << p a
// bound on the inputs of stage p, a+b < 2 B_p and a - b + B_p in (0, 2 B_p);
// after a phase (<= 8 stages) values are < 512q < 2^64 and are brought back
// to [0, 2q) once. 60-bit special primes take the corrected path.
template <bool SQ>
__device__ __forceinline__ void ct_bfly(u64& a, u64& b, u64 w, u64 ws, u64 q) {
    const u64 q2 = 2 * q;
    if constexpr (!SQ) {
        if (a >= q2) a -= q2;
    }
    const u64 t = shoup_lazy(b, w, ws, q);
    b = a - t + q2;
    a = a + t;
}

template <bool SQ>
__device__ __forceinline__ void gs_bfly(u64& a, u64& b, u64 w, u64 ws, u64 q, u64 bound) {
    const u64 q2 = 2 * q;
    u64 s = a + b;
    if constexpr (!SQ) {
        if (s >= q2) s -= q2;
    }
    const u64 d = a - b + (SQ ? bound : q2);
    b = shoup_lazy(d, w, ws, q);
    a = s;
}

// Bank-conflict-free twiddle runs. In stage p of a stage block with layout
// lo, lane l / register j reads group i = k0 >> (p+1): the low nj bits of i
// come from j and the rest from the lane's high bits, so consecutive lanes
// read entries 2^nj apart (64 B strides for nj = 2: 16 wavefronts per
// LDS.128 instead of 4). Each staged run of 2^u entries is therefore
// stored transposed, pos(i) = (i mod 2^nj) * 2^(u-nj) + (i >> nj), which puts
// one register's entries for consecutive lanes in consecutive slots.
template <int E, bool FWD>
__host__ __device__ constexpr int stage_lo(int p) {
    if constexpr (E == 8) return FWD ? (p >= 5 ? 5 : p >= 2 ? 2 : 0) : (p <= 2 ? 0 : p <= 5 ? 3 : 5);
    else return FWD ? (p >= 5 ? 5 : p >= 3 ? 3 : p >= 1 ? 1 : 0) : (p <= 1 ? 0 : p <= 3 ? 2 : p <= 5 ? 4 : 5);
}
template <int E, bool FWD>
__host__ __device__ constexpr int tw_nj(int u) {
    constexpr int LOGE = WGeo<E>::LOGE, LOGM = WGeo<E>::LOGM;
    const int p = LOGM - 1 - u, lo = stage_lo<E, FWD>(p);
    return LOGM - lo - LOGE > 0 ? lo + LOGE - p - 1 : 0;  // no lane-high bits: broadcast, keep order
}
template <int E, bool FWD>
__host__ __device__ constexpr u32 tw_nj_mask() {
    u32 m = 0;
    for (int u = 0; u < WGeo<E>::LOGM; ++u) m |= u32(tw_nj<E, FWD>(u)) << (2 * u);
    return m;
}
__device__ __forceinline__ u32 tw_pos(u32 u, u32 nj, u32 i) {
    return ((i & ((1u << nj) - 1)) << (u - nj)) | (i >> nj);
}
// inverse of tw_pos: the group index stored at position pl
__device__ __forceinline__ u32 tw_src(u32 u, u32 nj, u32 pl) {
    return ((pl & ((1u << (u - nj)) - 1)) << nj) | (pl >> (u - nj));
}

// Staged-twiddle index for group i of stage-unit u: CHUNK blocks use the
// per-u runs (8 chunks, this warp's chunk c), column blocks the raw index.
template <int E, bool FWD, bool CHUNK>
__device__ __forceinline__ u32 tw_slot(u32 u, u32 c, u32 i) {
    const u32 pi = tw_pos(u, u32(tw_nj<E, FWD>(int(u))), i);
    if constexpr (CHUNK) return 8 * ((1u << u) - 1) + (c << u) + pi;
    else return (1u << u) + pi;
}

// Cheap twiddle addressing. In layout LAY, lane l / register j of stage p
// reads group i = k0 >> (p+1) = (H << nj) | (j >> (p+1-LAY)) with
// H = l >> LAY the lane-high bits; its transposed slot is
// base_u + H + ((j >> (p+1-LAY)) << HB), HB = LOGM-LAY-LOGE. So one lane base
// per stage plus a compile-time offset per register: no per-butterfly index
// arithmetic (tw_slot computes the same slot generically).
template <int E, bool CHUNK, int LAY>
__device__ __forceinline__ u32 tw_lane_base(u32 u, u32 c, u32 lane) {
    constexpr int HB = WGeo<E>::LOGM - LAY - WGeo<E>::LOGE;
    const u32 H = HB > 0 ? (lane >> LAY) : 0u;
    return (CHUNK ? 8 * ((1u << u) - 1) + (c << u) : (1u << u)) + H;
}
template <int E, int LAY>
__host__ __device__ constexpr u32 tw_reg_off(int j, int p) {
    return u32(j >> (p + 1 - LAY)) << (WGeo<E>::LOGM - LAY - WGeo<E>::LOGE);
}

// Forward (CT) stages on bits HI..LO (descending) of layout LAY; stage s = LOGM-1-p.
template <int E, bool CHUNK, bool SQ, int LAY, int HI, int LO>
__device__ __forceinline__ void wfwd(u64 (&v)[E], u32 lane, const u64* sw, const u64* sws, u64 q, u32 c) {
    constexpr int LOGE = WGeo<E>::LOGE, LOGM = WGeo<E>::LOGM;
#pragma unroll
    for (int p = HI; p >= LO; --p) {
        const int b = p - LAY;
        const ulonglong2* tb = reinterpret_cast<const ulonglong2*>(sw) + tw_lane_base<E, CHUNK, LAY>(u32(LOGM - 1 - p), c, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if (j & (1 << b)) continue;
            const ulonglong2 tw = tb[tw_reg_off<E, LAY>(j, p)];
            ct_bfly<SQ>(v[j], v[j | (1 << b)], tw.x, tw.y, q);
        }
    }
}

// Inverse (GS) stages on bits LO..HI (ascending) of layout LAY; unit u = LOGM-1-p.
template <int E, bool CHUNK, bool SQ, int LAY, int LO, int HI>
__device__ __forceinline__ void winv(u64 (&v)[E], u32 lane, const u64* sw, const u64* sws, u64 q, u32 c) {
    constexpr int LOGE = WGeo<E>::LOGE, LOGM = WGeo<E>::LOGM;
#pragma unroll
    for (int p = LO; p <= HI; ++p) {
        const int b = p - LAY;
        const ulonglong2* tb = reinterpret_cast<const ulonglong2*>(sw) + tw_lane_base<E, CHUNK, LAY>(u32(LOGM - 1 - p), c, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if (j & (1 << b)) continue;
            const ulonglong2 tw = tb[tw_reg_off<E, LAY>(j, p)];
            gs_bfly<SQ>(v[j], v[j | (1 << b)], tw.x, tw.y, q, (2 * q) << p);
        }
    }
}

template <int E, class T>
__device__ __forceinline__ void wxchg(T (&v)[E], u64* colw, u32 lane, u32 lo_from, u32 lo_to) {
    constexpr int LOGE = WGeo<E>::LOGE;
    T* col = reinterpret_cast<T*>(colw);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) col[wpad(wins<LOGE>(lane, u32(j), lo_from))] = v[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = col[wpad(wins<LOGE>(lane, u32(j), lo_to))];
}

// ---- FP64 path (q < 1.2 * 2^50; tg_fp64.cuh) ------------------------------
// Staged twiddle pairs are (w, fl(w/q)) doubles. Forward blocks hold at most
// 3 stages; with the centred twiddles and bounds of tg_fp64.cuh six forward
// stages run between reductions from centred inputs (|v| <= q/2 + 1; the
// column phase centres canonical inputs with c2d), so only the second and the
// last radix-8 block end in fp_reduce (RED). Inverse butterflies reduce the
// sum after odd stages only (|x - y| <= 2.4q < 2^52 in between).
// NP independent transforms of the same modulus and position (NP polys) run
// interleaved: each staged twiddle feeds NP butterflies and the FP64
// dependency chains of one transform hide behind the other's.
template <int NP, int E, bool CHUNK, int LAY, int HI, int LO, bool RED = true>
__device__ __forceinline__ void wfwd_fp(double (&v)[NP][E], u32 lane, const u64* sw, double q, double qi, u32 c) {
    constexpr int LOGE = WGeo<E>::LOGE, LOGM = WGeo<E>::LOGM;
#pragma unroll
    for (int p = HI; p >= LO; --p) {
        const int b = p - LAY;
        const double2* tb = reinterpret_cast<const double2*>(sw) + tw_lane_base<E, CHUNK, LAY>(u32(LOGM - 1 - p), c, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if (j & (1 << b)) continue;
            const double2 tw = tb[tw_reg_off<E, LAY>(j, p)];
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                const double x = fp_mulmod(v[n][j | (1 << b)], tw.x, tw.y, q);
                const double a = v[n][j];
                v[n][j] = __dadd_rn(a, x);
                v[n][j | (1 << b)] = __dsub_rn(a, x);
            }
        }
    }
    if constexpr (RED) {  // block-final reduction (skipped where tg_fp64.cuh's bound allows)
#pragma unroll
        for (int n = 0; n < NP; ++n)
#pragma unroll
            for (int j = 0; j < E; ++j) v[n][j] = fp_reduce(v[n][j], q, qi);
    }
}

template <int NP, int E, bool CHUNK, int LAY, int LO, int HI>
__device__ __forceinline__ void winv_fp(double (&v)[NP][E], u32 lane, const u64* sw, double q, double qi, u32 c) {
    constexpr int LOGE = WGeo<E>::LOGE, LOGM = WGeo<E>::LOGM;
#pragma unroll
    for (int p = LO; p <= HI; ++p) {
        const int b = p - LAY;
        const double2* tb = reinterpret_cast<const double2*>(sw) + tw_lane_base<E, CHUNK, LAY>(u32(LOGM - 1 - p), c, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) {
            if (j & (1 << b)) continue;
            const double2 tw = tb[tw_reg_off<E, LAY>(j, p)];
#pragma unroll
            for (int n = 0; n < NP; ++n) {
                const double a = v[n][j], bb = v[n][j | (1 << b)];
                // sums reduced after odd stages and the last one (tg_fp64.cuh)
                if ((p & 1) == 1 || p == LOGM - 1) v[n][j] = fp_reduce(__dadd_rn(a, bb), q, qi);
                else v[n][j] = __dadd_rn(a, bb);
                v[n][j | (1 << b)] = fp_mulmod(__dsub_rn(a, bb), tw.x, tw.y, q);
            }
        }
    }
}

// NP warp-private exchange columns, `cs` words apart.
template <int NP, int E>
__device__ __forceinline__ void wxchg_fp(double (&v)[NP][E], u64* colw, u32 cs, u32 lane, u32 lo_from, u32 lo_to) {
    constexpr int LOGE = WGeo<E>::LOGE;
    __syncwarp();
#pragma unroll
    for (int n = 0; n < NP; ++n) {
        double* col = reinterpret_cast<double*>(colw + n * cs);
#pragma unroll
        for (int j = 0; j < E; ++j) col[wpad(wins<LOGE>(lane, u32(j), lo_from))] = v[n][j];
    }
    __syncwarp();
#pragma unroll
    for (int n = 0; n < NP; ++n) {
        const double* col = reinterpret_cast<const double*>(colw + n * cs);
#pragma unroll
        for (int j = 0; j < E; ++j) v[n][j] = col[wpad(wins<LOGE>(lane, u32(j), lo_to))];
    }
}

// NP = 2 exchange with both transforms' values of element k moved as one
// 16-byte word, in the warp's contiguous 2*CS-word region: half the shared-
// memory instructions of two separate columns, conflict-free (wpad).
template <int E>
__device__ __forceinline__ void wxchg_fp_pair(double (&v)[2][E], u64* colw, u32 lane, u32 lo_from, u32 lo_to) {
    constexpr int LOGE = WGeo<E>::LOGE;
    double2* pr = reinterpret_cast<double2*>(colw);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) pr[wpad(wins<LOGE>(lane, u32(j), lo_from))] = make_double2(v[0][j], v[1][j]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) {
        const double2 t = pr[wpad(wins<LOGE>(lane, u32(j), lo_to))];
        v[0][j] = t.x;
        v[1][j] = t.y;
    }
}
template <int NP, int E, bool PX>
__device__ __forceinline__ void wxchg_any(double (&v)[NP][E], u64* col, u32 cs, u32 lane, u32 lo_from, u32 lo_to) {
    if constexpr (PX && NP == 2) wxchg_fp_pair<E>(v, col, lane, lo_from, lo_to);
    else wxchg_fp<NP, E>(v, col, cs, lane, lo_from, lo_to);
}

template <int NP, int E, bool CHUNK, bool PX = false>
__device__ __forceinline__ void wfwd_all_fp(double (&v)[NP][E], u64* col, u32 cs, u32 lane, const u64* sw, double q,
                                            double qi, u32 c) {
    if constexpr (E == 8) {
        wfwd_fp<NP, 8, CHUNK, 5, 7, 5, false>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 8, PX>(v, col, cs, lane, 5, 2);
        wfwd_fp<NP, 8, CHUNK, 2, 4, 2>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 8, PX>(v, col, cs, lane, 2, 0);
        wfwd_fp<NP, 8, CHUNK, 0, 1, 0>(v, lane, sw, q, qi, c);
    } else {
        wfwd_fp<NP, 4, CHUNK, 5, 6, 5, false>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 5, 3);
        wfwd_fp<NP, 4, CHUNK, 3, 4, 3, false>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 3, 1);
        wfwd_fp<NP, 4, CHUNK, 1, 2, 1>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 1, 0);
        wfwd_fp<NP, 4, CHUNK, 0, 0, 0>(v, lane, sw, q, qi, c);
    }
}

template <int NP, int E, bool CHUNK, bool PX = false>
__device__ __forceinline__ void winv_all_fp(double (&v)[NP][E], u64* col, u32 cs, u32 lane, const u64* sw, double q,
                                            double qi, u32 c) {
    if constexpr (E == 8) {
        winv_fp<NP, 8, CHUNK, 0, 0, 2>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 8, PX>(v, col, cs, lane, 0, 3);
        winv_fp<NP, 8, CHUNK, 3, 3, 5>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 8, PX>(v, col, cs, lane, 3, 5);
        winv_fp<NP, 8, CHUNK, 5, 6, 7>(v, lane, sw, q, qi, c);
    } else {
        winv_fp<NP, 4, CHUNK, 0, 0, 1>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 0, 2);
        winv_fp<NP, 4, CHUNK, 2, 2, 3>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 2, 4);
        winv_fp<NP, 4, CHUNK, 4, 4, 5>(v, lane, sw, q, qi, c);
        wxchg_any<NP, 4, PX>(v, col, cs, lane, 4, 5);
        winv_fp<NP, 4, CHUNK, 5, 6, 6>(v, lane, sw, q, qi, c);
    }
}

// Full forward sub-transform: layout 5 (k = lane + 32 j) -> layout 0.
template <int E, bool CHUNK, bool SQ>
__device__ __forceinline__ void wfwd_all(u64 (&v)[E], u64* col, u32 lane, const u64* sw, const u64* sws, u64 q, u32 c) {
    if constexpr (E == 8) {
        wfwd<8, CHUNK, SQ, 5, 7, 5>(v, lane, sw, sws, q, c);
        wxchg<8>(v, col, lane, 5, 2);
        wfwd<8, CHUNK, SQ, 2, 4, 2>(v, lane, sw, sws, q, c);
        wxchg<8>(v, col, lane, 2, 0);
        wfwd<8, CHUNK, SQ, 0, 1, 0>(v, lane, sw, sws, q, c);
    } else {
        wfwd<4, CHUNK, SQ, 5, 6, 5>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 5, 3);
        wfwd<4, CHUNK, SQ, 3, 4, 3>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 3, 1);
        wfwd<4, CHUNK, SQ, 1, 2, 1>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 1, 0);
        wfwd<4, CHUNK, SQ, 0, 0, 0>(v, lane, sw, sws, q, c);
    }
}

// Full inverse sub-transform: layout 0 -> layout 5.
template <int E, bool CHUNK, bool SQ>
__device__ __forceinline__ void winv_all(u64 (&v)[E], u64* col, u32 lane, const u64* sw, const u64* sws, u64 q, u32 c) {
    if constexpr (E == 8) {
        winv<8, CHUNK, SQ, 0, 0, 2>(v, lane, sw, sws, q, c);
        wxchg<8>(v, col, lane, 0, 3);
        winv<8, CHUNK, SQ, 3, 3, 5>(v, lane, sw, sws, q, c);
        wxchg<8>(v, col, lane, 3, 5);
        winv<8, CHUNK, SQ, 5, 6, 7>(v, lane, sw, sws, q, c);
    } else {
        winv<4, CHUNK, SQ, 0, 0, 1>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 0, 2);
        winv<4, CHUNK, SQ, 2, 2, 3>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 2, 4);
        winv<4, CHUNK, SQ, 4, 4, 5>(v, lane, sw, sws, q, c);
        wxchg<4>(v, col, lane, 4, 5);
        winv<4, CHUNK, SQ, 5, 6, 6>(v, lane, sw, sws, q, c);
    }
}

// Stage the 8-chunk twiddle runs of block bx: for u < LOGM,
// sw[8(2^u-1) + t] = tab[2^(logN1+u) + 8 bx 2^u + t], t < 8*2^u.
template <int E, bool FWD>
__device__ __forceinline__ void stage_chunk_twiddles(u64* sw, u64* sws, const u64* __restrict__ w,
                                                     const u64* __restrict__ ws, u32 logN1, u32 bx) {
    // flattened slot e -> (u, t): all of a thread's loads are issued before
    // any store, so the staging costs one memory latency, not LOGM of them
    constexpr int TOT = WGeo<E>::TW_CHUNK;
    constexpr int PER = (TOT + 255) / 256;
    u64 a[PER], b[PER];
    u32 d[PER];
    constexpr u32 NJ = tw_nj_mask<E, FWD>();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const u32 e = threadIdx.x + 256u * k;
        d[k] = u32(TOT);
        if (e < u32(TOT)) {
            const u32 u = 31 - __clz((e >> 3) + 1);  // e in [8(2^u - 1), 8(2^(u+1) - 1))
            // thread e fills slot e (conflict-free stores) from the group
            // index whose transposed position it is
            const u32 t = e - 8 * ((1u << u) - 1), pl = t & ((1u << u) - 1);
            const u32 src = (1u << (logN1 + u)) + ((8 * bx) << u) + (t - pl) + tw_src(u, (NJ >> (2 * u)) & 3, pl);
            a[k] = __ldg(w + src);
            b[k] = __ldg(ws + src);
            d[k] = e;
        }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k)
        if (d[k] < u32(TOT)) reinterpret_cast<ulonglong2*>(sw)[d[k]] = make_ulonglong2(a[k], b[k]);
}

template <int E, bool FWD>
__device__ __forceinline__ void stage_col_twiddles(u64* sw, u64* sws, const u64* __restrict__ w,
                                                   const u64* __restrict__ ws) {
    constexpr u32 NJ = tw_nj_mask<E, FWD>();
    for (u32 d = threadIdx.x; d < u32(WGeo<E>::M); d += 256) {
        u32 t = 0;
        if (d > 0) {
            const u32 u = 31 - __clz(d);
            t = (1u << u) + tw_src(u, (NJ >> (2 * u)) & 3, d - (1u << u));
        }
        reinterpret_cast<ulonglong2*>(sw)[d] = make_ulonglong2(__ldg(w + t), __ldg(ws + t));
    }
}

// Which rows take the FP64 path: every q < kFpMaxQ row, except that one row
// in R.int_every (0: none) keeps the 64-bit integer path so the FP64 and the
// integer pipes work side by side. Both phases of a transform make the same
// choice (the inter-phase format differs).
__device__ __forceinline__ bool ntt_use_fp(const DevRing& R, u64 q, u32 r) {
    if (q >= kFpMaxQ) return false;
    return R.int_every == 0 || r % R.int_every != R.int_every - 1;
}

// ---- poly loop ------------------------------------------------------------
// Grid: x = column / chunk block, y = row r of a poly (modulus), z = group of
// `ppb` polys. A block transforms row r of each of its polys in turn: the
// staged twiddles (modulus r) are reused for every poly, and the next poly's
// input is fetched while the current one is computed (cp.async into a second
// tile for the column phase; registers for the chunk phase).
__device__ __forceinline__ u32 next_poly(u32 p, u32 pend, u32 r, u32 rpp, int level, u32 skip_gs) {
    while (p < pend && ntt_row_skipped(p * rpp + r, rpp, level, skip_gs)) ++p;
    return p;
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const u32 a = static_cast<u32>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory");
}

template <int E>
constexpr size_t col_smem() {  // two tiles + twiddles
    return size_t(8) * (16 * WGeo<E>::CS + 2 * WGeo<E>::TW_COL);
}
template <int E>
constexpr size_t chunk_smem() {  // exchange columns of two transforms per warp + twiddles (+ staging)
    return size_t(8) * (16 * WGeo<E>::CS + 2 * WGeo<E>::TW_CHUNK + (NTT_CHUNK_STAGE ? 16 * (WGeo<E>::M + WGeo<E>::M / 4) : 0));
}
// Chunk staging (NTT_CHUNK_STAGE): per warp two polys' chunks, prefetched by
// 16-byte cp.async while the current pair is transformed (forward: dense,
// read lane-strided; inverse: 2 pad words per 8, read as 16-byte vectors).
__device__ __forceinline__ u32 ipad(u32 k) { return k + 2 * (k >> 3); }
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const u32 a = static_cast<u32>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(a), "l"(gmem) : "memory");
}
template <int E, bool PAD>
__device__ __forceinline__ void stage_chunk(u64* s, const u64* g, u32 lane) {
#pragma unroll
    for (int i = 0; i < WGeo<E>::M / 64; ++i) {
        const u32 k = 2 * (lane + 32 * i);
        cp_async16(s + (PAD ? ipad(k) : k), g + k);
    }
}

// Column tile (8 columns x M1 rows, element (m, c) at c*CS + wpad(m)) of the
// row starting at rb (= row base + first column). N2 = M2 is the row stride
// of the M1 x N2 view: with it a compile-time constant every per-element
// address is the thread's base plus an immediate offset (thread t copies
// elements m = t/8 + 32i, c = t%8; wpad(m + 32i) = wpad(m) + 36i).
template <int OS, int OG>
__device__ __forceinline__ void cp_async8_imm(u32 sa, const u64* g) {
    asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], 8;\n" ::"r"(sa), "l"(g), "n"(OS), "n"(OG) : "memory");
}
template <int N2, int... I>
__device__ __forceinline__ void issue_col_elems(u32 sa, const u64* g, std::integer_sequence<int, I...>) {
    (cp_async8_imm<I * 36 * 8, I * 32 * N2 * 8>(sa, g), ...);
}
template <int E, int N2>
__device__ __forceinline__ void issue_col_tile(u64* tile, const u64* rb) {
    using Gm = WGeo<E>;
    const u32 t = threadIdx.x, c = t & 7, m0 = t >> 3;
    const u32 sa = static_cast<u32>(__cvta_generic_to_shared(tile + c * Gm::CS + wpad(m0)));
    issue_col_elems<N2>(sa, rb + size_t(m0) * N2 + c, std::make_integer_sequence<int, Gm::M / 32>{});
    cp_async_commit();
}
template <int E, int N2>
__device__ __forceinline__ void store_col_tile(const u64* tile, u64* rb) {
    using Gm = WGeo<E>;
    const u32 t = threadIdx.x, c = t & 7, m0 = t >> 3;
    const u64* sm = tile + c * Gm::CS + wpad(m0);
    u64* g = rb + size_t(m0) * N2 + c;
#pragma unroll
    for (int i = 0; i < Gm::M / 32; ++i) g[size_t(i) * 32 * N2] = sm[36 * i];
}

// Phase 1 forward: 8 columns x M1 rows, stages 0 .. log M1 - 1.
template <int E, int E2>
__global__ void __launch_bounds__(256, NTT_MIN_BLOCKS)
kw_fwd_cols(DevRing R, u64* data, const u64* src, u32 rpp, u32 npolys, u32 ppb, int level, u32 skip_gs,
            u32 row0) {
    using Gm = WGeo<E>;
    // row r of every poly (rows [row0, row0 + gridDim.y) are transformed)
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = next_poly(blockIdx.z * ppb, pend, r, rpp, level, skip_gs);
    if (p >= pend) return;
    extern __shared__ u64 dyn[];
    u64* tiles = dyn;
    u64* sw = dyn + 16 * Gm::CS;
    u64* sws = sw + Gm::TW_COL;
    constexpr u32 N = 32 * E * 32 * E2;  // == R.N (warp_plan)
    const u32 mi = mod_index(r, level, R.q_count);
    const u64 q = R.q[mi];
    const bool fp = ntt_use_fp(R, q, r);  // FP64 path; the other phase makes the same choice
    const u64* w = fp ? reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N) : R.tw + size_t(mi) * 4 * N;
    const u32 c0 = blockIdx.x * 8;
    issue_col_tile<E, 32 * E2>(tiles, src + size_t(p * rpp + r) * N + c0);
    stage_col_twiddles<E, true>(sw, sws, w, w + N);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (fp && NTT_COLS_PAIR) {  // polys in pairs on the block's two tiles: each staged twiddle feeds two interleaved transforms
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
        bool first = true;
        while (p < pend) {
            const u32 p2 = next_poly(p + 1, pend, r, rpp, level, skip_gs);
            const bool pair = p2 < pend;
            if (!first) issue_col_tile<E, 32 * E2>(tiles, src + size_t(p * rpp + r) * N + c0);
            if (pair) issue_col_tile<E, 32 * E2>(tiles + 8 * Gm::CS, src + size_t(p2 * rpp + r) * N + c0);
            first = false;
            cp_async_wait<0>();
            __syncthreads();
            u64* col = tiles + warp * Gm::CS;
            if (pair) {  // canonical u64 in, doubles (|v| <= q/2 + 1, raw bits) out to phase 2
                double v[2][E];
#pragma unroll
                for (int n = 0; n < 2; ++n)
#pragma unroll
                    for (int j = 0; j < E; ++j) v[n][j] = c2d(col[n * 8 * Gm::CS + wpad(lane + 32 * j)], q);
                wfwd_all_fp<2, E, false>(v, col, 8 * Gm::CS, lane, sw, qd, qi, 0);
                __syncwarp();
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    double* cold = reinterpret_cast<double*>(col + n * 8 * Gm::CS);
#pragma unroll
                    for (int j = 0; j < E; ++j) cold[wpad((lane << Gm::LOGE) | j)] = v[n][j];
                }
            } else {
                double v[1][E];
#pragma unroll
                for (int j = 0; j < E; ++j) v[0][j] = c2d(col[wpad(lane + 32 * j)], q);
                wfwd_all_fp<1, E, false>(v, col, 0, lane, sw, qd, qi, 0);
                __syncwarp();
                double* cold = reinterpret_cast<double*>(col);
#pragma unroll
                for (int j = 0; j < E; ++j) cold[wpad((lane << Gm::LOGE) | j)] = v[0][j];
            }
            __syncthreads();
            store_col_tile<E, 32 * E2>(tiles, data + size_t(p * rpp + r) * N + c0);
            if (pair) store_col_tile<E, 32 * E2>(tiles + 8 * Gm::CS, data + size_t(p2 * rpp + r) * N + c0);
            __syncthreads();
            p = pair ? next_poly(p2 + 1, pend, r, rpp, level, skip_gs) : p2;
        }
        return;
    }
    u32 cur = 0;
    while (p < pend) {
        const u32 pn = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        if (pn < pend) {
            issue_col_tile<E, 32 * E2>(tiles + (cur ^ 1) * 8 * Gm::CS, src + size_t(pn * rpp + r) * N + c0);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        u64* tile = tiles + cur * 8 * Gm::CS;
        u64* col = tile + warp * Gm::CS;
        if (fp) {  // canonical u64 in, doubles (|v| <= q/2 + 1, raw bits) out to phase 2
            const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
            double v[1][E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[0][j] = c2d(col[wpad(lane + 32 * j)], q);
            wfwd_all_fp<1, E, false>(v, col, 0, lane, sw, qd, qi, 0);
            __syncwarp();
            double* cold = reinterpret_cast<double*>(col);
#pragma unroll
            for (int j = 0; j < E; ++j) cold[wpad((lane << Gm::LOGE) | j)] = v[0][j];
        } else {
            u64 v[E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = col[wpad(lane + 32 * j)];
            if (q < kSmallQ) wfwd_all<E, false, true>(v, col, lane, sw, sws, q, 0);
            else wfwd_all<E, false, false>(v, col, lane, sw, sws, q, 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < E; ++j) col[wpad((lane << Gm::LOGE) | j)] = v[j];
        }
        __syncthreads();
        store_col_tile<E, 32 * E2>(tile, data + size_t(p * rpp + r) * N + c0);
        __syncthreads();  // the tile is the next prefetch target
        p = pn;
        cur ^= 1;
    }
}

// Chunk-phase loads/stores of one warp's chunk (lane-strided in, lane-
// contiguous 16-byte vectors out, or the reverse for the inverse).
template <int E>
__device__ __forceinline__ void ld_strided(u64 (&v)[E], const u64* x, u32 lane) {
#pragma unroll
    for (int j = 0; j < E; ++j) v[j] = x[lane + 32 * j];
}
template <int E>
__device__ __forceinline__ void st_strided(u64* x, const u64 (&v)[E], u32 lane) {
#pragma unroll
    for (int j = 0; j < E; ++j) x[lane + 32 * j] = v[j];
}
template <int E>
__device__ __forceinline__ void ld_vec(u64 (&v)[E], const u64* x, u32 lane) {
    const ulonglong2* x2 = reinterpret_cast<const ulonglong2*>(x + (lane << WGeo<E>::LOGE));
#pragma unroll
    for (int j = 0; j < E / 2; ++j) {
        const ulonglong2 t = x2[j];
        v[2 * j] = t.x;
        v[2 * j + 1] = t.y;
    }
}
template <int E>
__device__ __forceinline__ void st_vec(u64* x, const u64 (&v)[E], u32 lane) {
    ulonglong2* x2 = reinterpret_cast<ulonglong2*>(x + (lane << WGeo<E>::LOGE));
#pragma unroll
    for (int j = 0; j < E / 2; ++j) x2[j] = make_ulonglong2(v[2 * j], v[2 * j + 1]);
}

// FP64 chunk phase of NP polys: forward (phase-1 doubles in, canonical out)
template <int NP, int E, bool PX = false>
__device__ __forceinline__ void chunk_fwd_fp(u64 (&v)[NP][E], u64* col, u32 cs, u32 lane, const u64* sw, double qd,
                                             double qi, u32 warp, u64 q) {
    double vd[NP][E];
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int j = 0; j < E; ++j) vd[n][j] = __longlong_as_double(static_cast<long long>(v[n][j]));
    wfwd_all_fp<NP, E, true, PX>(vd, col, cs, lane, sw, qd, qi, warp);
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int j = 0; j < E; ++j) v[n][j] = fp_canon_small(vd[n][j], q);  // |vd| <= q/2 + 1 (fp_reduce)
}
// inverse (canonical in, doubles |v| <= 1.5q as raw bits out to phase B)
template <int NP, int E, bool PX = false>
__device__ __forceinline__ void chunk_inv_fp(u64 (&v)[NP][E], u64* col, u32 cs, u32 lane, const u64* sw, double qd,
                                             double qi, u32 warp, u64 q) {
    double vd[NP][E];
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int j = 0; j < E; ++j) vd[n][j] = c2d(v[n][j], q);  // centred: |v| <= q/2 (tg_fp64.cuh inverse bound)
    winv_all_fp<NP, E, true, PX>(vd, col, cs, lane, sw, qd, qi, warp);
#pragma unroll
    for (int n = 0; n < NP; ++n)
#pragma unroll
        for (int j = 0; j < E; ++j) v[n][j] = static_cast<u64>(__double_as_longlong(vd[n][j]));
}

// Phase 2 forward: one warp per contiguous chunk of M2, final canonical reduce.
// FP64 rows take the block's polys two at a time (interleaved transforms);
// integer rows one at a time with the next poly prefetched.
template <int E>
__global__ void __launch_bounds__(256, NTT_CHUNK_MIN_BLOCKS)
kw_fwd_chunks(DevRing R, u64* data, u32 rpp, u32 npolys, u32 ppb, int level, u32 logN1, u32 skip_gs,
              u32 row0) {
    using Gm = WGeo<E>;
    // row r of every poly (rows [row0, row0 + gridDim.y) are transformed)
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = next_poly(blockIdx.z * ppb, pend, r, rpp, level, skip_gs);
    if (p >= pend) return;
    extern __shared__ __align__(16) u64 dyn[];
    u64* sm = dyn;
    u64* sw = dyn + 16 * Gm::CS;
    u64* sws = sw + Gm::TW_CHUNK;
    const u32 N = R.N;
    const u32 mi = mod_index(r, level, R.q_count);
    const u64 q = R.q[mi];
    const bool fp = ntt_use_fp(R, q, r);
    const u64* w = fp ? reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N) : R.tw + size_t(mi) * 4 * N;
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t off = size_t(blockIdx.x * 8 + warp) * Gm::M;
    u64* col = sm + warp * Gm::CS;
    u64* colp = sm + warp * 2 * Gm::CS;  // FP64 paths: the warp's contiguous pair region
    constexpr u32 CS2 = 8 * Gm::CS;  // second transform's column
    auto row = [&](u32 pp) { return data + size_t(pp * rpp + r) * N + off; };
    if (fp && NTT_CHUNK_STAGE) {
        constexpr u32 SW = Gm::M + Gm::M / 4;
        u64* stg = dyn + 16 * Gm::CS + 2 * Gm::TW_CHUNK + warp * 2 * SW;
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
        u32 p2 = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        stage_chunk<E, false>(stg, row(p), lane);
        if (p2 < pend) stage_chunk<E, false>(stg + SW, row(p2), lane);
        cp_async_commit();
        stage_chunk_twiddles<E, true>(sw, sws, w, w + N, logN1, blockIdx.x);
        __syncthreads();
        while (true) {
            const bool pair = p2 < pend;
            cp_async_wait<0>();
            __syncwarp();
            u64 v[2][E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[0][j] = stg[lane + 32 * j];
            if (pair) {
#pragma unroll
                for (int j = 0; j < E; ++j) v[1][j] = stg[SW + lane + 32 * j];
            }
            __syncwarp();
            const u32 pn = pair ? next_poly(p2 + 1, pend, r, rpp, level, skip_gs) : pend;
            const u32 pn2 = pn < pend ? next_poly(pn + 1, pend, r, rpp, level, skip_gs) : pend;
            if (pn < pend) {  // the next pair is in flight during this pair's stages
                stage_chunk<E, false>(stg, row(pn), lane);
                if (pn2 < pend) stage_chunk<E, false>(stg + SW, row(pn2), lane);
            }
            cp_async_commit();
            if (pair) {
                chunk_fwd_fp<2, E, true>(v, colp, CS2, lane, sw, qd, qi, warp, q);
                st_vec<E>(row(p), v[0], lane);
                st_vec<E>(row(p2), v[1], lane);
            } else {
                chunk_fwd_fp<1, E>(reinterpret_cast<u64(&)[1][E]>(v[0]), colp, CS2, lane, sw, qd, qi, warp, q);
                st_vec<E>(row(p), v[0], lane);
            }
            if (pn >= pend) break;
            p = pn;
            p2 = pn2;
        }
        return;
    }
    if (fp) {
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
        u32 p2 = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        u64 v[2][E];
        ld_strided<E>(v[0], row(p), lane);
        if (p2 < pend) ld_strided<E>(v[1], row(p2), lane);
        stage_chunk_twiddles<E, true>(sw, sws, w, w + N, logN1, blockIdx.x);
        __syncthreads();
        while (true) {
            if (p2 < pend) {
                chunk_fwd_fp<2, E, true>(v, colp, CS2, lane, sw, qd, qi, warp, q);
                st_vec<E>(row(p), v[0], lane);
                st_vec<E>(row(p2), v[1], lane);
                p = next_poly(p2 + 1, pend, r, rpp, level, skip_gs);
            } else {
                chunk_fwd_fp<1, E>(reinterpret_cast<u64(&)[1][E]>(v[0]), colp, CS2, lane, sw, qd, qi, warp, q);
                st_vec<E>(row(p), v[0], lane);
                p = p2;
            }
            if (p >= pend) break;
            p2 = next_poly(p + 1, pend, r, rpp, level, skip_gs);
            ld_strided<E>(v[0], row(p), lane);
            if (p2 < pend) ld_strided<E>(v[1], row(p2), lane);
        }
        return;
    }
    u64 v[E], nx[E];
    ld_strided<E>(v, row(p), lane);
    stage_chunk_twiddles<E, true>(sw, sws, w, w + N, logN1, blockIdx.x);
    __syncthreads();
    while (p < pend) {
        const u32 pn = next_poly(p + 1, pend, r, rpp, level, skip_gs);
        if (pn < pend) ld_strided<E>(nx, row(pn), lane);  // in flight during this poly's stages
        if (q < kSmallQ) {
            wfwd_all<E, true, true>(v, col, lane, sw, sws, q, warp);
            const u64 one = R.one_shoup[mi];
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = shoup(v[j], 1, one, q);  // < 33q -> canonical
        } else {
            wfwd_all<E, true, false>(v, col, lane, sw, sws, q, warp);
            const u64 q2 = 2 * q;
#pragma unroll
            for (int j = 0; j < E; ++j) {
                u64 t = v[j];
                if (t >= q2) t -= q2;
                if (t >= q) t -= q;
                v[j] = t;
            }
        }
        st_vec<E>(row(p), v, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = nx[j];
        p = pn;
    }
}

// Phase A inverse: one warp per contiguous chunk (stages t = 1 .. M2/2).
// Tensor mode (tx != nullptr; FP64 rows, unstaged path): the source chunk is
// the product tx * ty (Evaluator::mul's c2 = x1 y1, eval form, ckks.hpp:236),
// written to c2e (ModUp's own-group rows) and transformed straight away --
// c2 makes one trip through HBM instead of two (tg_tensor_c2_inverse). With a
// second pair (tu, tv: lazy relinearisation of two products) the chunk is
// tx * ty + tu * tv.
template <int E>
__global__ void __launch_bounds__(256, NTT_CHUNK_MIN_BLOCKS)
kw_inv_chunks(DevRing R, u64* data, const u64* src, u32 rpp, u32 npolys, u32 ppb, int level, u32 logN1,
              u32 row0, const u64* tx = nullptr, const u64* ty = nullptr, u64* c2e = nullptr,
              const u64* tu = nullptr, const u64* tv = nullptr, u64 sx = 0, u64 sy = 0, u64 su = 0, u64 sv = 0) {
    using Gm = WGeo<E>;
    // row r of every poly (rows [row0, row0 + gridDim.y) are transformed)
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = blockIdx.z * ppb;
    if (p >= pend) return;
    extern __shared__ __align__(16) u64 dyn[];
    u64* sm = dyn;
    u64* sw = dyn + 16 * Gm::CS;
    u64* sws = sw + Gm::TW_CHUNK;
    const u32 N = R.N;
    const u32 mi = mod_index(r, level, R.q_count);
    const u64 q = R.q[mi];
    const bool fp = ntt_use_fp(R, q, r);
    const u64* w = fp ? reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N + 2 * size_t(N))
                      : R.tw + size_t(mi) * 4 * N + 2 * size_t(N);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t off = size_t(blockIdx.x * 8 + warp) * Gm::M;
    u64* col = sm + warp * Gm::CS;
    u64* colp = sm + warp * 2 * Gm::CS;  // FP64 paths: the warp's contiguous pair region
    constexpr u32 CS2 = 8 * Gm::CS;
    auto in = [&](u32 pp) { return src + size_t(pp * rpp + r) * N + off; };
    auto out = [&](u32 pp) { return data + size_t(pp * rpp + r) * N + off; };
    if (fp && NTT_CHUNK_STAGE) {
        constexpr u32 SW = Gm::M + Gm::M / 4;
        u64* stg = dyn + 16 * Gm::CS + 2 * Gm::TW_CHUNK + warp * 2 * SW;
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
        stage_chunk<E, true>(stg, in(p), lane);
        if (p + 1 < pend) stage_chunk<E, true>(stg + SW, in(p + 1), lane);
        cp_async_commit();
        stage_chunk_twiddles<E, false>(sw, sws, w, w + N, logN1, blockIdx.x);
        __syncthreads();
        const u32 base = ipad(lane << Gm::LOGE);
        while (true) {
            const bool pair = p + 1 < pend;
            cp_async_wait<0>();
            __syncwarp();
            u64 v[2][E];
#pragma unroll
            for (int n = 0; n < 2; ++n) {
                if (n == 1 && !pair) break;
                const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(stg + n * SW + base);
#pragma unroll
                for (int j = 0; j < E / 2; ++j) {
                    const ulonglong2 t = s2[j];
                    v[n][2 * j] = t.x;
                    v[n][2 * j + 1] = t.y;
                }
            }
            __syncwarp();
            const u32 pn = p + (pair ? 2 : 1);
            if (pn < pend) {
                stage_chunk<E, true>(stg, in(pn), lane);
                if (pn + 1 < pend) stage_chunk<E, true>(stg + SW, in(pn + 1), lane);
            }
            cp_async_commit();
            if (pair) {
                chunk_inv_fp<2, E, true>(v, colp, CS2, lane, sw, qd, qi, warp, q);
                st_strided<E>(out(p), v[0], lane);
                st_strided<E>(out(p + 1), v[1], lane);
            } else {
                chunk_inv_fp<1, E>(reinterpret_cast<u64(&)[1][E]>(v[0]), colp, CS2, lane, sw, qd, qi, warp, q);
                st_strided<E>(out(p), v[0], lane);
            }
            if (pn >= pend) break;
            p = pn;
        }
        return;
    }
    if (fp) {
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1];
        u64 v[2][E];
        // (tensor mode) chunk of c2 = x1 y1: exact FP64 product, canonical,
        // stored for ModUp's own rows
        auto tload = [&](u64 (&t)[E], u32 pp) {
            const size_t o = size_t(pp * rpp + r) * N + off, ro = size_t(r) * N + off;
            u64 yv[E];  // operand polys: sx .. sv words apart (level-dropped views read in place)
            ld_vec<E>(t, tx + size_t(pp) * sx + ro, lane);
            ld_vec<E>(yv, ty + size_t(pp) * sy + ro, lane);
            if (tu) {  // x1 y1 + u1 v1: |sum| < 1.62q
                u64 uv[E], vv[E];
                ld_vec<E>(uv, tu + size_t(pp) * su + ro, lane);
                ld_vec<E>(vv, tv + size_t(pp) * sv + ro, lane);
#pragma unroll
                for (int j = 0; j < E; ++j)
                    t[j] = fp_canonical(__dadd_rn(fp_mulmod_qi(u2d(t[j]), u2d(yv[j]), qd, qi),
                                                  fp_mulmod_qi(u2d(uv[j]), u2d(vv[j]), qd, qi)),
                                        qd);
            } else {
#pragma unroll
                for (int j = 0; j < E; ++j) t[j] = fp_canonical1(fp_mulmod_qi(u2d(t[j]), u2d(yv[j]), qd, qi), qd);
            }
            st_vec<E>(c2e + o, t, lane);
        };
        auto load = [&](u64 (&t)[E], u32 pp) {
            if (tx) tload(t, pp);
            else ld_vec<E>(t, in(pp), lane);
        };
        load(v[0], p);
        if (p + 1 < pend) load(v[1], p + 1);
        stage_chunk_twiddles<E, false>(sw, sws, w, w + N, logN1, blockIdx.x);
        __syncthreads();
        while (true) {
            if (p + 1 < pend) {
                chunk_inv_fp<2, E, true>(v, colp, CS2, lane, sw, qd, qi, warp, q);
                st_strided<E>(out(p), v[0], lane);
                st_strided<E>(out(p + 1), v[1], lane);
                p += 2;
            } else {
                chunk_inv_fp<1, E>(reinterpret_cast<u64(&)[1][E]>(v[0]), colp, CS2, lane, sw, qd, qi, warp, q);
                st_strided<E>(out(p), v[0], lane);
                p += 1;
            }
            if (p >= pend) break;
            load(v[0], p);
            if (p + 1 < pend) load(v[1], p + 1);
        }
        return;
    }
    u64 v[E], nx[E];
    ld_vec<E>(v, in(p), lane);
    stage_chunk_twiddles<E, false>(sw, sws, w, w + N, logN1, blockIdx.x);
    __syncthreads();
    for (; p < pend; ++p) {
        if (p + 1 < pend) ld_vec<E>(nx, in(p + 1), lane);
        if (q < kSmallQ) {
            winv_all<E, true, true>(v, col, lane, sw, sws, q, warp);
            const u64 one = R.one_shoup[mi];
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = shoup_lazy(v[j], 1, one, q);  // < 512q -> [0, 2q)
        } else {
            winv_all<E, true, false>(v, col, lane, sw, sws, q, warp);
        }
        st_strided<E>(out(p), v, lane);
#pragma unroll
        for (int j = 0; j < E; ++j) v[j] = nx[j];
    }
}

// Phase B inverse: 8 columns x M1 rows, then the N^-1 scaling.
template <int E, int E2>
__global__ void __launch_bounds__(256, NTT_MIN_BLOCKS)
kw_inv_cols(DevRing R, u64* data, u32 rpp, u32 npolys, u32 ppb, int level, u32 row0) {
    using Gm = WGeo<E>;
    // row r of every poly (rows [row0, row0 + gridDim.y) are transformed)
    const u32 r = row0 + blockIdx.y, pend = min(npolys, (blockIdx.z + 1) * ppb);
    u32 p = blockIdx.z * ppb;
    if (p >= pend) return;
    extern __shared__ u64 dyn[];
    u64* tiles = dyn;
    u64* sw = dyn + 16 * Gm::CS;
    u64* sws = sw + Gm::TW_COL;
    constexpr u32 N = 32 * E * 32 * E2;  // == R.N (warp_plan)
    const u32 mi = mod_index(r, level, R.q_count);
    const u64 q = R.q[mi];
    const bool fp = ntt_use_fp(R, q, r);
    const u64* w = fp ? reinterpret_cast<const u64*>(R.twd + size_t(mi) * 4 * N + 2 * size_t(N))
                      : R.tw + size_t(mi) * 4 * N + 2 * size_t(N);
    const u64 ninv = R.ninv[2 * mi], ninv_s = R.ninv[2 * mi + 1];
    const u32 c0 = blockIdx.x * 8;
    issue_col_tile<E, 32 * E2>(tiles, data + size_t(p * rpp + r) * N + c0);
    stage_col_twiddles<E, false>(sw, sws, w, w + N);
    const u32 warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (fp && NTT_COLS_PAIR) {  // polys in pairs on the block's two tiles (see kw_fwd_cols)
        const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1], nd = R.qd[4 * mi + 2], ndq = R.qd[4 * mi + 3];
        for (bool first = true; p < pend; first = false) {
            const bool pair = p + 1 < pend;
            if (!first) issue_col_tile<E, 32 * E2>(tiles, data + size_t(p * rpp + r) * N + c0);
            if (pair) issue_col_tile<E, 32 * E2>(tiles + 8 * Gm::CS, data + size_t((p + 1) * rpp + r) * N + c0);
            cp_async_wait<0>();
            __syncthreads();
            u64* col = tiles + warp * Gm::CS;
            if (pair) {
                double v[2][E];
#pragma unroll
                for (int n = 0; n < 2; ++n) {
                    const double* cold = reinterpret_cast<const double*>(col + n * 8 * Gm::CS);
#pragma unroll
                    for (int j = 0; j < E; ++j) v[n][j] = cold[wpad((lane << Gm::LOGE) | j)];
                }
                winv_all_fp<2, E, false>(v, col, 8 * Gm::CS, lane, sw, qd, qi, 0);
                __syncwarp();
#pragma unroll
                for (int n = 0; n < 2; ++n)
#pragma unroll
                    for (int j = 0; j < E; ++j)
                        col[n * 8 * Gm::CS + wpad(lane + 32 * j)] = fp_canon_small(fp_mulmod(v[n][j], nd, ndq, qd), q);
            } else {
                const double* cold = reinterpret_cast<const double*>(col);
                double v[1][E];
#pragma unroll
                for (int j = 0; j < E; ++j) v[0][j] = cold[wpad((lane << Gm::LOGE) | j)];
                winv_all_fp<1, E, false>(v, col, 0, lane, sw, qd, qi, 0);
                __syncwarp();
#pragma unroll
                for (int j = 0; j < E; ++j) col[wpad(lane + 32 * j)] = fp_canon_small(fp_mulmod(v[0][j], nd, ndq, qd), q);
            }
            __syncthreads();
            store_col_tile<E, 32 * E2>(tiles, data + size_t(p * rpp + r) * N + c0);
            if (pair) store_col_tile<E, 32 * E2>(tiles + 8 * Gm::CS, data + size_t((p + 1) * rpp + r) * N + c0);
            __syncthreads();
            p += pair ? 2 : 1;
        }
        return;
    }
    u32 cur = 0;
    for (; p < pend; ++p) {
        if (p + 1 < pend) {
            issue_col_tile<E, 32 * E2>(tiles + (cur ^ 1) * 8 * Gm::CS, data + size_t((p + 1) * rpp + r) * N + c0);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        u64* tile = tiles + cur * 8 * Gm::CS;
        u64* col = tile + warp * Gm::CS;
        if (fp) {  // phase-A doubles in, canonical u64 out (N^-1 applied in FP64)
            const double qd = R.qd[4 * mi], qi = R.qd[4 * mi + 1], nd = R.qd[4 * mi + 2], ndq = R.qd[4 * mi + 3];
            const double* cold = reinterpret_cast<const double*>(col);
            double v[1][E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[0][j] = cold[wpad((lane << Gm::LOGE) | j)];
            winv_all_fp<1, E, false>(v, col, 0, lane, sw, qd, qi, 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < E; ++j) col[wpad(lane + 32 * j)] = fp_canon_small(fp_mulmod(v[0][j], nd, ndq, qd), q);
        } else {
            u64 v[E];
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = col[wpad((lane << Gm::LOGE) | j)];
            if (q < kSmallQ) winv_all<E, false, true>(v, col, lane, sw, sws, q, 0);
            else winv_all<E, false, false>(v, col, lane, sw, sws, q, 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < E; ++j) col[wpad(lane + 32 * j)] = shoup(v[j], ninv, ninv_s, q);
        }
        __syncthreads();
        store_col_tile<E, 32 * E2>(tile, data + size_t(p * rpp + r) * N + c0);
        __syncthreads();  // the tile is the next prefetch target
        cur ^= 1;
    }
}

#include "tg_ntt_cols2.cuh"

// (E1, E2) for N = M1 * M2 handled by the warp kernels.
inline bool warp_plan(u32 logN, int& e1, int& e2) {
    switch (logN) {
        case 16: e1 = 8; e2 = 8; return true;
        case 15: e1 = 4; e2 = 8; return true;
        case 14: e1 = 4; e2 = 4; return true;
        default: return false;
    }
}

// TMA descriptor of a buffer of u64 rows viewed as [rows * M1][M2] (column
// index innermost, 2 KB row stride at N = 2^16), box 16 columns x M1 rows,
// 128-byte swizzle. cuTensorMapEncodeTiled comes from the driver through the
// runtime's entry-point query (no -lcuda); false if unavailable.
inline bool encode_col_tmap(CUtensorMap* m, const void* base, u64 matrix_rows, u32 cols, u32 box_rows) {
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<Encode>(f);
    }();
    if (!fn) return false;
    const cuuint64_t dims[2] = {cols, matrix_rows};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 8};
    const cuuint32_t box[2] = {16, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

inline bool ntt_tma_on() {
    static const bool on = [] {
        const char* e = getenv("TG_NTT_TMA");
        return !(e && *e == '0');
    }();
    return on;
}

template <int E1, int E2>
void set_smem_attrs() {
    // thread-safe one-time init (one process drives one device)
    static const bool done = [] {
        cudaFuncSetAttribute(kw_fwd_cols<E1, E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(col_smem<E1>()));
        cudaFuncSetAttribute(kw_inv_cols<E1, E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(col_smem<E1>()));
        cudaFuncSetAttribute(kw_fwd_chunks<E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(chunk_smem<E2>()));
        cudaFuncSetAttribute(kw_inv_chunks<E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(chunk_smem<E2>()));
        cudaFuncSetAttribute(kw_fwd_cols2<E1, E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pair_smem<E1>()));
        cudaFuncSetAttribute(kw_inv_cols2<E1, E2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(pair_smem<E1>()));
        cudaFuncSetAttribute(kw_inv_cols2<E1, E2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(pair_smem<E1>()));
        cudaFuncSetAttribute(kw_fwd_cols2_tma<E1, E2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(pair_tma_smem<E1>()));
        return true;
    }();
    (void)done;
}

// Polys per block: keep at least ~4 blocks per SM in the grid, otherwise let
// each block walk as many polys as possible (twiddle reuse, prefetch).
inline u32 polys_per_block(u32 blocks_per_row, u32 rpp, u32 npolys, int sms) {
    const u64 one = u64(blocks_per_row) * rpp * npolys, target = u64(sms) * 4;
    const u64 ppb = one / target;
    return u32(ppb < 1 ? 1 : ppb > npolys ? npolys : ppb);
}

// Column phases: the column-pair kernels when every row is FP64 (pair).
template <int E1, int E2>
void launch_fwd_cols_any(const DevRing& R, int sms, u64* data, const u64* src, u32 rpp, u32 npolys, int level,
                         cudaStream_t s, u32 skip_gs, u32 row0, u32 nrows, bool pair) {
    set_smem_attrs<E1, E2>();
    const u32 M2 = 32 * E2;
    if (pair && E1 == 8) {  // column pairs (tg_ntt_cols2.cuh), N = 2^16
        const u32 p1 = polys_per_block(M2 / 16, nrows, npolys, sms);
        CUtensorMap tm;
        if (ntt_tma_on() && encode_col_tmap(&tm, src, u64(rpp) * npolys * (32 * E1), M2, 32 * E1)) {
            kw_fwd_cols2_tma<E1, E2><<<dim3(M2 / 16, nrows, (npolys + p1 - 1) / p1), 256, pair_tma_smem<E1>(), s>>>(
                tm, R, data, rpp, npolys, p1, level, skip_gs, row0);
            return;
        }
        kw_fwd_cols2<E1, E2><<<dim3(M2 / 16, nrows, (npolys + p1 - 1) / p1), 256, pair_smem<E1>(), s>>>(
            R, data, src, rpp, npolys, p1, level, skip_gs, row0);
        return;
    }
    const u32 p1 = polys_per_block(M2 / 8, nrows, npolys, sms);
    kw_fwd_cols<E1, E2><<<dim3(M2 / 8, nrows, (npolys + p1 - 1) / p1), 256, col_smem<E1>(), s>>>(
        R, data, src, rpp, npolys, p1, level, skip_gs, row0);
}
template <int E1, int E2>
void launch_inv_cols_any(const DevRing& R, int sms, u64* data, u32 rpp, u32 npolys, int level, cudaStream_t s,
                         u32 row0, u32 nrows, bool pair, bool raw = false) {
    set_smem_attrs<E1, E2>();
    const u32 M2 = 32 * E2;
    if (pair && E1 == 8) {
        const u32 p1 = polys_per_block(M2 / 16, nrows, npolys, sms);
        const dim3 grid(M2 / 16, nrows, (npolys + p1 - 1) / p1);
        if (raw) kw_inv_cols2<E1, E2, true><<<grid, 256, pair_smem<E1>(), s>>>(R, data, rpp, npolys, p1, level, row0);
        else kw_inv_cols2<E1, E2><<<grid, 256, pair_smem<E1>(), s>>>(R, data, rpp, npolys, p1, level, row0);
        return;
    }
    const u32 p1 = polys_per_block(M2 / 8, nrows, npolys, sms);
    kw_inv_cols<E1, E2><<<dim3(M2 / 8, nrows, (npolys + p1 - 1) / p1), 256, col_smem<E1>(), s>>>(R, data, rpp, npolys,
                                                                                           p1, level, row0);
}

template <int E1, int E2>
void launch_fwd_w(const DevRing& R, int sms, u64* data, const u64* src, u32 rpp, u32 npolys, int level,
                  cudaStream_t s, u32 skip_gs, u32 row0, u32 nrows, bool pair = false) {
    set_smem_attrs<E1, E2>();
    const u32 M1 = 32 * E1;
    const u32 p2 = polys_per_block(M1 / 8, nrows, npolys, sms);
    launch_fwd_cols_any<E1, E2>(R, sms, data, src, rpp, npolys, level, s, skip_gs, row0, nrows, pair);
    kw_fwd_chunks<E2><<<dim3(M1 / 8, nrows, (npolys + p2 - 1) / p2), 256, chunk_smem<E2>(), s>>>(
        R, data, rpp, npolys, p2, level, WGeo<E1>::LOGM, skip_gs, row0);
}

// c2 = x1 y1 (written to c2e) and its inverse transform into data (level+1
// rows per poly; every row FP64, unstaged chunk phase)
template <int E1, int E2>
void launch_inv_tensor_w(const DevRing& R, int sms, u64* data, u64* c2e, const u64* x1, const u64* y1, u32 npolys,
                         int level, cudaStream_t s, bool pair, bool raw = false, const u64* u1 = nullptr,
                         const u64* v1 = nullptr, const u64* st = nullptr) {
    set_smem_attrs<E1, E2>();
    const u32 M1 = 32 * E1, rpp = u32(level) + 1;
    const u32 p2 = polys_per_block(M1 / 8, rpp, npolys, sms);
    kw_inv_chunks<E2><<<dim3(M1 / 8, rpp, (npolys + p2 - 1) / p2), 256, chunk_smem<E2>(), s>>>(
        R, data, nullptr, rpp, npolys, p2, level, WGeo<E1>::LOGM, 0, x1, y1, c2e, u1, v1, st ? st[0] : u64(rpp) * R.N,
        st ? st[1] : u64(rpp) * R.N, st ? st[2] : u64(rpp) * R.N, st ? st[3] : u64(rpp) * R.N);
    launch_inv_cols_any<E1, E2>(R, sms, data, rpp, npolys, level, s, 0, rpp, pair, raw);
}

template <int E1, int E2>
void launch_inv_w(const DevRing& R, int sms, u64* data, const u64* src, u32 rpp, u32 npolys, int level,
                  cudaStream_t s, u32 row0, u32 nrows, bool pair = false) {
    set_smem_attrs<E1, E2>();
    const u32 M1 = 32 * E1;
    const u32 p2 = polys_per_block(M1 / 8, nrows, npolys, sms);
    kw_inv_chunks<E2><<<dim3(M1 / 8, nrows, (npolys + p2 - 1) / p2), 256, chunk_smem<E2>(), s>>>(
        R, data, src, rpp, npolys, p2, level, WGeo<E1>::LOGM, row0);
    launch_inv_cols_any<E1, E2>(R, sms, data, rpp, npolys, level, s, row0, nrows, pair);
}
