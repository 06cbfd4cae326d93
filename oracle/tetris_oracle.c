/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement oracle (see tetris_oracle.h).
 * Straight-line scalar C, u128 `%` for every modular product: deliberately
 * the simplest correct restatement, not a fast one.
 */
#include "tetris_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef uint32_t u32;
typedef int64_t i64;

static u64 addm(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static u64 subm(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 mulm(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 powm(u64 b, u64 e, u64 q) {
    u64 r = 1;
    b %= q;
    while (e) {
        if (e & 1) r = mulm(r, b, q);
        b = mulm(b, b, q);
        e >>= 1;
    }
    return r;
}
static u64 invm(u64 a, u64 q) { return powm(a % q, q - 2, q); }
static u64 shoup_pre(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 shoup_mul(u64 a, u64 w, u64 ws, u64 q) { /* common.hpp:46-50 */
    u64 hi = (u64)(((u128)a * ws) >> 64);
    u64 r = a * w - hi * q;
    return r >= q ? r - q : r;
}
static i64 centered(u64 x, u64 q) { return x > q / 2 ? (i64)x - (i64)q : (i64)x; } /* common.hpp:84-86 */
static u64 uncentered(i64 x, u64 q) {                                               /* common.hpp:88-92 */
    i64 r = x % (i64)q;
    if (r < 0) r += (i64)q;
    return (u64)r;
}

/* ---------------- RNG (common.hpp:154-210) ---------------- */
u64 or_splitmix64(u64 x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* mt19937_64 (Matsumoto & Nishimura), the engine std::mt19937_64 specifies */
static void mt_seed(or_rng* r, u64 s) {
    r->mt[0] = s;
    for (int i = 1; i < 312; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (u64)i;
    r->mti = 312;
}
static u64 mt_next(or_rng* r) {
    static const u64 mag[2] = {0ULL, 0xB5026F5AA96619E9ULL};
    if (r->mti >= 312) {
        int i;
        u64 x;
        for (i = 0; i < 312 - 156; ++i) {
            x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ mag[x & 1];
        }
        for (; i < 311; ++i) {
            x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[i + 1] & 0x7FFFFFFFULL);
            r->mt[i] = r->mt[i + (156 - 312)] ^ (x >> 1) ^ mag[x & 1];
        }
        x = (r->mt[311] & 0xFFFFFFFF80000000ULL) | (r->mt[0] & 0x7FFFFFFFULL);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ mag[x & 1];
        r->mti = 0;
    }
    u64 y = r->mt[r->mti++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    return y;
}

void or_rng_init(or_rng* r, u64 seed) {
    r->seed = seed;
    r->have_spare = 0;
    r->spare = 0;
    mt_seed(r, or_splitmix64(seed));
}
u64 or_rng_next(or_rng* r) { return mt_next(r); }
u64 or_rng_uniform(or_rng* r, u64 bound) {
    u64 thr = (0 - bound) % bound;
    for (;;) {
        u64 x = mt_next(r);
        if (x >= thr) return x % bound;
    }
}
double or_rng_normal(or_rng* r) {
    if (r->have_spare) {
        r->have_spare = 0;
        return r->spare;
    }
    double u1 = ((double)(mt_next(r) >> 11) + 1.0) * 0x1p-53;
    double u2 = ((double)(mt_next(r) >> 11) + 1.0) * 0x1p-53;
    double rad = sqrt(-2.0 * log(u1));
    double th = 6.283185307179586476925 * u2;
    r->spare = rad * sin(th);
    r->have_spare = 1;
    return rad * cos(th);
}
void or_rng_split(const or_rng* r, u64 label, or_rng* child) {
    or_rng_init(child, or_splitmix64(r->seed ^ or_splitmix64(label ^ 0xa5a5a5a55a5a5a5aULL)));
}

/* ---------------- primes (common.hpp:103-147) ---------------- */
int or_is_prime(u64 n) {
    static const u64 B[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; ++i)
        if (n % B[i] == 0) return n == B[i];
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) {
        d >>= 1;
        ++s;
    }
    for (int k = 0; k < 12; ++k) {
        u64 x = powm(B[k], d, n);
        if (x == 1 || x == n - 1) continue;
        int wit = 1;
        for (int i = 1; i < s; ++i) {
            x = mulm(x, x, n);
            if (x == n - 1) {
                wit = 0;
                break;
            }
        }
        if (wit) return 0;
    }
    return 1;
}

static int taken(u64 p, const u64* ex, int nex, const u64* out, int nout) {
    for (int i = 0; i < nex; ++i)
        if (ex[i] == p) return 1;
    for (int i = 0; i < nout; ++i)
        if (out[i] == p) return 1;
    return 0;
}

int or_find_ntt_primes(int bits, int count, u64 modulus, const u64* ex, int nex, u64* out) {
    u64 center = 1ULL << bits;
    u64 lo = center - (center % modulus) + 1, hi = lo + modulus;
    int n = 0;
    while (n < count) {
        if (lo > modulus && or_is_prime(lo) && !taken(lo, ex, nex, out, n)) out[n++] = lo;
        if (n >= count) break;
        if (or_is_prime(hi) && !taken(hi, ex, nex, out, n)) out[n++] = hi;
        lo -= modulus;
        hi += modulus;
        if (hi - center > (center >> 2)) break;
    }
    return n;
}

/* ---------------- NTT (ring.hpp:25-101) ---------------- */
static u32 brev(u32 x, u32 bits) {
    u32 r = 0;
    for (u32 i = 0; i < bits; ++i, x >>= 1) r = (r << 1) | (x & 1);
    return r;
}

void or_ntt_tables(u64 q, u32 n, u32 idx, u64* psi_out, u64* w, u64* ws, u64* winv, u64* winvs, u64* ninv2) {
    u32 logn = 0;
    while ((1u << logn) < n) ++logn;
    or_rng root, r;
    or_rng_init(&root, 0x7e7215a1d2c3ULL);
    or_rng_split(&root, idx, &r);
    u64 psi;
    do {
        u64 x = or_rng_uniform(&r, q - 2) + 2;
        psi = powm(x, (q - 1) / (2 * (u64)n), q);
    } while (powm(psi, n, q) != q - 1);
    u64 pinv = invm(psi, q);
    for (u32 i = 0; i < n; ++i) {
        u32 e = brev(i, logn);
        w[i] = powm(psi, e, q);
        winv[i] = powm(pinv, e, q);
        ws[i] = shoup_pre(w[i], q);
        winvs[i] = shoup_pre(winv[i], q);
    }
    ninv2[0] = invm(n, q);
    ninv2[1] = shoup_pre(ninv2[0], q);
    *psi_out = psi;
}

void or_ntt_forward(u64* a, u32 n, u64 q, const u64* w, const u64* ws) {
    u32 t = n;
    for (u32 m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (u32 i = 0; i < m; ++i) {
            u64* x = a + 2 * i * t;
            for (u32 j = 0; j < t; ++j) {
                u64 u = x[j], v = shoup_mul(x[j + t], w[m + i], ws[m + i], q);
                x[j] = addm(u, v, q);
                x[j + t] = subm(u, v, q);
            }
        }
    }
}

void or_ntt_inverse(u64* a, u32 n, u64 q, const u64* winv, const u64* winvs, const u64* ninv2) {
    u32 t = 1;
    for (u32 m = n; m > 1; m >>= 1) {
        u32 h = m >> 1;
        for (u32 i = 0; i < h; ++i) {
            u64* x = a + 2 * i * t;
            for (u32 j = 0; j < t; ++j) {
                u64 u = x[j], v = x[j + t];
                x[j] = addm(u, v, q);
                x[j + t] = shoup_mul(subm(u, v, q), winv[h + i], winvs[h + i], q);
            }
        }
        t <<= 1;
    }
    for (u32 j = 0; j < n; ++j) a[j] = shoup_mul(a[j], ninv2[0], ninv2[1], q);
}

void or_eval_order(u32 n, u64 q0, const u64* w0, const u64* ws0, u64 psi0, u32* eval_exp, u32* slot_of_exp) {
    u64* a = calloc(n, 8);
    u64* pw = malloc(2 * (size_t)n * 8);
    a[1] = 1;
    or_ntt_forward(a, n, q0, w0, ws0);
    u64 v = 1;
    for (u32 e = 0; e < 2 * n; ++e) {
        pw[e] = v;
        slot_of_exp[e] = (u32)-1;
        v = mulm(v, psi0, q0);
    }
    for (u32 j = 0; j < n; ++j)
        for (u32 e = 0; e < 2 * n; ++e)
            if (pw[e] == a[j]) {
                eval_exp[j] = e;
                slot_of_exp[e] = j;
                break;
            }
    free(a);
    free(pw);
}

/* ---------------- element-wise (ring.hpp:250-325) ---------------- */
void or_poly_add(u64* out, const u64* a, const u64* b, const u64* mod, int rows, u32 n) {
    for (int r = 0; r < rows; ++r)
        for (u32 i = 0; i < n; ++i) out[(size_t)r * n + i] = addm(a[(size_t)r * n + i], b[(size_t)r * n + i], mod[r]);
}
void or_poly_sub(u64* out, const u64* a, const u64* b, const u64* mod, int rows, u32 n) {
    for (int r = 0; r < rows; ++r)
        for (u32 i = 0; i < n; ++i) out[(size_t)r * n + i] = subm(a[(size_t)r * n + i], b[(size_t)r * n + i], mod[r]);
}
void or_poly_neg(u64* out, const u64* a, const u64* mod, int rows, u32 n) {
    for (int r = 0; r < rows; ++r)
        for (u32 i = 0; i < n; ++i) {
            u64 x = a[(size_t)r * n + i];
            out[(size_t)r * n + i] = x ? mod[r] - x : 0;
        }
}
void or_poly_mul(u64* out, const u64* a, const u64* b, const u64* mod, int rows, u32 n) {
    for (int r = 0; r < rows; ++r)
        for (u32 i = 0; i < n; ++i) out[(size_t)r * n + i] = mulm(a[(size_t)r * n + i], b[(size_t)r * n + i], mod[r]);
}
void or_poly_mul_scalar(u64* out, const u64* a, const u64* scalar, const u64* mod, int rows, u32 n) {
    for (int r = 0; r < rows; ++r) {
        u64 s = scalar[r] % mod[r], ss = shoup_pre(s, mod[r]);
        for (u32 i = 0; i < n; ++i) out[(size_t)r * n + i] = shoup_mul(a[(size_t)r * n + i], s, ss, mod[r]);
    }
}

void or_automorphism(u64* out, const u64* in, u64 g, int eval_form, const u64* mod, int rows, u32 n,
                     const u32* eval_exp, const u32* slot_of_exp) {
    u64 two_n = 2 * (u64)n;
    g %= two_n;
    for (int r = 0; r < rows; ++r) {
        const u64* a = in + (size_t)r * n;
        u64* b = out + (size_t)r * n;
        if (!eval_form) {
            for (u32 i = 0; i < n; ++i) {
                u64 j = ((u64)i * g) % two_n;
                if (j < n) b[j] = a[i];
                else b[j - n] = a[i] ? mod[r] - a[i] : 0;
            }
        } else {
            for (u32 j = 0; j < n; ++j) b[j] = a[slot_of_exp[(u32)(((u64)eval_exp[j] * g) % two_n)]];
        }
    }
}

void or_rescale(u64* out, const u64* in, const u64* moduli, int level, u32 n) {
    u64 ql = moduli[level], half = ql >> 1;
    const u64* last = in + (size_t)level * n;
    for (int r = 0; r < level; ++r) {
        u64 q = moduli[r], qlq = ql % q, inv = invm(qlq, q), invs = shoup_pre(inv, q);
        for (u32 i = 0; i < n; ++i) {
            u64 t = last[i] % q;
            if (last[i] > half) t = subm(t, qlq, q);
            out[(size_t)r * n + i] = shoup_mul(subm(in[(size_t)r * n + i], t, q), inv, invs, q);
        }
    }
}

/* ---------------- key switching (rlwe.hpp) ---------------- */
static u64 row_modulus(const u64* moduli, int nq, int level, int r) { return moduli[r <= level ? r : nq + (r - level - 1)]; }

int or_modup(u64* digits, const u64* d, const u64* moduli, int nq, int K, int group, int level, u32 n) {
    int ngroups = (level + group) / group; /* group_count (rlwe.hpp:50-52) */
    int rows = level + 1 + K;
    for (int j = 0; j < ngroups; ++j) {
        int first = j * group;
        int cnt = nq - first < group ? nq - first : group;
        int active = cnt < level + 1 - first ? cnt : level + 1 - first;
        u64* dig = digits + (size_t)j * rows * n;
        memset(dig, 0, (size_t)rows * n * 8);
        for (int i = 0; i < active; ++i) {
            int src = first + i;
            u64 q = moduli[src], rest = 1;
            for (int t = 0; t < active; ++t)
                if (t != i) rest = mulm(rest, moduli[first + t] % q, q);
            u64 sc = invm(rest, q), scs = shoup_pre(sc, q);
            for (int r = 0; r < rows; ++r) {
                u64 qt = row_modulus(moduli, nq, level, r), w = 1;
                for (int u = 0; u < active; ++u)
                    if (u != i) w = mulm(w, moduli[first + u] % qt, qt);
                u64 wsh = shoup_pre(w, qt);
                for (u32 c = 0; c < n; ++c) {
                    u64 y = shoup_mul(d[(size_t)src * n + c], sc, scs, q);
                    dig[(size_t)r * n + c] = addm(dig[(size_t)r * n + c], shoup_mul(y % qt, w, wsh, qt), qt);
                }
            }
        }
    }
    return ngroups;
}

void or_key_inner(u64* acc0, u64* acc1, const u64* digits, int nd, const u64* const* key_b, const u64* const* key_a,
                  const u64* moduli, int nq, int K, int level, u32 n) {
    int rows = level + 1 + K;
    for (int r = 0; r < rows; ++r) {
        int m = r <= level ? r : nq + (r - level - 1);
        u64 q = moduli[m];
        for (u32 c = 0; c < n; ++c) {
            u128 s0 = 0, s1 = 0;
            for (int i = 0; i < nd; ++i) {
                u128 dv = digits[((size_t)i * rows + r) * n + c];
                s0 += dv * key_b[i][(size_t)m * n + c];
                s1 += dv * key_a[i][(size_t)m * n + c];
            }
            acc0[(size_t)r * n + c] = (u64)(s0 % q);
            acc1[(size_t)r * n + c] = (u64)(s1 % q);
        }
    }
}

void or_mod_down(u64* out, const u64* in, const u64* moduli, int nq, int K, int level, u32 n) {
    i64* y = malloc((size_t)K * n * sizeof(i64));
    for (int s = 0; s < K; ++s) {
        u64 ps = moduli[nq + s], rest = 1;
        for (int t = 0; t < K; ++t)
            if (t != s) rest = mulm(rest, moduli[nq + t] % ps, ps);
        u64 c = invm(rest, ps), cs = shoup_pre(c, ps);
        for (u32 i = 0; i < n; ++i) y[(size_t)s * n + i] = centered(shoup_mul(in[(size_t)(level + 1 + s) * n + i], c, cs, ps), ps);
    }
    for (int r = 0; r <= level; ++r) {
        u64 q = moduli[r], pinv = 1;
        for (int s = 0; s < K; ++s) pinv = mulm(pinv, moduli[nq + s] % q, q);
        pinv = invm(pinv, q);
        u64 pinvs = shoup_pre(pinv, q);
        for (u32 i = 0; i < n; ++i) {
            u64 conv = 0;
            for (int s = 0; s < K; ++s) {
                u64 ws = 1;
                for (int t = 0; t < K; ++t)
                    if (t != s) ws = mulm(ws, moduli[nq + t] % q, q);
                conv = addm(conv, mulm(uncentered(y[(size_t)s * n + i], q), ws, q), q);
            }
            out[(size_t)r * n + i] = shoup_mul(subm(in[(size_t)r * n + i], conv, q), pinv, pinvs, q);
        }
    }
    free(y);
}
