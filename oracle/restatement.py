"""TEST INFRASTRUCTURE ONLY — CPU restatement oracle, Python side.

Thin ctypes layer over oracle/_ref/libtetris_oracle.so (the plain-C
restatement, oracle/tetris_oracle.c) plus the evaluator-level composition of
the reference (ckks.hpp:195-615, rlwe.hpp:501-654, threshold.hpp:114-157)
restated over numpy residue arrays. Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg may import this, as the checker.

Pinned by tests/test_oracle_golden.py against golden vectors produced by the
compiled, unmodified reference (tests/golden/gen_golden.py).
"""
from __future__ import annotations

import ctypes
import math
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libtetris_oracle.so"

_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-s", "-C", str(HERE), "restatement"], check=True)
        L = ctypes.CDLL(str(LIB))
        L.or_ntt_tables.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, _u64p, _u64p, _u64p, _u64p,
                                    _u64p, _u64p]
        L.or_ntt_forward.argtypes = [_u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p, _u64p]
        L.or_ntt_inverse.argtypes = [_u64p, ctypes.c_uint32, ctypes.c_uint64, _u64p, _u64p, _u64p]
        L.or_eval_order.argtypes = [ctypes.c_uint32, ctypes.c_uint64, _u64p, _u64p, ctypes.c_uint64, _u32p, _u32p]
        for f in ("or_poly_add", "or_poly_sub", "or_poly_mul"):
            getattr(L, f).argtypes = [_u64p, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_uint32]
        L.or_poly_neg.argtypes = [_u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_uint32]
        L.or_poly_mul_scalar.argtypes = [_u64p, _u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_uint32]
        L.or_automorphism.argtypes = [_u64p, _u64p, ctypes.c_uint64, ctypes.c_int, _u64p, ctypes.c_int,
                                      ctypes.c_uint32, _u32p, _u32p]
        L.or_rescale.argtypes = [_u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_uint32]
        L.or_modup.argtypes = [_u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_uint32]
        L.or_modup.restype = ctypes.c_int
        L.or_key_inner.argtypes = [_u64p, _u64p, _u64p, ctypes.c_int, ctypes.POINTER(_u64p), ctypes.POINTER(_u64p),
                                   _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32]
        L.or_mod_down.argtypes = [_u64p, _u64p, _u64p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint32]
        L.or_find_ntt_primes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, _u64p, ctypes.c_int, _u64p]
        L.or_find_ntt_primes.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data_as(_u64p)


def _p32(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(_u32p)


def find_ntt_primes(bits, count, modulus, exclude=()):
    ex = np.array(list(exclude) or [0], dtype=np.uint64)
    out = np.zeros(count, dtype=np.uint64)
    n = lib().or_find_ntt_primes(bits, count, modulus, _p(ex), len(exclude), _p(out))
    return [int(x) for x in out[:n]]


def round_half_away(x: float) -> int:
    """llround semantics (common.hpp:95-97) for doubles."""
    a = abs(x)
    if a >= 2.0 ** 52:
        return int(x)
    r = math.floor(a)
    if a - r >= 0.5:  # exact: a < 2^52
        r += 1
    return int(r) if x >= 0 else -int(r)


def from_centered(v: int, q: int) -> int:
    return v % q


class Ring:
    """RingParams restated: NTT tables built by the C oracle (ring.hpp:118-140)."""

    def __init__(self, N: int, moduli, special_count: int):
        L = lib()
        self.N, self.moduli, self.K = N, [int(m) for m in moduli], special_count
        self.nq = len(self.moduli) - special_count
        self.tab = []
        for i, q in enumerate(self.moduli):
            w, ws, wi, wis = (np.zeros(N, np.uint64) for _ in range(4))
            ni = np.zeros(2, np.uint64)
            psi = ctypes.c_uint64()
            L.or_ntt_tables(q, N, i, ctypes.byref(psi), _p(w), _p(ws), _p(wi), _p(wis), _p(ni))
            self.tab.append(dict(q=q, psi=psi.value, w=w, w_shoup=ws, winv=wi, winv_shoup=wis, n_inv=int(ni[0]),
                                 n_inv_shoup=int(ni[1]), ni=ni))
        self.eval_exp = np.zeros(N, np.uint32)
        self.slot_of_exp = np.zeros(2 * N, np.uint32)
        t0 = self.tab[0]
        L.or_eval_order(N, t0["q"], _p(t0["w"]), _p(t0["w_shoup"]), t0["psi"], _p32(self.eval_exp),
                        _p32(self.slot_of_exp))

    def mod_index(self, r, level):
        return r if r <= level else self.nq + (r - level - 1)

    def row_moduli(self, level, nspecial=0):
        return np.array([self.moduli[self.mod_index(r, level)] for r in range(level + 1 + nspecial)], np.uint64)

    def ntt(self, a: np.ndarray, level: int, nspecial: int = 0, inverse: bool = False) -> np.ndarray:
        out = np.ascontiguousarray(a, dtype=np.uint64).copy()
        L = lib()
        for r in range(out.shape[0]):
            t = self.tab[self.mod_index(r, level)]
            row = out[r]
            if inverse:
                L.or_ntt_inverse(_p(row), self.N, t["q"], _p(t["winv"]), _p(t["winv_shoup"]), _p(t["ni"]))
            else:
                L.or_ntt_forward(_p(row), self.N, t["q"], _p(t["w"]), _p(t["w_shoup"]))
        return out


def _binop(fn, a, b, mods):
    out = np.empty_like(a)
    fn(_p(out), _p(np.ascontiguousarray(a)), _p(np.ascontiguousarray(b)), _p(mods), a.shape[0], a.shape[1])
    return out


@dataclass
class OCt:
    """Oracle ciphertext: parts as (rows, N) uint64 arrays + reference metadata."""
    parts: list
    level: int
    form: str  # "coeff" | "eval"
    scale: float
    domain: int = 1
    sk_id: int = 0
    noise_bound: float = 0.0

    def copy(self):
        return OCt([p.copy() for p in self.parts], self.level, self.form, self.scale, self.domain, self.sk_id,
                   self.noise_bound)


@dataclass
class OKey:
    """Switching key: b[i], a[i] as (nq+K, N) eval-form arrays."""
    b: list
    a: list
    to_id: int = 0


class Evaluator:
    """Evaluator restated over the C primitives (ckks.hpp:181-335)."""

    def __init__(self, ring: Ring, group: int):
        self.R, self.group = ring, group

    # --- form / level helpers (rlwe.hpp:287-298) ---
    def to_coeff(self, ct: OCt):
        if ct.form == "eval":
            ct.parts = [self.R.ntt(p, ct.level, inverse=True) for p in ct.parts]
            ct.form = "coeff"

    def to_eval(self, ct: OCt):
        if ct.form == "coeff":
            ct.parts = [self.R.ntt(p, ct.level) for p in ct.parts]
            ct.form = "eval"

    def drop(self, ct: OCt, lvl: int):
        ct.parts = [p[:lvl + 1].copy() for p in ct.parts]
        ct.level = lvl

    def align(self, a: OCt, b: OCt):
        lvl = min(a.level, b.level)
        for c in (a, b):
            if c.level != lvl:
                self.to_coeff(c)
                self.drop(c, lvl)

    @staticmethod
    def check_scales(a, b):
        if abs(a / b - 1.0) > 1e-4:
            raise RuntimeError("[ckks] scaling factors diverged beyond tolerance")

    def _addsub(self, a: OCt, b: OCt, sub: bool) -> OCt:
        x, y = a.copy(), b.copy()
        self.align(x, y)
        self.check_scales(x.scale, y.scale)
        if x.form != y.form:
            self.to_coeff(x)
            self.to_coeff(y)
        mods = self.R.row_moduli(x.level)
        f = lib().or_poly_sub if sub else lib().or_poly_add
        x.parts = [_binop(f, p, q, mods) for p, q in zip(x.parts, y.parts)]
        x.noise_bound += y.noise_bound
        return x

    def add(self, a, b):
        return self._addsub(a, b, False)

    def sub(self, a, b):
        return self._addsub(a, b, True)

    def add_inplace_raw(self, x: OCt, y: OCt, sub=False):
        mods = self.R.row_moduli(x.level)
        f = lib().or_poly_sub if sub else lib().or_poly_add
        x.parts = [_binop(f, p, q, mods) for p, q in zip(x.parts, y.parts)]
        x.noise_bound += y.noise_bound

    # --- products (ckks.hpp:220-283) ---
    def mul(self, a: OCt, b: OCt) -> OCt:
        x, y = a.copy(), b.copy()
        self.align(x, y)
        if x.level == 0:
            raise RuntimeError("[ckks] exhausted ciphertext: no level left to rescale")
        self.to_eval(x)
        self.to_eval(y)
        mods = self.R.row_moduli(x.level)
        mul, add = lib().or_poly_mul, lib().or_poly_add
        p0 = _binop(mul, x.parts[0], y.parts[0], mods)
        p1 = _binop(add, _binop(mul, x.parts[0], y.parts[1], mods), _binop(mul, x.parts[1], y.parts[0], mods), mods)
        p2 = _binop(mul, x.parts[1], y.parts[1], mods)
        return OCt([p0, p1, p2], x.level, "eval", x.scale * y.scale, x.domain, x.sk_id,
                   x.noise_bound * y.scale + y.noise_bound * x.scale)

    def mul_scalar(self, ct: OCt, c: float, scalar_scale: float) -> OCt:
        if abs(c) * scalar_scale >= 9.0e18:
            raise RuntimeError("[ckks] scalar multiplier exceeds the integer range")
        v = round_half_away(c * scalar_scale)
        out = ct.copy()
        mods = self.R.row_moduli(ct.level)
        sc = np.array([v % int(q) for q in mods], np.uint64)
        res = []
        for p in out.parts:
            o = np.empty_like(p)
            lib().or_poly_mul_scalar(_p(o), _p(p), _p(sc), _p(mods), p.shape[0], p.shape[1])
            res.append(o)
        out.parts = res
        out.scale = ct.scale * scalar_scale
        return out

    @staticmethod
    def scaled_residue(value: float, q: int) -> int:
        if abs(value) < 9.0e18:
            return round_half_away(value) % q
        r = np.fmod(np.longdouble(value), np.longdouble(q))
        ar = abs(r)
        mag = int(np.floor(ar + np.longdouble(0.5)))
        return (mag if r >= 0 else -mag) % q

    def add_scalar(self, ct: OCt, c: float) -> OCt:
        out = ct.copy()
        p0 = out.parts[0]
        for r in range(p0.shape[0]):
            q = int(self.R.moduli[self.R.mod_index(r, ct.level)])
            add = np.uint64(self.scaled_residue(c * ct.scale, q))
            if ct.form == "eval":
                row = p0[r].astype(object) + int(add)
                p0[r] = np.array([x - q if x >= q else x for x in row], dtype=np.uint64)
            else:
                v = int(p0[r, 0]) + int(add)
                p0[r, 0] = v - q if v >= q else v
        return out

    def rescale(self, ct: OCt) -> OCt:
        if ct.level == 0:
            raise RuntimeError("[ckks] cannot rescale at level 0")
        out = ct.copy()
        self.to_coeff(out)
        mods = np.array(self.R.moduli[:ct.level + 1], np.uint64)
        res = []
        for p in out.parts:
            o = np.empty((ct.level, self.R.N), np.uint64)
            lib().or_rescale(_p(o), _p(np.ascontiguousarray(p)), _p(mods), ct.level, self.R.N)
            res.append(o)
        ql = self.R.moduli[ct.level]
        return OCt(res, ct.level - 1, "coeff", ct.scale / float(ql), ct.domain, ct.sk_id, ct.noise_bound / float(ql) + 1.0)

    # --- key switching (rlwe.hpp:501-654) ---
    def decompose(self, d: np.ndarray, level: int):
        R = self.R
        ndig = (level + self.group) // self.group
        rows = level + 1 + R.K
        digs = np.zeros((ndig, rows, R.N), np.uint64)
        lib().or_modup(_p(digs), _p(np.ascontiguousarray(d)), _p(np.array(R.moduli, np.uint64)), R.nq, R.K,
                       self.group, level, R.N)
        return [R.ntt(digs[j], level, R.K) for j in range(ndig)]

    def mod_down(self, x: np.ndarray, level: int) -> np.ndarray:
        R = self.R
        out = np.zeros((level + 1, R.N), np.uint64)
        lib().or_mod_down(_p(out), _p(np.ascontiguousarray(x)), _p(np.array(R.moduli, np.uint64)), R.nq, R.K, level, R.N)
        return out

    def ks_inner(self, digits, key: OKey, level: int):
        R = self.R
        nd = len(digits)
        rows = level + 1 + R.K
        dig = np.ascontiguousarray(np.stack(digits))
        kb = (_u64p * nd)(*[_p(np.ascontiguousarray(key.b[i])) for i in range(nd)])
        ka = (_u64p * nd)(*[_p(np.ascontiguousarray(key.a[i])) for i in range(nd)])
        keep = [np.ascontiguousarray(key.b[i]) for i in range(nd)] + [np.ascontiguousarray(key.a[i]) for i in range(nd)]
        kb = (_u64p * nd)(*[_p(k) for k in keep[:nd]])
        ka = (_u64p * nd)(*[_p(k) for k in keep[nd:]])
        acc0 = np.zeros((rows, R.N), np.uint64)
        acc1 = np.zeros((rows, R.N), np.uint64)
        lib().or_key_inner(_p(acc0), _p(acc1), _p(dig), nd, kb, ka, _p(np.array(R.moduli, np.uint64)), R.nq, R.K,
                           level, R.N)
        acc0 = R.ntt(acc0, level, R.K, inverse=True)
        acc1 = R.ntt(acc1, level, R.K, inverse=True)
        return self.mod_down(acc0, level), self.mod_down(acc1, level)

    def switch_key_apply(self, d: np.ndarray, key: OKey, level: int):
        return self.ks_inner(self.decompose(d, level), key, level)

    def relinearize(self, ct: OCt, rlk: OKey, ks_noise: float) -> OCt:
        x = ct.copy()
        self.to_coeff(x)
        d0, d1 = self.switch_key_apply(x.parts[2], rlk, x.level)
        mods = self.R.row_moduli(x.level)
        add = lib().or_poly_add
        return OCt([_binop(add, x.parts[0], d0, mods), _binop(add, x.parts[1], d1, mods)], x.level, "coeff", ct.scale,
                   ct.domain, ct.sk_id, ct.noise_bound + ks_noise)

    def mul_relin(self, a, b, rlk, ks_noise):
        return self.relinearize(self.mul(a, b), rlk, ks_noise)

    def automorphism(self, p: np.ndarray, g: int, level: int, eval_form=False) -> np.ndarray:
        out = np.empty_like(p)
        mods = self.R.row_moduli(level, p.shape[0] - level - 1)
        lib().or_automorphism(_p(out), _p(np.ascontiguousarray(p)), g, 1 if eval_form else 0, _p(mods), p.shape[0],
                              self.R.N, _p32(self.R.eval_exp), _p32(self.R.slot_of_exp))
        return out

    def apply_galois(self, ct: OCt, g: int, key: OKey, ks_noise: float) -> OCt:
        x = ct.copy()
        self.to_coeff(x)
        c0g = self.automorphism(x.parts[0], g, x.level)
        c1g = self.automorphism(x.parts[1], g, x.level)
        d0, d1 = self.switch_key_apply(c1g, key, x.level)
        mods = self.R.row_moduli(x.level)
        return OCt([_binop(lib().or_poly_add, c0g, d0, mods), d1], x.level, "coeff", ct.scale, ct.domain, ct.sk_id,
                   ct.noise_bound + ks_noise)

    def rotate(self, ct: OCt, k: int, gkeys: dict, ks_noise: float) -> OCt:
        if k == 0:
            return ct
        g = pow(5, k, 2 * self.R.N)
        if g not in gkeys:
            raise RuntimeError(f"[ckks] missing rotation key for exponent {g}")
        return self.apply_galois(ct, g, gkeys[g], ks_noise)


def eval_chebyshev(ev: Evaluator, x: OCt, coeffs, rlk: OKey, ks_noise: float) -> OCt:
    """Memoised T_k ladder (ckks.hpp:515-579), same op order."""
    d = len(coeffs) - 1
    while d > 0 and coeffs[d] == 0.0:
        d -= 1
    if d == 0:
        return ev.add_scalar(ev.mul_scalar(x, 0.0, 1.0), coeffs[0])
    if x.level < math.ceil(math.log2(d)) + 1:
        raise RuntimeError("[ckks] insufficient levels for polynomial evaluation")
    T = {1: x}

    def get(k):
        if k in T:
            return T[k]
        a = k // 2
        b = k - a
        ta, tb = get(a), get(b)
        prod = ev.mul_relin(ta, tb, rlk, ks_noise)
        ev.to_coeff(prod)
        ev.add_inplace_raw(prod, prod.copy())
        if a == b:
            res = ev.rescale(ev.add_scalar(prod, -1.0))
        else:
            tc = get(b - a).copy()
            ev.to_coeff(tc)
            if tc.level > prod.level:
                ev.drop(tc, prod.level)
            tc = ev.mul_scalar(tc, 1.0, prod.scale / tc.scale)
            ev.check_scales(tc.scale, prod.scale)
            ev.add_inplace_raw(prod, tc, sub=True)
            res = ev.rescale(prod)
        T[k] = res
        return res

    k = d
    while k >= 1:
        get(k)
        k //= 2
    lvl = x.level
    for k in range(1, d + 1):
        if coeffs[k] != 0.0:
            lvl = min(lvl, get(k).level)
    comb = float(ev.R.moduli[lvl])
    acc = None
    for k in range(1, d + 1):
        if coeffs[k] == 0.0:
            continue
        term = get(k).copy()
        ev.to_coeff(term)
        if term.level > lvl:
            ev.drop(term, lvl)
        term = ev.mul_scalar(term, coeffs[k], comb)
        if acc is None:
            acc = term
        else:
            ev.check_scales(acc.scale, term.scale)
            ev.add_inplace_raw(acc, term)
    if coeffs[0] != 0.0:
        acc = ev.add_scalar(acc, coeffs[0])
    return ev.rescale(acc)


def inner_sum(ev: Evaluator, ct: OCt, n: int, gkeys: dict, ks_noise: float) -> OCt:
    acc = ct
    k = 1
    while k < n:
        acc = ev.add(acc, ev.rotate(acc, k, gkeys, ks_noise))
        k <<= 1
    return acc


def threshold_plain_norm(ev: Evaluator, scores: OCt, t: OCt, norm: float, stages_coeffs, levels_required: int,
                         epsilon: float, rlk: OKey, ks_noise: float) -> OCt:
    """eval_private_threshold_plain_norm (threshold.hpp:146-157); stages_coeffs
    = [chain.eval_coeffs(i) ...] from the (host-side) chain."""
    if scores.level < levels_required:
        raise RuntimeError(f"[threshold] insufficient levels: need {levels_required}, have {scores.level}")
    diff = ev.add_scalar(ev.sub(scores, t), epsilon / 2.0)
    ql = ev.R.moduli[diff.level]
    u = ev.rescale(ev.mul_scalar(diff, norm, float(ql)))
    for c in stages_coeffs:
        u = eval_chebyshev(ev, u, c, rlk, ks_noise)
    return ev.add_scalar(u, 0.5)
