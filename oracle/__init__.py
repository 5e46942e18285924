"""CPU oracle of arXiv 1606.07407 Algorithm 2 -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper around ``oracle/sfft_oracle.c`` (plain C, fp64, exact integer
phase reduction, direct O(p^2) DFT).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (``cpu_baseline`` and ``--impl reference``) may import this
package.  It never imports ``paper_1606_07407_b200`` and the CUDA library never
imports it.

Parity status of every function is listed in DESIGN.md ("Oracle pins"); each C
function cites the PAPER.md passage it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sfft_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

TRACE_COLS = 8      # ORACLE_TRACE_COLS (sfft_oracle.h)
OK, PARTIAL, EINVAL, EPRECISION, ECORRUPT, ENOMEM = 0, 1, -1, -2, -4, -6


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2, no fast-math).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "sfft_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fPIC", "-shared", "-o", tmp,
                               _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("d", ctypes.c_int32), ("k", ctypes.c_int32), ("N", ctypes.c_int64),
        ("r", ctypes.c_int32), ("blocks", ctypes.POINTER(ctypes.c_int32)),
        ("n_tilts", ctypes.c_int32), ("tilts", ctypes.POINTER(ctypes.c_int64)),
        ("E", ctypes.c_int64), ("c", ctypes.c_int32),
        ("tol", ctypes.c_double), ("bin_floor_rel", ctypes.c_double),
        ("prune_floor", ctypes.c_double), ("round_tol", ctypes.c_double),
        ("max_iter", ctypes.c_int32), ("stall_limit", ctypes.c_int32),
        ("extra_checks", ctypes.c_int32),
        ("n_primes", ctypes.c_int32), ("primes", ctypes.POINTER(ctypes.c_int64)),
        ("n_fallback", ctypes.c_int32), ("n_spec", ctypes.c_int32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        vp = ctypes.c_void_p
        L.oracle_unwrap_freq.argtypes = [i32, i64, i32, vp, vp, vp]
        L.oracle_wrap_freq.argtypes = [i32, i64, i32, vp, vp, vp]
        L.oracle_block_range.argtypes = [i64, i32, vp, vp]
        L.oracle_tilt_freq.argtypes = [i64, i64, i64, i64, vp]
        L.oracle_untilt_freq.argtypes = [i64, i64, i64, i64, i64, vp]
        L.oracle_unwrap_time.argtypes = [i32, i64, i32, vp, vp, vp]
        L.oracle_ith_prime_at_least.argtypes = [i64, i32]
        L.oracle_ith_prime_at_least.restype = i64
        L.oracle_prepare.argtypes = [ctypes.POINTER(_Params), vp, vp, vp]
        L.oracle_project.argtypes = [ctypes.POINTER(_Params), vp, i32, vp]
        L.oracle_eval_point.argtypes = [i32, i32, vp, vp, vp, vp]
        L.oracle_sample_line.argtypes = [i32, i32, vp, vp, i64, i32, i32, i64, vp]
        L.oracle_dft.argtypes = [i64, vp, vp]
        L.oracle_decode.argtypes = [ctypes.POINTER(_Params), i64, vp, vp, i64, i32, i32, vp, vp, vp,
                                    vp, vp]
        L.oracle_decode.restype = i32
        L.oracle_fallback_tilts.argtypes = [i32, i32, vp]
        L.oracle_fallback_tilts.restype = i32
        L.oracle_axis_order.argtypes = [i32, i32, vp]
        L.oracle_axis_order.restype = None
        L.oracle_solve.argtypes = [ctypes.POINTER(_Params), vp, vp, vp, vp, vp, vp, vp, i32, vp]
        L.oracle_solve_raw.argtypes = [ctypes.POINTER(_Params), vp, vp, vp, vp, vp]
        L.oracle_solve_batch.argtypes = [ctypes.POINTER(_Params), i32, vp, vp, vp, vp, vp, vp, vp,
                                         vp, i32, vp]
        _lib = L
    return _lib


def _p(x: np.ndarray):
    return ctypes.c_void_p(x.ctypes.data) if x is not None else None


@dataclass
class Params:
    """Algorithm 2 inputs + readings C3/C14/C15/C17-C19."""

    d: int
    N: int
    k: int
    blocks: Sequence[int]
    tilts: Sequence[Tuple[int, int, int, int, int]] = ()
    E: int = 0
    c: int = 5
    tol: float = 1e-6
    bin_floor_rel: float = 1e-8
    prune_floor: float = 1e-8
    round_tol: float = 0.01
    max_iter: int = 1000
    stall_limit: int = 0
    extra_checks: int = 3
    primes: Optional[Sequence[int]] = None
    n_fallback: int = 0
    n_spec: int = 0
    _keep: list = field(default_factory=list, repr=False)

    def c_struct(self) -> _Params:
        blocks = np.ascontiguousarray(np.asarray(self.blocks, dtype=np.int32))
        tilts = np.ascontiguousarray(np.asarray(self.tilts, dtype=np.int64).reshape(-1, 5)) \
            if len(self.tilts) else np.zeros((0, 5), np.int64)
        primes = np.ascontiguousarray(np.asarray(self.primes, dtype=np.int64)) \
            if self.primes is not None else None
        self._keep = [blocks, tilts, primes]
        s = _Params()
        s.d, s.k, s.N, s.r = self.d, self.k, self.N, len(self.blocks)
        s.blocks = blocks.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        s.n_tilts = tilts.shape[0]
        s.tilts = tilts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        s.E, s.c = self.E, self.c
        s.tol, s.bin_floor_rel, s.prune_floor, s.round_tol = (self.tol, self.bin_floor_rel,
                                                              self.prune_floor, self.round_tol)
        s.max_iter, s.stall_limit, s.extra_checks = self.max_iter, self.stall_limit, self.extra_checks
        s.n_primes = 0 if primes is None else primes.size
        s.primes = None if primes is None else primes.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        s.n_fallback = self.n_fallback
        s.n_spec = self.n_spec
        return s

    @property
    def r(self) -> int:
        return len(self.blocks)


def params_for(cfg, blocks=None, **kw) -> Params:
    return Params(d=cfg.d, N=cfg.N, k=cfg.k, blocks=tuple(blocks or cfg.blocks), **kw)


# ---------------------------------------------------------------- index maps
def unwrap_freq(w, N: int, blocks) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(w, dtype=np.int32))
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.int32))
    u = np.zeros(len(b), np.int64)
    rc = lib().oracle_unwrap_freq(w.size, N, len(b), _p(b), _p(w), _p(u))
    if rc:
        raise ValueError(f"unwrap_freq rc={rc}")
    return u


def wrap_freq(u, N: int, blocks) -> np.ndarray:
    u = np.ascontiguousarray(np.asarray(u, dtype=np.int64))
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.int32))
    w = np.zeros(int(b.sum()), np.int32)
    rc = lib().oracle_wrap_freq(w.size, N, len(b), _p(b), _p(u), _p(w))
    if rc:
        raise ValueError(f"wrap_freq rc={rc}")
    return w


def block_range(N: int, dq: int) -> Tuple[int, int]:
    lo, hi = np.zeros(1, np.int64), np.zeros(1, np.int64)
    lib().oracle_block_range(N, dq, _p(lo), _p(hi))
    return int(lo[0]), int(hi[0])


def tilt_freq(base, height, w1, w2) -> Tuple[int, int]:
    out = np.zeros(2, np.int64)
    lib().oracle_tilt_freq(base, height, w1, w2, _p(out))
    return int(out[0]), int(out[1])


def untilt_freq(base, height, hypo, v1, v2) -> Tuple[int, int]:
    out = np.zeros(2, np.int64)
    rc = lib().oracle_untilt_freq(base, height, hypo, v1, v2, _p(out))
    if rc:
        raise ValueError("untilt: not a tilted lattice point")
    return int(out[0]), int(out[1])


def unwrap_time(t_red, N: int, blocks) -> np.ndarray:
    t_red = np.ascontiguousarray(np.asarray(t_red, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(blocks, dtype=np.int32))
    t = np.zeros(int(b.sum()), np.float64)
    lib().oracle_unwrap_time(t.size, N, len(b), _p(b), _p(t_red), _p(t))
    return t


def ith_prime_at_least(x: int, i: int = 1) -> int:
    return int(lib().oracle_ith_prime_at_least(int(x), int(i)))


# ---------------------------------------------------------------- plan quantities
MAX_FALLBACK = 67   # ORACLE_MAX_FALLBACK


def axis_order(r: int, seed: int = 1):
    """Seeded axis order of the round-robin fallback levels (reading R24)."""
    pi = np.zeros(max(r, 1), np.int32)
    lib().oracle_axis_order(r, seed, _p(pi))
    return pi[:r].tolist()


def fallback_tilts(r: int, level: int):
    """Tilts of stall-fallback level `level` >= 1 (readings R23 / R24): list of (axis0, axis1, base, height, hypo)."""
    out = np.zeros((max(r // 2, 1), 5), np.int64)
    n = lib().oracle_fallback_tilts(r, level, _p(out))
    return [tuple(int(x) for x in row) for row in out[:n]]


def prepare(P: Params) -> Tuple[int, np.ndarray, np.ndarray]:
    """(E, lo[r], hi[r]) or raises with the status code."""
    lo, hi = np.zeros(P.r, np.int64), np.zeros(P.r, np.int64)
    E = np.zeros(1, np.int64)
    s = P.c_struct()
    rc = lib().oracle_prepare(ctypes.byref(s), _p(E), _p(lo), _p(hi))
    if rc:
        raise OracleError(rc)
    return int(E[0]), lo, hi


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle status {rc}")
        self.rc = rc


def project(P: Params, w: np.ndarray) -> np.ndarray:
    w = np.ascontiguousarray(w, dtype=np.int32)
    v = np.zeros((w.shape[0], P.r), np.int64)
    s = P.c_struct()
    rc = lib().oracle_project(ctypes.byref(s), _p(w), w.shape[0], _p(v))
    if rc:
        raise OracleError(rc)
    return v


# ---------------------------------------------------------------- evaluation, DFT, decode
def eval_point(w: np.ndarray, a: np.ndarray, t) -> complex:
    w = np.ascontiguousarray(np.atleast_2d(w), dtype=np.int32)
    a = np.ascontiguousarray(np.atleast_1d(a), dtype=np.complex128)
    t = np.ascontiguousarray(np.asarray(t, dtype=np.float64))
    out = np.zeros(2, np.float64)
    lib().oracle_eval_point(w.shape[1], w.shape[0], _p(w), _p(a.view(np.float64)), _p(t), _p(out))
    return complex(out[0], out[1])


def sample_line(v: np.ndarray, c: np.ndarray, p: int, m: int, n: int, E: int) -> np.ndarray:
    """s[h] = sum_j c_j e^{2 pi i v_j . ((h/p) e_m + (1/E) e_n)}, n < 0 -> unshifted."""
    v = np.ascontiguousarray(np.atleast_2d(v), dtype=np.int64)
    c = np.ascontiguousarray(np.atleast_1d(c), dtype=np.complex128)
    s = np.zeros(p, np.complex128)
    lib().oracle_sample_line(v.shape[0], v.shape[1], _p(v), _p(c.view(np.float64)), p, m, n, E,
                             _p(s.view(np.float64)))
    return s


def dft(s: np.ndarray) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.complex128)
    F = np.zeros_like(s)
    lib().oracle_dft(s.size, _p(s.view(np.float64)), _p(F.view(np.float64)))
    return F


def decode(P: Params, E: int, lo, hi, p: int, m: int, kstar: int, F: np.ndarray):
    """Select + test + decode of one iteration.  F complex128 [(r+1), p].
    Returns (n_candidates, acc_b int32[na], acc_v int64[na, r], acc_a complex128[na])."""
    F = np.ascontiguousarray(F, dtype=np.complex128)
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    hi = np.ascontiguousarray(hi, dtype=np.int64)
    cap = max(kstar, 1)
    acc_b = np.zeros(cap, np.int32)
    acc_v = np.zeros((cap, P.r), np.int64)
    acc_a = np.zeros(cap, np.complex128)
    nc = np.zeros(1, np.int32)
    s = P.c_struct()
    na = lib().oracle_decode(ctypes.byref(s), E, _p(lo), _p(hi), p, m, kstar,
                             _p(F.view(np.float64)), _p(nc), _p(acc_b), _p(acc_v),
                             _p(acc_a.view(np.float64)))
    return int(nc[0]), acc_b[:na].copy(), acc_v[:na].copy(), acc_a[:na].copy()


@dataclass
class SolveResult:
    status: int
    w: np.ndarray          # int32 [count, d], canonical lexicographic order
    a: np.ndarray          # complex128 [count]
    samples: int
    iterations: int
    trace: np.ndarray      # int64 [iterations, TRACE_COLS] = (i, p, m, n_candidates, n_accepted,
    #                        n_nonempty before the k* cap, n_accumulated, n_pruned)


def solve(P: Params, w: np.ndarray, a: np.ndarray, trace_cap: int = 1000) -> SolveResult:
    """Algorithm 2 end to end for one signal."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    a = np.ascontiguousarray(a, dtype=np.complex128)
    k, d = P.k, P.d
    out_w = np.zeros((k, d), np.int32)
    out_a = np.zeros(k, np.complex128)
    cnt = np.zeros(1, np.int32)
    samples = np.zeros(1, np.int64)
    iters = np.zeros(1, np.int32)
    trace = np.zeros((trace_cap, TRACE_COLS), np.int64)
    s = P.c_struct()
    st = lib().oracle_solve(ctypes.byref(s), _p(w), _p(a.view(np.float64)), _p(out_w),
                            _p(out_a.view(np.float64)), _p(cnt), _p(samples), _p(iters),
                            trace_cap, _p(trace))
    n = int(cnt[0])
    it = int(iters[0])
    return SolveResult(st, out_w[:n].copy(), out_a[:n].copy(), int(samples[0]), it,
                       trace[:min(it, trace_cap)].copy())


def solve_raw(P: Params, w: np.ndarray, a: np.ndarray):
    """Debugging aid: (status, registry keys int64 [n, r], coefficients complex128 [n]) before the wrap."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    a = np.ascontiguousarray(a, dtype=np.complex128)
    rv = np.zeros((P.k, P.r), np.int64)
    ra = np.zeros(P.k, np.complex128)
    n = np.zeros(1, np.int32)
    s = P.c_struct()
    st = lib().oracle_solve_raw(ctypes.byref(s), _p(w), _p(a.view(np.float64)), _p(rv), _p(ra.view(np.float64)),
                                _p(n))
    return st, rv[:int(n[0])].copy(), ra[:int(n[0])].copy()


def solve_batch(P: Params, w: np.ndarray, a: np.ndarray, n_threads: int = 0, times: bool = False):
    """Independent signals over host threads: returns (status[T], w[T,k,d], a[T,k], count[T],
    samples[T], iterations[T]) and, with times=True, ns int64 [T, 2] = (solve wall ns, sampling ns)."""
    w = np.ascontiguousarray(w, dtype=np.int32)
    a = np.ascontiguousarray(a, dtype=np.complex128)
    T = w.shape[0]
    k, d = P.k, P.d
    out_w = np.zeros((T, k, d), np.int32)
    out_a = np.zeros((T, k), np.complex128)
    cnt = np.zeros(T, np.int32)
    samples = np.zeros(T, np.int64)
    iters = np.zeros(T, np.int32)
    status = np.zeros(T, np.int32)
    if n_threads <= 0:
        n_threads = os.cpu_count() or 1
    ns = np.zeros((T, 2), np.int64) if times else None
    s = P.c_struct()
    lib().oracle_solve_batch(ctypes.byref(s), T, _p(w), _p(a.view(np.float64)), _p(out_w),
                             _p(out_a.view(np.float64)), _p(cnt), _p(samples), _p(iters),
                             _p(status), n_threads, _p(ns))
    if times:
        return status, out_w, out_a, cnt, samples, iters, ns
    return status, out_w, out_a, cnt, samples, iters
