"""Pins of the CPU oracle against what the paper and the mathematics fix (not against itself).

Every test names the passage it pins.  The sources of truth used here are:
  * worked values printed in / derived by hand from the paper (tests/golden/worked_examples.json);
  * closed forms written out independently in this file with Python integers /
    fractions (Eq. (3) aliasing identity, Eqs. (4)/(5) singleton bins, Eq. (36) duality);
  * library routines a special case reduces to (numpy.fft for the DFT);
  * brute force on tiny inputs (dense d-dimensional DFT of f on the N^d grid);
  * the paper's invariant that a noiseless k-sparse signal is recovered exactly.
"""
import cmath
import itertools
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ------------------------------------------------------------------ f evaluation (Eq. (9))
@pytest.mark.parametrize("ex", GOLD["eval_point"])
def test_eval_point_worked_values(ex):
    a = np.array([complex(*x) for x in ex["a"]])
    got = O.eval_point(np.array(ex["w"]), a, ex["t"])
    assert abs(got - complex(*ex["expect"])) < 1e-14


def _exact_phase_value(w_rows, a, x_frac):
    """sum_j a_j exp(2 pi i (w_j . x) mod 1) with w . x reduced exactly in rationals."""
    tot = 0j
    for wj, aj in zip(w_rows, a):
        ph = sum(Fraction(int(wl)) * xl for wl, xl in zip(wj, x_frac)) % 1
        tot += aj * cmath.exp(2j * math.pi * float(ph))
    return tot


@pytest.mark.parametrize("blocks,tilt", [((1, 1), None), ((2, 1), None), ((2,), None),
                                         ((1, 2, 1), None), ((1, 1), (0, 1, 3, 4, 5)),
                                         ((2, 2), (0, 1, 5, 12, 13))])
def test_sample_line_equals_f_at_unwrapped_point(blocks, tilt):
    """Eq. (41) + Eq. (36) (+ Eq. (27)): the oracle's exact-phase line sample equals the plain
    definition f(x) = sum a e^{2 pi i w . x} at the d-dimensional point x = unwrap_time(T^T t~),
    with w . x computed here in exact rationals from the ORIGINAL w (duality S:168)."""
    N, k = 8, 5
    d = sum(blocks)
    rng = np.random.default_rng(7)
    w = rng.integers(-N // 2, N // 2, size=(k, d))
    a = np.exp(2j * np.pi * rng.random(k))
    tilts = [tilt] if tilt else []
    P = O.Params(d=d, N=N, k=k, blocks=blocks, tilts=tilts)
    E, _, _ = O.prepare(P)
    v = O.project(P, w.astype(np.int32))
    r = len(blocks)
    p = 13
    for m in range(r):
        for n in [-1] + list(range(r)):
            s = O.sample_line(v, a, p, m, n, E)
            for h in (0, 1, 5, 12):
                t_red = [Fraction(0)] * r
                t_red[m] += Fraction(h, p)
                if n >= 0:
                    t_red[n] += Fraction(1, E)
                if tilt:   # t = T^T t~, T = [[b, -h], [h, b]] on (a0, a1)  (Eq. (27))
                    a0, a1, b, hh, _ = tilt
                    x0, x1 = t_red[a0], t_red[a1]
                    t_red[a0], t_red[a1] = b * x0 + hh * x1, -hh * x0 + b * x1
                # Eq. (36): x[off_q + s] = N^s t~_q
                x = []
                for q, dq in enumerate(blocks):
                    x += [t_red[q] * N ** s_ for s_ in range(dq)]
                ref = _exact_phase_value(w, a, x)
                assert abs(s[h] - ref) < 1e-12, (m, n, h)


def test_residual_of_truth_is_zero():
    """Residual oracle S:93: f - g with g = f (R = truth) vanishes."""
    c = W.CONFIGS["c2"]
    w, a = W.make_signal(c, 3)
    P = O.params_for(c)
    E, _, _ = O.prepare(P)
    v = O.project(P, w)
    vv = np.concatenate([v, v])
    cc = np.concatenate([a, -a])
    s = O.sample_line(vv, cc, 101, 1, 0, E)
    assert np.abs(s).max() < 1e-12 * c.k


# ------------------------------------------------------------------ index maps
@pytest.mark.parametrize("ex", GOLD["unwrap"])
def test_unwrap_worked(ex):
    assert O.unwrap_freq(ex["w"], ex["N"], ex["blocks"]).tolist() == ex["u"]
    assert O.wrap_freq(ex["u"], ex["N"], ex["blocks"]).tolist() == ex["w"]


def test_wrap_unwrap_exhaustive_bijection():
    """wrap o unwrap = id on the whole digit box N=4, d=4, (2,2), and unwrap is injective."""
    N, blocks = 4, (2, 2)
    seen = set()
    for w in itertools.product(range(-2, 2), repeat=4):
        u = O.unwrap_freq(w, N, blocks)
        # Eq. (35) written out independently
        assert u.tolist() == [w[0] + N * w[1], w[2] + N * w[3]]
        assert tuple(O.wrap_freq(u, N, blocks)) == w
        seen.add(tuple(u))
    assert len(seen) == 256


def test_wrap_rejects_out_of_image():
    lo, hi = O.block_range(20, 2)
    assert (lo, hi) == (-10 * 21, 9 * 21)    # [-(N/2)(N^2-1)/(N-1), (N/2-1)(N^2-1)/(N-1)]
    with pytest.raises(ValueError):
        O.wrap_freq([hi + 1], 20, (2,))


@pytest.mark.parametrize("ex", GOLD["unwrap_time"])
def test_unwrap_time_worked(ex):
    assert O.unwrap_time(ex["t_red"], ex["N"], ex["blocks"]).tolist() == ex["t"]


def test_tilt_worked_and_roundtrip():
    ex, rect = GOLD["tilt"]
    assert O.tilt_freq(ex["base"], ex["height"], *ex["w"]) == tuple(ex["v"])
    assert O.untilt_freq(ex["base"], ex["height"], ex["hypo"], *ex["v"]) == tuple(ex["w"])
    firsts = [O.tilt_freq(3, 4, *w)[0] for w in rect["rectangle"]]
    assert firsts == rect["first_coords"] and len(set(firsts)) == 4
    rng = np.random.default_rng(0)
    for (b, h, c) in [(3, 4, 5), (5, 12, 13), (8, 15, 17), (7, 24, 25)]:
        for w in rng.integers(-1000, 1000, size=(200, 2)):
            v = O.tilt_freq(b, h, int(w[0]), int(w[1]))
            assert O.untilt_freq(b, h, c, *v) == (int(w[0]), int(w[1]))
    with pytest.raises(ValueError):
        O.untilt_freq(3, 4, 5, 1, 0)      # not a tilted lattice point


def test_tilt_injective_small_box():
    """no two points of the N=8 box collide after tilting."""
    pts = {O.tilt_freq(3, 4, a, b) for a in range(-4, 4) for b in range(-4, 4)}
    assert len(pts) == 64


# ------------------------------------------------------------------ primes
@pytest.mark.parametrize("ex", GOLD["primes"])
def test_primes_worked(ex):
    assert O.ith_prime_at_least(ex["x"], ex["i"]) == ex["p"]


def test_primes_vs_sieve():
    M = 20000
    sieve = np.ones(M, bool)
    sieve[:2] = False
    for q in range(2, int(M ** 0.5) + 1):
        if sieve[q]:
            sieve[q * q::q] = False
    primes = np.nonzero(sieve)[0]
    for x in (0, 1, 2, 3, 100, 4999, 5000, 9973):
        after = primes[primes >= max(x, 2)]
        for i in (1, 2, 7):
            assert O.ith_prime_at_least(x, i) == after[i - 1]


# ------------------------------------------------------------------ DFT (Eq. (3))
def test_dft_worked_and_closed_forms():
    ex = GOLD["dft"][0]
    p = ex["p"]
    v = np.array([[m[0]] for m in ex["modes"]], np.int64)
    c = np.array([m[1] for m in ex["modes"]], np.complex128)
    F = O.dft(O.sample_line(v, c, p, 0, -1, 2))
    assert abs(F[ex["bin"]] - complex(*ex["value"])) < 1e-12
    assert np.abs(np.delete(F, ex["bin"])).max() < 1e-12
    # constant line -> (p a, 0, ..., 0)
    a = 0.3 - 1.7j
    F = O.dft(np.full(17, a))
    assert abs(F[0] - 17 * a) < 1e-12 and np.abs(F[1:]).max() < 1e-12


@pytest.mark.parametrize("p", [2, 3, 5, 23, 101, 503])
def test_dft_equals_library_fft(p):
    """The unnormalised forward DFT is numpy.fft.fft (a library special case) -- and Parseval."""
    rng = np.random.default_rng(p)
    s = rng.standard_normal(p) + 1j * rng.standard_normal(p)
    F = O.dft(s)
    ref = np.fft.fft(s)
    assert np.abs(F - ref).max() <= 1e-12 * np.abs(ref).max() * max(1, p / 50)
    assert abs(np.sum(np.abs(F) ** 2) - p * np.sum(np.abs(s) ** 2)) < 1e-9 * p * np.sum(np.abs(s) ** 2)


@pytest.mark.parametrize("name,blocks", [("c2", (2, 1)), ("c2", (1, 1, 1)), ("c1", (2,))])
def test_sampling_plus_dft_is_eq3_aliasing(name, blocks):
    """Eq. (3)/(41): the DFT of a sampled line equals p * sum_{v_m = b mod p} c_j e^{2 pi i v_n/E},
    written out here straight from the ground truth (never used by the product path)."""
    c = W.CONFIGS[name]
    w, a = W.make_signal(c, 1)
    P = O.params_for(c, blocks=blocks)
    E, _, _ = O.prepare(P)
    v = O.project(P, w)
    r = len(blocks)
    p = 103
    for m in range(r):
        for n in [-1] + list(range(r)):
            F = O.dft(O.sample_line(v, a, p, m, n, E))
            ref = np.zeros(p, np.complex128)
            for j in range(c.k):
                b = int(v[j, m]) % p
                ph = 0.0 if n < 0 else (int(v[j, n]) % E) / E
                ref[b] += p * a[j] * cmath.exp(2j * math.pi * ph)
            assert np.abs(F - ref).max() < 1e-9 * p * np.abs(a).sum()


# ------------------------------------------------------------------ collision test + decode
def _one_iteration_F(v, c, p, m, E, r):
    return np.stack([O.dft(O.sample_line(v, c, p, m, n, E)) for n in [-1] + list(range(r))])


def test_collision_ratio_worked():
    ex = GOLD["collision"][0]
    v = np.array([[m[0]] for m in ex["modes"]], np.int64)
    c = np.array([m[1] for m in ex["modes"]], np.complex128)
    F = _one_iteration_F(v, c, ex["p"], 0, ex["E"], 1)
    ratio = abs(F[1, ex["bin"]]) / abs(F[0, ex["bin"]])
    assert abs(ratio - ex["ratio"]) < 1e-12
    assert abs(ex["ratio"] - abs(math.cos(11 * math.pi / 16))) < 1e-15
    # the decoder rejects that bin (Eq. (8)) ...
    P = O.Params(d=1, N=16, k=2, blocks=(1,), E=ex["E"])
    E, lo, hi = O.prepare(P)
    nc, acc_b, _, _ = O.decode(P, E, lo, hi, ex["p"], 0, 2, F)
    assert nc == 1 and acc_b.size == 0


@pytest.mark.parametrize("ex", GOLD["decode"])
def test_decode_singleton_worked(ex):
    """Eqs. (4), (5), (7): a singleton bin decodes to its frequency and coefficient."""
    P = O.Params(d=1, N=16, k=1, blocks=(1,), E=ex["E"])
    E, lo, hi = O.prepare(P)
    a = complex(*ex["a"])
    F = _one_iteration_F(np.array([[ex["w"]]]), np.array([a]), ex["p"], 0, E, 1)
    b = ex["w"] % ex["p"]
    assert abs(F[0, b] - ex["p"] * a) < 1e-12                             # Eq. (5)
    assert abs(F[1, b] - ex["p"] * a * cmath.exp(2j * math.pi * ex["w"] / E)) < 1e-12   # Eq. (4)
    nc, acc_b, acc_v, acc_a = O.decode(P, E, lo, hi, ex["p"], 0, 1, F)
    assert acc_b.tolist() == [b] and acc_v.tolist() == [[ex["w"]]]
    assert abs(acc_a[0] - a) < 1e-12


def test_decode_random_singletons():
    """random single-mode lines over w in [-8, 8), eps = 1/16 decode exactly."""
    P = O.Params(d=1, N=16, k=1, blocks=(1,), E=16)
    E, lo, hi = O.prepare(P)
    rng = np.random.default_rng(5)
    for w in range(-8, 8):
        a = complex(*rng.standard_normal(2))
        F = _one_iteration_F(np.array([[w]]), np.array([a]), 7, 0, E, 1)
        _, _, acc_v, acc_a = O.decode(P, E, lo, hi, 7, 0, 1, F)
        assert acc_v.tolist() == [[w]] and abs(acc_a[0] - a) < 1e-12


def test_collision_detection_rate():
    """S:308 / S:541: random two-mode collisions are rejected by Eq. (8) (false-pass rate < 1%)."""
    P = O.Params(d=1, N=1 << 20, k=2, blocks=(1,))
    E, lo, hi = O.prepare(P)
    rng = np.random.default_rng(11)
    p, passes, n = 31, 0, 1000
    for _ in range(n):
        w1 = int(rng.integers(-(1 << 19), 1 << 19))
        w2 = w1 + p * int(rng.integers(1, 1000))
        if w2 >= (1 << 19):
            w2 = w1 - p * int(rng.integers(1, 1000))
        c = np.exp(2j * np.pi * rng.random(2))
        F = _one_iteration_F(np.array([[w1], [w2]]), c, p, 0, E, 1)
        _, acc_b, _, _ = O.decode(P, E, lo, hi, p, 0, 2, F)
        passes += acc_b.size
    assert passes / n < 0.01


# ------------------------------------------------------------------ Algorithm 2 end to end
@pytest.mark.parametrize("ex", GOLD["sample_count"])
def test_sample_count_closed_form(ex):
    d, N = ex["d"], ex["N"]
    blocks = tuple([ex["blocks_d1"]] * (d // ex["blocks_d1"]))
    c = W.custom_config(d, N, ex["k"], blocks, cfg=77)
    w, a = W.make_signal(c, 0)
    res = O.solve(O.params_for(c), w, a)
    assert res.status == O.OK and res.iterations == 1
    assert res.trace[0, 1] == ex["p"] and res.samples == ex["samples"]


def test_example_4d():
    ex = GOLD["example_4d"][0]
    for u, w in zip(ex["u"], ex["w"]):
        assert O.wrap_freq(u, ex["N"], ex["blocks"]).tolist() == w
    w = np.array(ex["w"], np.int32)
    a = np.array([1.0 + 0.5j, -0.25 + 1j])
    res = O.solve(O.Params(d=4, N=ex["N"], k=2, blocks=ex["blocks"]), w, a)
    ws, as_ = W.canonical_sort(w, a)
    assert res.status == O.OK and (res.w == ws).all() and np.abs(res.a - as_).max() < 1e-13


def test_fig2_projection_order():
    """Fig. 2 / P:134: with collisions on both axes, one mode is recovered on the first axis and
    the other two after subtracting it and switching axis (adaptive subtraction)."""
    ex = GOLD["fig2"][0]
    w = np.array(ex["w"], np.int32)
    a = np.exp(2j * np.pi * np.array([0.1, 0.4, 0.7]))
    res = O.solve(O.Params(d=2, N=ex["N"], k=3, blocks=(1, 1), primes=ex["primes"]), w, a)
    assert res.status == O.OK
    assert res.trace[:, 4].tolist() == ex["accepted_per_iteration"]
    ws, as_ = W.canonical_sort(w, a)
    assert (res.w == ws).all()


def test_rectangle_stalls_untilted_and_tilt_recovers():
    """P:119 worst case stalls under parallel projection; Eq. (27) tilt (3,4,5) separates it."""
    ex = GOLD["rectangle"][0]
    w = np.array(ex["w"], np.int32)
    a = np.exp(2j * np.pi * np.array([0.1, 0.3, 0.6, 0.8]))
    res = O.solve(O.Params(d=2, N=ex["N"], k=4, blocks=(1, 1)), w, a)
    assert res.status == O.PARTIAL and res.w.shape[0] == 0
    res = O.solve(O.Params(d=2, N=ex["N"], k=4, blocks=(1, 1), tilts=[tuple(ex["tilt"])]), w, a)
    ws, as_ = W.canonical_sort(w, a)
    assert res.status == O.OK and (res.w == ws).all() and np.abs(res.a - as_).max() < 1e-12


def _brute_force_modes(w, a, N):
    """Dense d-dim DFT of f sampled on the N^d grid (textbook Fourier-series coefficients)."""
    d = w.shape[1]
    grid = np.stack(np.meshgrid(*[np.arange(N)] * d, indexing="ij"), -1).reshape(-1, d)
    ph = (grid @ w.T.astype(np.int64)) % N                    # exact (w . x) mod N
    f = (np.exp(2j * np.pi * ph / N) * a[None, :]).sum(1).reshape([N] * d)
    coef = np.fft.fftn(f) / N ** d
    idx = np.argwhere(np.abs(coef) > 1e-8)
    wb = ((idx + N // 2) % N) - N // 2                       # bin index -> frequency in [-N/2, N/2)
    return W.canonical_sort(wb.astype(np.int32), coef[tuple(idx.T)])


def test_config1_vs_brute_force_dft():
    """BASELINE configs[0]: the 4096-point DFT on the 64x64 grid and the oracle agree exactly."""
    c = W.CONFIGS["c1"]
    for t in range(20):
        w, a = W.make_signal(c, t)
        wb, ab = _brute_force_modes(w, a, c.N)
        for blocks in (c.blocks, c.alt_blocks):
            res = O.solve(O.params_for(c, blocks=blocks), w, a)
            assert res.status == O.OK
            assert res.w.shape == wb.shape and (res.w == wb).all()
            assert np.abs(res.a - ab).max() < 1e-10


def test_small_instances_vs_brute_force():
    """d=2, N=8, k <= 6, 200 instances; plus d=3, N=8, partition (2,1)."""
    fails = 0
    for t in range(200):
        k = 1 + t % 6
        c = W.custom_config(2, 8, k, (1, 1), cfg=50)
        w, a = W.make_signal(c, t)
        wb, ab = _brute_force_modes(w, a, 8)
        res = O.solve(O.params_for(c), w, a)
        if res.status != O.OK:
            fails += 1       # a stall on a tiny box (axis-aligned worst case)
            continue
        assert (res.w == wb).all() and np.abs(res.a - ab).max() < 1e-10
    assert fails <= 20
    for t in range(30):
        c = W.custom_config(3, 8, 5, (2, 1), cfg=51)
        w, a = W.make_signal(c, t)
        wb, ab = _brute_force_modes(w, a, 8)
        res = O.solve(O.params_for(c), w, a)
        assert res.status == O.OK and (res.w == wb).all() and np.abs(res.a - ab).max() < 1e-10


@pytest.mark.parametrize("name,trials", [("c1", range(100)), ("c2", range(4)), ("c4", range(1))])
def test_exact_recovery_invariant(name, trials):
    """P:426 'recover the frequency vectors perfectly': noiseless inputs are recovered exactly."""
    c = W.CONFIGS[name]
    for t in trials:
        w, a = W.make_signal(c, t)
        ws, as_ = W.canonical_sort(w, a)
        for blocks in ((c.blocks, c.alt_blocks) if name != "c4" else (c.blocks,)):
            res = O.solve(O.params_for(c, blocks=blocks), w, a)
            assert res.status == O.OK, (name, t, blocks)
            assert (res.w == ws).all()
            assert np.abs(res.a - as_).max() <= 1e-12 * np.abs(as_).max()


def test_paper_config_small_k():
    """P:422-426 (N=20, d1=5, d=100): exact recovery and l2 error far below 1e-9 (SPEC crit. 1)."""
    for k in (1, 2, 4, 8):
        c = W.paper_config(100, k)
        for t in range(2):
            w, a = W.make_signal(c, t)
            res = O.solve(O.params_for(c), w, a)
            ws, as_ = W.canonical_sort(w, a)
            assert res.status == O.OK and (res.w == ws).all()
            assert np.sqrt(np.sum(np.abs(res.a - as_) ** 2)) < 1e-12


def test_partial_when_sparsity_overstated():
    """Alg. 2 loops while |R| < k: with k larger than the true sparsity the stall rule (C19)
    ends the solve with PARTIAL and the true modes in the registry."""
    w = np.array([[3, -2], [1, 5], [0, 0]], np.int32)
    a = np.array([1.0, 1j, 0.0])          # the third term has a zero coefficient: 2-sparse signal
    res = O.solve(O.Params(d=2, N=16, k=3, blocks=(1, 1)), w, a)
    assert res.status == O.PARTIAL
    ws, _ = W.canonical_sort(w[:2], a[:2])
    assert (res.w == ws).all()


# ------------------------------------------------------------------ stall fallback (reading R23)
def test_fallback_tilt_schedule():
    """Four Pythagorean triples (Eq. (25): b^2 + h^2 = c^2, gcd = 1) on disjoint reduced-axis pairs."""
    assert O.fallback_tilts(1, 1) == []
    assert O.fallback_tilts(2, 1) == [(0, 1, 3, 4, 5)]
    assert O.fallback_tilts(2, 2) == [(0, 1, 5, 12, 13)]
    assert O.fallback_tilts(3, 2) == [(1, 2, 5, 12, 13)]
    assert O.fallback_tilts(3, 3) == [(0, 2, 8, 15, 17)]
    assert O.fallback_tilts(5, 4) == [(0, 3, 7, 24, 25), (1, 4, 7, 24, 25)]
    for r in range(2, 9):
        pairs = set()
        for lvl in range(1, 5):
            ts = O.fallback_tilts(r, lvl)
            axes = [x for t in ts for x in t[:2]]
            assert len(axes) == len(set(axes))                        # disjoint pairs
            for (a0, a1, b, h, c) in ts:
                assert b * b + h * h == c * c and np.gcd(b, c) == 1 and np.gcd(h, c) == 1
                pairs.add((a0, a1))
        if r <= 4:                                                    # every axis pair tilted at some level
            assert pairs == {(i, j) for i in range(r) for j in range(i + 1, r)}


@pytest.mark.parametrize("d,N,k,blocks,structure", [(2, 16, 8, (1, 1), "rectangles"), (2, 16, 8, (1, 1), "rect_mix"),
                                                    (3, 16, 16, (1, 1, 1), "rectangles"),
                                                    (4, 8, 8, (2, 2), "rect_mix")])
def test_stall_fallback_recovers_worst_case(d, N, k, blocks, structure):
    """P:119 rectangles stall under parallel projection (PARTIAL without the fallback); with the fallback
    (tilting after a stall, keeping what was found) the recovered set and coefficients equal the
    brute-force dense d-dimensional DFT of f on the N^d grid."""
    c = W.custom_config(d, N, k, blocks, structure=structure)
    n_done = 0
    for t in range(8):
        try:
            w, a = W.make_signal(c, t)
        except AssertionError:
            continue
        r0 = O.solve(O.Params(d=d, N=N, k=k, blocks=blocks), w, a)
        r4 = O.solve(O.Params(d=d, N=N, k=k, blocks=blocks, n_fallback=4), w, a)
        wb, ab = _brute_force_modes(w, a, N)
        assert r4.status == O.OK and np.array_equal(r4.w, wb) and np.abs(r4.a - ab).max() < 1e-11
        if r0.status == O.PARTIAL:
            # the trace shows the stall: stall_limit zero-accept iterations right before the switch
            sl = max(2 * len(blocks), 16)
            acc = r4.trace[:, 4]
            runs = [len(x) for x in "".join("0" if v == 0 else "1" for v in acc).split("1")]
            assert max(runs) >= sl
            assert r4.samples > r0.samples
        n_done += 1
    assert n_done >= 5


def test_stall_fallback_keeps_found_modes():
    """Entries found before the switch are mapped exactly into the tilted coordinates: a mixed signal needs
    fewer iterations after the switch than a solve that starts tilted from scratch would need for all k."""
    c = W.custom_config(2, 64, 12, (1, 1), structure="rect_mix")
    w, a = W.make_signal(c, 3)
    r0 = O.solve(O.Params(d=2, N=64, k=12, blocks=(1, 1)), w, a)
    assert r0.status == O.PARTIAL and 0 < r0.w.shape[0] < 12
    r1 = O.solve(O.Params(d=2, N=64, k=12, blocks=(1, 1), n_fallback=1), w, a)
    ws, as_ = W.canonical_sort(w, a)
    assert r1.status == O.OK and np.array_equal(r1.w, ws) and np.abs(r1.a - as_).max() < 1e-12
    # after the switch the first prime is the first prime >= c k* with k* = k - (modes kept), not c k
    sw = r0.trace.shape[0]
    assert r1.trace[sw, 1] == O.ith_prime_at_least(5 * (12 - r0.w.shape[0]), 1)


# ------------------------------------------------------------------ Alg. 2 decision branches: cap, accumulate, prune
def _cap_fixture(E):
    """Hand-made bins of one p = 11 iteration (r = 1): singletons at b = 3, 5, 9 with |F_0| = 33, 22, 22 EXACTLY
    (F_0 = 33, 22, 22i: the two 22s are an exact magnitude tie), shifted line F_1[b] = F_0[b] e^{2 pi i v/E}
    (Eq. (4)) with v = 3, 5, -2 (v = b mod 11)."""
    p = 11
    F = np.zeros((2, p), np.complex128)
    for b, f0, v in ((3, 33.0, 3), (5, 22.0, 5), (9, 22.0j, -2)):
        F[0, b] = f0
        F[1, b] = f0 * cmath.exp(2j * math.pi * v / E)
    return p, F


def test_select_cap_keeps_largest_ties_to_smaller_b():
    """Alg. 2 l.18 SORT with readings C5/C6: when more than k* bins are non-empty only the k* largest
    |F_0| are examined, ties going to the smaller b; the examined bins are then processed in ascending b.
    Fails if the cap keeps the smallest bins, breaks ties towards the larger b, or does not bind."""
    P = O.Params(d=1, N=16, k=3, blocks=(1,))
    E, lo, hi = O.prepare(P)
    p, F = _cap_fixture(E)
    nc, acc_b, acc_v, acc_a = O.decode(P, E, lo, hi, p, 0, 3, F)
    assert nc == 3 and acc_b.tolist() == [3, 5, 9] and acc_v[:, 0].tolist() == [3, 5, -2]
    nc, acc_b, acc_v, acc_a = O.decode(P, E, lo, hi, p, 0, 2, F)
    assert nc == 2 and acc_b.tolist() == [3, 5] and acc_v[:, 0].tolist() == [3, 5]    # 22 vs 22i: smaller b
    assert abs(acc_a[0] - 3.0) < 1e-15 and abs(acc_a[1] - 2.0) < 1e-15               # a = F_0 / p (Eq. (7))
    nc, acc_b, _, _ = O.decode(P, E, lo, hi, p, 0, 1, F)
    assert nc == 1 and acc_b.tolist() == [3]
    # swap the tie's phases: still the smaller b wins; make b = 9 strictly larger: it is kept instead of b = 5
    F2 = F.copy()
    F2[:, 9] *= (22.0 + 1e-9) / 22.0
    _, acc_b, _, _ = O.decode(P, E, lo, hi, p, 0, 2, F2)
    assert acc_b.tolist() == [3, 9]


# Workloads that force false accepts (pins of Alg. 2 l.30 / l.33): tau = 0.5 and round_tol = 0.5 let collided bins
# pass Eq. (42), extra_checks = 0 drops the range and bin-consistency rejections (2: bin consistency only).  A false entry
# puts a spurious mode -a' at v' into the residual; a later iteration finds it isolated, decodes v' again and the
# accumulation R[v'] += -a' cancels it to rounding, which the prune removes.  The wrong residual also holds more
# non-empty bins than k*, so the cap binds.  Seeds listed here are ones where the oracle ends with the exact
# input spectrum (seeds where a false entry survives to |R| = k exist too: the method then returns a wrong set,
# which the GPU must reproduce -- tests/test_gpu_parity.py).
FFA_CASES = [((2, 128, 40, (1, 1)), (2, 7, 26, 32)), ((3, 32, 30, (1, 1, 1)), (13, 28, 29)),
             ((3, 16, 20, (2, 1)), (6, 7, 36))]
FFA_PARAMS = dict(tol=0.5, round_tol=0.5, extra_checks=0, max_iter=60)


def ffa_config(d, N, k, blocks):
    return W.custom_config(d, N, k, blocks, cfg=81, rho="uniform1_10")


@pytest.mark.parametrize("extra", [0, 2])
@pytest.mark.parametrize("case,seeds", FFA_CASES)
def test_forced_false_accepts_accumulate_prune_exact(case, seeds, extra):
    """Alg. 2 l.30 'R <- R u (w, a)' read as R[v] += a (C16) and l.33 prune (C17): with forced false accepts
    the oracle still ends with the brute-force dense DFT's spectrum, and its trace shows the k* cap binding,
    keys found again (accumulated) and entries pruned.  Replacing instead of accumulating leaves the spurious
    entry with a non-zero coefficient (never pruned, so the set is wrong); dropping the prune keeps it too."""
    d, N, k, blocks = case
    c = ffa_config(d, N, k, blocks)
    for t in seeds:
        w, a = W.make_signal(c, t)
        res = O.solve(O.params_for(c, **dict(FFA_PARAMS, extra_checks=extra)), w, a)
        wb, ab = _brute_force_modes(w, a, N)
        assert res.status == O.OK, t
        assert res.w.shape == wb.shape and np.array_equal(res.w, wb), t
        assert np.all(np.abs(res.a - ab) <= 1e-10 * np.abs(ab)), t
        tr = res.trace
        assert (tr[:, 5] > tr[:, 3]).any(), t           # more non-empty bins than k*: the cap bound
        assert (tr[:, 3] == np.minimum(tr[:, 5], k - np.concatenate([[0], np.cumsum(tr[:-1, 4] - tr[:-1, 6]
                                                                                   - tr[:-1, 7])]))).all(), t
        assert tr[:, 6].sum() > 0 and tr[:, 7].sum() > 0, t


# ------------------------------------------------------------------ randomized axis order (reading R24)
def test_round_robin_levels_cover_every_axis_pair():
    """Levels 5.. tilt the pairs of the circle-method round robin over a seeded axis order: disjoint pairs per
    level, r - 1 rounds (r even; r for odd r), every pair of axes exactly once, then the schedule ends."""
    for r in range(2, 11):
        pi = O.axis_order(r)
        assert sorted(pi) == list(range(r))
        n = r + (r & 1)
        seen = []
        for j in range(n - 1):
            ts = O.fallback_tilts(r, 5 + j)
            axes = [x for t in ts for x in t[:2]]
            assert len(axes) == len(set(axes)) and len(ts) == r // 2
            tri = [(3, 4, 5), (5, 12, 13), (8, 15, 17), (7, 24, 25)][j % 4]
            assert all(tuple(t[2:]) == tri for t in ts)
            seen += [tuple(sorted(t[:2])) for t in ts]
        assert sorted(seen) == [(i, j) for i in range(r) for j in range(i + 1, r)]
        assert O.fallback_tilts(r, 5 + n - 1) == []


@pytest.mark.parametrize("d,N,k,seeds,brute", [(6, 8, 8, range(3), True), (8, 16, 8, range(3), False),
                                                (20, 16, 8, range(2), False)])
def test_far_apart_rectangles_need_the_round_robin(d, N, k, seeds, brute):
    """Rectangles on axes at least 4 apart are never tilted by the fixed-stride levels 1-4: the solve stalls
    through them and ends PARTIAL; with the round-robin levels some level tilts their pair and the solve
    recovers the input spectrum exactly -- for d = 6, N = 8 also the brute-force dense DFT's."""
    c = W.custom_config(d, N, k, (1,) * d, cfg=85, structure="rect_far")
    for t in seeds:
        w, a = W.make_signal(c, t)
        r4 = O.solve(O.params_for(c, n_fallback=4), w, a)
        assert r4.status == O.PARTIAL, t
        rr = O.solve(O.params_for(c, n_fallback=O.MAX_FALLBACK), w, a)
        ws, as_ = W.canonical_sort(w, a)
        assert rr.status == O.OK and np.array_equal(rr.w, ws), t
        assert np.all(np.abs(rr.a - as_) <= 1e-12 * np.abs(as_)), t
        if brute:
            wb, ab = _brute_force_modes(w, a, N)
            assert np.array_equal(rr.w, wb) and np.all(np.abs(rr.a - ab) <= 1e-10 * np.abs(ab))


# ------------------------------------------------------------------ multi-prime speculation (NEXT #3, reading R26)
@pytest.mark.parametrize("name,trials", [("c1", range(40)), ("c2", range(3))])
def test_speculation_exact_and_fewer_iterations(name, trials):
    """Reading R26: G primes per iteration against one snapshot of the registry, merged in prime order.  Noiseless
    inputs are still recovered exactly -- a key two primes of one iteration both isolate is counted once
    (double counting would leave 2 a_j); G = 1 is Alg. 2 itself (identical trace); the iterations never exceed
    G = 1's."""
    c = W.CONFIGS[name]
    for t in trials:
        w, a = W.make_signal(c, t)
        ws, as_ = W.canonical_sort(w, a)
        base = O.solve(O.params_for(c), w, a)
        one = O.solve(O.params_for(c, n_spec=1), w, a)
        assert np.array_equal(base.trace, one.trace) and base.samples == one.samples
        for G in (2, 3, 4):
            res = O.solve(O.params_for(c, n_spec=G), w, a)
            assert res.status == O.OK, (name, t, G)
            assert np.array_equal(res.w, ws)
            assert np.abs(res.a - as_).max() <= 1e-12 * np.abs(as_).max(), (name, t, G)
            assert res.iterations <= base.iterations, (name, t, G)


def test_speculation_two_primes_isolating_one_mode_count_it_once():
    """k = 1: both primes of iteration 1 isolate the single mode; the merge keeps one entry with a_0 (not 2 a_0),
    one iteration, f evaluated on both primes' lines."""
    c = W.custom_config(3, 64, 1, (1, 1, 1), cfg=82)
    for t in range(10):
        w, a = W.make_signal(c, t)
        res = O.solve(O.params_for(c, n_spec=2), w, a)
        assert res.status == O.OK and res.iterations == 1
        assert np.array_equal(res.w, w) and abs(res.a[0] - a[0]) <= 1e-12 * abs(a[0])
        assert res.trace[0, 4] == 2 and res.trace[0, 6] == 0       # two accepted bins, no accumulation
        assert res.samples == 4 * (5 + 7)                           # primes 5 and 7 (counters 1, 2 from c k* = 5)


SPEC_FFA_CASE, SPEC_FFA_SEEDS = (3, 32, 30, (1, 1, 1)), (2, 13, 15, 27, 36)


def test_speculation_forced_false_accepts_exact():
    """R26 with forced false accepts (keys re-found and accumulated, entries pruned): on these seeds the G = 2
    schedule ends with the brute-force dense DFT's spectrum (on others the false entries fill R to k first, as
    they can under Alg. 2 itself); its trace shows accumulations and prunes.  (A key re-found inside one prime's
    own set -- R25, kept accumulating -- did not occur on 240 seeds of the three FFA cases, so the same-set
    distinction of the merge is not observable here.)"""
    d, N, k, blocks = SPEC_FFA_CASE
    c = ffa_config(d, N, k, blocks)
    for t in SPEC_FFA_SEEDS:
        w, a = W.make_signal(c, t)
        wb, ab = _brute_force_modes(w, a, N)
        res = O.solve(O.params_for(c, **dict(FFA_PARAMS, n_spec=2)), w, a)
        assert res.status == O.OK, t
        assert res.w.shape == wb.shape and np.array_equal(res.w, wb), t
        assert np.all(np.abs(res.a - ab) <= 1e-10 * np.abs(ab)), t
        assert res.trace[:, 6].sum() > 0 and res.trace[:, 7].sum() > 0, t
