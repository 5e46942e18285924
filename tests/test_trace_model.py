"""Pins the oracle's iteration traces and sample totals (previously "parity unpinned") against a
second route to the same iteration, written from the paper and independent of the oracle's sampling and DFT.

By Eq. (3) the length-p DFT of line n's samples of the residual f - g holds, in bin b,
p * sum of c_j e^{2 pi i (u_{j,n} mod E)/E} over the residual spectrum's modes j with u_{j,m} = b (mod p), where u_j
is the unwrapped frequency of Eq. (35) and the line-0 factor is 1.  So Alg. 2 (PAPER.md:
369-417) can be run without evaluating f at all: the bins come straight from the residual spectrum (truth minus the
registry).  On those bins the model applies Alg. 2's own rules -- threshold 1e-8 p and the k* cap (C5, C18), the
Eq. (42) ratio test with tau = 1e-6 (C3, C4), the Eq. (41) phase decode rounded within 0.01 (C14), the image-range and
bin checks (C15), R[u] += F_0 / p in ascending b (C12, C16), the 1e-8 prune (C17), p = the i-th prime >= c k* on axis
m = i mod r (C10, C11), r + 1 lines of p samples per iteration (C22), PARTIAL after max(2r, 16) iterations without an
accept (C19).  The decode rules are restated (they have their own worked-value pins in test_oracle_pins.py); what
this pins is the sampling + DFT route and the iteration bookkeeping: the oracle's per-iteration prime, axis,
candidates, accepts, accumulations and prunes, its sample totals and statuses must equal the model's -- including
C5's genuine false accepts (two modes in one bin whose shifted-line phases differ by less than the ratio test
resolves) and their later correction."""
import os

import numpy as np
import pytest

import workloads as W

GOLD_DIR = os.path.join(os.path.dirname(__file__), "golden")


def _primes_upto(n):
    sieve = bytearray([1]) * (n + 1)
    sieve[0:2] = b"\x00\x00"
    for q in range(2, int(n ** 0.5) + 1):
        if sieve[q]:
            sieve[q * q::q] = bytearray(len(sieve[q * q::q]))
    return np.array([q for q in range(n + 1) if sieve[q]])


_PRIMES = _primes_upto(300000)


def _ith_prime_at_least(i, x):
    return int(_PRIMES[np.searchsorted(_PRIMES, x) + i - 1])


def alg2_frequency_domain(w, a, N, blocks, c=5, tau=1e-6, floor=1e-8, prune=1e-8, rtol=0.01, max_iter=1000,
                          extra=3):
    """Trace rows (i, p, m, candidates, accepted, non-empty, accumulated, pruned), samples, 'OK' / 'PARTIAL'."""
    offs = np.concatenate([[0], np.cumsum(blocks)]).astype(int)
    r, k = len(blocks), len(a)
    # Eq. (35): u_{j,q} = sum_{t < d_q} w_{j, off_q + t} N^t (exact in int64: N^{d_q} <= 2^40)
    U = np.zeros((k, r), np.int64)
    for q in range(r):
        for t in range(blocks[q]):
            U[:, q] += np.asarray(w)[:, offs[q] + t].astype(np.int64) * N ** t
    B = max(N ** d for d in blocks)
    E = 2 * B                                                                  # P:422, C2
    lo = np.array([-(N // 2) * (N ** d - 1) // (N - 1) for d in blocks])     # image of block q
    hi = np.array([(N // 2 - 1) * (N ** d - 1) // (N - 1) for d in blocks])
    truth = {tuple(U[j]): complex(a[j]) for j in range(k)}
    R = {}
    rows, samples, stall, i = [], 0, 0, 1
    while len(R) < k and i <= max_iter:
        kstar = k - len(R)
        p = _ith_prime_at_least(i, max(2, c * kstar))
        m = i % r
        resid = dict(truth)
        for key, v in R.items():
            resid[key] = resid.get(key, 0.0) - v
        keys = np.array(list(resid.keys()), np.int64).reshape(-1, r)
        coef = np.array(list(resid.values()), complex)
        b_of = np.mod(keys[:, m], p)
        # Eq. (3) bins of line 0 and of the r shifted lines: p sum c e^{2 pi i (u_n mod E) / E}
        F0 = np.zeros(p, complex)
        np.add.at(F0, b_of, p * coef)
        fac = np.exp(2j * np.pi * (np.mod(keys, E).astype(np.float64) / E))   # [modes, r]
        Fn = np.zeros((p, r), complex)
        np.add.at(Fn, b_of, p * coef[:, None] * fac)
        mag = np.abs(F0)
        nonempty = np.nonzero(mag >= floor * p)[0]
        if len(nonempty) > kstar:                       # the k* largest, ties to the smaller b (C5, C6)
            order = sorted(nonempty, key=lambda b: (-mag[b], b))[:kstar]
            cand = np.sort(np.array(order))
        else:
            cand = nonempty
        accepted = []
        for b in cand:                                   # ascending b
            f0 = F0[b]
            rho = np.abs(Fn[b]) / abs(f0)
            if not np.all(np.abs(rho - 1.0) < tau):
                continue
            x = np.angle(Fn[b] * np.conj(f0)) * E / (2 * np.pi)
            v = np.rint(x)
            if np.any(np.abs(x - v) > rtol):
                continue
            v = v.astype(np.int64)
            if (extra & 1) and (np.any(v < lo) or np.any(v > hi)):    # C15 (i)
                continue
            if (extra & 2) and v[m] % p != b:                          # C15 (ii)
                continue
            accepted.append((tuple(int(t) for t in v), f0 / p))
        n_acc = 0
        for key, val in accepted:
            if key in R:
                n_acc += 1
            R[key] = R.get(key, 0.0) + val
        n_pruned = 0
        for key in [key for key, v in R.items() if abs(v) < prune]:
            del R[key]
            n_pruned += 1
        rows.append((i, p, m, len(cand), len(accepted), len(nonempty), n_acc, n_pruned))
        samples += (r + 1) * p
        stall = 0 if accepted else stall + 1
        if len(R) < k and stall >= max(2 * r, 16):
            return np.array(rows, np.int64), samples, "PARTIAL"
        i += 1
    return np.array(rows, np.int64), samples, "OK" if len(R) >= k else "PARTIAL"


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_golden_traces_match_frequency_domain_model(name):
    """Every golden oracle run (both partitions): the full 8-column trace, the sample total and the status equal
    the frequency-domain model's."""
    import oracle as O
    c = W.CONFIGS[name]
    g = np.load(os.path.join(GOLD_DIR, f"oracle_{name}.npz"))
    keys = sorted({k.rsplit("_", 1)[0] for k in g.keys() if k.endswith("_trace")})
    assert keys
    for key in keys:
        tag, t = key.rsplit("_", 1)
        w, a = W.make_signal(c, int(t))
        rows, samples, status = alg2_frequency_domain(w, a, c.N, c.blocks if tag == "primary" else c.alt_blocks)
        tr = g[key + "_trace"]
        assert tr.shape == rows.shape and np.array_equal(tr, rows), key
        assert int(g[key + "_samples"]) == samples, key
        assert int(g[key + "_status"]) == (O.OK if status == "OK" else O.PARTIAL), key


def test_live_oracle_traces_match_frequency_domain_model():
    """Live oracle runs: C1 (40 seeds, both partitions) and C2 (4 seeds)."""
    import oracle as O
    for name, seeds in (("c1", range(40)), ("c2", range(4))):
        c = W.CONFIGS[name]
        for blocks in (c.blocks, c.alt_blocks):
            for t in seeds:
                w, a = W.make_signal(c, t)
                res = O.solve(O.params_for(c, blocks=blocks), w, a)
                rows, samples, status = alg2_frequency_domain(w, a, c.N, blocks)
                assert np.array_equal(res.trace, rows), (name, blocks, t)
                assert res.samples == samples and (res.status == O.OK) == (status == "OK"), (name, blocks, t)


@pytest.mark.parametrize("extra", [0, 2])
def test_forced_false_accept_traces_match_frequency_domain_model(extra):
    """The forced-false-accept workloads of test_oracle_pins (tau = 0.5, round_tol = 0.5: the k* cap binds, false
    keys are accepted, found again and pruned) give the model's trace, samples and status, every column."""
    import oracle as O
    from test_oracle_pins import FFA_CASES, FFA_PARAMS, ffa_config
    for (d, N, k, blocks), seeds in FFA_CASES:
        c = ffa_config(d, N, k, blocks)
        for t in seeds:
            w, a = W.make_signal(c, t)
            res = O.solve(O.params_for(c, **dict(FFA_PARAMS, extra_checks=extra)), w, a)
            rows, samples, status = alg2_frequency_domain(w, a, N, blocks, tau=FFA_PARAMS["tol"],
                                                          rtol=FFA_PARAMS["round_tol"],
                                                          max_iter=FFA_PARAMS["max_iter"], extra=extra)
            assert np.array_equal(res.trace, rows), (d, N, k, blocks, t, res.trace, rows)
            assert res.samples == samples and (res.status == O.OK) == (status == "OK"), (d, N, k, blocks, t)


def test_model_worked_example():
    """Hand-checkable: d = 2, N = 8, blocks (1, 1), modes (1, 2), (1, -3), (3, 2), unit coefficients.
    Iteration 1: k* = 3, p = 17 (the first prime >= 15), axis 1: u = 2, -3, 2 -> bin 2 holds two modes whose
    axis-0 shift phases differ (ratio |1 + e^{2 pi i 2/16}| / 2 = cos(pi/8) = 0.924: rejected), bin 14 one mode
    (accepted).  Iteration 2: k* = 2, p = 13 (the second prime >= 10: 11, 13), axis 0: u = 1, 3 -> two singletons.
    Samples 3 (17 + 13) = 90."""
    rows, samples, status = alg2_frequency_domain(np.array([[1, 2], [1, -3], [3, 2]]), np.ones(3), 8, (1, 1))
    assert rows[:, :5].tolist() == [[1, 17, 1, 2, 1], [2, 13, 0, 2, 2]] and samples == 90 and status == "OK"
