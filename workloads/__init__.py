"""Seeded synthetic workloads for the multidimensional phase-shift sparse FFT.

This module is the ONE place that both the CPU oracle (``oracle/``) and the CUDA
path (``paper_1606_07407_b200``) take their inputs from.  It holds none of the
method's arithmetic: it only draws ground-truth spectra {(omega_j, a_j)} the way
the paper's experiments do (Sec. 5: "We randomly choose k frequency
vectors ... and corresponding coefficients a_j = e^{2 pi i theta_j} ... from
randomly chosen angles theta_j in [0,1)") and names the BASELINE.json configs
with their partitions.

Recipe:
  * rng = numpy Generator(PCG64(seed)), seed = 1_000_000 * cfg + trial.
  * omega rows ~ integers(-N/2, N/2, (k, d)); duplicate rows are redrawn (first
    occurrence kept) until all k rows are distinct (Eq. (9): distinct modes).
  * theta ~ random(k); a = rho * exp(2 pi i theta) with rho = 1, or rho ~
    uniform(1, 10, k) for config 3 (BASELINE.json configs[2]).
  * config 5 ("collinear groups"): G groups of k/G modes; each group draws a
    base vector ~ integers(-N/2, N/2, d), an axis alpha ~ integers(0, d) and
    k/G distinct values on that axis (choice(N, k/G, replace=False) - N/2).
  * "rectangles" (SURVEY NEXT #2, P:119 / P:213): axis-aligned 2x2 rectangles
    in a random pair of coordinates, the paper's worst case; "rect_far": the same
    with the two coordinates at least 4 axes apart.

Arrays: omega int32 [k, d] (C-contiguous), a complex128 [k].
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    """One workload: BASELINE.json configs[idx] plus the partition used by both sides."""

    cfg: int                      # 1-based BASELINE config number (seed namespace)
    name: str
    d: int
    N: int
    k: int
    blocks: Tuple[int, ...]       # primary partition (d_1, ..., d_r), SURVEY 8(d) / C21
    alt_blocks: Tuple[int, ...]   # alternate partition exercised in parity tests
    trials: int                   # signals per batch (bench step)
    rho: str = "unit"             # "unit" or "uniform1_10"
    structure: str = "uniform"    # "uniform", "collinear", "rectangles", "rect_mix"
    groups: int = 0               # collinear groups (config 5)

    def seed(self, trial: int) -> int:
        return 1_000_000 * self.cfg + int(trial)


def _uniform_blocks(d: int, d1: int) -> Tuple[int, ...]:
    assert d % d1 == 0
    return tuple([d1] * (d // d1))


# BASELINE.json "configs" (index = cfg - 1); partitions from SURVEY.md 8(d).
CONFIGS = {
    "c1": Config(1, "c1", d=2, N=64, k=4, blocks=(1, 1), alt_blocks=(2,), trials=100),
    "c2": Config(2, "c2", d=3, N=4096, k=100, blocks=(2, 1), alt_blocks=(1, 1, 1), trials=1024),
    "c3": Config(3, "c3", d=100, N=65536, k=1000, blocks=_uniform_blocks(100, 2),
                 alt_blocks=_uniform_blocks(100, 1), trials=100, rho="uniform1_10"),
    "c4": Config(4, "c4", d=1000, N=4096, k=100, blocks=_uniform_blocks(1000, 2),
                 alt_blocks=_uniform_blocks(1000, 1), trials=100),
    "c5": Config(5, "c5", d=20, N=65536, k=500, blocks=_uniform_blocks(20, 1),
                 alt_blocks=_uniform_blocks(20, 2), trials=100, structure="collinear", groups=10),
}


def paper_config(d: int, k: int, trials: int = 100) -> Config:
    """The paper's own sweep: N=20, d1=5, d in {100, 1000}, k = 2^0..2^10."""
    return Config(10 + (0 if d == 100 else 1), f"paper_d{d}_k{k}", d=d, N=20, k=k,
                  blocks=_uniform_blocks(d, 5), alt_blocks=_uniform_blocks(d, 4 if d % 4 == 0 else 5),
                  trials=trials)


def custom_config(d: int, N: int, k: int, blocks: Sequence[int], cfg: int = 99,
                  trials: int = 1, rho: str = "unit", structure: str = "uniform",
                  groups: int = 0) -> Config:
    return Config(cfg, f"custom_d{d}_N{N}_k{k}", d=d, N=N, k=k, blocks=tuple(blocks),
                  alt_blocks=tuple(blocks), trials=trials, rho=rho, structure=structure,
                  groups=groups)


def _distinct_uniform_rows(rng: np.random.Generator, N: int, k: int, d: int) -> np.ndarray:
    lo, hi = -N // 2, N // 2
    w = rng.integers(lo, hi, size=(k, d), dtype=np.int64)
    while True:
        _, first = np.unique(w, axis=0, return_index=True)
        if first.size == k:
            return w
        dup = np.setdiff1d(np.arange(k), first)
        w[dup] = rng.integers(lo, hi, size=(dup.size, d), dtype=np.int64)


def _collinear_rows(rng: np.random.Generator, N: int, k: int, d: int, groups: int) -> np.ndarray:
    assert groups > 0 and k % groups == 0 and k // groups <= N
    per = k // groups
    rows = []
    for _ in range(groups):
        base = rng.integers(-N // 2, N // 2, size=d, dtype=np.int64)
        axis = int(rng.integers(0, d))
        vals = rng.choice(N, size=per, replace=False).astype(np.int64) - N // 2
        g = np.repeat(base[None, :], per, axis=0)
        g[:, axis] = vals
        rows.append(g)
    w = np.concatenate(rows, axis=0)
    # cross-group coincidences are redrawn as whole groups are not allowed to merge
    _, first = np.unique(w, axis=0, return_index=True)
    if first.size != k:
        dup = np.setdiff1d(np.arange(k), first)
        w[dup] = _distinct_uniform_rows(rng, N, dup.size, d)
        _, first = np.unique(w, axis=0, return_index=True)
        assert first.size == k
    return w


def _rectangle_rows(rng: np.random.Generator, N: int, k: int, d: int, min_gap: int = 0) -> np.ndarray:
    """k/4 axis-aligned rectangles: 4 modes sharing all but two coordinates; min_gap > 0: the two
    coordinates are at least min_gap axes apart (pairs the fixed-stride tilt levels never tilt)."""
    assert k % 4 == 0 and d >= 2
    rows = []
    for _ in range(k // 4):
        base = rng.integers(-N // 2, N // 2, size=d, dtype=np.int64)
        i, j = rng.choice(d, size=2, replace=False)
        while min_gap and abs(int(i) - int(j)) < min_gap:
            i, j = rng.choice(d, size=2, replace=False)
        xi = rng.choice(N, size=2, replace=False) - N // 2
        xj = rng.choice(N, size=2, replace=False) - N // 2
        for a in xi:
            for b in xj:
                r = base.copy()
                r[i], r[j] = a, b
                rows.append(r)
    w = np.stack(rows)
    _, first = np.unique(w, axis=0, return_index=True)
    assert first.size == k, "rectangle generator produced duplicates; choose another seed"
    return w


def _rect_mix_rows(rng: np.random.Generator, N: int, k: int, d: int) -> np.ndarray:
    """k/2 modes in axis-aligned rectangles plus k/2 uniform distinct modes (stall-fallback tests)."""
    kr = (k // 2) // 4 * 4
    rect = _rectangle_rows(rng, N, kr, d)
    rest = []
    seen = {tuple(r) for r in rect}
    while len(rest) < k - kr:
        r = tuple(rng.integers(-N // 2, N // 2, size=d, dtype=np.int64))
        if r not in seen:
            seen.add(r)
            rest.append(r)
    return np.concatenate([rect, np.array(rest, np.int64).reshape(-1, d)])


def make_signal(c: Config, trial: int = 0, seed: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
    """Ground truth (omega int32 [k,d], a complex128 [k]) for one trial of config c."""
    s = c.seed(trial) if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(s))
    if c.structure == "uniform":
        w = _distinct_uniform_rows(rng, c.N, c.k, c.d)
    elif c.structure == "collinear":
        w = _collinear_rows(rng, c.N, c.k, c.d, c.groups)
    elif c.structure == "rectangles":
        w = _rectangle_rows(rng, c.N, c.k, c.d)
    elif c.structure == "rect_mix":
        w = _rect_mix_rows(rng, c.N, c.k, c.d)
    elif c.structure == "rect_far":
        w = _rectangle_rows(rng, c.N, c.k, c.d, min_gap=4)
    else:
        raise ValueError(c.structure)
    theta = rng.random(c.k)
    if c.rho == "unit":
        rho = np.ones(c.k)
    elif c.rho == "uniform1_10":
        rho = rng.uniform(1.0, 10.0, c.k)
    else:
        raise ValueError(c.rho)
    a = rho * np.exp(2j * np.pi * theta)
    return np.ascontiguousarray(w.astype(np.int32)), np.ascontiguousarray(a.astype(np.complex128))


def make_batch(c: Config, trials: Sequence[int]) -> Tuple[np.ndarray, np.ndarray]:
    """Stacked ground truth for several trials: omega int32 [T,k,d], a complex128 [T,k]."""
    ws, as_ = [], []
    for t in trials:
        w, a = make_signal(c, t)
        ws.append(w)
        as_.append(a)
    return np.ascontiguousarray(np.stack(ws)), np.ascontiguousarray(np.stack(as_))


def canonical_sort(w: np.ndarray, a: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Lexicographic order of frequency rows (the output order of both sides)."""
    if w.shape[0] == 0:
        return w, a
    order = np.lexsort(w.T[::-1])
    return w[order], a[order]
