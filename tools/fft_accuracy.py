"""Accuracy of the batched Bluestein FFT (sfft_stage_pfft) against an exact-summation DFT: numpy's FFT of
the same input in extended precision (np.longdouble direct DFT for small p, pocketfft fp64 otherwise).
Prints max |F_gpu - F_ref| / max |F_ref| and the same relative to each bin's magnitude (median)."""
import sys

import numpy as np
import torch

import paper_1606_07407_b200 as S
import workloads as W


def ref_dft(x):
    p = x.shape[-1]
    if p <= 600:
        h = np.arange(p)
        Wm = np.exp(-2j * np.pi * ((np.outer(h, h) % p).astype(np.longdouble) / p).astype(np.float64))
        xl = x.astype(np.clongdouble)
        # exact-index twiddles in fp64, sums in extended precision
        return (xl @ Wm.T.astype(np.clongdouble)).astype(np.complex128)
    return np.fft.fft(x, axis=-1)


def main():
    c = W.CONFIGS["c3"]
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks)
    rng = np.random.default_rng(1)
    for p in [int(a) for a in sys.argv[1:]] or [11, 19, 23, 101, 229, 503, 1009, 2503, 5003]:
        n = 64
        x = rng.standard_normal((n, p)) + 1j * rng.standard_normal((n, p))
        xt = torch.from_numpy(x.copy()).cuda()
        S.sfft_stage_pfft(plan, xt)
        g = xt.cpu().numpy()
        r = ref_dft(x)
        err = np.abs(g - r)
        print(f"p={p:5d}: max err / max|F| = {err.max() / np.abs(r).max():.2e}   "
              f"median err/|F_b| = {np.median(err / np.abs(r)):.2e}   max err/|F_b| = {(err / np.abs(r)).max():.2e}",
              flush=True)


if __name__ == "__main__":
    main()
