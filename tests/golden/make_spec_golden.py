"""Writes tests/golden/oracle_spec.npz: the CPU oracle's multi-prime speculation (reading R26, n_spec = G) on
seeded full-size signals of BASELINE's configs.

Calls only oracle/ and workloads/ (never the CUDA path).  Re-run after any change to the oracle's arithmetic:

    python tests/golden/make_spec_golden.py
"""
import hashlib
import os
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O      # noqa: E402
import workloads as W   # noqa: E402

CASES = [("c3", 0, 2), ("c3", 1, 4), ("c5", 0, 4), ("c4", 0, 2), ("c4", 1, 8)]


def run(name, trial, G):
    c = W.CONFIGS[name]
    w, a = W.make_signal(c, trial)
    return O.solve(O.params_for(c, n_spec=G), w, a)


def main():
    out = {}
    with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
        jobs = [(name, t, G, ex.submit(run, name, t, G)) for name, t, G in CASES]
        for name, t, G, fut in jobs:
            res = fut.result()
            key = f"{name}_{t}_G{G}"
            out[key + "_status"] = np.int32(res.status)
            out[key + "_w_sha256"] = np.frombuffer(hashlib.sha256(np.ascontiguousarray(res.w).tobytes()).digest(),
                                                   np.uint8)
            out[key + "_count"] = np.int32(res.w.shape[0])
            out[key + "_a"] = res.a
            out[key + "_samples"] = np.int64(res.samples)
            out[key + "_trace"] = res.trace
            print(key, res.status, res.iterations, res.samples, flush=True)
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_spec.npz"), **out)


if __name__ == "__main__":
    main()
