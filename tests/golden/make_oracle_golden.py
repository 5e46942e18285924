"""Writes tests/golden/oracle_<cfg>.npz: the CPU oracle's results on seeded configs.

Calls only oracle/ and workloads/ (never the CUDA path).  The GPU parity tests compare
the CUDA path against these files at full BASELINE sizes, where re-running the oracle
on the GPU box would take minutes.  Re-run after any change to the oracle's arithmetic:

    python tests/golden/make_oracle_golden.py c3 c4 c5
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

TRIALS = {"c1": range(16), "c2": range(16), "c3": range(4), "c4": range(4), "c5": range(4)}


def run(name, trial, blocks):
    c = W.CONFIGS[name]
    w, a = W.make_signal(c, trial)
    res = O.solve(O.params_for(c, blocks=blocks), w, a)
    return res


def main(names):
    for name in names:
        c = W.CONFIGS[name]
        out = {}
        jobs = []
        with ThreadPoolExecutor(max_workers=os.cpu_count()) as ex:
            for tag, blocks in (("primary", c.blocks), ("alt", c.alt_blocks)):
                for t in TRIALS[name]:
                    if tag == "alt" and name in ("c3", "c4", "c5") and t > 0:
                        continue
                    jobs.append((tag, t, ex.submit(run, name, t, blocks)))
            for tag, t, fut in jobs:
                res = fut.result()
                key = f"{tag}_{t}"
                out[key + "_status"] = np.int32(res.status)
                out[key + "_w_sha256"] = np.frombuffer(
                    hashlib.sha256(np.ascontiguousarray(res.w).tobytes()).digest(), np.uint8)
                out[key + "_count"] = np.int32(res.w.shape[0])
                out[key + "_a"] = res.a
                out[key + "_samples"] = np.int64(res.samples)
                out[key + "_trace"] = res.trace
                if name in ("c1", "c2"):
                    out[key + "_w"] = res.w
                print(name, key, res.status, res.iterations, res.samples, flush=True)
        np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                         f"oracle_{name}.npz"), **out)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"])
