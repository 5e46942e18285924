"""Experiment: a batch split over two plans driven from two host threads on two CUDA streams (host round trips of
one half hidden behind the other half's kernels) vs one plan over the whole batch.  Device time with CUDA events
on the default stream after a cross-stream join."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1606_07407_b200 as S  # noqa: E402
import workloads as W  # noqa: E402


def run(name, T, nsplit, steps=5):
    c = W.CONFIGS[name]
    w, a = W.make_batch(c, list(range(T)))
    wd, ad = torch.from_numpy(w).cuda(), torch.from_numpy(a).cuda()
    per = T // nsplit
    streams = [torch.cuda.Stream() for _ in range(nsplit)]
    plans, sigs = [], []
    for i in range(nsplit):
        with torch.cuda.stream(streams[i]):
            pl = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=per, stream=streams[i])
            plans.append(pl)
            sigs.append(S.sfft_signal_expsum(pl, wd[i * per:(i + 1) * per].contiguous(),
                                             ad[i * per:(i + 1) * per].contiguous()))
    torch.cuda.synchronize()

    def one(i):
        S.sfft_execute(plans[i], sigs[i])

    for _ in range(2):
        ths = [threading.Thread(target=one, args=(i,)) for i in range(nsplit)]
        [t.start() for t in ths]
        [t.join() for t in ths]
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for s in streams:
            s.wait_event(e0)
        ths = [threading.Thread(target=one, args=(i,)) for i in range(nsplit)]
        [t.start() for t in ths]
        [t.join() for t in ths]
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = sorted(ts)[len(ts) // 2]
    print(f"{name} T={T} split={nsplit}: {ms:.3f} ms  {T * c.k / ms / 1e3:.2f} M modes/s", flush=True)


if __name__ == "__main__":
    for name, T in (("c3", 100), ("c5", 100), ("c4", 100)):
        for ns in (1, 2, 4):
            run(name, T, ns)
