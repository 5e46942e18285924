"""Host-buffer pipeline: effect of CPU writes to the pinned output buffers between calls (debugging aid)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_1606_07407_b200 as S
import workloads as W

for name in sys.argv[1:] or ["c2"]:
    c = W.CONFIGS[name]
    T = 1024 if name == "c2" else 100
    nb = 10
    w, a = W.make_batch(c, range(T))
    plan = S.sfft_plan(c.d, c.N, c.k, blocks=c.blocks, batch=T)
    wh, ah = torch.from_numpy(w).pin_memory(), torch.from_numpy(a).pin_memory()
    wb = wh.unsqueeze(0).expand(nb, *wh.shape).contiguous().pin_memory()
    ab = ah.unsqueeze(0).expand(nb, *ah.shape).contiguous().pin_memory()
    bo = (torch.empty((nb, T, c.k, c.d), dtype=torch.int32).pin_memory(),
          torch.empty((nb, T, c.k, 2), dtype=torch.float64).pin_memory(),
          torch.empty((nb, T), dtype=torch.int32).pin_memory(), torch.empty((nb, T), dtype=torch.int32).pin_memory())
    def call(tag):
        t = time.perf_counter()
        S.sfft_solve_host_batches(plan, wb, ab, bo)
        print(name, tag, "%.3f ms/step" % ((time.perf_counter() - t) * 1e3 / nb), flush=True)
    for i in range(3):
        call("plain")
    for i in range(3):
        bo[0].fill_(-1); call("after fill of out freqs")
    for i in range(3):
        call("plain")
    for i in range(3):
        bo[0].fill_(-1); time.sleep(0.2); call("after fill + 0.2 s sleep")
    for i in range(3):
        x = bo[0].sum(); call("after a CPU read of out freqs")
    for i in range(3):
        time.sleep(0.2); call("after 0.2 s sleep")
