"""Summarise ncu outputs into profiles/ (tracked): kernel shares from a launch list, key metrics of a
full capture, and profiles/expsum_ncu.json (DRAM bytes per launch, read by bench.py for `traffic`)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": n, "total_us": t / 1e3, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]


def full_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    units = next(r)
    res = []
    for row in r:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        item = {"kernel": d.get("Kernel Name")}
        for k in KEYS:
            if k in d:
                item[k] = f"{d[k]} {u.get(k, '')}".strip()
        st = {}
        for k, v in d.items():
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    st[k.split("stalled_")[-1]] = float(v)
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        item["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        res.append(item)
    return res


def _bytes(s):
    v, unit = s.split()[0], (s.split() + [""])[1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * mult


if __name__ == "__main__":
    tag = sys.argv[1]
    launches, full = sys.argv[2], sys.argv[3]
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    shares = launch_shares(launches)
    json.dump(shares, open(os.path.join(prof, f"{tag}_launch_shares.json"), "w"), indent=1)
    summ = full_summary(full)
    json.dump(summ, open(os.path.join(prof, f"{tag}_expsum_ncu_full.json"), "w"), indent=1)
    s0 = summ[0]
    dram = _bytes(s0["dram__bytes_read.sum"]) + _bytes(s0["dram__bytes_write.sum"])
    json.dump({"source": f"profiles/{tag}_expsum_ncu_full.json", "kernel": s0["kernel"],
               "dram_bytes_per_launch": dram,
               "note": "one ncu --set full capture of the iteration-1 exp-sum launch of the bench workload"},
              open(os.path.join(prof, "expsum_ncu.json"), "w"), indent=1)
    for s in shares:
        print(f"{s['kernel'][:60]:60s} n={s['launches']:4d} {s['total_us']:10.1f} us  {100 * s['share']:5.1f}%")
    print(json.dumps(summ, indent=1)[:2000])
