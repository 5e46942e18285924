"""Copy the evidence of one GPU call (gpurun_out/<TAG>_*) into profiles/ (tracked): bench JSON lines, the ncu
launch list and its per-kernel shares, the ncu --set full summary (tools/ncu_json.py), and profiles/expsum_ncu.json
(DRAM bytes per launch of the exp-sum capture, read by bench.py for roofline.traffic).
Usage: python tools/collect_profiles.py TAG"""
import glob
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_profiles import launch_shares  # noqa: E402
from ncu_json import summarise  # noqa: E402


def main(tag):
    src, dst = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
    for f in sorted(glob.glob(os.path.join(src, f"{tag}_bench_*.json"))):
        lines = [l for l in open(f).read().splitlines() if l.startswith("{")]
        if lines:
            open(os.path.join(dst, os.path.basename(f) + "l"), "w").write(lines[-1] + "\n")
    lc = os.path.join(src, f"{tag}_launches.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(dst, f"{tag}_launches.csv"))
        json.dump(launch_shares(lc), open(os.path.join(dst, f"{tag}_launch_shares.json"), "w"), indent=1)
    rep = os.path.join(src, f"{tag}_full.ncu-rep")
    if os.path.exists(rep):
        s = summarise(rep)
        json.dump(s, open(os.path.join(dst, f"{tag}_ncu_full.json"), "w"), indent=1)
        for k in s:
            if "pfft_kernel<1" in k["kernel"] and "dram_bytes_per_launch" in k:
                # C3 iteration 1: 100 signals x 51 lines of p = 5003 (the bench workload's first FFT launch)
                lines = int(k.get("grid", 0))
                json.dump({"source": f"profiles/{tag}_ncu_full.json", "kernel": k["kernel"],
                           "dram_bytes_per_launch": k["dram_bytes_per_launch"],
                           "algorithmic_bytes_per_launch": 32 * 5003 * lines,
                           "note": "one ncu --set full capture of the iteration-1 FFT launch of the bench workload "
                                   "(C3: grid = lines, p = 5003; algorithmic 32 B per sample)"},
                          open(os.path.join(dst, "fft_ncu.json"), "w"), indent=1)
            if "expsum_i8" in k["kernel"] and "dram_bytes_per_launch" in k:
                json.dump({"source": f"profiles/{tag}_ncu_full.json", "kernel": k["kernel"],
                           "dram_bytes_per_launch": k["dram_bytes_per_launch"],
                           "note": "one ncu --set full capture of the iteration-1 exp-sum launch of the bench workload"},
                          open(os.path.join(dst, "expsum_ncu.json"), "w"), indent=1)
    print("collected", tag)


if __name__ == "__main__":
    main(sys.argv[1])
