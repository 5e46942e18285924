"""Summarise an ncu report: key throughput metrics, stall reasons, hottest source lines."""
import csv
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    hdr = next(r)
    next(r)
    return [dict(zip(hdr, row)) for row in r]


KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__cycles_elapsed.avg.per_second"]


def main(rep, top=20):
    for d in raw(rep):
        for k in KEYS:
            if k in d:
                print(f"{k:75s} {d[k]}")
        st = []
        for k, v in d.items():
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    st.append((k.split("stalled_")[-1], float(v)))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1
        print("stalls:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st, key=lambda x: -x[1])[:8]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    next(r)
    hdr = next(r)
    rows = list(r)
    iw = hdr.index("Warp Stall Sampling (All Samples)")
    isrc = hdr.index("Source")
    tot = sum(int(x[iw]) for x in rows) or 1
    for x in sorted(rows, key=lambda x: -int(x[iw]))[:top]:
        print(f"{int(x[iw]):7d} {100 * int(x[iw]) / tot:5.1f}%  {x[isrc][:100]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
