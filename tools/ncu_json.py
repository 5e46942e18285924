"""Summarise an ncu --set full report as JSON (per kernel): duration, occupancy, pipe utilisation (tensor / FP64 /
ALU), shared-memory wavefronts and bank conflicts, DRAM bytes, FP64 instruction mix, stall reasons, hottest
source lines.  Usage: python tools/ncu_json.py report.ncu-rep [out.json]"""
import csv
import json
import subprocess
import sys

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "grid": "launch__grid_size", "block": "launch__block_size", "registers": "launch__registers_per_thread",
    "smem_per_block_bytes": "launch__shared_mem_per_block_dynamic",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "tensor_pipe_active_pct_elapsed": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tensor_mem_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "imma_inst_pct": "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "tmem_inst_pct": "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
    "tc_smem_wavefronts": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum",
    "tc_smem_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_smem_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "lsu_smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_read_bytes": "dram__bytes_read.sum", "dram_write_bytes": "dram__bytes_write.sum",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "dfma_thread_inst": "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "dadd_thread_inst": "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "dmul_thread_inst": "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
}
SCALE = {"dram__bytes_read.sum": ("MB", 1e6), "dram__bytes_write.sum": ("MB", 1e6)}


def _num(v, unit):
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return v
    u = unit.strip()
    if u in ("Mbyte", "MB"):
        x *= 1e6
    elif u in ("Kbyte", "KB"):
        x *= 1e3
    elif u in ("Gbyte", "GB"):
        x *= 1e9
    elif u == "msecond":
        pass
    elif u == "usecond":
        x /= 1e3
    elif u == "nsecond":
        x /= 1e6
    elif u in ("cycle/nsecond", "Ghz", "GHz"):
        pass
    elif u == "cycle/usecond":
        x /= 1e3
    return x


def summarise(rep, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for row in data:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for k, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                d[k] = _num(row[i], units[i])
        if "dram_read_bytes" in d:
            d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((h.split("stalled_")[-1], float(row[i])))
                except ValueError:
                    pass
        tot = sum(v for _, v in st) or 1.0
        d["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda x: -x[1])[:8]}
        res.append(d)
    # hottest source lines of each kernel (source page lists one kernel after another)
    try:
        src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                             capture_output=True, text=True).stdout
        lines = list(csv.reader(src.splitlines()))
        hot = []
        cur = None
        for l in lines:
            if len(l) == 1 or (l and l[0].startswith("Kernel")):
                continue
            if l and l[0] == "#":
                cur = l
                continue
            if cur is None or len(l) != len(cur):
                continue
            try:
                iw = cur.index("Warp Stall Sampling (All Samples)")
                isrc = cur.index("Source")
                v = l[iw]
                if v:
                    hot.append((int(v), l[isrc].strip()[:110]))
            except (ValueError, IndexError):
                continue
        tot = sum(v for v, _ in hot) or 1
        if res:
            res[-1]["hot_lines_all_kernels"] = [f"{100 * v / tot:.1f}% {s}" for v, s in sorted(hot, reverse=True)[:top]]
    except Exception as e:  # noqa: BLE001
        if res:
            res[-1]["hot_lines_error"] = str(e)
    return res


if __name__ == "__main__":
    r = summarise(sys.argv[1])
    s = json.dumps(r, indent=1)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(s + "\n")
    print(s)
