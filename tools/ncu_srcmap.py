"""Aggregate an ncu report's per-instruction warp-stall samples by CUDA source line.

ncu's source page (SASS view) lists the kernel's instructions in address order with their samples; nvdisasm
with line info (-g, the library is built with -lineinfo) lists the same instructions with the source line
they came from.  Instruction i of one is instruction i of the other.

usage: python tools/ncu_srcmap.py REPORT.ncu-rep CUBIN KERNEL_SUBSTRING [top]
(CUBIN: `cuobjdump -xelf all paper_1606_07407_b200/libsfft.so` in a scratch directory.)
"""
import collections
import csv
import re
import subprocess
import sys


def ncu_rows(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv"]
    if kernel:
        cmd += ["--kernel-name", "regex:" + re.escape(kernel.split("<")[0])]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    r = csv.reader(out.splitlines())
    next(r)
    hdr = next(r)
    col = __import__("os").environ.get("SRCMAP_COL", "Warp Stall Sampling (All Samples)")   # or "Instructions Executed"
    iw, isrc = hdr.index(col), hdr.index("Source")
    rows = []
    for x in r:                                   # several launches: the first launch's listing only
        if x and x[0] in ("Kernel Name", "Address"):
            break
        if len(x) > max(iw, isrc):
            rows.append((int(x[iw]) if x[iw] else 0, x[isrc]))
    return rows


def sass_lines(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    fn, cur, res, inside = None, "?", [], False
    for line in out.splitlines():
        m = re.match(r"^\.text\.(\S+):", line.strip())
        if m:
            if inside:
                break
            if kernel in m.group(1):
                fn, inside = m.group(1), True
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        if re.search(r"/\*[0-9a-f]{4,}\*/", line) and not line.strip().startswith("//"):
            res.append((cur, line.split("*/", 1)[1].strip()))
    if fn is None:
        sys.exit(f"no function matching {kernel}")
    return fn, res


def main():
    rep, cubin, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    rows = ncu_rows(rep, sys.argv[5] if len(sys.argv) > 5 else kernel)   # argv[5]: function-name filter for ncu
    fn, ins = sass_lines(cubin, kernel)
    if len(ins) != len(rows):
        print(f"warning: {len(rows)} ncu rows vs {len(ins)} disassembled instructions ({fn})")
    agg = collections.Counter()
    for (n, _), (src, _) in zip(rows, ins):
        agg[src] += n
    tot = sum(agg.values()) or 1
    for src, n in agg.most_common(top):
        print(f"{n:8d} {100 * n / tot:5.1f}%  {src}")


if __name__ == "__main__":
    main()
