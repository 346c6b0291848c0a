#!/usr/bin/env python
"""Warp-stall samples of one ncu capture per CUDA source line (and per stall reason).

  ncu_lines.py <report.ncu-rep> <lib.so> <kernel mangled-name substring> [top N]

ncu's SASS page gives samples per instruction address; nvdisasm -g gives the source line of
each instruction offset of the same cubin (built with -lineinfo).  Inlined helpers are
attributed to their own lines (mbar_wait, dmma, ...)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def line_table(lib, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, check=True, capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.startswith("cv_kernel")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    table, cur, inside = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith(".text."):
            inside = kernel_sub in ln
            continue
        if not inside:
            continue
        m = re.search(r'//## File ".*?", line (\d+)', ln)
        if m:
            cur = int(m.group(1))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            table[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return table


def main():
    rep, lib, ksub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    table = line_table(lib, ksub)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                          capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(sass)))
    hdr, data = rows[1], rows[2:]
    iS = hdr.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    base = int(data[0][0], 16)
    per = collections.defaultdict(lambda: [0.0, collections.Counter(), collections.Counter()])
    tot = 0.0
    for r in data:
        off = int(r[0], 16) - base
        line, ins = table.get(off, (None, r[1]))
        v = float(r[iS] or 0)
        tot += v
        p = per[line]
        p[0] += v
        for i, h in reasons:
            x = float(r[i] or 0)
            if x:
                p[1][h[6:]] += x
        p[2][ins.split()[1] if ins.startswith("@") else ins.split()[0]] += v
    src = open(os.path.join(os.path.dirname(os.path.abspath(lib)), "csrc", "cv_kernel.cu")).read().splitlines()
    print(f"# {rep}: warp-stall samples per source line of cv_kernel.cu ({int(tot)} samples)")
    cum = 0.0
    for line, (v, rs, ops) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        cum += v
        text = src[line - 1].strip()[:70] if line and line <= len(src) else "?"
        rtop = ", ".join(f"{k} {100 * x / tot:.1f}" for k, x in rs.most_common(3))
        otop = ", ".join(f"{k} {100 * x / tot:.1f}" for k, x in ops.most_common(2))
        print(f"{100 * v / tot:6.2f}% (cum {100 * cum / tot:5.1f}) line {line}: {text}\n          reasons[{rtop}] ops[{otop}]")


if __name__ == "__main__":
    main()
