#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (the judged copies; gpurun_out/ is scratch).

  summarize_ncu.py launches <launches.csv> <header line>      -> per-kernel launch table
  summarize_ncu.py full <report.ncu-rep> <kernel label> <out.json> [sass_top.txt] [configs in the launch]
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, header):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}.get(r["Metric Unit"], 1e-6)
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + float(r["Metric Value"].replace(",", "")) * scale)
    total = sum(t for _, t in agg.values())
    print(f"# {header}")
    print("# kernel, launches, total ms, share of GPU time (cold-cache, serialised)")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:72]:72s} {n:5d} {t:12.3f} {100 * t / total:6.2f}%")


def full(rep, label, out, sass_out=None, configs="1"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def num(name, scale_to=None):
        v, u = get[name]
        x = float(v.replace(",", ""))
        mult = {"Tbyte": 1e12, "Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "s": 1.0, "ms": 1e-3,
                "us": 1e-6, "ns": 1e-9}.get(u, 1.0)
        return x * mult
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    d = {"kernel": label, "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
         "dram_bytes_per_config": (rd + wr) / int(configs),
         "duration_s": num("gpu__time_duration.sum"),
         "dmma_pipe_active_pct": num("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
         "fp64_pipe_active_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
         "l2_hit_rate_pct": num("lts__t_sector_hit_rate.pct"),
         "registers_per_thread": num("launch__registers_per_thread"),
         "warp_stalls_per_issue": {h.split("issue_stalled_")[1].split("_per_issue")[0]: float(v)
                                   for h, v in zip(hdr, vals) if h.startswith("smsp__average_warps_issue_stalled_")
                                   and h.endswith("_per_issue_active.ratio") and v and float(v) > 0.05},
         "source": f"ncu --set full --import-source on --clock-control none, {rep}"}
    json.dump(d, open(out, "w"), indent=1)
    if sass_out:
        sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                              capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(sass)))
        hdr, data = rows[1], rows[2:]
        iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        tot = sum(float(r[iS] or 0) for r in data)
        cls = collections.defaultdict(lambda: [0.0, 0, collections.Counter()])
        for r in data:
            e = int(float(r[iE] or 0))
            c = cls[e]
            c[0] += float(r[iS] or 0)
            c[1] += 1
            opc = r[1].split()[1] if r[1].startswith("@") else r[1].split()[0]
            c[2][opc] += float(r[iS] or 0)
        with open(sass_out, "w") as f:
            f.write(f"# {label}: warp-stall samples grouped by SASS execution count (instructions that run\n"
                    "# equally often belong to the same loop level); share of all samples, top opcodes\n")
            for e, (v, n, ops) in sorted(cls.items(), key=lambda kv: -kv[1][0])[:20]:
                top = ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in ops.most_common(4))
                f.write(f"exec {e:>14d}  instrs {n:5d}  samples {100 * v / tot:6.2f}%  [{top}]\n")
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(*sys.argv[2:])
