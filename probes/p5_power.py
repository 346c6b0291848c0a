"""P5 driver: runs probes/p5_stream (the cv_kernel update loop alone) and the P0 register-only
DMMA loop while sampling power and SM clock with NVML every 50 ms; prints one JSON object.
Variants: operands L2-resident (32 MB) vs DRAM-streamed (16 GB), B chunks shared by CTA
pairs or not."""
import json
import os
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))


def sample(stop, out):
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
        time.sleep(0.05)


def run(cmd):
    stop, smp = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, smp), daemon=True)
    th.start()
    r = subprocess.run(cmd, capture_output=True, text=True)
    stop.set()
    th.join()
    tail = smp[len(smp) // 4:] or smp  # skip the ramp
    res = {"cmd": " ".join(os.path.basename(c) for c in cmd), "rc": r.returncode}
    try:
        res.update(json.loads(r.stdout.strip().splitlines()[-1]))
    except Exception:
        res["stdout"] = r.stdout[-500:] + r.stderr[-500:]
    if tail:
        res["power_w_median"] = sorted(p for p, _ in tail)[len(tail) // 2]
        res["sm_mhz_median"] = sorted(c for _, c in tail)[len(tail) // 2]
    return res


def main():
    exe = os.path.join(HERE, "p5_stream")
    if not os.path.exists(exe):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-o", exe, os.path.join(HERE, "p5_stream.cu")])
    out = {"what": "cv_kernel update loop alone (p5_stream) and power", "runs": []}
    for args in (["32", "5", "0"], ["16384", "5", "0"], ["16384", "5", "1"], ["32", "5", "1"]):
        out["runs"].append(run([exe] + args))
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    p0 = os.path.join(HERE, "p0_fp64_peak")
    if os.path.exists(p0):
        out["p0_register_dmma"] = run([p0])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
