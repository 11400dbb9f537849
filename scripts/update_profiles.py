#!/usr/bin/env python3
"""Copy the evidence of a GPU check run (scripts/gpu_check.sh) from gpurun_out/
into profiles/ for round RR: launch list + its summary, the ncu --set full
summary of the fused kernel, its DRAM traffic per launch, the bench line."""
import csv
import collections
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RR = sys.argv[1] if len(sys.argv) > 1 else "r01"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
N = 1920 * 1080
B = 64


def launches():
    rows = [r for r in csv.reader(open(os.path.join(G, "launches.csv"))) if len(r) > 10]
    h, data = rows[0], rows[1:]
    iK, iV, iU, iID = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("ID")
    t = collections.defaultdict(list)
    for r in data:
        v = float(r[iV].replace(",", ""))
        v = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}[r[iU]]
        name = r[iK].split("(")[0].replace("void ", "")
        t[name].append(v)
    shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{RR}_launches.csv"))
    lines = [f"# {RR} ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)",
             "# command: python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline",
             f"{'kernel':45s} {'launches':>8s} {'mean_us':>9s}"]
    for k, v in t.items():
        lines.append(f"{k[:45]:45s} {len(v):8d} {sum(v) / len(v):9.2f}")
    path = [k for k in t if k.startswith("fizi::") and not any(
        s in k for s in ("lut_table", "tstate", "learn", "skin_table", "env_"))]
    tot = sum(sum(t[k]) / len(t[k]) for k in path)
    lines += ["", "# share of one call's serialised kernel time, from the launch list:"]
    for k in path:
        m = sum(t[k]) / len(t[k])
        lines.append(f"{k[:45]:45s} {m:9.2f} us {100 * m / tot:6.1f}%")
    open(os.path.join(P, f"{RR}_launches_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full():
    rep = os.path.join(G, "prof.ncu-rep")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    hdr = (f"# {RR} ncu --set full --clock-control none, one launch of the fused segmentation kernel "
           "(64 frames C3)\n# command: ncu --set full ... -k regex:seg_fast -s 4 -c 1 python bench.py "
           "--steps 3 --warmup 2 --no-e2e --no-cpu-baseline\n")
    open(os.path.join(P, f"{RR}_seg_fast_ncu_full.txt"), "w").write(hdr + out)
    shutil.copy(rep, os.path.join(P, f"{RR}_seg_fast.ncu-rep"))
    vals = {}
    for line in out.splitlines():
        parts = line.split()
        if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                            "gpu__time_duration.sum"):
            v = float(parts[1])
            unit = parts[2]
            v *= {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "us": 1, "usecond": 1,
                  "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1)
            vals[parts[0]] = v
    alg = B * (3 * N + N / 8) + 6 * N
    traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
    j = {"kernel": "seg_fast_kernel", "round": int(RR[1:]), "source": f"profiles/{RR}_seg_fast_ncu_full.txt (ncu --set full)",
         "dram_bytes_per_launch": traffic, "algorithmic_bytes_per_launch": alg,
         "traffic_over_algorithmic": traffic / alg, "ncu_duration_us": vals["gpu__time_duration.sum"]}
    json.dump(j, open(os.path.join(P, f"{RR}_seg_fast_traffic.json"), "w"), indent=1)
    print(out)
    print(j)


def bench():
    line = [l for l in open(os.path.join(G, "bench.log")) if l.startswith("{")][-1]
    open(os.path.join(P, f"{RR}_bench.jsonl"), "a").write(line)


if __name__ == "__main__":
    launches()
    full()
    bench()
