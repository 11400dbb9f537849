#!/usr/bin/env python3
"""Copy the final run's bench lines and checks (scripts/gpu_final_r02.sh) from
gpurun_out/ into profiles/r02_*."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def line(name):
    rows = [l for l in open(os.path.join(G, name + ".log")) if l.startswith("{")]
    return rows[-1].strip()


with open(os.path.join(P, "r02_bench_configs.jsonl"), "w") as f:
    for c in ("bench_c1", "bench_c2", "bench_c3", "bench_c4", "bench_c5"):
        f.write(line(c) + "\n")
for src, dst in (("final_driver_c3", "r02_bench_driver_cmd.json"),
                 ("bench_c3_300", "r02_bench_c3_300steps.json"),
                 ("bench_c3_fg", "r02_bench_c3_fg.json"),
                 ("bench_c5_fg", "r02_bench_c5_fg.json"),
                 ("bench_ref", "r02_bench_reference.json")):
    json.dump(json.loads(line(src)), open(os.path.join(P, dst), "w"))


def tail(name, skip_dots=True):
    out = []
    for l in open(os.path.join(G, name + ".log")):
        if skip_dots and l.strip().startswith(".") and "passed" not in l:
            continue
        out.append(l.rstrip("\n"))
    return "\n".join(out[-6:])


txt = f"""# r02 sanitizer substitute (compute-sanitizer is closed on this GPU pool: every tool exits 86 with
# 'compute-sanitizer is closed on this pool and stays closed: runs under it have left GPUs needing a reset')
# final run: scripts/gpu_final_r02.sh -> scripts/gpu_checks.sh

## 1. GPU test suite on libfizi_checked.so (-DFIZI_DEVICE_CHECKS: bounds of every queue / run / list index trap)
# FIZI_LIB=checked python -m pytest tests -m gpu
{tail("checked_pytest")}

## 2. scripts/sanitize_driver.py on the checked build (C1 joined + debug stages, C2 pipelined with LUT re-test frames, C5 multi-stream kernel)
{tail("checked_driver")}

## 3. race detection by repetition: scripts/race_stress.py (pipelined calls in flight vs joined calls, bit for bit)
{tail("race_stress")}

## normal build, same run
{tail("final_pytest")}
{tail("final_smoke")}
"""
if os.path.exists(os.path.join(G, "race_stress50.log")):
    txt += ("\n## 3b. race stress with 50 repetitions (REPS=50 scripts/race_stress.py, same code)\n"
            + open(os.path.join(G, "race_stress50.log")).read().strip() + "\n")
open(os.path.join(P, "r02_checks.txt"), "w").write(txt)
print("ok")
