#!/usr/bin/env python3
"""Copy round-2 evidence from gpurun_out/ (scripts/gpu_profile_r02.sh) into
profiles/: the C3 launch list + per-kernel summary, one ncu --set full
summary per captured kernel, and the DRAM traffic per launch of the fused
kernels (read by bench.py's roofline.traffic when the per-launch workload
matches)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
RR = "r02"
sys.path.insert(0, os.path.join(ROOT, "scripts"))
from launch_summary import main as launch_main  # noqa: E402

CAPTURES = {  # name: (kernel, config, command)
    "c3_seg": ("seg_fast_kernel", "C3 1920x1080, 64 frames", "bench.py --steps 3 --warmup 2"),
    "c3_morph": ("morph_rows_kernel", "C3 1920x1080, 64 frames", "bench.py --steps 3 --warmup 2"),
    "c3_ccl": ("ccl_kernel", "C3 1920x1080, 64 frames", "bench.py --steps 3 --warmup 2"),
    "c3_slow": ("slow_words_kernel", "C3 1920x1080, 64 frames", "bench.py --steps 3 --warmup 2"),
    "c5_seg": ("seg_multi_kernel", "C5 256 streams x 640x480, one frame each",
               "bench.py --config 5 --steps 3 --warmup 2"),
    "c4_seg": ("seg_fast_kernel", "C4 3840x2160, 64 frames", "bench.py --config 4 --steps 3 --warmup 2"),
    "c4_slow": ("slow_words_kernel", "C4 3840x2160, 64 frames",
                "bench.py --config 4 --steps 3 --warmup 2"),
    "c4_ccl": ("ccl_kernel", "C4 3840x2160, 64 frames", "bench.py --config 4 --steps 3 --warmup 2"),
    "c4_morph": ("morph_rows_kernel", "C4 3840x2160, 64 frames",
                 "bench.py --config 4 --steps 3 --warmup 2"),
}
ALG = {  # algorithmic bytes per launch of the fused kernels
    "c3_seg": 64 * (3 + 1 / 8) * 1920 * 1080 + 6 * 1920 * 1080,
    "c5_seg": 256 * (3 + 1 / 8 + 6) * 640 * 480,
    "c4_seg": 64 * (3 + 1 / 8) * 3840 * 2160 + 6 * 3840 * 2160,
}


def summary(name):
    rep = os.path.join(G, f"prof_{name}.ncu-rep")
    if not os.path.exists(rep):
        return None
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), rep],
                         capture_output=True, text=True).stdout
    kern, cfg, cmd = CAPTURES[name]
    hdr = (f"# {RR} ncu --set full --clock-control none, one launch of {kern} ({cfg})\n"
           f"# command: ncu --set full --clock-control none --import-source on -k regex:... -s 4 -c 1 "
           f"python {cmd} --no-e2e --no-cpu-baseline --no-spot-check\n")
    open(os.path.join(P, f"{RR}_ncu_{name}.txt"), "w").write(hdr + out)
    vals = {}
    for line in out.splitlines():
        parts = line.split()
        if len(parts) >= 3 and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                            "gpu__time_duration.sum"):
            v = float(parts[1]) * {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1, "us": 1,
                                   "usecond": 1, "ns": 1e-3, "nsecond": 1e-3, "ms": 1e3,
                                   "msecond": 1e3}.get(parts[2], 1)
            vals[parts[0]] = v
    if name in ALG:
        traffic = vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"]
        j = {"kernel": kern, "config": cfg, "round": 2,
             "source": f"profiles/{RR}_ncu_{name}.txt (ncu --set full)",
             "dram_bytes_per_launch": traffic, "algorithmic_bytes_per_launch": ALG[name],
             "traffic_over_algorithmic": traffic / ALG[name],
             "ncu_duration_us": vals["gpu__time_duration.sum"],
             "achieved_alone_gbs": ALG[name] / vals["gpu__time_duration.sum"] / 1e3}
        json.dump(j, open(os.path.join(P, f"{RR}_{name}_traffic.json"), "w"), indent=1)
        print(j)
    return out


if __name__ == "__main__":
    import contextlib
    import io
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        launch_main(os.path.join(G, "launches.csv"))
    txt = ("# r02 ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, "
           "serialised)\n# command: python bench.py --steps 3 --warmup 2 --no-e2e "
           "--no-cpu-baseline --no-spot-check (C3)\n" + buf.getvalue())
    open(os.path.join(P, f"{RR}_launches_summary.txt"), "w").write(txt)
    import shutil
    shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, f"{RR}_launches.csv"))
    print(txt)
    for n in CAPTURES:
        summary(n)
