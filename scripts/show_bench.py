import json, sys
for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if line.startswith("{"):
            d = json.loads(line)
            r = d.get("roofline", {})
            print(path, round(d["value"]), d["unit"], "seg", round(r.get("achieved") or 0), "GB/s",
                  round(r.get("frac") or 0, 3), "step_frac", round(r.get("step", {}).get("frac", 0), 3),
                  {k: round(v * 1000, 1) for k, v in r.get("stage_ms_per_step", {}).items()},
                  "e2e", d.get("e2e", {}).get("value"), "clk", d.get("clocks", {}).get("sm_mhz"), "ms", round(d["ms_per_step"],4), "host_ms", d.get("host_enqueue_ms_per_step"))
