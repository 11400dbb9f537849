#!/usr/bin/env python3
"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import collections
import sys


def main(path, skip_prefix=("<unnamed>",)):
    lines = open(path).read().splitlines()
    i = next(k for k, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.reader(lines[i:]))
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        d.setdefault(name, []).append(float(r[vi]) / 1e3)
    tot = 0.0
    print("%-45s %8s %10s" % ("kernel", "launches", "mean_us"))
    for k, v in d.items():
        print("%-45s %8d %10.2f" % (k[:45], len(v), sum(v) / len(v)))
    return d


if __name__ == "__main__":
    main(sys.argv[1])
