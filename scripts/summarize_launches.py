"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    tot = collections.defaultdict(lambda: [0.0, 0])
    for r in rows:
        if len(r) != len(hdr) or r is hdr or "Kernel Name" in r:
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        m = re.search(r"\b(k_\w+|at::\w+)", d["Kernel Name"])
        name = m.group(1) if m else d["Kernel Name"][:40]
        m2 = re.search(r"k_\w+<(\d+)>", d["Kernel Name"])
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(d["Metric Unit"], 1.0)
        tot[name][0] += v
        tot[name][1] += 1
    S = sum(v[0] for v in tot.values())
    print(f"total {S:.1f} us over {sum(v[1] for v in tot.values())} launches (cold-cache, serialised)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1][0]):
        print(f"{k:32s} {v[0]:9.1f} us {v[1]:4d} launches {100 * v[0] / S:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
