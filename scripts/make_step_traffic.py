"""ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
--csv launch list of ONE step (scripts/prof_step.py, --profile-from-start off)
-> profiles/r01_step_traffic.json: per kernel, launches and mean DRAM bytes
per launch (bench.py's roofline "traffic")."""
import collections
import csv
import json
import re
import sys


def main(path, out="profiles/r01_step_traffic.json"):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if "Kernel Name" in r][0]
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    for r in rows:
        if len(r) != len(hdr) or "Kernel Name" in r:
            continue
        d = dict(zip(hdr, r))
        m = re.search(r"\b(k_\w+|at::\w+)", d["Kernel Name"])
        name = m.group(1) if m else d["Kernel Name"][:40]
        v = float(d["Metric Value"].replace(",", "") or 0)
        per[name][d["Metric Name"]] += v
        ids[name].add(d["ID"])
    ks = {}
    for name, mets in per.items():
        n = len(ids[name])
        ks[name] = {"launches": n,
                    "dram_bytes_per_launch": (mets["dram__bytes_read.sum"] + mets["dram__bytes_write.sum"]) / n,
                    "ns_per_launch": mets["gpu__time_duration.sum"] / n}
    with open(out, "w") as f:
        json.dump({"source": f"ncu launch list of one eager MLP step ({path})", "kernels": ks}, f, indent=1)
    print(json.dumps(ks, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
