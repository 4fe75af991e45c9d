"""Sum an ncu --csv launch list (gpu__time_duration.sum) per kernel name:
python tools/ncu_group.py a.csv [b.csv] -> per-kernel totals in us (side by side)."""
import csv
import sys
from collections import defaultdict


def load(path):
    rows = open(path).read().splitlines()
    start = next(i for i, r in enumerate(rows) if r.startswith('"ID"'))
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in csv.DictReader(rows[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        v = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        tot[name] += v
        cnt[name] += 1
    return tot, cnt


tabs = [load(p) for p in sys.argv[1:]]
names = sorted(set().union(*[t[0] for t in tabs]), key=lambda k: -max(t[0].get(k, 0) for t in tabs))
print("%-36s" % "kernel" + "".join("%14s %6s" % ("us", "n") for _ in tabs))
for k in names:
    print("%-36s" % k[:36] + "".join("%14.1f %6d" % (t[0].get(k, 0), t[1].get(k, 0)) for t in tabs))
print("%-36s" % "TOTAL" + "".join("%14.1f %6d" % (sum(t[0].values()), sum(t[1].values())) for t in tabs))
