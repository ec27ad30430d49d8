"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, re, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
hdr = rows[0]; data = rows[1:]
ik = hdr.index("Kernel Name"); iv = hdr.index("Metric Value"); iu = hdr.index("Metric Unit")
tot = defaultdict(float); cnt = defaultdict(int)
for r in data:
    v = float(r[iv].replace(",", "")); u = r[iu]
    ms = v / 1e6 if u in ("nsecond", "ns") else v / 1e3 if u in ("usecond", "us") else v if u in ("msecond", "ms") else v
    name = re.sub(r"\(.*", "", r[ik])[:80]
    tot[name] += ms; cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':82s} {'launches':>8s} {'total ms':>10s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{k:82s} {cnt[k]:8d} {v:10.2f} {100*v/T:5.1f}%")
print(f"{'TOTAL':82s} {sum(cnt.values()):8d} {T:10.2f}")
