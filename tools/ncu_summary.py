"""Summarise an ncu report: SOL/occupancy/scheduler sections + stall reasons by opcode."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = csv.reader(out.splitlines()); hdr = next(r)
keep = ('GPU Speed Of Light Throughput', 'Compute Workload Analysis', 'Occupancy', 'Scheduler Statistics', 'Memory Workload Analysis')
for row in r:
    d = dict(zip(hdr, row))
    if d.get('Section Name', '') in keep and d.get('Metric Name'):
        print(f"{d['Section Name'][:18]:18s} {d['Metric Name'][:48]:48s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
if len(rows) > 2:
    hdr = rows[1]; data = rows[2:]
    i_src = hdr.index('Source'); i_st = hdr.index('Warp Stall Sampling (All Samples)'); i_ex = hdr.index('Instructions Executed')
    cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
    def fl(v):
        try: return float(v or 0)
        except ValueError: return 0.0
    data = [x for x in data if len(x) > max(i_src, i_st, i_ex)]
    tot = sum(fl(x[i_st]) for x in data) or 1
    c = Counter(); ce = Counter(); reasons = Counter()
    for x in data:
        toks = x[i_src].split()
        if not toks: continue
        op = (toks[1] if toks[0].startswith('@') else toks[0]).split('.')[0]
        c[op] += fl(x[i_st]); ce[op] += fl(x[i_ex])
        for h in cols:
            try: reasons[h] += float(x[hdr.index(h)] or 0)
            except ValueError: pass
    for op, v in c.most_common(14): print(f"  {op:10s} stall%={100*v/tot:5.1f}  exec={ce[op]:.3g}")
    rt = sum(reasons.values()) or 1
    for k, v in reasons.most_common(8): print(f"    {k:25s} {100*v/rt:5.1f}%")
