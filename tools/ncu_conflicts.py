"""Per-CUDA-source-line shared-memory wavefronts of an ncu report (--set full, --import-source on,
-lineinfo): actual vs ideal, i.e. where the bank conflicts are.  usage: ncu_conflicts.py rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []; fname = None; hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] in ("File Name", "File Path"): fname = r[1].split("/")[-1]; hdr = None; continue
    if r[0] == "Line No":
        hdr = r
        cols = {h: i for i, h in enumerate(hdr)}
        if not rows and "--cols" in sys.argv: print([h for h in hdr if "hared" in h or "avefront" in h])
        continue
    if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
        def g(name):
            i = cols.get(name)
            try: return float(r[i] or 0) if i is not None else 0.0
            except ValueError: return 0.0
        w = g("L1 Wavefronts Shared"); wi = g("L1 Wavefronts Shared Ideal")
        ex = g("L1 Wavefronts Shared Excessive") or max(0.0, w - wi)
        rows.append((fname, int(r[0]), r[1][:90], w, wi, ex, g("Instructions Executed")))
tw = sum(x[3] for x in rows) or 1; te = sum(x[5] for x in rows)
print(f"shared wavefronts {tw:.4g}, excessive (bank conflicts) {te:.4g} = {100*te/tw:.1f}%")
print(f"{'file:line':22s} {'wavefr%':>7s} {'excess%':>7s} {'x ideal':>7s}  source")
for f, ln, src, w, wi, ex, ie in sorted(rows, key=lambda x: -x[5])[:top]:
    print(f"{f}:{ln:<10d} {100*w/tw:7.1f} {100*ex/tw:7.1f} {w/max(wi,1):7.2f}  {src.strip()}")
