"""Per-CUDA-source-line instruction / stall totals from an ncu report (--import-source on, -lineinfo)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []; fname = None; hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r: continue
    if r[0] in ("File Name", "File Path"): fname = r[1].split("/")[-1]; hdr = None; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr and r[0].isdigit() and len(r) > 4 and r[2] == "-":
        iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            ie = float(r[iI] or 0); st = float(r[iS] or 0)
        except ValueError: continue
        rows.append((fname, int(r[0]), r[1][:90], ie, st))
ti = sum(x[3] for x in rows) or 1; ts = sum(x[4] for x in rows) or 1
print(f"{'file:line':22s} {'instr%':>6s} {'stall%':>6s}  source")
for f, ln, src, ie, st in sorted(rows, key=lambda x: -x[4])[:top]:
    print(f"{f}:{ln:<10d} {100*ie/ti:6.1f} {100*st/ts:6.1f}  {src.strip()}")
