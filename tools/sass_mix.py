"""Instruction-class counts of the hot kernels in libscurve_b200.so (static SASS,
cuobjdump -sass): FP64 tensor (DMMA), other FP64, shared loads/stores, async
copies (LDGSTS), TMA (UTMALDG/UTMASTG/UBLKCP), global loads/stores, barriers,
mbarrier (SYNCS), setmaxnreg (USETMAXREG).  usage: sass_mix.py [lib.so] [regex]"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1511_05578_b200/libscurve_b200.so"
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else
                 r"k_pfa_rows_pILi2047|k_ana_colgen_pILi2047|k_syn_gamma_qpILi2047|k_pfa_rows_pILi1023ELin1ELi1|k_bq_gemm|k_sht_contract_w|k_sht_bins_w")
CLASSES = [("DMMA", r"^DMMA"), ("DFMA/DADD/DMUL", r"^(DFMA|DADD|DMUL)"), ("MUFU/exp", r"^MUFU"),
           ("LDS", r"^LDS"), ("STS", r"^STS"), ("LDGSTS (cp.async)", r"^LDGSTS"),
           ("TMA (UTMALDG/UTMASTG/UBLKCP)", r"^(UTMALDG|UTMASTG|UBLKCP)"), ("LDG", r"^LDG"), ("STG", r"^STG"),
           ("RED/ATOM", r"^(RED|ATOM)"), ("LDL/STL (spills)", r"^(LDL|STL)"), ("BAR", r"^BAR"),
           ("SYNCS (mbarrier)", r"^SYNCS"), ("USETMAXREG", r"^USETMAXREG"), ("SHFL", r"^SHFL"),
           ("integer/other", r".")]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
fn, counts = None, {}
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1) if pat.search(m.group(1)) else None
        if fn:
            counts[fn] = collections.Counter()
        continue
    if fn is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(1)
    for name, rx in CLASSES:
        if re.match(rx, op):
            counts[fn][name] += 1
            break
for fn, c in counts.items():
    tot = sum(c.values())
    short = subprocess.run(["c++filt", fn], capture_output=True, text=True).stdout.strip()
    short = re.sub(r"\(anonymous namespace\)::", "", short).split("(")[0]
    print(f"== {short}  ({tot} SASS instructions)")
    for name, _ in CLASSES:
        if c[name]:
            print(f"   {name:32s} {c[name]:6d}  {100.0 * c[name] / tot:5.1f}%")
