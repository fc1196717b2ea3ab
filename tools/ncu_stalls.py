"""Where the warps of one kernel wait (dev tool): samples per mbarrier / per address range from an
ncu --set full --import-source report's SASS source page.

    python tools/ncu_stalls.py report.ncu-rep
"""
import collections
import csv
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h, data = rows[hi], rows[hi + 1:]
iS, iSrc, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(r[iS] or 0) for r in data) or 1.0
agg = collections.Counter()
last = None
for r in data:
    s = r[iSrc]
    m = re.search(r"TRYWAIT \w+, \[(\w+)\+URZ(\+0x[0-9a-f]+)?\]", s)
    if m:
        last = m.group(2) or m.group(1)
    if "TRYWAIT" in s or ("BRA" in s and last) or "YIELD" in s:
        agg["wait " + str(last)] += float(r[iS] or 0)
    else:
        agg["other"] += float(r[iS] or 0)
        last = None if "BRA" not in s else last
for k, v in agg.most_common(12):
    print(f"{v / tot * 100:5.1f}%  {k}")
print("top instructions:")
for r in sorted(data, key=lambda r: -float(r[iS] or 0))[:12]:
    st = sorted(((float(r[h.index(c)] or 0), c[6:]) for c in cols), reverse=True)[:2]
    print(f"{float(r[iS] or 0) / tot * 100:5.1f}%  {r[0][-5:]}  {r[iSrc][:70]:70s} exec={r[iE]} {st}")
