"""Per-opcode executed instructions (per work unit) and stall share from an
ncu source-page export: ncu -i X.ncu-rep --page source --csv --print-source sass > f.csv
usage: python scripts/sass_hist.py f.csv UNITS"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
hdr = rows[1]
ie, src, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, stall, tot, stot = collections.Counter(), collections.Counter(), 0, 0
for r in rows[2:]:
    if len(r) <= ie:
        continue
    try:
        n, s = int(r[ie]), int(r[st])
    except ValueError:
        continue
    op = r[src].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    op = op.split()[0].split(".")[0]
    cnt[op] += n
    stall[op] += s
    tot += n
    stot += s
print("total warp-instrs", tot, "per unit", round(tot / units, 1))
for op, n in cnt.most_common(32):
    print(f"{op:10s} {n / units:8.1f}/unit  stall-samples {100 * stall[op] / max(stot, 1):5.1f}%")
