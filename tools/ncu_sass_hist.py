"""Summarise an ncu source page (SASS) export: executed warp instructions by
opcode and the stall samples by reason.
  ncu -i rep --page source --csv -k regex:K | python tools/ncu_sass_hist.py"""
import collections
import csv
import sys

rows = list(csv.reader(sys.stdin))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
src = hdr.index("Source")
samp = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ops = collections.Counter()
stalls = collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        n = float(r[ie])
    except (ValueError, IndexError):
        continue
    op = r[src].split()[0] if r[src].split() else "?"
    if op.startswith("@"):
        op = r[src].split()[1]
    ops[op.split(".")[0]] += n
    tot += n
    for i, h in stall_cols:
        try:
            stalls[h] += float(r[i])
        except ValueError:
            pass
print(f"warp instructions: {tot:.0f}")
for op, n in ops.most_common(25):
    print(f"  {op:12s} {100 * n / tot:5.1f}%")
st = sum(stalls.values())
print("stall samples:")
for h, n in stalls.most_common(10):
    print(f"  {h:24s} {100 * n / st:5.1f}%")
