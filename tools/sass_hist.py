"""Summarise an ncu --page source --csv --print-source sass dump: executed instructions and
stall samples per opcode (used to write profiles/*.md)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
src, ex, st = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
inst = collections.Counter()
stall = collections.Counter()
tot_i = tot_s = 0
for r in rows[2:]:
    if len(r) <= ex or not r[ex].isdigit():
        continue
    op = r[src].strip().split()[0] if r[src].strip() else "?"
    if op.startswith("@"):
        op = r[src].strip().split()[1]
    op = op.split(".")[0]
    inst[op] += int(r[ex])
    stall[op] += int(r[st] or 0)
    tot_i += int(r[ex])
    tot_s += int(r[st] or 0)
print(f"total warp-instructions {tot_i}, stall samples {tot_s}")
for op, n in inst.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} {n:10d} {100*n/tot_i:5.1f}%  stall {100*stall[op]/max(1,tot_s):5.1f}%")
