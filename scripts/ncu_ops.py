"""Opcode histogram (executed warp-instructions) of an ncu report's profiled kernel.
    python scripts/ncu_ops.py report.ncu-rep [units_for_per_unit_count]"""
import collections
import csv
import io
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ia, ie, isrc = h.index("Address"), h.index("Instructions Executed"), h.index("Source")
op = collections.Counter()
for r in rows[hi + 1:]:
    if not (r and r[ia].startswith("0x")):
        continue
    t = r[isrc].split()
    if not t:
        continue
    s = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    op[s.split(".")[0]] += float(r[ie] or 0)
tot = sum(op.values())
print(" ".join(f"{k}:{100 * v / tot:.1f}%" for k, v in op.most_common(20)))
print(f"total warp-instructions {tot:.4g}")
if len(sys.argv) > 2:
    print(f"lane-instructions per unit: {tot * 32 / float(sys.argv[2]):.3f}")
