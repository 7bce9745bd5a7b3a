"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

    python scripts/stall_by_line.py <report.ncu-rep> <lib.so> <kernel-substring> [top]

ncu's SASS source page gives absolute addresses; the kernel's first instruction is offset 0 of
the function in the cubin, whose line table (`nvdisasm -g`) maps offsets to source lines.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_lines(lib, kname):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    for f in sorted(os.listdir(tmp)):
        if not f.endswith(".cubin"):
            continue
        out = subprocess.run(["nvdisasm", "-c", "-g", os.path.join(tmp, f)], capture_output=True, text=True).stdout
        cur_fn, line, table = None, None, {}
        for ln in out.splitlines():
            m = re.match(r"^(\S+):\s*$", ln)
            if m:
                if not m.group(1).startswith(".L"):
                    cur_fn = m.group(1)
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
            if m and cur_fn and kname in cur_fn:
                table[int(m.group(1), 16)] = (line, m.group(2).strip())
        if table:
            return table
    return {}


def main():
    rep, lib, kname = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hi]
    ia, iw = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    sidx = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    data = []
    for r in rows[hi + 1:]:
        if r and r[ia].startswith("0x"):
            st = {n: float(r[i] or 0) for i, n in sidx}
            data.append((int(r[ia], 16), float(r[iw] or 0), st))
    base = min(a for a, _, _ in data)
    table = sass_lines(lib, kname)
    per_line = collections.Counter()
    per_reason = collections.defaultdict(collections.Counter)
    total = sum(w for _, w, _ in data) or 1.0
    for a, w, st in data:
        line = table.get(a - base, ("?", ""))[0]
        per_line[line] += w
        per_reason[line].update(st)
    for line, w in per_line.most_common(top):
        rs = ", ".join(f"{n} {100 * v / total:.1f}" for n, v in per_reason[line].most_common(3) if v > 0)
        print(f"{100 * w / total:6.2f}%  {line:28s} {rs}")


if __name__ == "__main__":
    main()
