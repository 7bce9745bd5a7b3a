"""Instruction histogram of the backward-branch loops of a kernel's SASS (A/B check of hot loops).

    python scripts/sass_loops.py file.o|file.so name_substring
"""
import collections
import re
import subprocess
import sys

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
fn, code = None, {}
for ln in out.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        fn = m.group(1)
        code[fn] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", ln)
    if m and fn:
        code[fn].append((int(m.group(1), 16), m.group(2)))
for fn, c in code.items():
    if sys.argv[2] not in fn:
        continue
    print(fn, len(c))
    for a, ins in c:
        m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", ins)
        if m and int(m.group(1), 16) < a:
            t = int(m.group(1), 16)
            body = [i for (x, i) in c if t <= x <= a]
            ops = collections.Counter((i.split()[1] if i.split()[0].startswith("@") else i.split()[0]).split(".")[0] for i in body)
            print(f"  loop {t:#x}-{a:#x}: {len(body)} instr", dict(ops.most_common(8)))
