"""Instruction counts of the backward-branch loops of one kernel's SASS.
usage: python tools/sass_loops.py <mangled-name-substring>"""
import re, subprocess, sys
out = subprocess.run([sys.executable, "tools/sass_fn.py", sys.argv[1], "--body"], capture_output=True, text=True).stdout
lines = out.split("\n")
print(lines[0])
addr = []
for l in lines[1:]:
    m = re.match(r"\s*/\*([0-9a-f]{4,5})\*/\s*(.*?);", l)
    if m:
        addr.append((int(m.group(1), 16), m.group(2)))
for a, ins in addr:
    m = re.search(r"BRA.*?0x([0-9a-f]+)", ins)
    if m and int(m.group(1), 16) < a:
        t = int(m.group(1), 16)
        body = [i for x, i in addr if t <= x <= a]
        print(f"loop {t:#x}-{a:#x}: {len(body)} instr, MUFU {sum('MUFU' in i for i in body)}, "
              f"LDG {sum('LDG' in i for i in body)}, BRA {sum('BRA' in i for i in body)}")
