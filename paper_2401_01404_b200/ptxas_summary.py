"""Summarise `nvcc -Xptxas -v` output: one line per kernel (registers, spills)."""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
rows = []
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
        rows.append([cur, spill, None])
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and rows and rows[-1][2] is None:
        rows[-1][2] = int(m.group(1))
names = [r[0] for r in rows]
try:
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
except Exception:
    dem = names
for (n, sp, rg), d in zip(rows, dem):
    d = re.sub(r"\(.*", "", d)
    print(f"{rg:>4} regs  spill {sp[0]:>4}/{sp[1]:<4} {d}")
