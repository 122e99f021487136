"""Registers / stack / spills per kernel from `nvcc -Xptxas -v` (stdin)."""
import re
import sys

cur = st = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = re.sub(r".*?(k_\w+?I\w+?E)E.*", r"\1", m.group(1))
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        st = m.groups()
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        print(f"{cur:40s} regs {m2.group(1):>4s} stack {st[0]:>5s} spill st/ld {st[1]}/{st[2]}")
        cur = None
