"""Summarise `nvcc -Xptxas -v` output: kernel -> registers, spill bytes."""
import re, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)))
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        if len(sys.argv) < 3 or re.search(sys.argv[2], cur):
            print(f"{m2.group(1):>4} regs spill {spill[0]:>4}/{spill[1]:<4} {cur}")
        cur = None
