"""Registers / spills per kernel from build/fembatch_b200/ptxas.log."""
import re
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "build/fembatch_b200/ptxas.log"
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
rows = {}
for line in open(path):
    m = re.search(r"Compiling entry function '(\S+)' for", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        rows.setdefault(cur, {})["spill"] = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.setdefault(cur, {})["regs"] = int(m.group(1))
for k, v in sorted(rows.items()):
    if pat in k:
        m = re.search(r"fb_(\w+?)I([fd])Li(\d)ELi(\d)E(.*)EEvNS", k)
        name = f"{m.group(1)}<{m.group(2)},{m.group(3)}D,op{m.group(4)},{m.group(5)}>" if m else k
        print(f"{name:60s} regs={v.get('regs')} spill={v.get('spill')}")
