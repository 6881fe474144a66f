"""Per-kernel registers / spills from `nvcc -Xptxas=-v` output (stdin)."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        k = re.search(r"k_conv_tcILi(\d+)ELi(\d)ELb([01])E", cur)
        cur = f"conv BN={k.group(1)} MODE={k.group(2)} FUSE={k.group(3)}" if k else re.sub(r"_ZN.*?(k_\w+?)E.*", r"\1", cur)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = m.group(0)
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:40s} regs={m.group(1)} {spill}")
        cur = None
