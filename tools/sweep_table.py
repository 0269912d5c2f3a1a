"""Pivot a '== cfg' / 'layer time' sweep log into one table: python tools/sweep_table.py LOG"""
import sys

blocks = open(sys.argv[1]).read().split("== ")[1:]
tab, cfgs = {}, []
for b in blocks:
    lines = b.strip().split("\n")
    cfgs.append(lines[0].strip())
    for ln in lines[1:]:
        parts = ln.split()
        if len(parts) >= 2:
            tab.setdefault(parts[0], {})[cfgs[-1]] = parts[1]
print("layer".ljust(22), *[c.rjust(8) for c in cfgs])
for n, d in tab.items():
    print(n.ljust(22), *[d.get(c, "").rjust(8) for c in cfgs])
