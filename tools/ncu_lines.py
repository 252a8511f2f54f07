"""Aggregate an ncu SASS source page (CSV) per CUDA source line using nvdisasm
line info (diagnostics): python tools/ncu_lines.py <sass.csv> <nvdisasm -g output> <function> [top]"""
import collections
import csv
import re
import sys

csv_path, dis_path, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
r = list(csv.reader(open(csv_path)))
h, rows = r[1], r[2:]
ia, iall, iex = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
addr = [int(x[ia], 16) for x in rows]
base = min(addr)
samples = {a - base: float(x[iall] or 0) for a, x in zip(addr, rows)}
execs = {a - base: float(x[iex] or 0) for a, x in zip(addr, rows)}
where = {}
cur = None
inside = False
for line in open(dis_path):
    if line.startswith("//----") and ".text." in line:
        inside = ("." + fn + " ") in line or line.rstrip().endswith("." + fn + " --------------------------")
        inside = fn in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        where[int(m.group(1), 16)] = cur
agg = collections.Counter()
agge = collections.Counter()
for off, s in samples.items():
    k = where.get(off, ("?", 0))
    agg[k] += s
    agge[k] += execs[off]
tot = sum(agg.values())
src = {}
for k, s in agg.most_common(top):
    f, ln = k
    if f not in src and f != "?":
        try:
            src[f] = open(next(p for p in ["paper_2208_12964_b200/csrc/" + f] if p)).read().split("\n")
        except OSError:
            src[f] = []
    text = src.get(f, [])[ln - 1].strip()[:70] if f in src and 0 < ln <= len(src[f]) else ""
    print(f"{100 * s / tot:5.1f}%  {agge[k]:14.0f}  {f}:{ln}  {text}")
