"""Per-source-line totals of an ncu SASS source export, mapped through the
cubin's line table (nvdisasm -g):

    ncu -i rep --page source --csv --print-source sass > x.csv
    python tools/ncu_sass_lines.py x.csv lib.so kernel_substring [top]
"""
import collections
import csv
import re
import subprocess
import sys

csvf, binf, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = "/tmp/_ncu_sass_lines"
subprocess.run(["cuobjdump", "-xelf", "all", binf], cwd="/tmp", capture_output=True)
import glob
cubins = glob.glob("/tmp/*.sm_100a.cubin")
lines = {}
for cb in cubins:
    out = subprocess.run(["nvdisasm", "-g", cb], capture_output=True, text=True).stdout
    inside = False
    cur = None
    for line in out.splitlines():
        if line.startswith(".") and not line.startswith(".L"):
            inside = line.startswith(".text.") and fn in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+[A-Z@]', line)
        if m:
            lines[int(m.group(1), 16)] = cur
    if lines:
        break
rows = list(csv.reader(open(csvf, encoding="latin-1")))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
base = None
samp = collections.Counter()
inst = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) - 1:
        continue
    a = int(r[0], 16)
    if base is None:
        base = a
    key = lines.get(a - base, ("?", 0))
    samp[key] += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    inst[key] += int(r[ci["Instructions Executed"]] or 0)
ts, ti = sum(samp.values()), sum(inst.values())
print(f"samples {ts} warp-insts {ti}")
for k, v in samp.most_common(top):
    print(f"{100 * v / ts:5.1f}% samp {100 * inst[k] / ti:5.1f}% inst  {k[0]}:{k[1]}")
