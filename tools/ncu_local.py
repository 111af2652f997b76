"""Executed local-memory (spill) instructions per source line of one kernel:
    ncu -i rep --page source --csv --print-source sass > x.csv
    python tools/ncu_local.py x.csv lib.so kernel_substring"""
import collections, csv, glob, os, re, subprocess, sys
csvf, binf, fn = sys.argv[1], sys.argv[2], sys.argv[3]
os.system(f"cd /tmp && rm -f *.cubin && cuobjdump -xelf all {os.path.abspath(binf)} > /dev/null")
lines = {}
for cb in glob.glob("/tmp/*.cubin"):
    out = subprocess.run(["nvdisasm", "-g", cb], capture_output=True, text=True).stdout
    inside, cur = False, None
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
base = int(rows[2][0], 16)
loc, allc = collections.Counter(), collections.Counter()
for r in rows[2:]:
    if not r or not r[0].startswith("0x"):
        continue
    k = lines.get(int(r[0], 16) - base)
    n = int(r[ci["Instructions Executed"]] or 0)
    allc[k] += n
    if "STL" in r[1] or "LDL" in r[1]:
        loc[k] += n
print("local", sum(loc.values()), "all", sum(allc.values()))
for k, v in loc.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 25):
    print(v, k)
