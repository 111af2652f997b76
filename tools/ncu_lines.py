"""Aggregate ncu source-page stall samples by CUDA source line:
   python tools/ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr = None, None
agg = collections.defaultdict(collections.Counter)
text = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    text[(cur, ln)] = r[1]
    wi = hdr.index("Warp Stall Sampling (All Samples)")
    v = r[wi] if len(r) > wi else ""
    if v and v.replace(".", "").isdigit():
        agg[(cur, ln)]["all"] += float(v)
        for i, name in enumerate(hdr):
            if name.startswith("stall_") and "Not Issued" not in name:
                x = r[i]
                if x and x.replace(".", "").isdigit():
                    agg[(cur, ln)][name[6:]] += float(x)
tot = sum(c["all"] for c in agg.values())
print("total samples", tot)
for k, c in sorted(agg.items(), key=lambda kv: -kv[1]["all"])[:top]:
    st = sorted([(n, v) for n, v in c.items() if n != "all"], key=lambda x: -x[1])[:3]
    print(f"{c['all']:6.0f} {100*c['all']/tot:5.1f}% {k[0]}:{k[1]} {text.get(k,'').strip()[:60]} | " +
          " ".join(f"{n}={v:.0f}" for n, v in st))
