"""Top source lines of an ncu source export (--page source --csv --print-source cuda,sass)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
f = None; out = []; hdr = None
for r in rows:
    if r and r[0] == "File Path": f = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if hdr and len(r) > 8 and r[2] == "-":
        try: out.append((int(r[4]), int(r[7]), f, r[0], r[1][:90]))
        except ValueError: pass
tot = sum(o[0] for o in out); ti = sum(o[1] for o in out)
print("total samples", tot, "warp insts", ti)
for s, i, f, ln, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{100*s/tot:5.1f}% {100*i/ti:5.1f}%i {f}:{ln} {src}")
if len(sys.argv) > 3:
    import collections
    agg = collections.defaultdict(lambda: [0, 0])
    for s, i, f, ln, src in out:
        key = f
        if f == "persist.cu":
            l = int(ln)
            for lo, hi, name in [(0, 150, "setup"), (150, 200, "p1 wait/fft"), (200, 295, "p1 thomas"), (295, 365, "p2"), (365, 418, "p3 setup"), (418, 505, "p3 thomas"), (505, 540, "p3 fft")]:
                if lo <= l < hi: key = "persist.cu " + name
        agg[key][0] += s; agg[key][1] += i
    for k, (s, i) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{100*s/tot:5.1f}% {100*i/ti:5.1f}%i {k}")
