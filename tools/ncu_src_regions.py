"""Per-source-line and per-region warp-stall samples from an ncu source export
(`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`).
usage: python tools/ncu_src_regions.py src.csv [top] [regions-spec]
regions-spec: file:lo-hi=name,... (line ranges of one file)"""
import csv, sys, collections

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
spec = sys.argv[3] if len(sys.argv) > 3 else ""
regions = []
for part in filter(None, spec.split(",")):
    f, rest = part.split(":")
    rng, name = rest.split("=")
    lo, hi = map(int, rng.split("-"))
    regions.append((f, lo, hi, name))
f = None
hdr = None
out = []
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        idx = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r and r[0] and len(r) > 8 and r[2] == "-":
        try:
            s = int(r[idx["Warp Stall Sampling (All Samples)"]])
            ins = int(r[idx["Instructions Executed"]])
        except ValueError:
            continue
        stalls = {}
        for h, i in idx.items():
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    stalls[h[6:]] = int(r[i])
                except ValueError:
                    pass
        out.append((s, ins, f, int(r[0]), r[1][:80], stalls))
tot = sum(o[0] for o in out) or 1
ti = sum(o[1] for o in out) or 1
print("total samples", tot, "warp insts", ti)
for s, i, fn, ln, src, st in sorted(out, key=lambda o: -o[0])[:top]:
    tops = sorted(st.items(), key=lambda x: -x[1])[:3]
    print(f"{100*s/tot:5.1f}% {100*i/ti:5.1f}%i {fn}:{ln} {src}  | " + " ".join(f"{k}={v}" for k, v in tops))
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
for s, i, fn, ln, src, st in out:
    key = fn
    for rf, lo, hi, name in regions:
        if fn == rf and lo <= ln <= hi:
            key = name
    agg[key][0] += s
    agg[key][1] += i
    agg[key][2].update(st)
print("--- regions")
for k, (s, i, st) in sorted(agg.items(), key=lambda x: -x[1][0]):
    tops = st.most_common(4)
    print(f"{100*s/tot:5.1f}% {100*i/ti:5.1f}%i {k} | " + " ".join(f"{a}={100*b/max(1,s):.0f}%" for a, b in tops))
