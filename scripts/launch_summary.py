"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(list)
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] == "gpu__time_duration.sum":
            v = float(d["Metric Value"]) / (1e3 if d["Metric Unit"] == "nsecond" else 1.0)
            agg[d["Kernel Name"][:70]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{100*sum(v)/tot:5.1f}% {sum(v):9.1f} us  n={len(v):3d} mean={sum(v)/len(v):8.1f}  {k}")
