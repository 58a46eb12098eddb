"""Hot-spot table of an ncu '--page source --print-source sass --csv' export: top instructions by
warp-stall samples, with their dominant stall reasons, and per-opcode instruction counts.
    python tools/sass_hot.py gpurun_out/k3_c3.sass.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[i_s] or 0) for r in data)
print(f"samples {tot:.0f}")
for r in sorted(data, key=lambda r: -float(r[i_s] or 0))[:top]:
    reasons = sorted(((float(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:2]
    print(f"{r[0][-5:]} {float(r[i_s]) / tot:6.3f} {float(r[i_e] or 0):10.0f}  {r[1][:60]:60s} "
          + " ".join(f"{n}:{v:.0f}" for v, n in reasons if v))
agg = collections.Counter()
for r in data:
    for i in st:
        agg[hdr[i][6:]] += float(r[i] or 0)
print("stall reasons:", ", ".join(f"{k} {v / tot:.3f}" for k, v in agg.most_common(8)))
