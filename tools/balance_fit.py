"""Fit K3 per-CTA end times (tools/gpu_balance.sh output: cta smid tiles segs start end per line)
against work (tiles, segments) and show what the residual correlates with (SM id, TPC, CTA index)."""
import sys

import numpy as np

rows = []
for line in open(sys.argv[1]):
    p = line.split("]")[-1].split()
    rows.append([int(x) for x in p])
a = np.array(rows[-int(sys.argv[2]) if len(sys.argv) > 2 else -148:], dtype=float)
cta, smid, tiles, segs, st, en = a.T
X = np.stack([np.ones_like(tiles), tiles, segs], 1)
coef, *_ = np.linalg.lstsq(X, en, rcond=None)
res = en - X @ coef
print(f"n={len(a)} end: min {en.min():.0f} med {np.median(en):.0f} max {en.max():.0f} ns (spread {100*(en.max()-en.min())/en.max():.1f} %)")
print(f"fit end = {coef[0]:.0f} + {coef[1]:.1f}*tiles + {coef[2]:.0f}*segs ns; per-seg = {coef[2]/coef[1]:.1f} tiles; resid sd {res.std():.0f} ns")
print(f"start: max {st.max():.0f} ns; corr(resid, start) {np.corrcoef(res, st)[0,1]:.2f}")
print(f"tiles {tiles.min():.0f}-{tiles.max():.0f}, segs {segs.min():.0f}-{segs.max():.0f}")
# residual by smid groups
order = np.argsort(smid)
for grp, name in ((2, "TPC"), (16, "16-SM block")):
    g = (smid // grp).astype(int)
    means = [res[g == k].mean() for k in np.unique(g)]
    print(f"resid by {name}: sd of group means {np.std(means):.0f} ns over {len(means)} groups "
          f"(min {min(means):.0f}, max {max(means):.0f})")
print("smid  resid(ns) sorted by smid:")
print(" ".join(f"{int(smid[i])}:{res[i]:+.0f}" for i in order))
print("slowest 10 (cta smid tiles segs resid):")
for i in np.argsort(-res)[:10]:
    print(f"  {int(cta[i])} {int(smid[i])} {int(tiles[i])} {int(segs[i])} {res[i]:+.0f}")
