"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py.

Keeps the library's kernels (namespace tpla::), drops the prefill cache-fill launches (append
launches with more rows than the decode batch), and reports per kernel: launches, mean/min/max
duration and the share of the summed decode-step time.  ncu serialises launches and runs them
cold-cache, so absolute times differ from bench.py's in-step CUDA-event times; the SHARES are
what must agree (B200_PROFILING.md).

    python tools/ncu_summary.py gpurun_out/launches.csv [--decode-grid 8] > profiles/...md
"""
import argparse
import collections
import csv
import re


def short(name):
    m = re.search(r"tpla::<unnamed>::(\w+)(<[^>(]*>)?", name)
    return (m.group(1) + (m.group(2) or "")) if m else name[:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--decode-grid", type=int, default=8, help="append launches with grid.x <= this are decode K1")
    ap.add_argument("--cap", type=int, default=0,
                    help="count at most this many launches per kernel (the first ones): drops launches outside "
                         "the decode steps, e.g. bench.py's K3-alone graph")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 14 and r[0] != "ID" and "tpla::" in r[4]]
    per = collections.defaultdict(list)
    grids = {}
    for r in rows:
        name = short(r[4])
        gx = int(r[8].strip("()").split(",")[0])
        if name.startswith("append_kernel") and gx > a.decode_grid:
            continue                          # prefill cache fill, not part of the decode step
        if a.cap and len(per[name]) >= a.cap:
            continue
        per[name].append(float(r[14]) / 1e3)  # ns -> us
        grids[name] = (r[8], r[7])
    tot = sum(sum(v) for v in per.values())
    print("| kernel | grid | block | launches | mean us | min us | max us | share of decode time |")
    print("|---|---|---|---|---|---|---|---|")
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {name} | {grids[name][0]} | {grids[name][1]} | {len(v)} | {sum(v)/len(v):.1f} | {min(v):.1f} | "
              f"{max(v):.1f} | {sum(v)/tot:.3f} |")


if __name__ == "__main__":
    main()
