"""configs[4] sweep on one GPU: TPLA (g = k = TP: one latent shard per GPU) against the
replicated-MLA baseline (g = 1 with the heads split over the same k, the paper's MLA TP), DeepSeek-V3
shape, over batch x context.  All k ranks run on the one GPU (one stream per co-located rank), so the
step is what k GPUs of a TP group spend together; the step ratio MLA/TPLA is the decode speedup the
paper reports as 1.79x (TP = 2) and 1.93x (TP = 4) at 32K (FlashAttention-3 on its own
hardware).  Writes a markdown table and a JSON file.

    python tools/sweep.py [--tp 2] [--batches 1,8,32,128,256] [--contexts 4096,8192,32768,65536] [--steps 30]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bench(workload, B, S, steps, g, k):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--workload", workload, "--batch", str(B), "--seq-len",
           str(S), "--steps", str(steps), "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-headline",
           "--g", str(g), "--k", str(k)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    if r.returncode:
        raise RuntimeError(r.stderr[-2000:])
    d = json.loads(r.stdout.strip().splitlines()[-1])
    rf = d["roofline"]
    return {"us_per_step": d["ms_per_step"] * 1e3, "tokens_s": d["value"], "k3_us": rf["avg_launch_us"],
            "k3_hbm_frac": rf["hbm_frac"], "sm_mhz": d["clocks"]["sm_mhz"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--batches", default="1,8,32,128,256")
    ap.add_argument("--contexts", default="4096,8192,32768,65536")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for S in [int(x) for x in a.contexts.split(",")]:
        for B in [int(x) for x in a.batches.split(",")]:
            t = bench("c1", B, S, a.steps, a.tp, a.tp)
            m = bench("mla2", B, S, a.steps, 1, a.tp)
            rows.append({"tp": a.tp, "B": B, "S": S, "tpla": t, "mla": m,
                         "speedup": m["us_per_step"] / t["us_per_step"]})
            print(f"B={B:4d} S={S:6d}  TPLA {t['us_per_step']:8.1f} us (K3 {t['k3_us']:7.1f}, "
                  f"{t['k3_hbm_frac']:.2f} HBM)  MLA {m['us_per_step']:8.1f} us (K3 {m['k3_us']:7.1f}, "
                  f"{m['k3_hbm_frac']:.2f} HBM)  speedup {rows[-1]['speedup']:.2f}x", flush=True)
    out = a.out or os.path.join(ROOT, "gpurun_out", f"sweep_tp{a.tp}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(rows, open(out, "w"), indent=1)
    print(f"\nTP = {a.tp}:\n")
    print("| context | batch | TPLA us/step | MLA us/step | speedup | TPLA K3 HBM frac | MLA K3 HBM frac |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['S']} | {r['B']} | {r['tpla']['us_per_step']:.1f} | {r['mla']['us_per_step']:.1f} | "
              f"{r['speedup']:.2f}x | {r['tpla']['k3_hbm_frac']:.2f} | {r['mla']['k3_hbm_frac']:.2f} |")


if __name__ == "__main__":
    main()
