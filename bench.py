#!/usr/bin/env python
"""TPLA decode-step benchmark (BASELINE.json metric: decode tokens/s & µs/layer at 32K ctx, DSV3 shape).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c3] [--impl tpla|reference]
    torchrun --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole hot path for one batch:
K1 append of the new token's latent row (every sequence), then K2 absorb, K3 split-K attention,
K4 combine, K5 W^UV + W^O up-projection and C1 all-reduce, on every one of the k TPLA ranks.

Workload (default c1 = BASELINE configs[1]): DeepSeek-V3 attention layer, 128 heads, latent
512 + RoPE 64, 32K cached tokens per sequence, batch 32, TPLA g = 2 on k = max(2, N) ranks.
The total work is fixed, so scaling over N is "strong": N=1 runs both g=2 ranks on one GPU
(they accumulate into y, standing in for the all-reduce), N=2 is the paper's TP=2 deployment
(P:499), N=4/8 further split the heads inside each latent group.  Every N
produces the same numbers.  The per-step cache (1.34 GB at N=1) exceeds L2 (126 MB), so
every read comes from HBM without an explicit flush.

Prints one JSON line (rank 0).  --impl reference times the fp64 oracle (oracle/) on the
host cores instead: the one other place this file runs oracle code besides cpu_baseline.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "decode tokens/s & µs/layer at 32K ctx (DSV3 shape); HBM GB/s vs peak @1/2/4/8"

WORKLOADS = {
    "c1": dict(desc="configs[1]: DeepSeek-V3 attention layer decode, 128 heads, latent 512 + RoPE 64, "
                    "32K context, batch 32, TPLA g=2", model="dsv3", B=32, S=32768, g=2, xform="hadamard"),
    "c2": dict(desc="configs[2]: Kimi-K2 attention layer decode, 64 heads, latent 512 + RoPE 64, 32K context, "
                    "batch 64, TPLA g=4", model="kimi", B=64, S=32768, g=4, xform="hadamard"),
    "c3": dict(desc="configs[3]: DeepSeek-V3 decode at 128K context, batch 16, g=8, Hadamard-rotated cache",
               model="dsv3", B=16, S=131072, g=8, xform="hadamard"),
    # SURVEY §8(d) headline shape: one latent shard per GPU on 8 GPUs (all k=8 shards on one GPU here)
    "h8": dict(desc="SURVEY 8(d) headline shape: DeepSeek-V3 32K context, batch 32, g=8 (one latent shard per GPU "
                    "at 8 GPUs)", model="dsv3", B=32, S=32768, g=8, xform="hadamard"),
    # the same 8-GPU 32K shape with the paper's TP > 2 recipe: g = 2 latent shards, heads
    # split 4 ways (H_loc = 32, W = 320): all k = 8 ranks on one GPU
    "h8g2": dict(desc="SURVEY 8(d) headline, paper's TP>2 recipe: DeepSeek-V3 32K context, batch 32, g=2 with heads "
                      "split over k=8 (H_loc=32; the 8-GPU per-GPU shard)", model="dsv3", B=32, S=32768, g=2, k=8,
                 xform="hadamard"),
    # configs[4] baseline: replicated-MLA cache (g = 1); "mla2" = the paper's MLA TP=2 (heads split)
    "mla1": dict(desc="configs[4] baseline: MLA (g=1, replicated 576-wide cache), DeepSeek-V3 32K, batch 32, "
                      "all heads on one rank", model="dsv3", B=32, S=32768, g=1, xform="identity"),
    "mla2": dict(desc="configs[4] baseline: MLA (g=1) with heads split over k=2 (the paper's MLA TP=2), "
                      "DeepSeek-V3 32K, batch 32", model="dsv3", B=32, S=32768, g=1, k=2, xform="identity"),
    # two query tokens per sequence per step (MTP / speculative decode); with Kimi's
    # 64 heads per device the tokens x heads rows fill the 128-row MMA
    "c2mtp": dict(desc="SURVEY f3: Kimi-K2 shape, 32K context, batch 64, g=4, 2 query tokens per sequence per step "
                       "(multi-token decode)", model="kimi", B=64, S=32768, g=4, n_q=2, xform="hadamard"),
}
SEED = 1001   # seed = 1000 + config index


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--workload", default="c1", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="tpla", choices=["tpla", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--e2e-diag", action="store_true", help="stderr: per-step graph replay timings behind e2e")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-headline", action="store_true", help="skip the h8 K3 headline record")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the cpu_baseline sample")
    p.add_argument("--batch", type=int, default=None, help="override the workload batch (sweep)")
    p.add_argument("--seq-len", type=int, default=None, help="override the workload context length (sweep)")
    p.add_argument("--g", type=int, default=None, help="override the workload's latent groups g (sweep)")
    p.add_argument("--k", type=int, default=None, help="override the workload's TP ranks k (sweep)")
    p.add_argument("--no-graph", action="store_true", help="issue the timed steps eagerly instead of a CUDA graph")
    p.add_argument("--wo", default="auto", choices=["auto", "rank", "shared"],
                   help="up-projection: 'rank' = every rank multiplies its own v_j by its W^O rows (P:139-141); "
                        "'shared' = the g ranks of a head block sum v first and read W^O once, reduce-scattered "
                        "across processes (SURVEY f2(ii)); auto = shared when g > 1")
    p.add_argument("--fused-ar", action="store_true",
                   help="N > 1: the fused one-shot all-reduce in the W^O epilogue (SURVEY f2(i); validated at world "
                        "1 only) instead of the plain ncclAllReduce")
    p.add_argument("--no-fused-ar", action="store_true", help="(default; kept for compatibility)")
    p.add_argument("--watchdog", type=float, default=1200.0,
                   help="N > 1: seconds after which a run that has not finished prints why and exits 3 "
                        "(a collective that never completes would otherwise hang the launcher)")
    p.add_argument("--rank-streams", default="auto", choices=["auto", "off", "full", "pre"],
                   help="co-located ranks of a latent group: off = serially on one stream; full = one stream per rank "
                        "(separate v accumulators summed in tpla_project_out_sum); pre = each rank's K1 / K3p / K2 on "
                        "its own stream, the attention stages (K3, K45) in rank order on the main stream; auto = full "
                        "for groups of more than 2 ranks, off otherwise")
    p.add_argument("--no-rank-streams", action="store_true", help="= --rank-streams off")
    p.add_argument("--profile-region", action="store_true",
                   help="cudaProfilerStart/Stop around the timed region (for ncu --profile-from-start off)")
    return p.parse_args()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), float(pk.get("bf16_tflops_sustained", 0)), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML SM clock / throttle-reason sampler running during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.0):
        self.samples, self.reasons = [], 0
        self.ok = False
        self.period = period_s
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            if self.period > 0:         # (0: poll back to back — a sub-10 ms region still gets samples)
                time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self, seconds=None):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        out = {"sm_mhz": float(np.median(self.samples)) if self.samples else None, "sm_max_mhz": self.max_mhz,
               "samples": len(self.samples), "reasons": names}
        if self.samples:
            out["sm_mhz_min"] = float(np.min(self.samples))
            out["sm_mhz_p10"] = float(np.percentile(self.samples, 10))
        if seconds is not None:
            out["window_s"] = seconds
        return out


# ----------------------------------------------------------------------------------- CPU oracle leg
class OracleLeg:
    """The fp64 oracle (oracle/, as it stands) decoding ONE sequence of the workload on every one
    of the k ranks, summed over the ranks (the all-reduce).

    Inputs are bf16 bit patterns: the sequence's raw latent rows with their row modes (prompt rows
    EXACT, decode rows SLICED: reading R11), k^PE rows, and one query token (all heads).  The
    offline parts — weight conversion (a1) and the cache rows (a2, rounded to bf16: reading R19) —
    are prepared once, untimed; `run()` times the per-token decode (Q' absorption, shard attention,
    W^UV, W^O, sum over ranks) and returns (y [D], seconds)."""

    def __init__(self, wl, k, g, c_raw_bits, modes, k_pe_bits, q_bits, qpe_bits, sign_seed):
        from oracle import numerics, plan as oplan, reparam, tpla
        self.tpla = tpla
        dims = synth.PRESETS[wl["model"]]
        f64 = numerics.bf16_to_f64
        U = reparam.hadamard_U(dims.d_c, sign_seed) if wl["xform"] == "hadamard" else np.eye(dims.d_c)
        alpha = reparam.uniform_alpha(g)
        w = synth.gen_weights(dims, SEED)
        self.plans = [oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, r) for r in range(k)]
        W_UK_new, W_UV_new = tpla.reparam_weights(f64(w.W_UK), f64(w.W_UV), f64(w.gamma), U)
        eye, W_O = np.eye(dims.d_c), f64(w.W_O)
        self.dws = [tpla.convert_weights(W_UK_new, W_UV_new, np.ones(dims.d_c), W_O, eye, pl, alpha[pl.shard],
                                         d_h=dims.d_h) for pl in self.plans]
        c_raw, k_pe = f64(c_raw_bits), f64(k_pe_bits)
        modes = np.asarray(modes)
        self.rows = {}
        for pl in self.plans:
            if pl.shard in self.rows:
                continue
            rows = np.empty((c_raw.shape[0], pl.row_width))
            for m in (tpla.EXACT, tpla.SLICED):
                sel = modes == m
                if sel.any():
                    rows[sel] = tpla.cache_rows(c_raw[sel], k_pe[sel], U, pl, alpha[pl.shard], 1e-6, m)
            self.rows[pl.shard] = numerics.round_bf16(rows)
        self.q, self.qpe = f64(q_bits)[None], f64(qpe_bits)[None]
        self.sm = 1.0 / math.sqrt(dims.d_h + dims.d_r)

    def run(self):
        t0 = time.perf_counter()
        ys = [self.tpla.decode_device(self.q, self.qpe, [self.rows[pl.shard]], dw, pl, sm_scale=self.sm)
              for pl, dw in zip(self.plans, self.dws)]
        y = self.tpla.all_reduce(ys)[0]
        return y, time.perf_counter() - t0


def host_inputs(wl, nq=1):
    """The workload's sequence 0 generated on the host (reference arm: no GPU)."""
    dims = synth.PRESETS[wl["model"]]
    S = wl["S"]
    q, qpe = synth.gen_queries(dims, 1, SEED)
    return dict(c_raw=synth.gen_raw_ckv(dims, S, SEED, 0), k_pe=synth.gen_kpe(dims, S, SEED, 0),
                modes=["exact"] * (S - nq) + ["sliced"] * nq, q=q[0], qpe=qpe[0])


def time_oracle(leg, budget_s: float, max_reps: int = 50):
    """Repeat the one-sequence decode for ~budget_s on all cores, then once on one thread."""
    reps, total = 0, 0.0
    y = None
    while (total < budget_s or reps == 0) and reps < max_reps:
        y, t = leg.run()
        total += t
        reps += 1
    t1 = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            _, t1 = leg.run()
    except Exception:
        pass
    return y, total / reps, reps, t1


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        n = max((i.get("num_threads", 1) for i in info), default=1)
    except Exception:
        n = None
    return n or len(os.sched_getaffinity(0))


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def config_of(wl, N, k, g):
    return {"workload": wl["desc"], "global_batch": wl["B"], "seq_len": wl["S"], "heads": synth.PRESETS[wl["model"]].h_q,
            "latent": 512, "rope": 64, "g": g, "k": k, "ranks_per_gpu": k // N, "transform": wl["xform"],
            "query_tokens_per_seq": wl.get("n_q", 1),
            "parallelism": f"tpla k={k} g={g} over {N} GPU(s)",
            "l2": "no flush: per-step cache reads (>=0.5 GB) exceed the 126 MB L2",
            "data": "synthetic (seeded bf16; DESIGN.md input recipe)"}


def run_reference(args):
    """The reference arm for this tier: the fp64 oracle as it stands, on the host cores, rank 0 only.
    Each step is ONE sequence's full decode (all heads, all k ranks, summed) of the workload —
    a bounded sample of the batch; tokens/s = sequences decoded / time (no extrapolation)."""
    wl = WORKLOADS[args.workload]
    N = args.gpus
    k = max(N, wl.get("k", wl["g"]))
    g = wl["g"]
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    nq = wl.get("n_q", 1)
    inp = host_inputs(wl, nq)
    t_setup = time.perf_counter()
    leg = OracleLeg(wl, k, g, inp["c_raw"], inp["modes"], inp["k_pe"], inp["q"], inp["qpe"], SEED)
    t_setup = time.perf_counter() - t_setup
    for _ in range(args.warmup):
        leg.run()
    total = 0.0
    for _ in range(args.steps):
        total += leg.run()[1]
    sec = total / max(1, args.steps)
    value = 1.0 / sec
    sample = (f"each step: the fp64 oracle's decode of ONE sequence of the batch (all {synth.PRESETS[wl['model']].h_q} "
              f"heads, all k={k} ranks summed) at {wl['S']} context, on the workload's inputs generated on the host; "
              f"the batch's sequences are independent, so tokens/s = sequences / time (measured, not extrapolated); "
              f"untimed setup (weight conversion, cache rows) {t_setup:.1f}s")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_of(wl, N, k, g),
            "tokens_per_step": 1, "extrapolated": False,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
                             "sample": sample, "host": {"affinity_cores": len(os.sched_getaffinity(0)),
                                                        "cpu": _cpu_name()}},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------- GPU leg
def headline_k3(args, dev, torch, abi, TplaRank, LayerSpec, hbm):
    """SURVEY 8(d)'s headline: TPLA decode attention at 32K on 8 x B200, one latent shard per GPU
    (DeepSeek-V3, g = 8: H_loc 128, W_lat 64, W 128), batch 32.  One GPU holds one such shard: K3
    alone, K launches back to back in a CUDA graph between two CUDA events.  The cache holds N(0, 1)
    bf16 rows (normalised-latent statistics); bytes = Σ_b S_b · W · 2 per launch."""
    dims = synth.PRESETS["dsv3"]
    B, S, k, g = 32, 32768, 8, 8
    rk = TplaRank(LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D), k=k, g=g, rank=k - 1, batch=B,
                  max_seq_len=S, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED + 8)
    rk.cache_buf[..., :rk.plan.row_width].normal_(generator=gen)
    q_lat = torch.randn((B, rk.plan.h_loc, rk.plan.w_lat), generator=gen, device=dev).to(torch.bfloat16)
    q_pe = torch.randn((B, dims.h_q, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    for _ in range(3):
        rk.decode_attention(q_lat, q_pe, lens, None)            # (K3p + K3: leaves the schedule in ws)
    torch.cuda.synchronize()
    n = max(args.steps, 20)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, capture_error_mode="relaxed"):
        for _ in range(n):
            rk.decode_attention(q_lat, q_pe, lens, None, reuse_plan=True)   # K3 alone
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as cs:
        e0.record()
        gr.replay()
        e1.record()
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    nbytes = B * S * rk.plan.row_width * 2
    gbs = nbytes / (us * 1e-6) / 1e9
    out = {"workload": "SURVEY 8(d) headline: DeepSeek-V3 32K, batch 32, g=8 (one latent shard per GPU of 8), K3 alone",
           "kernel": "K3_attn_tc (W_lat=64)", "launches": n, "us_per_launch": us,
           "algorithmic_bytes_per_launch": nbytes, "hbm_gbs": gbs, "hbm_frac": gbs / hbm,
           "hbm_frac_of_8tbs": gbs / 8000.0, "target_frac": 0.70, "meets_target": gbs / hbm >= 0.70,
           "clocks": cs.summary(us * n * 1e-6)}
    del rk, gr
    torch.cuda.empty_cache()
    return out



def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_2508_15881_b200 import abi
    from paper_2508_15881_b200.runtime import (LayerSpec, TplaRank, bf16_from_bits, bits_from_bf16, group_process_sets,
                                               head_block_groups)

    wl = dict(WORKLOADS[args.workload])
    if args.batch:
        wl["B"] = args.batch
    if args.seq_len:
        wl["S"] = args.seq_len
    if args.g:
        wl["g"] = args.g
        wl["xform"] = "hadamard" if args.g > 1 else "identity"
    if args.k:
        wl["k"] = args.k
    N = args.gpus
    world = int(os.environ.get("WORLD_SIZE", "1"))
    proc = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == N, f"--gpus {N} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        def watchdog():
            time.sleep(args.watchdog)
            print(json.dumps({"error": f"rank {proc}: no result after {args.watchdog:.0f} s (watchdog)"}), file=sys.stderr,
                  flush=True)
            os._exit(3)
        threading.Thread(target=watchdog, daemon=True).start()
        dist.init_process_group("nccl", device_id=dev)
    dims = synth.PRESETS[wl["model"]]
    g = wl["g"]
    k = max(N, wl.get("k", g))
    if k % N or dims.h_q % (k // g):
        raise SystemExit(f"k={k} ranks cannot be spread over {N} GPUs")
    m = k // N
    my_ranks = list(range(proc * m, (proc + 1) * m))
    B, S = wl["B"], wl["S"]
    nq = wl.get("n_q", 1)                    # query tokens per sequence per step (multi-token decode)
    spec = LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D)

    # ---- setup (untimed): weights, converted per rank; cache prefilled through K1 (EXACT rows)
    w = synth.gen_weights(dims, SEED)
    ranks = []
    for r in my_ranks:
        rk = TplaRank(spec, k=k, g=g, rank=r, batch=B, max_seq_len=S, device=dev, n_q=nq)
        xf = abi.XFORM_HADAMARD if wl["xform"] == "hadamard" else abi.XFORM_IDENTITY
        rk.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=SEED)
        ranks.append(rk)
    del w
    gen = torch.Generator(device=dev)
    gen.manual_seed(SEED)
    sig = torch.tensor(synth.latent_spectrum(dims.d_c, dims.n_outlier), dtype=torch.float32, device=dev)
    pos_all = torch.arange(S - nq, dtype=torch.int32, device=dev)
    seq0 = None                              # sequence 0's raw prompt rows: the oracle leg's inputs
    for b in range(B):
        ck = (torch.randn((S - nq, dims.d_c), generator=gen, device=dev) * sig).to(torch.bfloat16)
        kp = torch.randn((S - nq, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
        sq = torch.full((S - nq,), b, dtype=torch.int32, device=dev)
        if b == 0 and proc == 0 and N == 1 and not args.no_cpu_baseline:
            seq0 = (bits_from_bf16(ck), bits_from_bf16(kp))
        for rk in ranks:
            rk.prefill(ck, kp, sq, pos_all)
    del ck, kp, sq, pos_all
    # per-step inputs: new latent row + RoPE key of every sequence at position S-1, queries
    NP = 4
    qshape = (B, dims.h_q) if nq == 1 else (B, nq, dims.h_q)
    new_ck = [(torch.randn((B * nq, dims.d_c), generator=gen, device=dev) * sig).to(torch.bfloat16) for _ in range(NP)]
    new_kp = [torch.randn((B * nq, dims.d_r), generator=gen, device=dev).to(torch.bfloat16) for _ in range(NP)]
    qn = [torch.randn(qshape + (dims.d_h,), generator=gen, device=dev).to(torch.bfloat16) for _ in range(NP)]
    qp = [torch.randn(qshape + (dims.d_r,), generator=gen, device=dev).to(torch.bfloat16) for _ in range(NP)]
    seq_idx = torch.arange(B, dtype=torch.int32, device=dev).repeat_interleave(nq)
    pos_new = (S - nq + torch.arange(nq, dtype=torch.int32, device=dev)).repeat(B)
    seq_lens = torch.full((B,), S, dtype=torch.int32, device=dev)
    y = torch.zeros((B * nq, dims.D), dtype=torch.float32, device=dev)
    out = torch.empty((B * nq, dims.D), dtype=torch.bfloat16, device=dev)
    comm = None
    ar_mode = 0
    if N > 1:
        obj = [abi.tpla_comm_unique_id() if proc == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = abi.tpla_comm_init(obj[0], N, proc)
        if args.fused_ar and not args.no_fused_ar:
            try:        # the all-reduce inside the K5 reduce (symmetric window, LSA / NVLS)
                abi.tpla_comm_enable_fused_allreduce(comm, B * nq * dims.D)
            except abi.TplaError as e:
                print(f"[bench] fused all-reduce unavailable, plain ncclAllReduce: {e}", file=sys.stderr)
        ar_mode = abi.tpla_comm_fused_allreduce_mode(comm)
    wo = args.wo if args.wo != "auto" else ("shared" if g > 1 else "rank")
    groups = head_block_groups(k, g, N, proc) if wo == "shared" else []
    gcomms = {}
    if wo == "shared":
        for ps in group_process_sets(k, g, N):               # one communicator per process set, global order
            obj = [abi.tpla_comm_unique_id() if proc == ps[0] else None]
            dist.broadcast_object_list(obj, src=ps[0])
            if proc in ps:
                gcomms[ps] = abi.tpla_comm_init(obj[0], len(ps), ps.index(proc))
    by_id = {rk.rank: rk for rk in ranks}
    v_acc = [torch.zeros(by_id[grp.local_ranks[0]].v_acc_shape(B * nq, grp.n_chunks), dtype=torch.float32, device=dev)
             for grp in groups]
    # A latent group held entirely by this process (all N = 1 runs): each rank's K1 + decode_v on its own
    # stream into its own accumulator (the ranks are independent devices in the deployment),
    # summed in rank order by tpla_project_out_sum.  Groups spanning processes keep the in-place sum
    # that the reduce-scatter needs.
    rs_mode = "off" if args.no_rank_streams else args.rank_streams
    par = [wo == "shared" and rs_mode != "off" and gcomms.get(grp.procs) is None and len(grp.local_ranks) > 1
           for grp in groups]
    # auto: one stream per rank for groups of more than two ranks (h8 666 -> 586 us, c3 / c2 a few %) or
    # when a rank's attention is short (batch 1 at 32K: 155 -> 125 us); two ranks with long K3s (c1)
    # gain nothing from either overlap (A/B: off 344-348, pre 349, full 347-352 us)
    short_k3 = B * S * (dims.d_c // g + dims.d_r) * 2 < (128 << 20)
    par = [p and (rs_mode != "auto" or len(grp.local_ranks) > 2 or short_k3) for p, grp in zip(par, groups)]
    par_mode = ["full" if rs_mode == "auto" else rs_mode for grp in groups]
    v_sep = [[torch.zeros_like(v_acc[gi]) for _ in grp.local_ranks] if par[gi] else None
             for gi, grp in enumerate(groups)]
    rank_streams = {r: torch.cuda.Stream(device=dev) for gi, grp in enumerate(groups) if par[gi] for r in grp.local_ranks}
    stream = torch.cuda.current_stream()

    def step(i, ck=None, kp=None, q=None, qq=None, o=None, serial=False):
        ck = new_ck[i % NP] if ck is None else ck
        kp = new_kp[i % NP] if kp is None else kp
        q = qn[i % NP] if q is None else q
        qq = qp[i % NP] if qq is None else qq
        o = out if o is None else o
        if wo == "shared":
            main = torch.cuda.current_stream()
            for gi, (grp, va) in enumerate(zip(groups, v_acc)):
                if par[gi] and not serial and par_mode[gi] == "full":     # one stream per co-located rank
                    for j, r in enumerate(grp.local_ranks):
                        st = rank_streams[r]
                        st.wait_stream(main)
                        with torch.cuda.stream(st):
                            by_id[r].append(ck, kp, seq_idx, pos_new, abi.RMS_SLICED)
                            by_id[r].decode_v(q, qq, seq_lens, v_sep[gi][j], n_chunks=grp.n_chunks)
                    for r in grp.local_ranks:
                        main.wait_stream(rank_streams[r])
                elif par[gi] and not serial:               # the query stages early, the attention in order
                    for j, r in enumerate(grp.local_ranks):
                        st = rank_streams[r]
                        st.wait_stream(main)
                        with torch.cuda.stream(st):
                            by_id[r].append(ck, kp, seq_idx, pos_new, abi.RMS_SLICED)
                            by_id[r].decode_v(q, qq, seq_lens, v_sep[gi][j], n_chunks=grp.n_chunks, stage="pre")
                    for j, r in enumerate(grp.local_ranks):
                        main.wait_stream(rank_streams[r])
                        by_id[r].decode_v(q, qq, seq_lens, v_sep[gi][j], n_chunks=grp.n_chunks, stage="attn")
                else:
                    for j, r in enumerate(grp.local_ranks):
                        by_id[r].append(ck, kp, seq_idx, pos_new, abi.RMS_SLICED)
                        by_id[r].decode_v(q, qq, seq_lens, va, n_chunks=grp.n_chunks, accumulate=j > 0)
            for gi, (grp, va) in enumerate(zip(groups, v_acc)):
                last = gi == len(groups) - 1
                rk0 = by_id[grp.local_ranks[0]]
                if par[gi] and not serial:
                    rk0.project_out_sum(v_sep[gi], y, o if last else None, chunk=grp.chunk, accumulate=gi > 0,
                                        comm=comm if last else None)
                else:
                    rk0.project_out(va, y, o if last else None, chunk=grp.chunk, accumulate=gi > 0,
                                    group_comm=gcomms.get(grp.procs), comm=comm if last else None)
            return
        for rk in ranks:
            rk.append(ck, kp, seq_idx, pos_new, abi.RMS_SLICED)
        for j, rk in enumerate(ranks):
            last = j == len(ranks) - 1
            if nq == 1:
                rk.decode(q, qq, seq_lens, y, o if last else None, accumulate=j > 0, comm=comm if last else None)
            else:
                rk.decode_mtp(q, qq, seq_lens, y, o if last else None, accumulate=j > 0, comm=comm if last else None)

    def barrier():
        if N > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if N == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- the north-star headline shape in the same run, before the main timed region (a cool GPU, as
    # for every other kernel time of this line): K3 alone on one 8-GPU shard (DeepSeek-V3, 32K, batch 32,
    # g = 8: W_lat = 64, W = 128), back to back in a CUDA graph, CUDA events
    headline = None
    if proc == 0 and not args.no_headline:
        headline = headline_k3(args, dev, torch, abi, TplaRank, LayerSpec, load_peaks()[0])

    for i in range(args.warmup):
        step(i)
    abi.tpla_sync(stream.cuda_stream)

    # ---- timed region (device-timed with CUDA events on the launching stream)
    # The K steps are captured once as a CUDA graph (every library call is async on the stream,
    # NCCL included) and replayed: no host launch overhead inside the region.  The library's
    # per-kernel profile events are captured too, as event nodes between the kernels.
    # Two identical captures: `graph` (no profiling) times the value; `graph_prof` (with the
    # library's event nodes around every kernel) is replayed right after for the per-kernel times.
    abi.tpla_profile_reset()
    n0 = abi.tpla_launch_count()
    graph = graph_prof = breakdown = None
    k3_q = [torch.randn((B, rk.plan.h_loc, rk.plan.w_lat), generator=gen, device=dev).to(torch.bfloat16) for rk in ranks]
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            for i in range(args.steps):
                step(i)
        launches = abi.tpla_launch_count() - n0           # kernels in the K timed steps
        abi.tpla_profile_enable(1)                       # events around every kernel (breakdown)
        graph_all = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph_all, capture_error_mode="relaxed"):
            for i in range(args.steps):
                step(i, serial=True)                     # (one stream: per-kernel durations stay defined)
        abi.tpla_profile_enable(False)
        # the event nodes add gaps between kernels, so these durations are upper bounds
        graph_all.replay()
        torch.cuda.synchronize()
        breakdown = abi.profile_table()
        abi.tpla_profile_reset()
        # K3 alone: the attention launches of the K steps (same kernel, same cache, Q' of the
        # same shape), back to back with no event nodes; outer events give its launch duration
        graph_prof = torch.cuda.CUDAGraph() if nq == 1 else None     # (K3 alone: single-token only)
        if graph_prof is not None:
            with torch.cuda.graph(graph_prof, capture_error_mode="relaxed"):
                for i in range(args.steps):
                    for j, rk in enumerate(ranks):
                        rk.decode_attention(k3_q[j], qp[i % NP], seq_lens, None, reuse_plan=True)   # K3 alone
                                                 # (on the schedule the step's K3p left in the rank's ws)
        stream = torch.cuda.current_stream()
        graph.replay()                                   # untimed warm replay
        torch.cuda.synchronize()
    else:
        abi.tpla_profile_enable(True)
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if args.profile_region:
        torch.cuda.cudart().cudaProfilerStart()
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for i in range(args.steps):
                step(i)
        ev1.record(stream)
        torch.cuda.synchronize()
    if args.profile_region:
        torch.cuda.cudart().cudaProfilerStop()
    barrier()
    # the same graph replayed back to back for >= 0.5 s: the clock record of a sustained run (the
    # timed region itself may be a few ms; its own samples are in `clocks`)
    clocks_sust = None
    if graph is not None and not args.profile_region:
        with ClockSampler(local, period_s=0.002) as cs:
            t_end = time.perf_counter() + 0.5
            n_rep = 0
            while time.perf_counter() < t_end or n_rep == 0:
                graph.replay()
                n_rep += 1
                if n_rep % 4 == 0:
                    torch.cuda.synchronize()
            torch.cuda.synchronize()
        clocks_sust = cs.summary()
        clocks_sust["replays"] = n_rep
    ms_prof = None
    if graph is not None:
        if graph_prof is not None:
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            graph_prof.replay()
            p1.record(stream)
            torch.cuda.synchronize()
            ms_prof = p0.elapsed_time(p1) / (args.steps * len(ranks))   # ms per isolated K3 launch
        prof = breakdown                                 # in-step durations (roofline)
    else:
        launches = abi.tpla_launch_count() - n0
        prof = abi.profile_table()
        breakdown = prof
    abi.tpla_profile_enable(False)
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    ms_step = ms / args.steps
    value = B * nq * args.steps / (ms / 1e3)
    abi.tpla_sync(stream.cuda_stream)

    # ---- roofline of the dominant kernel (K3 attention), per launch = one rank's shard
    hbm, tf_burst, tf_sust, peak_src = load_peaks()
    k3_name = next((n for n in prof if n.startswith("K3_attn")), None)
    plan0 = ranks[0].plan
    bytes_k3 = B * S * plan0.row_width * 2                       # Σ_b S_b · W · 2
    flops_k3 = 2 * B * nq * S * plan0.h_loc * (2 * plan0.w_lat + dims.d_r)   # (MTP: ~S keys per token)
    k3_ms, k3_n = prof.get(k3_name, (float("nan"), 1))
    k3_avg_s = k3_ms / max(k3_n, 1) / 1e3
    gbs = bytes_k3 / k3_avg_s / 1e9
    tfs = flops_k3 / k3_avg_s / 1e12
    # The tensor peak follows the run's own clock record (B200_PROFILING.md): a sub-second timed
    # region that saw no sw_power_cap runs at burst clocks -> the burst bf16 figure; otherwise the
    # sustained one.  The binding roofline is the slower of bytes / HBM and FLOPs / tensor peak.
    clk = clocks.summary(ms / 1e3)
    burst = ms < 1000.0 and "sw_power_cap" not in clk.get("reasons", [])
    tf_peak = tf_burst if (burst or tf_sust <= 0) else tf_sust
    t_hbm_s, t_tc_s = bytes_k3 / (hbm * 1e9), flops_k3 / (tf_peak * 1e12)
    bound = "hbm" if t_hbm_s >= t_tc_s else "tensor"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if k3_name in tr and tr[k3_name].get("workload") == args.workload:
            traffic = tr[k3_name]["dram_bytes_per_launch"]
    except Exception:
        pass
    step_gpu_ms = ms_step                                  # clean (unprofiled) step time
    roofline = {"bound": bound, "achieved": gbs if bound == "hbm" else tfs, "peak": hbm if bound == "hbm" else tf_peak,
                "unit": "GB/s" if bound == "hbm" else "TFLOP/s", "frac": (gbs / hbm) if bound == "hbm" else (tfs / tf_peak),
                "traffic": traffic, "kernel": k3_name,
                "peak_source": (f"{peak_src} MEASURED_PEAKS.json: hbm_gbs and "
                                f"{'bf16_tflops (burst: timed region < 1 s, no sw_power_cap)' if tf_peak == tf_burst else 'bf16_tflops_sustained (long or power-capped region)'}"),
                "tensor_peak_choice": "burst" if tf_peak == tf_burst else "sustained",
                "roofline_time_us": {"hbm": t_hbm_s * 1e6, "tensor": t_tc_s * 1e6,
                                     "tensor_burst": flops_k3 / (tf_burst * 1e12) * 1e6,
                                     "tensor_sustained": flops_k3 / (max(tf_sust, 1e-9) * 1e12) * 1e6},
                "hbm_gbs": gbs, "hbm_frac": gbs / hbm, "hbm_frac_of_8tbs": gbs / 8000.0,
                "algorithmic_bytes_per_launch": bytes_k3, "algorithmic_flops_per_launch": flops_k3,
                "avg_launch_us": k3_avg_s * 1e6, "launches": k3_n,
                "isolated_avg_launch_us": ms_prof * 1e3 if ms_prof else None,
                "tensor_tflops": tfs, "tensor_frac_of_burst": tfs / tf_burst,
                "tensor_frac_of_sustained": tfs / tf_sust if tf_sust > 0 else None,
                "share_of_step": (k3_ms / args.steps) / step_gpu_ms if step_gpu_ms > 0 else None}
    kernels = {n: {"us_per_step": v[0] / args.steps * 1e3, "launches_per_step": v[1] / args.steps}
               for n, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0])}

    # ---- end to end through the public API with host buffers (pinned), copies inside the region
    e2e = None
    if not args.no_e2e:
        # A step's inputs (new latent rows, RoPE keys, queries) travel as ONE packed pinned buffer and
        # one copy (a serving engine stages its batch the same way); the device views unpack them.
        parts = (new_ck, new_kp, qn, qp)
        nbytes = [t[0].numel() * t[0].element_size() for t in parts]
        offs = [sum(nbytes[:i]) for i in range(len(nbytes))]
        h_in = []
        for j in range(NP):
            hb = torch.empty(sum(nbytes), dtype=torch.uint8).pin_memory()
            for t, o_, n_ in zip(parts, offs, nbytes):
                hb[o_:o_ + n_].copy_(t[j].contiguous().view(-1).view(torch.uint8).cpu())
            h_in.append(hb)
        d_buf = [torch.empty(sum(nbytes), dtype=torch.uint8, device=dev) for _ in range(2)]
        d_in = [tuple(d_buf[s_][o_:o_ + n_].view(t[0].dtype).view(t[0].shape) for t, o_, n_ in zip(parts, offs, nbytes))
                for s_ in range(2)]
        # Serving-style pipeline: two input/output buffer sets; step i's host->device copy runs on a
        # copy stream while step i-1 computes, its output comes back on a second copy stream, and
        # the host consumes step i-1's output (waits for it) after enqueueing step i.
        h_out = [torch.empty((B * nq, dims.D), dtype=torch.bfloat16).pin_memory() for _ in range(2)]
        d_out = [torch.empty_like(out) for _ in range(2)]
        h2d = sum(nbytes)
        d2h = h_out[0].numel() * h_out[0].element_size()
        n_e2e = min(max(args.steps, 100), 200)           # (>= 100 steps: host jitter amortised)
        for i in range(3):
            step(i, *d_in[i & 1], o=d_out[i & 1])
        g1 = [None, None]
        if not args.no_graph:                         # one decode step (K1..K5) per buffer set
            for s in range(2):
                g1[s] = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g1[s], capture_error_mode="relaxed"):
                    step(0, *d_in[s], o=d_out[s])
            stream = torch.cuda.current_stream()
            for s in range(2):                        # first replays upload the graphs: keep them untimed
                g1[s].replay()
            torch.cuda.synchronize()
        cs_in, cs_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        barrier()
        torch.cuda.synchronize()
        # (a second of idle first: the sustained-clock replays above hold the board at its power cap, and
        # the e2e region should see the same clocks as the main timed region; its own clocks are reported)
        time.sleep(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ce = ClockSampler(local, period_s=0.002).__enter__()
        e0.record(stream)
        cs_in.wait_event(e0)
        for i in range(n_e2e):
            s, j = i & 1, i % NP
            with torch.cuda.stream(cs_in):
                if i >= 2:
                    cs_in.wait_event(ev_done[s])     # buffer set s is free (step i-2 computed)
                d_buf[s].copy_(h_in[j], non_blocking=True)
                ev_in[s].record(cs_in)
            stream.wait_event(ev_in[s])
            if g1[s] is not None:
                g1[s].replay()
            else:
                step(i, *d_in[s], o=d_out[s])
            ev_done[s].record(stream)
            with torch.cuda.stream(cs_out):
                cs_out.wait_event(ev_done[s])
                h_out[s].copy_(d_out[s], non_blocking=True)
                ev_out[s].record(cs_out)
            if i >= 1:
                ev_out[s ^ 1].synchronize()          # the host consumes step i-1's output
        ev_out[(n_e2e - 1) & 1].synchronize()
        e1.record(cs_out)
        torch.cuda.synchronize()
        ce.__exit__(None, None, None)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1))
        if args.e2e_diag and g1[0] is not None:
            # where the e2e time goes: per-step graph replays back to back (no copies, no host waits),
            # then with the cross-stream event waits, then with the host waiting for every output
            def timed(fn):
                torch.cuda.synchronize()
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                fn()
                a1.record(stream)
                torch.cuda.synchronize()
                return a0.elapsed_time(a1) / n_e2e * 1e3
            def replays():
                for i in range(n_e2e):
                    g1[i & 1].replay()
            def replays_ev():
                for i in range(n_e2e):
                    s = i & 1
                    with torch.cuda.stream(cs_in):
                        ev_in[s].record(cs_in)
                    stream.wait_event(ev_in[s])
                    g1[s].replay()
                    ev_done[s].record(stream)
            def replays_sync():
                for i in range(n_e2e):
                    s = i & 1
                    g1[s].replay()
                    ev_done[s].record(stream)
                    if i >= 1:
                        ev_done[s ^ 1].synchronize()
            print(json.dumps({"e2e_diag_us_per_step": {"graph_per_step": timed(replays),
                                                       "with_event_waits": timed(replays_ev),
                                                       "with_host_wait": timed(replays_sync),
                                                       "e2e": ems / n_e2e * 1e3}}), file=sys.stderr)
        e2e = {"value": B * nq * n_e2e / (ems / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": n_e2e, "ms_per_step": ems / n_e2e,
               "pipeline": "double-buffered: H2D of step i and D2H of step i-1 on copy streams, "
                           "overlapping compute; host waits for every step's output",
               "clocks": ce.summary(ems / 1e3)}

    # ---- parity of this run's own step against the fp64 oracle, and the oracle timed (cpu_baseline)
    cpu = None
    if seq0 is not None:
        y.zero_()
        step(0)                                              # one step: new rows new_ck[0], queries qn[0]
        torch.cuda.synchronize()
        row = nq - 1                                         # sequence 0's last query token sees every row
        gpu_y = y[row].double().cpu().numpy()
        ck0 = np.concatenate([seq0[0], bits_from_bf16(new_ck[0][:nq])])
        kp0 = np.concatenate([seq0[1], bits_from_bf16(new_kp[0][:nq])])
        q0 = bits_from_bf16(qn[0][0] if nq == 1 else qn[0][0, nq - 1])
        qp0 = bits_from_bf16(qp[0][0] if nq == 1 else qp[0][0, nq - 1])
        t_setup = time.perf_counter()
        leg = OracleLeg(wl, k, g, ck0, ["exact"] * (S - nq) + ["sliced"] * nq, kp0, q0, qp0, SEED)
        t_setup = time.perf_counter() - t_setup
        ref_y, sec, reps, sec1 = time_oracle(leg, args.cpu_seconds)
        err = float(np.max(np.abs(gpu_y - ref_y)) / np.max(np.abs(ref_y)))
        cpu = {"value": 1.0 / sec, "unit": "tokens/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": (f"fp64 oracle decode of sequence 0 of this run's batch (its {S} cache rows from the same "
                          f"device-generated raw latents the GPU cache was written from, the step's new row and "
                          f"query; all {dims.h_q} heads, all k={k} ranks summed), repeated {reps}x; "
                          f"{sec * 1e3:.0f} ms per token; untimed setup {t_setup:.1f}s"),
               "same_inputs": True, "parity_max_row_rel_err": err, "parity_tol": 1e-2,
               "one_thread": {"value": 1.0 / sec1, "unit": "tokens/s", "cores": 1} if sec1 else None,
               "us_per_layer_batch": sec * B * 1e6,
               "host": {"affinity_cores": len(os.sched_getaffinity(0)), "cpu": _cpu_name()}}

    if comm is not None:
        abi.tpla_comm_destroy(comm)
    for c in gcomms.values():
        abi.tpla_comm_destroy(c)
    if proc == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "us_per_layer": ms_step * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic", "impl": "tpla", "config": config_of(wl, N, k, g),
                "up_projection": ("shared: the latent group's v_j summed first (co-located ranks: one stream per rank "
                                  "into separate accumulators, summed in rank order by tpla_project_out_sum; across "
                                  "GPUs a reduce-scatter over column chunks), W^O read once per head block "
                                  "(SURVEY f2(ii); Σ_j v_j W^O_i = (Σ_j v_j) W^O_i, P:363)" if wo == "shared" else
                                  "rank: every rank multiplies its own v_j by its W^O rows (P:139-141)"),
                "roofline": roofline, "headline": headline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "gpu_launches_per_step": launches / args.steps, "clocks": clk, "clocks_sustained": clocks_sust,
                "kernels": kernels,
                "cuda_graph": graph is not None,
                "rank_streams": sorted({m for m, p in zip(par_mode, par) if p}) or "off",
                "all_reduce": ({0: "ncclAllReduce", 1: "fused into the K5 reduce (LSA peer loads)",
                                2: "fused into the K5 reduce (NVLS multimem.ld_reduce)"}[ar_mode]
                               if N > 1 else "none (N = 1)"),
                "kernel_timing": ("library CUDA events (on the launching stream) captured as graph event nodes "
                                  "around every kernel of the K timed steps, replayed right after the timed "
                                  "replay, with the co-located ranks on ONE stream (the timed graph overlaps them "
                                  "on per-rank streams; the nodes add small gaps: durations are upper bounds); "
                                  "roofline.isolated_avg_launch_us: a graph of the K3 launches alone"
                                  if graph is not None else "library CUDA events inside the timed region"),
                "hbm_gbs_per_gpu_k3": gbs, "kv_bytes_per_gpu_per_step": bytes_k3 * len(ranks)}
        print(json.dumps(line), flush=True)
    if N > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
