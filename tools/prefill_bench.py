"""prefill attention time of one prompt (TTFT of one attention layer), DSV3 shape, the k
ranks of the TP group on this GPU (per-device time = total / k):
  mla_fwd   the PD-separated MLA prefill in its non-absorbed form (tpla_prefill_mla_forward: RMSNorm,
            k/v up-projection GEMMs, the K8 causal attention kernel, W^O), heads split over k, g = 1,
            plus the K1 write of the prompt's decode-cache rows (EXACT rows);
  mla_abs   the same MLA prefill through the absorbed decode kernels (tpla_prefill_attention, g = 1);
  tpla_abs  the TPLA prefill (g = k) through the absorbed decode kernels.
The paper reports TTFT 1.4x in favour of the PD-separated MLA prefill at 1K context (its
hardware).  Also reports the K8 forward's achieved TFLOP/s on its algorithmic FLOPs (the k/v
up-projections, the causal attention with head dim 192 / 128, W^O).

    python tools/prefill_bench.py [--L 1024 4096] [--k 2] [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2508_15881_b200 import abi  # noqa: E402
from paper_2508_15881_b200.runtime import LayerSpec, PrefillRank, TplaRank  # noqa: E402


def inputs(L, dev):
    dims = synth.PRESETS["dsv3"]
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    sig = torch.tensor(synth.latent_spectrum(dims.d_c, dims.n_outlier), dtype=torch.float32, device=dev)
    ck = (torch.randn((L, dims.d_c), generator=gen, device=dev) * sig).to(torch.bfloat16)
    kp = torch.randn((L, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    q = torch.randn((L, dims.h_q, dims.d_h), generator=gen, device=dev).to(torch.bfloat16)
    qp = torch.randn((L, dims.h_q, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    return ck, kp, q, qp


def timed(step, iters):
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def run_fwd(L, k, iters, dev):
    """The non-absorbed MLA prefill (K8) + the K1 cache write of the prompt, per device."""
    dims = synth.PRESETS["dsv3"]
    spec = LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D)
    w = synth.gen_weights(dims, 7)
    ck, kp, q, qp = inputs(L, dev)
    seq = torch.zeros(L, dtype=torch.int32, device=dev)
    pos = torch.arange(L, dtype=torch.int32, device=dev)
    prs, caches = [], []
    for r in range(k):
        pr = PrefillRank(spec, k=k, rank=r, max_len=L, device=dev)
        pr.convert(w.W_UK, w.W_UV, w.gamma, w.W_O)
        prs.append(pr)
        rk = TplaRank(spec, k=k, g=k, rank=r, batch=1, max_seq_len=L, device=dev)   # the TPLA decode cache
        rk.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=7)
        caches.append(rk)
    y = torch.zeros((L, dims.D), dtype=torch.float32, device=dev)
    out = torch.empty((L, dims.D), dtype=torch.bfloat16, device=dev)

    def step():
        for j, (pr, rk) in enumerate(zip(prs, caches)):
            rk.prefill(ck, kp, seq, pos)                       # K1: the prompt's decode rows (EXACT)
            pr.forward(ck, kp, q, qp, y, out if j == k - 1 else None, accumulate=j > 0)

    def fwd_only():
        for j, pr in enumerate(prs):
            pr.forward(ck, kp, q, qp, y, out if j == k - 1 else None, accumulate=j > 0)

    ms = timed(step, iters)
    ms_fwd = timed(fwd_only, iters)
    abi.tpla_profile_reset()
    abi.tpla_profile_enable(1)                               # per-kernel device time of one forward (all ranks)
    fwd_only()
    torch.cuda.synchronize()
    prof = abi.profile_table()
    abi.tpla_profile_enable(0)
    abi.tpla_profile_reset()
    kernels = {n: round(v[0] * 1e3 / k, 1) for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}
    H = dims.h_q // k
    flops = (2 * 2 * L * dims.d_c * H * dims.d_h                       # k, v up-projections
             + 2 * (L * (L + 1) // 2) * H * (dims.d_h + dims.d_r + dims.d_h)   # causal QK (192) + PV (128)
             + 2 * L * H * dims.d_h * dims.D)                          # W^O
    return {"L": L, "k": k, "us_all_ranks": ms * 1e3, "us_per_device": ms * 1e3 / k,
            "fwd_us_per_device": ms_fwd * 1e3 / k, "fwd_tflops": flops / (ms_fwd / k / 1e3) / 1e12,
            "fwd_gflop_per_device": flops / 1e9, "prompt_tokens_per_s_per_device": L / (ms / k / 1e3),
            "fwd_kernels_us_per_device": kernels,
            "attn_tflops": 2 * (L * (L + 1) // 2) * H * (dims.d_h + dims.d_r + dims.d_h) /
                           (kernels.get("K8_prefill_fa", float("nan")) * 1e-6) / 1e12}


def run(L, k, g, iters, dev):
    dims = synth.PRESETS["dsv3"]
    spec = LayerSpec(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D)
    w = synth.gen_weights(dims, 7)
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    sig = torch.tensor(synth.latent_spectrum(dims.d_c, dims.n_outlier), dtype=torch.float32, device=dev)
    ck = (torch.randn((L, dims.d_c), generator=gen, device=dev) * sig).to(torch.bfloat16)
    kp = torch.randn((L, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    q = torch.randn((L, dims.h_q, dims.d_h), generator=gen, device=dev).to(torch.bfloat16)
    qp = torch.randn((L, dims.h_q, dims.d_r), generator=gen, device=dev).to(torch.bfloat16)
    seq = torch.zeros(L, dtype=torch.int32, device=dev)
    pos = torch.arange(L, dtype=torch.int32, device=dev)
    xf = abi.XFORM_HADAMARD if g > 1 else abi.XFORM_IDENTITY
    ranks = []
    for r in range(k):
        rk = TplaRank(spec, k=k, g=g, rank=r, batch=1, max_seq_len=L, device=dev)
        rk.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=7)
        ranks.append(rk)
    y = torch.zeros((L, dims.D), dtype=torch.float32, device=dev)
    out = torch.empty((L, dims.D), dtype=torch.bfloat16, device=dev)

    def step():
        for j, rk in enumerate(ranks):
            rk.prefill(ck, kp, seq, pos)                       # K1: the prompt's rows (EXACT)
            rk.prefill_attention(q, qp, 0, y, out if j == k - 1 else None, accumulate=j > 0)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return {"L": L, "k": k, "g": g, "us_all_ranks": ms * 1e3, "us_per_device": ms * 1e3 / k,
            "prompt_tokens_per_s_per_device": L / (ms / k / 1e3)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, nargs="+", default=[1024, 4096])
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--fwd-only", action="store_true", help="only the non-absorbed MLA forward (A/B runs)")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    rows = []
    for L in a.L:
        fwd = run_fwd(L, a.k, a.iters, dev)
        if a.fwd_only:
            print(json.dumps({"L": L, "mla_fwd": fwd}), flush=True)
            continue
        mla = run(L, a.k, 1, a.iters, dev)
        tp = run(L, a.k, a.k, a.iters, dev)
        rows.append({"L": L, "mla_fwd": fwd, "mla_abs": mla, "tpla_abs": tp,
                     "tpla_abs_over_mla_fwd_time": tp["us_per_device"] / fwd["us_per_device"],
                     "mla_abs_over_mla_fwd_time": mla["us_per_device"] / fwd["us_per_device"]})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
