"""slicing-mode ablation on synthetic data (the mechanism behind the paper's
Fig. 3), computed with the fp64 oracle (test infrastructure; this is a study, not the
product path):

  TPLA (norm only)     sliced RMSNorm, exact softmax (partial logits summed before it)
  TPLA (softmax only)  exact RMSNorm, per-shard softmax
  TPLA                 sliced RMSNorm and per-shard softmax (mu = alpha, and mu = 1)
  GLA                  MLA -> GLA conversion: heads block i sees latent shard i only
  x  U in {identity ("Original"), Hadamard, PCA},  g = 2

Error = per-row ||o - o_MLA||_inf / ||o_MLA||_inf against absorbed MLA (g = 1, exact), median
over the batch.  Latents: the input recipe's concentrated spectrum with outlier channels
 expressed in a random orthogonal basis V (the PCA basis handed over is V sorted
by eigenvalue, as in the parity tests); queries and weights as in the recipe.

    python tools/ablation.py [--heads 16] [--seq 256] [--batch 4] [--natural-basis]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import mla, numerics, reparam, tpla  # noqa: E402

MODES = ["norm only", "softmax only", "TPLA (mu=alpha)", "TPLA (mu=1)", "GLA"]
BASES = ["identity", "hadamard", "pca"]


def problem(dims, U, alpha, mu, c_raw, k_pe, q, qpe, modes):
    f = numerics.bf16_to_f64
    w = synth.gen_weights(dims, 11)
    return tpla.Problem(W_UK=f(w.W_UK), W_UV=f(w.W_UV), gamma=f(w.gamma), W_O=f(w.W_O), U=U,
                        alpha=np.asarray(alpha, float), mu=np.asarray(mu, float), c_raw=c_raw, k_pe=k_pe,
                        modes=modes, q_nope=q, q_pe=qpe, h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                        sm_scale=1.0 / np.sqrt(dims.d_h + dims.d_r))


def run(heads=16, seq=256, batch=4, g=2, natural_basis=False, seed=3):
    base = synth.PRESETS["dsv3"]
    dims = synth.ModelDims("ablation", h_q=heads, d_c=base.d_c, d_r=base.d_r, d_h=base.d_h, D=512)
    f = numerics.bf16_to_f64
    V = np.eye(dims.d_c) if natural_basis else synth.random_orthogonal(dims.d_c, seed)
    lam = synth.latent_spectrum(dims.d_c, dims.n_outlier) ** 2
    order = np.argsort(-lam, kind="stable")
    c_raw = [f(synth.gen_raw_ckv(dims, seq, seed, b, basis=None if natural_basis else V)) for b in range(batch)]
    k_pe = [f(synth.gen_kpe(dims, seq, seed, b)) for b in range(batch)]
    qb, qpeb = synth.gen_queries(dims, batch, seed)
    q, qpe = f(qb), f(qpeb)
    w = synth.gen_weights(dims, 11)
    o_mla = np.stack([mla.mla_decode_absorbed(q[b], qpe[b], c_raw[b], k_pe[b], f(w.W_UK), f(w.W_UV), f(w.gamma),
                                              f(w.W_O), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                                              sm_scale=1.0 / np.sqrt(dims.d_h + dims.d_r))[0]
                      for b in range(batch)])
    table = {}
    for kind in BASES:
        if kind == "identity":
            U, alpha = np.eye(dims.d_c), np.full(g, float(g))
        elif kind == "hadamard":
            U, alpha = reparam.hadamard_U(dims.d_c, 7), np.full(g, float(g))
        else:
            U = V[:, order]
            alpha = np.asarray(reparam.pca_alpha(lam[order], g), float)
        sl = [[tpla.SLICED] * seq] * batch
        ex = [[tpla.EXACT] * seq] * batch
        outs = {
            "norm only": tpla.tpla_decode_exact_logits(problem(dims, U, alpha, alpha, c_raw, k_pe, q, qpe, sl), g),
            "softmax only": tpla.tpla_decode_step(problem(dims, U, alpha, alpha, c_raw, k_pe, q, qpe, ex), g, g),
            "TPLA (mu=alpha)": tpla.tpla_decode_step(problem(dims, U, alpha, alpha, c_raw, k_pe, q, qpe, sl), g, g),
            "TPLA (mu=1)": tpla.tpla_decode_step(problem(dims, U, alpha, np.ones(g), c_raw, k_pe, q, qpe, sl), g, g),
            "GLA": tpla.gla_decode_step(problem(dims, U, alpha, np.ones(g), c_raw, k_pe, q, qpe, sl), g),
        }
        for m, o in outs.items():
            e = np.max(np.abs(o - o_mla), axis=1) / np.max(np.abs(o_mla), axis=1)
            table[(kind, m)] = float(np.median(e))
    return table


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--natural-basis", action="store_true", help="latents not rotated (outliers on fixed channels)")
    a = ap.parse_args()
    t = run(a.heads, a.seq, a.batch, natural_basis=a.natural_basis)
    print("| U \\ slicing | " + " | ".join(MODES) + " |")
    print("|---|" + "---|" * len(MODES))
    for kind in BASES:
        print(f"| {kind} | " + " | ".join(f"{t[(kind, m)]:.4f}" for m in MODES) + " |")


if __name__ == "__main__":
    main()
