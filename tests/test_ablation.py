"""slicing-mode ablation on synthetic data (tools/ablation.py, fp64 oracle).

The paper's Fig. 3 findings are measured on trained checkpoints; on the synthetic
recipe only the mechanisms that do not depend on trained attention patterns are expected to
carry over, and those are what these tests pin:

* slicing the RMSNorm alone costs least, slicing the softmax costs more (finding 1);
* with outlier channels in the natural basis, the per-slice RMS of the identity split is far
  off while Hadamard balances it (finding 2; the imbalance argument of P:274-276), and
  PCA with its alpha_j does as well;
* for the per-shard softmax PCA beats Hadamard (finding 3), and with both sliced PCA is
  the best basis (finding 4).

Not reproduced on random data (reported in DESIGN.md, not asserted): "both sliced" being worse
than "softmax only" — random attention is nearly uniform, so the relative errors of the two are
of the same size.
"""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import ablation  # noqa: E402


@pytest.fixture(scope="module")
def rotated():
    return ablation.run(heads=8, seq=128, batch=3, natural_basis=False)


@pytest.fixture(scope="module")
def natural():
    return ablation.run(heads=8, seq=128, batch=3, natural_basis=True)


def test_norm_slicing_costs_less_than_softmax_slicing(rotated, natural):
    for t in (rotated, natural):
        for u in ablation.BASES:
            assert t[(u, "norm only")] < t[(u, "softmax only")], u


def test_hadamard_and_pca_balance_the_sliced_norm(natural):
    ident, had, pca = (natural[(u, "norm only")] for u in ablation.BASES)
    assert had < 0.3 * ident and pca < 0.3 * ident


def test_pca_best_for_sliced_softmax(rotated, natural):
    for t in (rotated, natural):
        assert t[("pca", "softmax only")] < t[("hadamard", "softmax only")]
        assert t[("pca", "TPLA (mu=alpha)")] == min(t[(u, "TPLA (mu=alpha)")] for u in ablation.BASES)
