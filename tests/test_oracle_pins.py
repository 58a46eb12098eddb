"""Pins of the fp64 oracle against what PAPER.md and mathematics fix (pins c1-c14).

None of these tests retypes the oracle's formula: each compares it with a value
the paper prints (tests/golden), a closed form, a library routine the paper names
(scipy.linalg.hadamard), an independent formulation (non-absorbed MLA), or an
invariant that a dropped term / wrong index / transposed operand would break.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg

import synth
from oracle import cost, mla, numerics, plan, reparam, tpla

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def f64(bits):
    return numerics.bf16_to_f64(bits)


def make_problem(dims, *, S=37, B=2, seed=3, U=None, g=2, transform="identity", mu=None, modes="sliced",
                 gamma_one=False, basis=None, alpha=None):
    w = synth.gen_weights(dims, seed, gamma_one=gamma_one)
    if U is None:
        if transform == "identity":
            U = np.eye(dims.d_c)
        elif transform == "hadamard":
            U = reparam.hadamard_U(dims.d_c, 1234)
    if alpha is None:
        alpha = reparam.uniform_alpha(g)
    if mu is None:
        mu = alpha.copy()
    q, qpe = synth.gen_queries(dims, B, seed)
    c_raw = [f64(synth.gen_raw_ckv(dims, S, seed, b, basis=basis)) for b in range(B)]
    k_pe = [f64(synth.gen_kpe(dims, S, seed, b)) for b in range(B)]
    return tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O), U=U,
                        alpha=np.asarray(alpha, float), mu=np.asarray(mu, float), c_raw=c_raw, k_pe=k_pe,
                        modes=[[modes] * S for _ in range(B)], q_nope=f64(q), q_pe=f64(qpe),
                        h_q=dims.h_q, d_h=dims.d_h, eps=1e-6, sm_scale=1.0 / np.sqrt(dims.d_h + dims.d_r))


def mla_ref(pb, absorbed=False):
    f = mla.mla_decode_absorbed if absorbed else mla.mla_decode_full
    outs = []
    for b in range(len(pb.c_raw)):
        r = f(pb.q_nope[b], pb.q_pe[b], pb.c_raw[b], pb.k_pe[b], pb.W_UK, pb.W_UV, pb.gamma, pb.W_O,
              h_q=pb.h_q, d_h=pb.d_h, eps=pb.eps, sm_scale=pb.sm_scale)
        outs.append(r[0])
    return np.stack(outs)


def rel(a, b):
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


DIMS = [synth.PRESETS["tiny"], synth.PRESETS["odd"]]


# ---------------------------------------------------------------- numerics
def test_rms_closed_forms():
    # RMS((3,4), 0) = sqrt(12.5); RMS((c), 0) = |c|; ε enters under the root
    assert numerics.rms(np.array([3.0, 4.0]), 0.0) == pytest.approx(np.sqrt(12.5), rel=1e-15)
    assert numerics.rms(np.array([-7.0]), 0.0) == pytest.approx(7.0, rel=1e-15)
    assert numerics.rms(np.zeros(4), 0.25) == pytest.approx(0.5, rel=1e-15)
    out = numerics.rmsnorm(np.array([2.0, 3.0]), np.array([3.0, 4.0]), 0.0)
    assert np.allclose(out, np.array([3.0 * 2, 4.0 * 3]) / np.sqrt(12.5), rtol=1e-15, atol=0)


def test_softmax_brute_force():
    s = np.array([[0.3, -1.2, 2.0], [5.0, 5.0, 5.0]])
    e = np.exp(np.array([0.3, -1.2, 2.0]))
    assert np.allclose(numerics.softmax(s)[0], e / e.sum(), rtol=1e-15)
    assert np.allclose(numerics.softmax(s)[1], 1.0 / 3.0, rtol=1e-15)


def test_round_bf16_against_bit_truncation():
    # every value exactly representable in bf16 is a fixed point; midpoints go to even
    rng = np.random.default_rng(0)
    x = rng.standard_normal(10000).astype(np.float32)
    exact = numerics.bf16_to_f64(synth.bf16_bits(x))
    assert np.array_equal(numerics.round_bf16(exact), exact)
    assert numerics.round_bf16(np.array([1.0 + 2.0 ** -8]))[0] == 1.0               # tie -> even
    assert numerics.round_bf16(np.array([1.0 + 3 * 2.0 ** -8]))[0] == 1.0 + 2.0 ** -6  # tie -> even (up)
    assert numerics.round_bf16(np.array([1.0 + 2.0 ** -8 + 2.0 ** -20]))[0] == 1.0 + 2.0 ** -7


def test_splitmix64_reference_vector():
    # Vigna's splitmix64.c reference output for seed 1234567
    assert numerics.splitmix64(1234567, 5) == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                                              4593380528125082431, 16408922859458223821]


# ---------------------------------------------------------------- c5: Hadamard
def test_c5_hadamard_worked_example():
    gd = golden("hadamard_worked_example.json")
    H = reparam.hadamard_U(4, None)
    assert np.array_equal(H, np.array(gd["H4_normalised"]))
    assert np.array_equal(np.array(gd["c"], float) @ H, np.array(gd["c_prime"], float))


@pytest.mark.parametrize("d", [1, 2, 4, 64, 512])
def test_c5_sylvester_equals_scipy(d):
    # P:274 names scipy.linalg.hadamard as the generator of the Sylvester matrix
    assert np.array_equal(reparam.sylvester(d), scipy.linalg.hadamard(d).astype(float))


def test_hadamard_orthonormal_with_signs():
    U = reparam.hadamard_U(64, 99)
    assert np.max(np.abs(U @ U.T - np.eye(64))) < 1e-14
    s = numerics.sign_vector(99, 64)
    assert set(np.unique(s)) <= {-1.0, 1.0} and 10 < np.sum(s > 0) < 54
    # D multiplies on the left: row i of U is s_i times row i of H/sqrt(d)
    assert np.array_equal(U, s[:, None] * scipy.linalg.hadamard(64) / 8.0)


# ---------------------------------------------------------------- c6: counterexample
def test_c6_hadamard_counterexample():
    gd = golden("hadamard_counterexample.json")
    H = reparam.hadamard_U(4, None)
    Qp = np.array(gd["Q"], float) @ H
    cp = np.array(gd["c"], float) @ H
    assert np.array_equal(Qp, np.array(gd["Q_prime"], float))
    assert np.array_equal(cp, np.array(gd["c_prime"], float))
    prod = Qp * cp
    # corrected arithmetic (the printed (200,..)/400 is garbled, reading R8); the sign pattern survives
    assert np.array_equal(prod, np.array(gd["product_corrected"], float))
    halves = [prod[:2].sum(), prod[2:].sum()]
    assert halves == gd["half_sums_corrected"]
    assert prod.sum() == gd["total"] == np.dot(gd["Q"], gd["c"])


# ---------------------------------------------------------------- c7: PCA constants
def test_c7_pca_alpha_from_eigenvalues():
    gd = golden("pca_constants.json")
    lam = np.array(gd["eigenvalues"], float)
    a = reparam.pca_alpha(lam, gd["g"])
    assert np.allclose(a, [10 / 7, 10 / 3], rtol=1e-15)
    assert np.allclose(a, gd["alpha"], rtol=1e-15)


def test_c7_pca_recovers_planted_basis():
    # features with exact second moment V diag(4,3,2,1) Vᵀ: rows ±sqrt(n λ_i/2) v_i
    V = synth.random_orthogonal(4, 5)
    lam = np.array([4.0, 3.0, 2.0, 1.0])
    rows = []
    for i in range(4):
        for sgn in (1, -1):
            rows.append(sgn * np.sqrt(8 * lam[i] / 2) * V[:, i])
    F = np.array(rows)
    U, lam_hat = reparam.pca(F)
    assert np.allclose(lam_hat, lam, rtol=1e-12)
    for i in range(4):
        assert abs(abs(U[:, i] @ V[:, i]) - 1) < 1e-12
    assert np.allclose(reparam.pca_alpha(lam_hat, 2), [10 / 7, 10 / 3], rtol=1e-12)


def test_pca_isotropic_alpha_is_g():
    lam = np.ones(64)
    for g in (1, 2, 4, 8):
        assert np.allclose(reparam.pca_alpha(lam, g), g)


# ---------------------------------------------------------------- Prop. 1
def test_prop1_rmsnorm_orthogonal_invariance():
    rng = np.random.default_rng(1)
    c = rng.standard_normal((9, 64)) * synth.latent_spectrum(64, 4)
    for U in (reparam.hadamard_U(64, 3), synth.random_orthogonal(64, 4)):
        lhs = numerics.rmsnorm(np.ones(64), c, 0.0)
        rhs = numerics.rmsnorm(np.ones(64), c @ U, 0.0) @ U.T
        assert np.max(np.abs(lhs - rhs)) < 1e-13
        # "when and only when W_gamma = I": a non-trivial gamma breaks it
        gam = 1 + 0.3 * rng.standard_normal(64)
        bad = numerics.rmsnorm(gam, c @ U, 0.0) @ U.T
        assert np.max(np.abs(numerics.rmsnorm(gam, c, 0.0) - bad)) > 1e-2


# ---------------------------------------------------------------- c2: absorbed == non-absorbed
@pytest.mark.parametrize("dims", DIMS, ids=lambda d: d.name)
def test_c2_absorbed_equals_full(dims):
    pb = make_problem(dims)
    a = mla_ref(pb, absorbed=True)
    f = mla_ref(pb, absorbed=False)
    assert rel(a, f) < 1e-12


def test_c2_brute_force_two_tokens():
    # h_q = 1, d_h = 1, d_c = 2, d_r = 2, S = 2: everything by hand
    c = np.array([[3.0, 4.0], [1.0, -1.0]])
    kpe = np.array([[0.5, 0.0], [0.0, 2.0]])
    q = np.array([[2.0]])
    qpe = np.array([[1.0, 1.0]])
    W_UK = np.array([[1.0], [2.0]])
    W_UV = np.array([[-1.0], [0.5]])
    gam = np.array([1.0, 2.0])
    W_O = np.array([[3.0, -1.0]])
    sc = 0.5
    chat = np.array([[3.0 / np.sqrt(12.5), 4.0 * 2 / np.sqrt(12.5)], [1.0, -2.0]])
    k = chat @ W_UK
    v = chat @ W_UV
    s0 = (2.0 * k[0, 0] + 0.5) * sc
    s1 = (2.0 * k[1, 0] + 2.0) * sc
    p0 = np.exp(s0) / (np.exp(s0) + np.exp(s1))
    o = p0 * v[0, 0] + (1 - p0) * v[1, 0]
    want = o * W_O[0]
    for f in (mla.mla_decode_full, mla.mla_decode_absorbed):
        got = f(q, qpe, c, kpe, W_UK, W_UV, gam, W_O, h_q=1, d_h=1, eps=0.0, sm_scale=sc)[0]
        assert np.allclose(got, want, rtol=1e-14, atol=0)


# ---------------------------------------------------------------- c1: g = 1 TPLA == MLA
@pytest.mark.parametrize("dims", DIMS, ids=lambda d: d.name)
@pytest.mark.parametrize("k", [1, 2])
def test_c1_g1_tpla_equals_mla(dims, k):
    pb = make_problem(dims, g=1)
    if dims.h_q % k:
        pytest.skip("heads not divisible")
    o = tpla.tpla_decode_step(pb, k=k, g=1)
    assert rel(o, mla_ref(pb, absorbed=True)) < 1e-13
    assert rel(o, mla_ref(pb, absorbed=False)) < 1e-12


# ---------------------------------------------------------------- c3: U invariance at g = 1
@pytest.mark.parametrize("dims", DIMS, ids=lambda d: d.name)
def test_c3_g1_invariant_under_U(dims):
    pb = make_problem(dims, g=1)
    base = tpla.tpla_decode_step(pb, 1, 1)
    feats = np.concatenate(pb.c_raw)
    U_pca, _ = reparam.pca(feats)
    for U in (reparam.hadamard_U(dims.d_c, 7), U_pca, synth.random_orthogonal(dims.d_c, 8)):
        pb.U = U
        assert rel(tpla.tpla_decode_step(pb, 1, 1), base) < 1e-12


def test_logit_invariance_under_U():
    # Q ĉᵀ = QU (ĉU)ᵀ  (Eq. absorb_softmax)
    rng = np.random.default_rng(2)
    Q = rng.standard_normal((5, 64))
    c = rng.standard_normal((7, 64))
    U = reparam.hadamard_U(64, 11)
    assert np.max(np.abs(Q @ c.T - (Q @ U) @ (c @ U).T)) < 1e-12


# ---------------------------------------------------------------- c4: per-shard softmax
@pytest.mark.parametrize("k,g", [(2, 2), (4, 2), (4, 4)])
def test_c4_shard_softmax_rows_and_rope(k, g):
    dims = synth.PRESETS["tiny"]
    pb = make_problem(dims, g=g, transform="hadamard")
    _, _, parts = tpla.tpla_decode_step(pb, k, g, return_parts=True)
    for pr in parts:
        for p in pr["P"]:
            assert np.max(np.abs(p.sum(axis=1) - 1)) < 1e-12
            assert np.all(p > 0)
    # RoPE logits identical on every device holding the same heads (k^PE replicated)
    by_block = {}
    for pr in parts:
        by_block.setdefault(pr["plan"].head_block, []).append(pr["rope_logits"])
    for lst in by_block.values():
        for other in lst[1:]:
            for a, b in zip(lst[0], other):
                assert np.array_equal(a, b)


# ---------------------------------------------------------------- c8: duplicated slices
def _dup_problem(dims, mu, g=2):
    """c' = [a ‖ a ‖ ... ‖ a] and W^UK / W^UV rows repeated the same way (g copies), gamma = 1:
    every slice carries 1/g of the energy, so alpha = g makes the sliced RMS the full RMS
    (Condition 1 with equality) and each shard's NoPE logit is 1/g of MLA's, which
    mu = g restores (Condition 2 with equality)."""
    pb = make_problem(dims, g=g, S=29)
    w = dims.d_c // g
    pb.gamma = np.ones(dims.d_c)
    for arr in (pb.W_UK, pb.W_UV):
        for j in range(1, g):
            arr[j * w:(j + 1) * w] = arr[:w]     # Q' = [b ‖ b ‖ ...]
    pb.c_raw = [np.concatenate([c[:, :w]] * g, axis=1) for c in pb.c_raw]   # c' = [a ‖ a ‖ ...]
    pb.mu = np.full(g, float(mu))
    pb.alpha = np.full(g, float(g))
    return pb


@pytest.mark.parametrize("dims", DIMS, ids=lambda d: d.name)
def test_c8_duplicated_halves_closed_form(dims):
    # Conditions 1 and 2 hold with equality => sliced TPLA == MLA, eps included
    pb = _dup_problem(dims, mu=2.0)
    o = tpla.tpla_decode_step(pb, 2, 2)
    assert rel(o, mla_ref(pb, absorbed=False)) < 1e-12
    # the literal-§4 reading mu = 1 (no logit scaling) does not reach MLA
    pb1 = _dup_problem(dims, mu=1.0)
    assert rel(tpla.tpla_decode_step(pb1, 2, 2), mla_ref(pb1)) > 1e-2


@pytest.mark.parametrize("g", [4, 8])
@pytest.mark.parametrize("k_per_g", [1, 2])
def test_c8_duplicated_slices_g4_g8(g, k_per_g):
    """The alpha = g sliced-RMS / mu = alpha chain at g > 2 (configs C2, C3, the 8-GPU headline):
    with g duplicated slices TPLA(k, g) equals MLA exactly (eps included); with mu = 1 each shard's
    NoPE logits are 1/g too small and the output is O(1) off."""
    dims = synth.PRESETS["odd"] if g == 4 else synth.PRESETS["tiny"]
    if dims.h_q % k_per_g:
        pytest.skip("heads do not split")
    k = g * k_per_g
    pb = _dup_problem(dims, mu=float(g), g=g)
    assert rel(tpla.tpla_decode_step(pb, k, g), mla_ref(pb, absorbed=False)) < 1e-12
    pb1 = _dup_problem(dims, mu=1.0, g=g)
    assert rel(tpla.tpla_decode_step(pb1, k, g), mla_ref(pb1)) > 1e-2


# ---------------------------------------------------------------- shard_attention's lse
def test_lse_two_token_hand_case():
    """Logits (0, ln 3) by construction (one head, one latent, no RoPE, scale 1):
    lse = ln(1 + 3) = ln 4, p = (1/4, 3/4), O = 3/4 · 1 (hand-computed)."""
    Qp = np.array([[np.log(3.0)]])
    rows = np.array([[0.0], [1.0]])                       # ĉ_0 = 0, ĉ_1 = 1; d_r = 0
    O, lse, p, _ = tpla.shard_attention(Qp, np.zeros((1, 0)), rows, 1, 1.0)
    assert lse[0] == pytest.approx(np.log(4.0), rel=1e-15)
    assert np.allclose(p[0], [0.25, 0.75], rtol=1e-15, atol=0)
    assert O[0, 0] == pytest.approx(0.75, rel=1e-15)


@pytest.mark.parametrize("S", [1, 7, 4096])
def test_lse_uniform_logits_is_log_S(S):
    """All logits equal to c (q = 0 and q^PE = 0 give c = 0; a constant RoPE logit shifts it):
    lse = c + ln S, p = 1/S, O = the mean row."""
    rng = np.random.default_rng(S)
    H, W_lat, d_r = 3, 8, 4
    rows = np.concatenate([rng.standard_normal((S, W_lat)), np.ones((S, d_r))], axis=1)
    qpe = np.zeros((H, d_r))
    qpe[1] = 0.5                                          # head 1: RoPE logit 4 * 0.5 = 2 on every token
    O, lse, p, _ = tpla.shard_attention(np.zeros((H, W_lat)), qpe, rows, W_lat, 1.0)
    assert np.allclose(lse, [np.log(S), 2.0 + np.log(S), np.log(S)], rtol=1e-14, atol=1e-14)
    assert np.allclose(p, 1.0 / S, rtol=1e-12, atol=0)
    assert np.allclose(O, rows[:, :W_lat].mean(axis=0)[None, :], rtol=1e-10, atol=1e-12)


def test_lse_shift_and_large_logits():
    """lse(s + c) = lse(s) + c, finite for logits near 700 where exp overflows (the stable form)."""
    rng = np.random.default_rng(5)
    rows = rng.standard_normal((50, 4))
    Qp = rng.standard_normal((2, 4))
    _, l0, _, _ = tpla.shard_attention(Qp, np.zeros((2, 0)), rows, 4, 1.0)
    rows_c = np.concatenate([rows, np.full((50, 1), 1.0)], axis=1)
    _, l1, _, _ = tpla.shard_attention(Qp, np.full((2, 1), 700.0), rows_c, 4, 1.0)
    assert np.all(np.isfinite(l1))
    assert np.allclose(l1 - l0, 700.0, rtol=1e-14, atol=1e-9)


# ---------------------------------------------------------------- c9: degenerate softmax
@pytest.mark.parametrize("mu", [1.0, 2.0, 3.7])
def test_c9_single_token_exact_rms(mu):
    dims = synth.PRESETS["odd"]
    pb = make_problem(dims, g=2, S=1, mu=[mu, mu], modes="exact", transform="hadamard")
    assert rel(tpla.tpla_decode_step(pb, 2, 2), mla_ref(pb)) < 1e-12


def test_c9_uniform_logits_exact_rms():
    dims = synth.PRESETS["tiny"]
    pb = make_problem(dims, g=2, S=23, modes="exact", transform="hadamard")
    pb.q_nope[:] = 0
    pb.q_pe[:] = 0
    assert rel(tpla.tpla_decode_step(pb, 2, 2), mla_ref(pb)) < 1e-12


# ---------------------------------------------------------------- c10: exact logits
@pytest.mark.parametrize("g", [2, 4])
def test_c10_exact_logits_exact_rms_is_mla(g):
    dims = synth.PRESETS["odd"]
    pb = make_problem(dims, g=g, modes="exact", transform="hadamard")
    assert rel(tpla.tpla_decode_exact_logits(pb, g), mla_ref(pb)) < 1e-12


def test_sliced_tpla_differs_from_mla_generically():
    # TPLA is an approximation: generic inputs do NOT give MLA
    dims = synth.PRESETS["tiny"]
    pb = make_problem(dims, g=2, transform="hadamard")
    assert rel(tpla.tpla_decode_step(pb, 2, 2), mla_ref(pb)) > 1e-3


# ---------------------------------------------------------------- exactness of the head split
@pytest.mark.parametrize("g,ks", [(2, [2, 4]), (1, [1, 2])])
def test_head_split_is_exact(g, ks):
    # splitting heads within a latent group is a plain row-parallel decomposition
    dims = synth.PRESETS["tiny"]
    pb = make_problem(dims, g=g, transform="hadamard")
    outs = [tpla.tpla_decode_step(pb, k, g) for k in ks]
    assert rel(outs[1], outs[0]) < 1e-13


def test_row_parallel_identity():
    rng = np.random.default_rng(4)
    X, A = rng.standard_normal((3, 8)), rng.standard_normal((8, 5))
    assert np.max(np.abs(X @ A - (X[:, :4] @ A[:4] + X[:, 4:] @ A[4:]))) < 1e-13


# ---------------------------------------------------------------- cache rows (K1 oracle)
def test_cache_rows_worked_example():
    # c = (100,0,0,0), H_4/2: c' = (50,50,50,50); sliced RMS of device 0 with alpha = 2:
    # sqrt(2/4 * 5000) = 50, the exact RMS is also 50 (Condition 1 with equality)
    pl = plan.make_plan(2, 2, 4, 4, 2, 0)
    U = reparam.hadamard_U(4, None)
    for mode in (tpla.SLICED, tpla.EXACT):
        r = tpla.cache_rows(np.array([[100.0, 0, 0, 0]]), np.array([[0.25, -0.5]]), U, pl, 2.0, 0.0, mode)
        assert np.array_equal(r, np.array([[1.0, 1.0, 0.25, -0.5]]))
    r = tpla.cache_rows(np.array([[3.0, 4.0, 0, 0]]), np.zeros((1, 2)), np.eye(4), pl, 2.0, 0.0, tpla.SLICED)
    assert np.allclose(r[0, :2], np.array([3.0, 4.0]) / np.sqrt(2 / 4 * 25), rtol=1e-15)
    r = tpla.cache_rows(np.array([[3.0, 4.0, 0, 0]]), np.zeros((1, 2)), np.eye(4), pl, 2.0, 0.0, tpla.EXACT)
    assert np.allclose(r[0, :2], np.array([3.0, 4.0]) / np.sqrt(25 / 4), rtol=1e-15)


def test_hadamard_balances_slice_energy():
    # Condition 1 holds better after Hadamard on outlier-heavy latents
    dims = synth.PRESETS["dsv3"]
    c = f64(synth.gen_raw_ckv(dims, 256, 1, 0))
    U = reparam.hadamard_U(512, 5)

    def imbalance(x):
        e0 = np.sum(x[:, :256] ** 2, 1)
        e1 = np.sum(x[:, 256:] ** 2, 1)
        return np.mean(np.abs(e0 - e1) / (e0 + e1))
    assert imbalance(c @ U) < 0.5 * imbalance(c)


def test_pca_beats_identity_on_planted_basis():
    # PCA puts the leading energy in shard 0 and calibrates alpha; on latents drawn
    # in a rotated power-law basis, sliced RMS with PCA alpha is closer to the true RMS than
    # identity slicing with alpha = g
    dims = synth.PRESETS["tiny"]
    V = synth.random_orthogonal(dims.d_c, 3)
    c = f64(synth.gen_raw_ckv(dims, 400, 1, 0, basis=V))
    U, lam = reparam.pca(c)
    a = reparam.pca_alpha(lam, 2)
    true_r = numerics.rms(c, 0.0)

    def err(Ux, al):
        x = c @ Ux
        r0 = np.sqrt(al / dims.d_c * np.sum(x[:, :32] ** 2, 1))
        return np.median(np.abs(r0 / true_r - 1))
    assert err(U, a[0]) < err(np.eye(dims.d_c), 2.0)


# ---------------------------------------------------------------- c12-c14: integer facts
def test_c12_kv_widths():
    gd = golden("kv_dims.json")
    assert cost.kv_width_mla(512, 64) == gd["mla_width"]
    for g, w in gd["tpla_width"].items():
        assert cost.kv_width_tpla(512, 64, int(g)) == w
    for g, ratio in gd["byte_ratio_vs_mla"].items():
        assert cost.kv_width_mla(512, 64) / cost.kv_width_tpla(512, 64, int(g)) == ratio
    assert cost.kv_width_gqa(8, 128, 1) == gd["gqa_llama3_70b"]["total"]
    assert cost.kv_width_gqa(8, 128, 4) == gd["gqa_llama3_70b"]["tp4"]
    # latent part falls exactly g-fold
    for g in (1, 2, 4, 8):
        assert (cost.kv_width_tpla(512, 64, g) - 64) * g == 512


def test_c13_nope_flops_equal():
    # "These two complexities are arithmetically equivalent", exhaustively on a grid
    for h_q in (16, 64, 128):
        for d_h in (16, 64, 128):
            for S in (1, 4096, 32768):
                assert cost.nope_flops_tpla(1, S, h_q, d_h, 2) == cost.nope_flops_mla(1, S, h_q, d_h, 2)


def test_c14_plan_examples():
    gd = golden("plan_examples.json")
    for case in gd["cases"]:
        for row in case["ranks"]:
            p = plan.make_plan(case["k"], case["g"], case["h_q"], case["d_c"], case["d_r"], row[0])
            assert [p.rank, p.shard, p.head_block, p.head_begin, p.head_end, p.lat_begin, p.lat_end,
                    p.row_width] == row


def test_plan_partitions_exactly_once():
    for k, g in [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (8, 2), (8, 8)]:
        plans = plan.all_plans(k, g, 128, 512, 64)
        for j in range(g):
            heads = sorted(h for p in plans if p.shard == j for h in range(p.head_begin, p.head_end))
            assert heads == list(range(128))
        lat = sorted({(p.lat_begin, p.lat_end) for p in plans})
        assert [x for a, b in lat for x in range(a, b)] == list(range(512))


@pytest.mark.parametrize("bad", [(3, 2), (4, 3), (2, 4)])
def test_plan_rejects_indivisible(bad):
    with pytest.raises(ValueError):
        plan.make_plan(bad[0], bad[1], 128, 512, 64, 0)


# ---------------------------------------------------------------- c11: TPLA == GLA with 2 h_q heads
@pytest.mark.parametrize("g", [2, 4])
def test_c11_tpla_is_gla_with_duplicated_heads(g):
    """TPLA(k = g) is algebraically a GLA system whose heads are g copies of the
    original heads (Q' stacks Q g times; every copy keeps its W^UK / W^UV / W^O): GLA device i
    pairs head copy i with latent shard i — exactly TPLA's device i (all heads, shard i)."""
    dims = synth.PRESETS["odd"] if g == 2 else synth.PRESETS["tiny"]
    pb = make_problem(dims, g=g, transform="hadamard", mu=[1.0] * g)
    dup = tpla.Problem(W_UK=np.concatenate([pb.W_UK] * g, axis=1), W_UV=np.concatenate([pb.W_UV] * g, axis=1),
                       gamma=pb.gamma, W_O=np.concatenate([pb.W_O] * g, axis=0), U=pb.U, alpha=pb.alpha,
                       mu=pb.mu, c_raw=pb.c_raw, k_pe=pb.k_pe, modes=pb.modes,
                       q_nope=np.concatenate([pb.q_nope] * g, axis=1), q_pe=np.concatenate([pb.q_pe] * g, axis=1),
                       h_q=g * pb.h_q, d_h=pb.d_h, eps=pb.eps, sm_scale=pb.sm_scale)
    assert rel(tpla.gla_decode_step(dup, g), tpla.tpla_decode_step(pb, g, g)) < 1e-12


def test_gla_drops_the_off_diagonal_blocks():
    """GLA is not MLA: with the cross blocks Q_{0,1}, Q_{1,0} dropped the output is O(1)
    off ("significant performance degradation"); but on a model whose heads block i lives
    only in latent shard i (W^UK / W^UV zero outside the diagonal blocks, the GLA architecture
    itself) with per-shard exact RMS rows it is exactly that model's attention (softmax over a
    block's own shard = softmax over the full latent, whose other shard contributes nothing)."""
    dims = synth.PRESETS["odd"]
    g = 2
    pb = make_problem(dims, g=g, modes="sliced")
    assert rel(tpla.gla_decode_step(pb, g), mla_ref(pb)) > 1e-1
    # block-diagonal model: heads block i only reads latent shard i
    w = dims.d_c // g
    hb = dims.h_q // g
    for arr in (pb.W_UK, pb.W_UV):
        for i in range(g):
            for j in range(g):
                if i != j:
                    arr[j * w:(j + 1) * w, i * hb * dims.d_h:(i + 1) * hb * dims.d_h] = 0.0
    pb.gamma = np.ones(dims.d_c)
    # per-head reference: head h in block i attends over RMSNorm(shard i) with its own W^UK rows
    out = np.zeros((len(pb.c_raw), pb.W_O.shape[1]))
    for b in range(len(pb.c_raw)):
        for i in range(g):
            c_i = pb.c_raw[b][:, i * w:(i + 1) * w]
            chat = c_i / np.sqrt(np.sum(c_i * c_i, axis=1) / w + pb.eps)[:, None]
            for h in range(i * hb, (i + 1) * hb):
                cols = slice(h * dims.d_h, (h + 1) * dims.d_h)
                k = chat @ pb.W_UK[i * w:(i + 1) * w, cols]
                v = chat @ pb.W_UV[i * w:(i + 1) * w, cols]
                s = (k @ pb.q_nope[b, h] + pb.k_pe[b] @ pb.q_pe[b, h]) * pb.sm_scale
                p = np.exp(s - s.max())
                p /= p.sum()
                out[b] += (p @ v) @ pb.W_O[cols]
    assert rel(tpla.gla_decode_step(pb, g), out) < 1e-12
