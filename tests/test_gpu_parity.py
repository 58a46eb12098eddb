"""GPU parity: libtpla.so (through the C-ABI) against the fp64 oracle on the same seeded bf16 inputs.

Tolerances: integer layout bit-exact; cache rows within 1 bf16 ulp;
attention / end-to-end outputs per row ‖gpu − ref‖_∞ / ‖ref‖_∞ ≤ 1e-2 (reading R18, the
north-star bound), also reported as relative L2.
"""
import numpy as np
import pytest

import synth
from oracle import mla, numerics, plan as oplan, reparam, tpla

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2508_15881_b200 import _abi as abi
    from paper_2508_15881_b200.runtime import LayerSpec, TplaRank, bf16_from_bits, bits_from_bf16

TOL = 1e-2


def f64(b):
    return numerics.bf16_to_f64(b)


def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda:0")


def row_rel_err(got, ref):
    got = np.asarray(got, np.float64).reshape(ref.shape[0], -1)
    ref = np.asarray(ref, np.float64).reshape(ref.shape[0], -1)
    return np.max(np.max(np.abs(got - ref), axis=1) / np.max(np.abs(ref), axis=1))


def spec_of(d: synth.ModelDims):
    return LayerSpec(d.h_q, d.d_c, d.d_r, d.d_h, d.D)


def transform_inputs(kind, dims, seed, g):
    """(xform id, sign seed, U fp64, U_pca fp32 host or None, alpha[g])."""
    if kind == "identity":
        return abi.XFORM_IDENTITY, 0, np.eye(dims.d_c), None, np.full(g, float(g))
    if kind == "hadamard":
        return abi.XFORM_HADAMARD, seed, reparam.hadamard_U(dims.d_c, seed), None, np.full(g, float(g))
    # PCA basis planted by the generator (population eigenvectors V, eigenvalues sigma^2)
    V = synth.random_orthogonal(dims.d_c, seed)
    lam = synth.latent_spectrum(dims.d_c, dims.n_outlier) ** 2
    order = np.argsort(-lam, kind="stable")
    U = V[:, order]
    U32 = U.astype(np.float32)
    return abi.XFORM_PCA, 0, U32.astype(np.float64), U32, abi.tpla_pca_alpha(lam[order], g).astype(np.float64)


def upload_rows(rank, b, rows_bits):
    """Write [S, W] bf16 rows of sequence b into the paged cache (test setup)."""
    S, W = rows_bits.shape
    img = torch.from_numpy(rows_bits.view(np.int16)).view(torch.bfloat16).to(rank.cache_buf.device)
    for t0 in range(0, S, rank.page_size):
        page = int(rank.block_table_host[b, t0 // rank.page_size])
        n = min(rank.page_size, S - t0)
        rank.cache_buf[page, :n, :W] = img[t0:t0 + n]


# ----------------------------------------------------------------------------- K1 layout
@pytest.mark.parametrize("dname", ["tiny", "dsv3"])
def test_append_layout_bit_exact(dname):
    """identity + RMS_NONE: the cache image is a byte copy of (c_j ‖ k_pe) at the paged address."""
    d = dev()
    dims = synth.PRESETS[dname]
    k = g = 2
    B, S = 3, 150
    for rank_id in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rank_id, batch=B, max_seq_len=256, device=d, page_perm_seed=7,
                     extra_pages=3)
        w = synth.gen_weights(dims, 1)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_IDENTITY)
        rng = np.random.default_rng(3)
        seq = np.repeat(np.arange(B), S).astype(np.int32)
        pos = np.tile(np.arange(S), B).astype(np.int32)
        perm = rng.permutation(seq.size)                     # arbitrary append order
        ckv = np.concatenate([synth.gen_raw_ckv(dims, S, 5, b) for b in range(B)])
        kpe = np.concatenate([synth.gen_kpe(dims, S, 5, b) for b in range(B)])
        r.append(bf16_from_bits(ckv[perm], d), bf16_from_bits(kpe[perm], d),
                 torch.from_numpy(seq[perm]).to(d), torch.from_numpy(pos[perm]).to(d), abi.RMS_NONE)
        torch.cuda.synchronize()
        pl = oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, rank_id)
        expect = np.zeros_like(bits_from_bf16(r.cache_buf))
        for b in range(B):
            for t in range(S):
                page = r.block_table_host[b, t // r.page_size]
                expect[page, t % r.page_size, :pl.w_lat] = ckv[b * S + t, pl.lat_begin:pl.lat_end]
                expect[page, t % r.page_size, pl.w_lat:pl.row_width] = kpe[b * S + t]
        assert np.array_equal(bits_from_bf16(r.cache_buf), expect)


def test_append_drops_out_of_range():
    d = dev()
    dims = synth.PRESETS["tiny"]
    r = TplaRank(spec_of(dims), k=2, g=2, rank=0, batch=2, max_seq_len=64, device=d)
    w = synth.gen_weights(dims, 1)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_IDENTITY)
    ckv = bf16_from_bits(synth.gen_raw_ckv(dims, 4, 1, 0), d)
    kpe = bf16_from_bits(synth.gen_kpe(dims, 4, 1, 0), d)
    seq = torch.tensor([0, 5, -1, 1], dtype=torch.int32, device=d)
    pos = torch.tensor([0, 0, 0, 64], dtype=torch.int32, device=d)
    nd = torch.zeros(1, dtype=torch.int32, device=d)
    r.append(ckv, kpe, seq, pos, abi.RMS_SLICED, n_dropped=nd)
    torch.cuda.synchronize()
    assert int(nd.item()) == 3
    img = bits_from_bf16(r.cache_buf)
    assert np.count_nonzero(img) > 0 and np.count_nonzero(img[r.block_table_host[1]]) == 0


# ----------------------------------------------------------------------------- K1 values
@pytest.mark.parametrize("dname", ["tiny", "odd", "dsv3"])
@pytest.mark.parametrize("kind", ["identity", "hadamard", "pca"])
@pytest.mark.parametrize("mode", ["sliced", "exact"])
@pytest.mark.parametrize("g", [2, 4])
def test_append_rows_match_oracle(dname, kind, mode, g):
    d = dev()
    dims = synth.PRESETS[dname]
    k = g
    xf, seed, U, U32, alpha = transform_inputs(kind, dims, 11, g)
    basis = U if kind == "pca" else None
    n = 70
    ckv = synth.gen_raw_ckv(dims, n, 9, 0, basis=basis)
    kpe = synth.gen_kpe(dims, n, 9, 0)
    w = synth.gen_weights(dims, 2)
    for rank_id in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rank_id, batch=1, max_seq_len=128, device=d)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=seed, U_pca=U32, alpha=alpha)
        mode_id = abi.RMS_SLICED if mode == "sliced" else abi.RMS_EXACT
        r.append(bf16_from_bits(ckv, d), bf16_from_bits(kpe, d), torch.zeros(n, dtype=torch.int32, device=d),
                 torch.arange(n, dtype=torch.int32, device=d), mode_id)
        torch.cuda.synchronize()
        pl = oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, rank_id)
        ref = tpla.cache_rows(f64(ckv), f64(kpe), U, pl, alpha[pl.shard], 1e-6, mode)
        got = f64(r.cache_rows_bits(0, n)[:, :pl.row_width])
        # within one bf16 ulp of the fp64 value (fp32 arithmetic on the GPU, RNE store)
        ulp = np.abs(numerics.round_bf16(ref)) * 2.0 ** -7
        assert np.all(np.abs(got - ref) <= ulp + 1e-30), np.max(np.abs(got - ref) / (ulp + 1e-30))


# ----------------------------------------------------------------------------- K3+K4
def attention_case(d, dims, g, B, S_list, seed=0, peak=1.0, needle=False, page_perm=None, stale=False, page_size=64):
    k = g
    r = TplaRank(spec_of(dims), k=k, g=g, rank=g - 1, batch=B, max_seq_len=max(S_list), device=d,
                 page_perm_seed=page_perm, page_size=page_size)
    if stale:   # finite junk in every row past the lengths: must be masked, never reach O
        r.cache_buf.copy_(torch.randn(r.cache_buf.shape, generator=torch.Generator(device=d).manual_seed(seed),
                                      device=d).mul_(300.0).to(torch.bfloat16))
    pl = oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, g - 1)
    rng = np.random.default_rng(seed)
    rows = []
    for b, S in enumerate(S_list):
        rb = synth.bf16_bits(rng.standard_normal((S, pl.row_width)).astype(np.float32))
        rows.append(rb)
        upload_rows(r, b, rb)
    q_lat = rng.standard_normal((B, pl.h_loc, pl.w_lat)).astype(np.float32) * peak
    if needle:
        q_lat *= 0.2
    q_lat_b = synth.bf16_bits(q_lat)
    qpe_b = synth.bf16_bits(rng.standard_normal((B, dims.h_q, dims.d_r)).astype(np.float32) * peak)
    if needle:   # a few very large logits late in the sequence: exercises the running-max rescale
        for b, S in enumerate(S_list):
            t = S - 1 - rng.integers(0, max(1, S // 8))
            rows[b][t, :pl.w_lat] = synth.bf16_bits(np.sign(f64(q_lat_b[b, 0])) * 4.0)
            upload_rows(r, b, rows[b])
    O = torch.zeros((B, pl.h_loc, pl.w_lat), dtype=torch.float32, device=d)
    lse = torch.zeros((B, pl.h_loc), dtype=torch.float32, device=d)
    r.decode_attention(bf16_from_bits(q_lat_b, d), bf16_from_bits(qpe_b, d),
                       torch.tensor(S_list, dtype=torch.int32, device=d), O, lse)
    torch.cuda.synchronize()
    heads = slice(pl.head_begin, pl.head_end)
    for b, S in enumerate(S_list):
        Oref, lref, _, _ = tpla.shard_attention(f64(q_lat_b[b]), f64(qpe_b[b, heads]), f64(rows[b]), pl.w_lat,
                                                 dims_scale(dims))
        e = row_rel_err(O[b].cpu().numpy(), Oref)
        assert e <= TOL, (b, S, e)
        assert np.max(np.abs(lse[b].cpu().numpy() - lref)) < 1e-2 * max(1.0, np.max(np.abs(lref)))


def dims_scale(dims):
    return 1.0 / np.sqrt(dims.d_h + dims.d_r)


@pytest.mark.parametrize("dname,g", [("tiny", 2), ("odd", 2), ("dsv3", 1), ("dsv3", 2), ("dsv3", 4), ("dsv3", 8),
                                     ("kimi", 1), ("kimi", 4)])
def test_attention_parity_small(dname, g):
    d = dev()
    attention_case(d, synth.PRESETS[dname], g, 3, [1, 77, 300], page_perm=3)


def test_attention_parity_edge_lengths():
    d = dev()
    attention_case(d, synth.PRESETS["dsv3"], 2, 6, [1, 63, 64, 65, 128, 129], seed=1, stale=True)
    attention_case(d, synth.PRESETS["dsv3"], 2, 2, [4097, 2000], seed=2, needle=True)
    attention_case(d, synth.PRESETS["dsv3"], 8, 2, [1500, 3], seed=4, peak=3.0)
    # g = 1 (plain MLA, CTA pairs exchanging partial logits): ragged, needle, stale rows
    attention_case(d, synth.PRESETS["dsv3"], 1, 6, [1, 63, 64, 65, 129, 700], seed=12, stale=True)
    attention_case(d, synth.PRESETS["dsv3"], 1, 2, [2500, 90], seed=13, needle=True)
    # 128-token tiles (W_lat <= 128): ragged lengths around the 64-row box and 128-row tile edges
    attention_case(d, synth.PRESETS["dsv3"], 8, 9, [1, 63, 64, 65, 127, 128, 129, 192, 255], seed=7, stale=True)
    attention_case(d, synth.PRESETS["dsv3"], 4, 5, [64, 65, 191, 193, 256], seed=8, page_perm=5)
    # 64 heads per device: TMEM lane quadrants 2-3 hold no head rows
    attention_case(d, synth.PRESETS["kimi"], 4, 4, [1, 64, 129, 640], seed=9)


@pytest.mark.parametrize("page_size", [128, 256])
def test_attention_parity_page_sizes(page_size):
    """Pages larger than the 64-row TMA box: boxes are looked up individually (64- and 128-token tiles)."""
    d = dev()
    for g in (2, 8):
        attention_case(d, synth.PRESETS["dsv3"], g, 4, [63, 129, 300, 513], seed=10 + g, page_perm=page_size,
                       page_size=page_size, stale=True)


def test_attention_parity_divergent_rescale():
    """Large logit spread over many sequences: the running max of different heads (TMEM lanes of
    one warp) is raised at different tiles, so O rescales are per-row and warp-divergent."""
    d = dev()
    attention_case(d, synth.PRESETS["dsv3"], 2, 32, [2048] * 31 + [777], seed=5, peak=2.5)
    attention_case(d, synth.PRESETS["dsv3"], 4, 16, [1000 + 37 * b for b in range(16)], seed=6, peak=3.0)


# ----------------------------------------------------------------------------- end to end (K1..K5)
def e2e_case(d, dims, k, g, kind, S_list, *, seed=0, modes=("exact", "sliced"), check_rank_parts=True, wo="rank",
             mu=None):
    """All k ranks of a (k, g) plan run on this GPU, each accumulating into y (k-shard emulation);
    compared with the oracle's full step (sum over ranks).
    wo: "rank"   every rank projects its own v_j through W^O (tpla_decode);
        "shared" the g ranks of a head block add their v_j into one v_acc, projected once (f2(ii));
        "split"  as if each rank of a group were its own process: v_acc in g column chunks per rank,
                 the group sum formed here (the reduce-scatter's arithmetic), each rank projecting
                 its chunk's K-slice of W^O.
    mu: None = mu_j = alpha_j (reading R6), else a scalar for every shard (1.0: the literal §4 reading)."""
    B = len(S_list)
    xf, sseed, U, U32, alpha = transform_inputs(kind, dims, 21, g)
    mu = np.asarray(alpha, float) if mu is None else np.full(g, float(mu))
    basis = U if kind == "pca" else None
    w = synth.gen_weights(dims, seed + 1)
    q, qpe = synth.gen_queries(dims, B, seed + 2)
    # prompt rows (EXACT, PD-separated prefill P:421) then decode rows (SLICED) appended one by one
    n_prompt = [max(1, S - 3) for S in S_list]
    c_raw = [synth.gen_raw_ckv(dims, S, seed + 3, b, basis=basis) for b, S in enumerate(S_list)]
    k_pe = [synth.gen_kpe(dims, S, seed + 3, b) for b, S in enumerate(S_list)]
    y = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    ranks = []
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=max(S_list), device=d,
                     page_perm_seed=rid)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=sseed, U_pca=U32, alpha=alpha, mu=mu)
        seq = np.concatenate([np.full(n, b, np.int32) for b, n in enumerate(n_prompt)])
        pos = np.concatenate([np.arange(n, dtype=np.int32) for n in n_prompt])
        ck = np.concatenate([c_raw[b][:n] for b, n in enumerate(n_prompt)])
        kp = np.concatenate([k_pe[b][:n] for b, n in enumerate(n_prompt)])
        r.prefill(bf16_from_bits(ck, d), bf16_from_bits(kp, d), torch.from_numpy(seq).to(d),
                  torch.from_numpy(pos).to(d))
        for step in range(3):
            sel = [b for b, S in enumerate(S_list) if n_prompt[b] + step < S]
            if not sel:
                continue
            ck = np.stack([c_raw[b][n_prompt[b] + step] for b in sel])
            kp = np.stack([k_pe[b][n_prompt[b] + step] for b in sel])
            r.append(bf16_from_bits(ck, d), bf16_from_bits(kp, d), torch.tensor(sel, dtype=torch.int32, device=d),
                     torch.tensor([n_prompt[b] + step for b in sel], dtype=torch.int32, device=d), abi.RMS_SLICED)
        if wo == "rank":
            r.decode(bf16_from_bits(q, d), bf16_from_bits(qpe, d), torch.tensor(S_list, dtype=torch.int32, device=d),
                     y, accumulate=True)
        ranks.append(r)
    if wo != "rank":
        lens = torch.tensor(S_list, dtype=torch.int32, device=d)
        n_ch = 1 if wo == "shared" else g
        blocks = sorted({r.plan.head_block for r in ranks})
        for hb in blocks:
            grp = [r for r in ranks if r.plan.head_block == hb]
            assert len(grp) == g
            accs = [torch.full(grp[0].v_acc_shape(B, n_ch), float("nan"), device=d) for _ in range(len(grp))]
            for j, r in enumerate(grp):
                if wo == "shared":     # co-located: one accumulator for the group
                    r.decode_v(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, accs[0], accumulate=j > 0)
                else:
                    r.decode_v(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, accs[j], n_chunks=n_ch)
            if wo == "shared":
                grp[0].project_out(accs[0], y, accumulate=True)
            else:
                tot = torch.stack(accs).sum(0)
                for j, r in enumerate(grp):
                    a = torch.full_like(tot, float("nan"))   # only chunk j is read by rank j
                    a[j] = tot[j]
                    r.project_out(a, y, chunk=j, accumulate=True)
    out = torch.empty((B, dims.D), dtype=torch.bfloat16, device=d)
    abi.tpla_sync(0)
    torch.cuda.synchronize()
    pb = tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O), U=U,
                      alpha=np.asarray(alpha, float), mu=mu,
                      c_raw=[f64(c) for c in c_raw], k_pe=[f64(x) for x in k_pe],
                      modes=[[tpla.EXACT] * n + [tpla.SLICED] * (S - n) for S, n in zip(S_list, n_prompt)],
                      q_nope=f64(q), q_pe=f64(qpe), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                      sm_scale=dims_scale(dims))
    # the latent cache is bf16 by specification (north_star): the oracle stores its fp64 rows
    # rounded to bf16 too (reading R19) — with PCA's large alpha_1/mu_1 (~34 here) that storage
    # rounding alone moves the output by ~1e-2, so it must be on both sides of the comparison
    ref = tpla.tpla_decode_step(pb, k, g, round_rows=numerics.round_bf16)
    got = y.cpu().numpy()
    e = row_rel_err(got, ref)
    l2 = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert e <= TOL, (e, l2)
    return e, l2


@pytest.mark.parametrize("dname", ["tiny", "odd"])
@pytest.mark.parametrize("k,g", [(2, 2), (4, 2), (4, 4), (2, 1)])
@pytest.mark.parametrize("kind", ["identity", "hadamard", "pca"])
def test_e2e_parity_tiny(dname, k, g, kind):
    dims = synth.PRESETS[dname]
    if dims.h_q % (k // g) or (dims.d_c // g) % 32:
        pytest.skip("shape outside the plan / kernels")
    e2e_case(dev(), dims, k, g, kind, [1, 77, 130])


@pytest.mark.parametrize("k,g,kind", [(2, 2, "hadamard"), (2, 2, "pca"), (4, 4, "hadamard"), (8, 8, "hadamard"),
                                      (4, 2, "identity"), (8, 2, "hadamard"), (1, 1, "identity"), (2, 1, "hadamard")])
def test_e2e_parity_dsv3_shape(k, g, kind):
    e2e_case(dev(), synth.PRESETS["dsv3"], k, g, kind, [5, 200, 333])


def test_e2e_parity_kimi_shape():
    e2e_case(dev(), synth.PRESETS["kimi"], 4, 4, "hadamard", [64, 129])


@pytest.mark.parametrize("dname,k,g,kind", [("dsv3", 2, 2, "hadamard"), ("dsv3", 4, 2, "pca"), ("dsv3", 8, 8, "hadamard"),
                                            ("kimi", 8, 4, "hadamard"), ("dsv3", 8, 2, "identity")])
@pytest.mark.parametrize("wo", ["shared", "split"])
def test_e2e_parity_group_shared_wo(dname, k, g, kind, wo):
    """the latent group sums v before one W^O product (co-located or reduce-scattered)."""
    e2e_case(dev(), synth.PRESETS[dname], k, g, kind, [5, 200, 333], wo=wo)


def test_project_out_rejects_bad_chunking():
    d = dev()
    dims = synth.PRESETS["dsv3"]
    r = TplaRank(spec_of(dims), k=8, g=8, rank=0, batch=2, max_seq_len=64, device=d)
    w = synth.gen_weights(dims, 1)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD)
    y = torch.zeros((2, dims.D), dtype=torch.float32, device=d)
    v = torch.zeros((3, 2, dims.h_q * dims.d_h // 3 + 1), dtype=torch.float32, device=d)
    with pytest.raises(abi.TplaError) as ei:            # 3 chunks of 64-multiples do not tile K = 16384
        r.project_out(v, y, chunk=0)
    assert ei.value.status == abi.ERR_DIVISIBILITY
    v = torch.zeros(r.v_acc_shape(2, 2), dtype=torch.float32, device=d)
    with pytest.raises(abi.TplaError) as ei:
        r.project_out(v, y, chunk=2)
    assert ei.value.status == abi.ERR_INVALID_ARG


def mtp_case(d, dims, k, g, n_q, S_list, *, seed=0, kind="hadamard"):
    """Multi-token decode: the n_q newest tokens of each sequence are decoded in one
    step.  Pinned against the oracle's single-token step over each token's causal prefix: token i
    of sequence b sees the first S_b - n_q + 1 + i rows (P:137-141 per token)."""
    B = len(S_list)
    xf, sseed, U, U32, alpha = transform_inputs(kind, dims, 31, g)
    basis = U if kind == "pca" else None
    w = synth.gen_weights(dims, seed + 1)
    qb, qpeb = synth.gen_queries(dims, B * n_q, seed + 2)
    qb = qb.reshape(B, n_q, dims.h_q, dims.d_h)
    qpeb = qpeb.reshape(B, n_q, dims.h_q, dims.d_r)
    c_raw = [synth.gen_raw_ckv(dims, S, seed + 3, b, basis=basis) for b, S in enumerate(S_list)]
    k_pe = [synth.gen_kpe(dims, S, seed + 3, b) for b, S in enumerate(S_list)]
    n_prompt = [S - n_q for S in S_list]
    y = torch.zeros((B * n_q, dims.D), dtype=torch.float32, device=d)
    out = torch.empty((B * n_q, dims.D), dtype=torch.bfloat16, device=d)
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=max(S_list), device=d, n_q=n_q,
                     page_perm_seed=rid + 3)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=sseed, U_pca=U32, alpha=alpha)
        # prompt rows EXACT (prefill), the n_q new rows SLICED (appended by the decode step's K1)
        seq = np.concatenate([np.full(n, b, np.int32) for b, n in enumerate(n_prompt)])
        pos = np.concatenate([np.arange(n, dtype=np.int32) for n in n_prompt])
        r.prefill(bf16_from_bits(np.concatenate([c[:n] for c, n in zip(c_raw, n_prompt)]), d),
                  bf16_from_bits(np.concatenate([x[:n] for x, n in zip(k_pe, n_prompt)]), d),
                  torch.from_numpy(seq).to(d), torch.from_numpy(pos).to(d))
        seq = np.repeat(np.arange(B, dtype=np.int32), n_q)
        pos = np.concatenate([np.arange(n, n + n_q, dtype=np.int32) for n in n_prompt])
        r.append(bf16_from_bits(np.concatenate([c[n:] for c, n in zip(c_raw, n_prompt)]), d),
                 bf16_from_bits(np.concatenate([x[n:] for x, n in zip(k_pe, n_prompt)]), d),
                 torch.from_numpy(seq).to(d), torch.from_numpy(pos).to(d), abi.RMS_SLICED)
        r.decode_mtp(bf16_from_bits(qb, d), bf16_from_bits(qpeb, d), lens, y, out if rid == k - 1 else None,
                     accumulate=rid > 0)
    torch.cuda.synchronize()
    got = y.cpu().numpy().reshape(B, n_q, dims.D)
    for i in range(n_q):
        lim = [S - n_q + 1 + i for S in S_list]
        pb = tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O), U=U,
                          alpha=np.asarray(alpha, float), mu=np.asarray(alpha, float),
                          c_raw=[f64(c[:L]) for c, L in zip(c_raw, lim)], k_pe=[f64(x[:L]) for x, L in zip(k_pe, lim)],
                          modes=[[tpla.EXACT] * n + [tpla.SLICED] * (L - n) for n, L in zip(n_prompt, lim)],
                          q_nope=f64(qb[:, i]), q_pe=f64(qpeb[:, i]), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                          sm_scale=dims_scale(dims))
        ref = tpla.tpla_decode_step(pb, k, g, round_rows=numerics.round_bf16)
        e = row_rel_err(got[:, i], ref)
        assert e <= TOL, (i, e)
    assert torch.equal(out, y.to(torch.bfloat16))


@pytest.mark.parametrize("dname,k,g,n_q", [("kimi", 4, 4, 2), ("dsv3", 4, 2, 2), ("dsv3", 8, 2, 4), ("kimi", 8, 4, 4),
                                           ("dsv3", 2, 1, 2)])
def test_multi_token_decode(dname, k, g, n_q):
    # lengths around tile edges: a segment may hold no visible token for the earlier rows
    mtp_case(dev(), synth.PRESETS[dname], k, g, n_q, [n_q, 65, 129, 300])


def test_multi_token_decode_rejects_too_many_rows():
    d = dev()
    dims = synth.PRESETS["dsv3"]
    r = TplaRank(spec_of(dims), k=2, g=2, rank=0, batch=1, max_seq_len=64, device=d, n_q=2)
    w = synth.gen_weights(dims, 1)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD)
    q = torch.zeros((1, 2, dims.h_q, dims.d_h), dtype=torch.bfloat16, device=d)
    qpe = torch.zeros((1, 2, dims.h_q, dims.d_r), dtype=torch.bfloat16, device=d)
    y = torch.zeros((2, dims.D), dtype=torch.float32, device=d)
    with pytest.raises(abi.TplaError) as ei:            # 2 tokens x 128 heads > 128 MMA rows
        r.decode_mtp(q, qpe, torch.tensor([64], dtype=torch.int32, device=d), y)
    assert ei.value.status == abi.ERR_UNSUPPORTED


def test_deterministic_graph_replay_and_fused_bf16_out():
    """DSV3 shape, k = g = 2 on this GPU: the decode is bitwise deterministic, a CUDA-graph capture
    of it (PDL launches inside) replays to the same bits, and the bf16 output written by the W^O
    segment reduce (no all-reduce) is exactly the RNE rounding of y."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    k = g = 2
    S_list = [100, 257, 64]
    B = len(S_list)
    w = synth.gen_weights(dims, 5)
    q, qpe = synth.gen_queries(dims, B, 6)
    q, qpe = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    ranks = []
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=max(S_list), device=d)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=9)
        for b, S in enumerate(S_list):
            r.prefill(bf16_from_bits(synth.gen_raw_ckv(dims, S, 7, b), d), bf16_from_bits(synth.gen_kpe(dims, S, 7, b), d),
                      torch.full((S,), b, dtype=torch.int32, device=d), torch.arange(S, dtype=torch.int32, device=d))
        ranks.append(r)

    def run(y, out):
        for j, r in enumerate(ranks):
            r.decode(q, qpe, lens, y, out if j == k - 1 else None, accumulate=j > 0)

    ys = [torch.zeros((B, dims.D), dtype=torch.float32, device=d) for _ in range(3)]
    outs = [torch.empty((B, dims.D), dtype=torch.bfloat16, device=d) for _ in range(3)]
    run(ys[0], outs[0])
    run(ys[1], outs[1])
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
        run(ys[2], outs[2])
    ys[2].zero_()
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    for i in (1, 2):
        assert torch.equal(ys[i], ys[0]) and torch.equal(outs[i], outs[0])
    assert torch.equal(outs[0], ys[0].to(torch.bfloat16))
    assert torch.isfinite(ys[0]).all() and ys[0].abs().max() > 0


def test_bf16_output_and_nccl_world1():
    """tpla_decode with a 1-rank NCCL communicator (the C1 call path) and the bf16 output cast."""
    d = dev()
    dims = synth.PRESETS["tiny"]
    r = TplaRank(spec_of(dims), k=1, g=1, rank=0, batch=2, max_seq_len=64, device=d)
    w = synth.gen_weights(dims, 4)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=3)
    n = 40
    ck = bf16_from_bits(np.concatenate([synth.gen_raw_ckv(dims, n, 1, b) for b in range(2)]), d)
    kp = bf16_from_bits(np.concatenate([synth.gen_kpe(dims, n, 1, b) for b in range(2)]), d)
    seq = torch.repeat_interleave(torch.arange(2, dtype=torch.int32), n).to(d)
    pos = torch.arange(n, dtype=torch.int32).repeat(2).to(d)
    r.append(ck, kp, seq, pos, abi.RMS_SLICED)
    q, qpe = synth.gen_queries(dims, 2, 5)
    lens = torch.tensor([n, n - 7], dtype=torch.int32, device=d)
    y0 = torch.zeros((2, dims.D), dtype=torch.float32, device=d)
    r.decode(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, y0)
    comm = abi.tpla_comm_init(abi.tpla_comm_unique_id(), 1, 0)
    y1 = torch.zeros_like(y0)
    out = torch.empty((2, dims.D), dtype=torch.bfloat16, device=d)
    r.decode(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, y1, out, comm=comm)
    torch.cuda.synchronize()
    abi.tpla_comm_destroy(comm)
    assert torch.equal(y0, y1)
    assert torch.equal(out, y1.to(torch.bfloat16))


def test_decode_v_project_out_nccl_world1_equals_decode():
    """One rank: tpla_decode_v + tpla_project_out (with 1-rank group and TP communicators: the
    reduce-scatter and all-reduce call path) is bit-identical to tpla_decode — same bf16 v, same
    W^O kernel and reduction order."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    B, n = 3, 150
    r = TplaRank(spec_of(dims), k=2, g=2, rank=1, batch=B, max_seq_len=n, device=d)
    w = synth.gen_weights(dims, 6)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=5)
    ck = bf16_from_bits(np.concatenate([synth.gen_raw_ckv(dims, n, 2, b) for b in range(B)]), d)
    kp = bf16_from_bits(np.concatenate([synth.gen_kpe(dims, n, 2, b) for b in range(B)]), d)
    seq = torch.repeat_interleave(torch.arange(B, dtype=torch.int32), n).to(d)
    pos = torch.arange(n, dtype=torch.int32).repeat(B).to(d)
    r.append(ck, kp, seq, pos, abi.RMS_SLICED)
    q, qpe = synth.gen_queries(dims, B, 7)
    q, qpe = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
    lens = torch.tensor([n, n - 7, 64], dtype=torch.int32, device=d)
    y0 = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    r.decode(q, qpe, lens, y0)
    gcomm = abi.tpla_comm_init(abi.tpla_comm_unique_id(), 1, 0)
    comm = abi.tpla_comm_init(abi.tpla_comm_unique_id(), 1, 0)
    v = torch.empty(r.v_acc_shape(B), dtype=torch.float32, device=d)
    r.decode_v(q, qpe, lens, v)
    y1 = torch.zeros_like(y0)
    out = torch.empty((B, dims.D), dtype=torch.bfloat16, device=d)
    r.project_out(v, y1, out, group_comm=gcomm, comm=comm)
    torch.cuda.synchronize()
    abi.tpla_comm_destroy(gcomm)
    abi.tpla_comm_destroy(comm)
    assert torch.equal(y0, y1)
    assert torch.equal(out, y1.to(torch.bfloat16))


@pytest.mark.parametrize("k,g,B,S", [(2, 2, 32, 32768), (8, 8, 32, 32768), (8, 2, 32, 32768), (8, 8, 16, 131072)])
def test_full_size_sampled_attention_c1(k, g, B, S):
    """Full-size shards in the bench's launch configuration: configs[1] (c1: H_loc=128, W=320),
    the 8-GPU 32K shape at g = 8 (h8: W_lat = 64, ping-pong softmax, split issuers) and with the
    paper's TP > 2 recipe (h8g2: H_loc = 32), configs[3] (c3: 128K); two sampled sequences checked
    against the oracle."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    r = TplaRank(spec_of(dims), k=k, g=g, rank=k - 1, batch=B, max_seq_len=S, device=d)
    pl = oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, k - 1)
    gen = torch.Generator(device=d)
    gen.manual_seed(123)
    r.cache_buf[..., :pl.row_width].normal_(generator=gen)
    q_lat = torch.randn((B, pl.h_loc, pl.w_lat), generator=gen, device=d).to(torch.bfloat16)
    qpe = torch.randn((B, dims.h_q, dims.d_r), generator=gen, device=d).to(torch.bfloat16)
    lens = torch.full((B,), S, dtype=torch.int32, device=d)
    lens[5] = S - 1000
    O = torch.zeros((B, pl.h_loc, pl.w_lat), dtype=torch.float32, device=d)
    r.decode_attention(q_lat, qpe, lens, O)
    torch.cuda.synchronize()
    for b in (5, B - 1):
        n = int(lens[b])
        rows = f64(r.cache_rows_bits(b, n)[:, :pl.row_width])
        Oref, _, _, _ = tpla.shard_attention(f64(bits_from_bf16(q_lat[b])),
                                              f64(bits_from_bf16(qpe[b, pl.head_begin:pl.head_end])), rows,
                                              pl.w_lat, dims_scale(dims))
        assert row_rel_err(O[b].cpu().numpy(), Oref) <= TOL


# ----------------------------------------------------------------------------- prefill (f1)
def prefill_case(d, dims, k, g, kind, L, *, sample=None, seed=0):
    """causal prefill attention of one prompt (cache sequence 1), every rank of a (k, g)
    plan on this GPU accumulating y.  Pinned to the oracle's decode step over each prefix: prompt
    token t attends to rows 0..t (P:137-141 per token; g = 1 is plain MLA)."""
    xf, sseed, U, U32, alpha = transform_inputs(kind, dims, 41, g)
    basis = U if kind == "pca" else None
    w = synth.gen_weights(dims, seed + 1)
    q, qpe = synth.gen_queries(dims, L, seed + 2)                # row t = prompt token t
    c_raw = synth.gen_raw_ckv(dims, L, seed + 3, 1, basis=basis)
    k_pe = synth.gen_kpe(dims, L, seed + 3, 1)
    junk = synth.gen_raw_ckv(dims, 64, seed + 4, 0, basis=basis)   # sequence 0: another prompt
    y = torch.zeros((L, dims.D), dtype=torch.float32, device=d)
    out = torch.empty((L, dims.D), dtype=torch.bfloat16, device=d)
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=2, max_seq_len=L + 64, device=d, page_perm_seed=rid + 5)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=sseed, U_pca=U32, alpha=alpha)
        r.prefill(bf16_from_bits(junk, d), bf16_from_bits(synth.gen_kpe(dims, 64, seed + 4, 0), d),
                  torch.zeros(64, dtype=torch.int32, device=d), torch.arange(64, dtype=torch.int32, device=d))
        r.prefill(bf16_from_bits(c_raw, d), bf16_from_bits(k_pe, d), torch.ones(L, dtype=torch.int32, device=d),
                  torch.arange(L, dtype=torch.int32, device=d))
        r.prefill_attention(bf16_from_bits(q, d), bf16_from_bits(qpe, d), 1, y, out if rid == k - 1 else None,
                            accumulate=rid > 0)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    ts = range(L) if sample is None else sorted(set(list(range(0, L, sample)) + [L - 1, L - 2]))
    for t in ts:
        pb = tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O), U=U,
                          alpha=np.asarray(alpha, float), mu=np.asarray(alpha, float),
                          c_raw=[f64(c_raw[:t + 1])], k_pe=[f64(k_pe[:t + 1])], modes=[[tpla.EXACT] * (t + 1)],
                          q_nope=f64(q[t:t + 1]), q_pe=f64(qpe[t:t + 1]), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                          sm_scale=dims_scale(dims))
        ref = tpla.tpla_decode_step(pb, k, g, round_rows=numerics.round_bf16)
        e = row_rel_err(got[t:t + 1], ref)
        assert e <= TOL, (t, e)
    assert torch.equal(out, y.to(torch.bfloat16))


@pytest.mark.parametrize("dname,k,g,kind,L", [("dsv3", 2, 1, "identity", 71), ("dsv3", 1, 1, "hadamard", 40),
                                              ("kimi", 4, 2, "hadamard", 45), ("dsv3", 2, 2, "hadamard", 66)])
def test_prefill_attention(dname, k, g, kind, L):
    """g = 1: the PD-separated MLA prefill (heads split over k); g > 1: TPLA prefill.  Ragged
    n_q remainders (L % n_q != 0)."""
    prefill_case(dev(), synth.PRESETS[dname], k, g, kind, L)


def test_prefill_attention_chunks():
    """More prompt rows than one decode call takes (256): two chunks plus a remainder, sampled."""
    prefill_case(dev(), synth.PRESETS["dsv3"], 2, 1, "hadamard", 517, sample=23)


def test_e2e_parity_ragged_combine_blocks():
    """B = 33 sequences: three 16-row K45 blocks per head, the last one ragged."""
    S_list = [1 + (7 * b) % 97 for b in range(33)]
    e2e_case(dev(), synth.PRESETS["dsv3"], 2, 2, "hadamard", S_list)
    e2e_case(dev(), synth.PRESETS["dsv3"], 2, 2, "hadamard", S_list, wo="shared")


# ----------------------------------------------------------------------------- round-2 parity cases
@pytest.mark.parametrize("k,g,S_list", [(2, 2, [12000]), (8, 8, [5000, 700, 9000]), (2, 2, [3000, 6000])])
def test_e2e_parity_small_batch_many_segments(k, g, S_list):
    """Small batch x long context: K3 splits each sequence over tens of CTAs (segments), and K45's
    16 warps share a CTA's few rows (16 / pow2ceil(rows) warps per row, merged through shared memory)."""
    e2e_case(dev(), synth.PRESETS["dsv3"], k, g, "hadamard", S_list)
    e2e_case(dev(), synth.PRESETS["dsv3"], k, g, "hadamard", S_list, wo="shared")


@pytest.mark.parametrize("dname,k,g,kind", [("dsv3", 2, 2, "hadamard"), ("dsv3", 8, 8, "hadamard"),
                                            ("kimi", 4, 4, "identity"), ("tiny", 2, 2, "pca")])
def test_e2e_parity_mu_one(dname, k, g, kind):
    """Reading R6's alternative: mu_j = 1 (the literal §4 equations, no NoPE logit scaling)."""
    e2e_case(dev(), synth.PRESETS[dname], k, g, kind, [5, 200, 333], mu=1.0)
    if dname != "tiny":                 # (the group-shared path needs the tcgen05 kernels' shapes)
        e2e_case(dev(), synth.PRESETS[dname], k, g, kind, [5, 200, 333], mu=1.0, wo="shared")


def dup_slices_case(d, dims, k, g, S_list, *, seed=0, wo="rank"):
    """Closed form (pin c8 at any g): c = [a ‖ a ‖ ... ‖ a] (g copies) and the W^UK / W^UV rows repeated
    the same way, gamma = 1, identity U, alpha = mu = g.  Conditions 1 and 2 hold with equality
    (P:201-209), so the GPU's sliced TPLA (every row appended SLICED by K1) must equal
    plain MLA (oracle mla_decode_full, non-absorbed, g = 1) up to the bf16 storage."""
    B = len(S_list)
    wl = dims.d_c // g
    w = synth.gen_weights(dims, seed + 1, gamma_one=True)
    W_UK, W_UV = w.W_UK.copy(), w.W_UV.copy()
    for j in range(1, g):
        W_UK[j * wl:(j + 1) * wl] = W_UK[:wl]
        W_UV[j * wl:(j + 1) * wl] = W_UV[:wl]
    q, qpe = synth.gen_queries(dims, B, seed + 2)
    c_raw = [np.concatenate([synth.gen_raw_ckv(dims, S, seed + 3, b)[:, :wl]] * g, axis=1) for b, S in enumerate(S_list)]
    k_pe = [synth.gen_kpe(dims, S, seed + 3, b) for b, S in enumerate(S_list)]
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    y = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    ranks = []
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=max(S_list), device=d,
                     page_perm_seed=rid + 11)
        r.convert(W_UK, W_UV, w.gamma, w.W_O, xform=abi.XFORM_IDENTITY, alpha=np.full(g, float(g)),
                  mu=np.full(g, float(g)))
        seq = np.concatenate([np.full(S, b, np.int32) for b, S in enumerate(S_list)])
        pos = np.concatenate([np.arange(S, dtype=np.int32) for S in S_list])
        r.append(bf16_from_bits(np.concatenate(c_raw), d), bf16_from_bits(np.concatenate(k_pe), d),
                 torch.from_numpy(seq).to(d), torch.from_numpy(pos).to(d), abi.RMS_SLICED)
        if wo == "rank":
            r.decode(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, y, accumulate=True)
        ranks.append(r)
    if wo == "shared":
        for hb in sorted({r.plan.head_block for r in ranks}):
            grp = [r for r in ranks if r.plan.head_block == hb]
            acc = torch.zeros(grp[0].v_acc_shape(B), dtype=torch.float32, device=d)
            for j, r in enumerate(grp):
                r.decode_v(bf16_from_bits(q, d), bf16_from_bits(qpe, d), lens, acc, accumulate=j > 0)
            grp[0].project_out(acc, y, accumulate=True)
    torch.cuda.synchronize()
    ref = np.stack([mla.mla_decode_full(f64(q[b]), f64(qpe[b]), f64(c_raw[b]), f64(k_pe[b]), f64(W_UK), f64(W_UV),
                                        f64(w.gamma), f64(w.W_O), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6,
                                        sm_scale=dims_scale(dims))[0] for b in range(B)])
    e = row_rel_err(y.cpu().numpy(), ref)
    assert e <= TOL, e
    return e


@pytest.mark.parametrize("k,g", [(2, 2), (4, 4), (8, 8), (8, 4)])
@pytest.mark.parametrize("wo", ["rank", "shared"])
def test_duplicated_slices_tpla_equals_mla(k, g, wo):
    """The alpha = g / mu = alpha chain at g = 4 and 8 (C2, C3, the 8-GPU headline) on the GPU,
    against MLA itself (DeepSeek-V3 shape)."""
    dup_slices_case(dev(), synth.PRESETS["dsv3"], k, g, [3, 130, 257], wo=wo)


@pytest.mark.parametrize("k,g", [(2, 2), (8, 8)])
def test_full_size_decode_v_project_out_all_sequences(k, g):
    """The production path at full size, in the bench's launch configuration: configs[1] (k = g = 2)
    and the 8-GPU 32K headline shape (k = g = 8), batch 32, 32K context, every rank co-located on
    this GPU: K2 -> K3 -> K45 (decode_v, the group's v summed in place) -> K5 (project_out).  The
    cache rows are seeded N(0, 1) bf16 rows (torch Philox); ALL 32 sequences are checked against
    the oracle (absorb, shard attention, W^UV, W^O, sum over ranks) on those rows."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    B, S = 32, 32768
    w = synth.gen_weights(dims, 77)
    q, qpe = synth.gen_queries(dims, B, 78)
    lens_h = np.full(B, S, np.int32)
    lens_h[5] = S - 1000
    lens_h[17] = 4097
    lens = torch.from_numpy(lens_h).to(d)
    U = reparam.hadamard_U(dims.d_c, 79)
    gen = torch.Generator(device=d)
    gen.manual_seed(80)
    ranks = []
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=S, device=d)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=79)
        r.cache_buf[..., :r.plan.row_width].normal_(generator=gen)
        ranks.append(r)
    y = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    acc = torch.zeros(ranks[0].v_acc_shape(B), dtype=torch.float32, device=d)
    qd, qped = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
    for j, r in enumerate(ranks):          # k = g: one head block, the whole latent group on this GPU
        r.decode_v(qd, qped, lens, acc, accumulate=j > 0)
    ranks[0].project_out(acc, y)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    W_UK_new, W_UV_new = tpla.reparam_weights(f64(w.W_UK), f64(w.W_UV), f64(w.gamma), U)
    alpha = np.full(g, float(g))
    eye = np.eye(dims.d_c)
    plans = [oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, r.rank) for r in ranks]
    W_O = f64(w.W_O)
    dws = [tpla.convert_weights(W_UK_new, W_UV_new, np.ones(dims.d_c), W_O, eye, pl, alpha[pl.shard], d_h=dims.d_h)
           for pl in plans]
    qf, qpef = f64(q), f64(qpe)
    ref = np.zeros((B, dims.D))
    for b in range(B):
        for r, pl, dw in zip(ranks, plans, dws):
            rows = f64(r.cache_rows_bits(b, int(lens_h[b]))[:, :pl.row_width])
            ref[b] += tpla.decode_device(qf[b:b + 1], qpef[b:b + 1], [rows], dw, pl, sm_scale=dims_scale(dims))[0]
    e = row_rel_err(got, ref)
    assert e <= TOL, e


def test_wo_large_batch_row_chunks():
    """B = 300 > 256 output rows: the tcgen05 W^O GEMM runs in 256-row chunks (decode and project_out)."""
    S_list = [1 + (13 * b) % 41 for b in range(300)]
    e2e_case(dev(), synth.PRESETS["dsv3"], 2, 2, "hadamard", S_list)
    e2e_case(dev(), synth.PRESETS["dsv3"], 2, 2, "hadamard", S_list, wo="shared")


def test_wo_mma_baseline_reads_blocked_layout(monkeypatch):
    """TPLA_WO=mma (the mma.sync W^O baseline) reads the blocked W^O layout tpla_convert_weights writes."""
    monkeypatch.setenv("TPLA_WO", "mma")
    e2e_case(dev(), synth.PRESETS["dsv3"], 2, 2, "hadamard", [5, 200, 333])
    e2e_case(dev(), synth.PRESETS["dsv3"], 8, 2, "identity", [64, 129])


# ----------------------------------------------------------------------------- f1: non-absorbed MLA prefill
def prefill_mla_forward_case(d, dims, k, L, *, sample=None, seed=0):
    """SURVEY f1, PD separation: the prompt's causal attention as MLA with the heads split over k
    devices and the latent unsliced, keys/values up-projected per head (K8), then W^O and the sum over
    the devices.  Pinned to the oracle's non-absorbed MLA (oracle/mla.py, Eq. isolate_rope)
    per prompt position t over the prefix 0..t."""
    from paper_2508_15881_b200.runtime import PrefillRank
    w = synth.gen_weights(dims, seed + 1)
    q, qpe = synth.gen_queries(dims, L, seed + 2)
    c_raw = synth.gen_raw_ckv(dims, L, seed + 3, 0)
    k_pe = synth.gen_kpe(dims, L, seed + 3, 0)
    y = torch.zeros((L, dims.D), dtype=torch.float32, device=d)
    out = torch.empty((L, dims.D), dtype=torch.bfloat16, device=d)
    args = [bf16_from_bits(x, d) for x in (c_raw, k_pe, q, qpe)]
    for r in range(k):
        pr = PrefillRank(spec_of(dims), k=k, rank=r, max_len=L, device=d)
        pr.convert(w.W_UK, w.W_UV, w.gamma, w.W_O)
        pr.forward(*args, y, out if r == k - 1 else None, accumulate=r > 0)
    torch.cuda.synchronize()
    got = y.cpu().numpy()
    ts = range(L) if sample is None else sorted(set(list(range(0, L, sample)) + [L - 1, 127, 128]) & set(range(L)))
    W = [f64(x) for x in (w.W_UK, w.W_UV, w.gamma, w.W_O)]
    for t in ts:
        ref = mla.mla_decode_full(f64(q[t]), f64(qpe[t]), f64(c_raw[:t + 1]), f64(k_pe[:t + 1]), *W, h_q=dims.h_q,
                                  d_h=dims.d_h, eps=1e-6, sm_scale=dims_scale(dims))[0]
        e = row_rel_err(got[t:t + 1], ref[None])
        assert e <= TOL, (t, e)
    assert torch.equal(out, y.to(torch.bfloat16))     # (k > 1: the bf16 cast after the reduce-added y)


@pytest.mark.parametrize("k,L", [(1, 129), (2, 300), (4, 77)])
def test_prefill_mla_forward(k, L):
    """Ragged query / key tiles (L % 128 != 0), two 256-row GEMM chunks, heads split 1 / 2 / 4 ways."""
    prefill_mla_forward_case(dev(), synth.PRESETS["dsv3"], k, L, sample=7)


def test_prefill_mla_forward_kimi_long():
    """Kimi-K2 heads (64), a 1100-token prompt: 9 query tiles, the longest attending to 9 key tiles."""
    prefill_mla_forward_case(dev(), synth.PRESETS["kimi"], 2, 1100, sample=97)


# ----------------------------------------------------------------------------- f2(i): fused W^O + all-reduce
def test_fused_allreduce_world1_bit_identical():
    """SURVEY f2(i) at world 1 (the only size one GPU can run): the K5 segment reduce writes Õ into the
    NCCL symmetric window, meets its peers at the LSA barrier and sums the ranks itself.  With one rank
    the sum is the rank's own rows: y and the bf16 output must be bit-identical to the decode without
    a communicator — for tpla_decode, for decode_v + project_out, repeatedly (the buffer halves
    alternate with the barrier epoch) and under CUDA-graph replay."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    B, n = 3, 150
    r = TplaRank(spec_of(dims), k=2, g=2, rank=1, batch=B, max_seq_len=n, device=d)
    w = synth.gen_weights(dims, 16)
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=5)
    ck = bf16_from_bits(np.concatenate([synth.gen_raw_ckv(dims, n, 2, b) for b in range(B)]), d)
    kp = bf16_from_bits(np.concatenate([synth.gen_kpe(dims, n, 2, b) for b in range(B)]), d)
    seq = torch.repeat_interleave(torch.arange(B, dtype=torch.int32), n).to(d)
    pos = torch.arange(n, dtype=torch.int32).repeat(B).to(d)
    r.append(ck, kp, seq, pos, abi.RMS_SLICED)
    q, qpe = synth.gen_queries(dims, B, 7)
    q, qpe = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
    lens = torch.tensor([n, n - 7, 64], dtype=torch.int32, device=d)
    y0 = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    r.decode(q, qpe, lens, y0)
    comm = abi.tpla_comm_init(abi.tpla_comm_unique_id(), 1, 0)
    try:
        abi.tpla_comm_enable_fused_allreduce(comm, 64 * dims.D)
    except abi.TplaError as e:
        abi.tpla_comm_destroy(comm)
        pytest.skip(f"no NCCL device API: {e}")
    assert abi.tpla_comm_fused_allreduce_mode(comm) == 1          # (world 1: peer loads, no multicast)
    n0 = abi.tpla_launch_count()
    ys = [torch.full_like(y0, float("nan")) for _ in range(3)]
    outs = [torch.empty((B, dims.D), dtype=torch.bfloat16, device=d) for _ in range(3)]
    for y, out in zip(ys, outs):
        r.decode(q, qpe, lens, y, out, comm=comm)
    torch.cuda.synchronize()
    for y, out in zip(ys, outs):
        assert torch.equal(y, y0) and torch.equal(out, y0.to(torch.bfloat16))
    # decode_v + project_out (the group-shared up-projection) on the same communicator
    v = torch.empty(r.v_acc_shape(B), dtype=torch.float32, device=d)
    r.decode_v(q, qpe, lens, v)
    y1 = torch.full_like(y0, float("nan"))
    out1 = torch.empty((B, dims.D), dtype=torch.bfloat16, device=d)
    r.project_out(v, y1, out1, comm=comm)
    # graph capture: two decodes per replay, replayed twice (the epoch parity keeps alternating)
    yg = [torch.zeros_like(y0) for _ in range(2)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
        for y in yg:
            r.decode(q, qpe, lens, y, comm=comm)
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    abi.tpla_comm_destroy(comm)
    assert torch.equal(y1, y0) and torch.equal(out1, y0.to(torch.bfloat16))
    for y in yg:
        assert torch.equal(y, y0)
    assert abi.tpla_launch_count() > n0


def test_decode_v_two_stages_bit_identical():
    """tpla_decode_v in two calls (STAGE_PRE: K3p + K2, then STAGE_ATTN: K3 + K45, as bench.py schedules
    co-located ranks) gives the same bits as the one-call decode_v; both flags together are rejected."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    B, n = 3, 300
    for k, g in ((2, 2), (8, 8)):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=k - 1, batch=B, max_seq_len=n, device=d)
        w = synth.gen_weights(dims, 17)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=abi.XFORM_HADAMARD, sign_seed=5)
        ck = bf16_from_bits(np.concatenate([synth.gen_raw_ckv(dims, n, 2, b) for b in range(B)]), d)
        kp = bf16_from_bits(np.concatenate([synth.gen_kpe(dims, n, 2, b) for b in range(B)]), d)
        seq = torch.repeat_interleave(torch.arange(B, dtype=torch.int32), n).to(d)
        pos = torch.arange(n, dtype=torch.int32).repeat(B).to(d)
        r.append(ck, kp, seq, pos, abi.RMS_SLICED)
        q, qpe = synth.gen_queries(dims, B, 7)
        q, qpe = bf16_from_bits(q, d), bf16_from_bits(qpe, d)
        lens = torch.tensor([n, n - 7, 64], dtype=torch.int32, device=d)
        v0 = torch.zeros(r.v_acc_shape(B), dtype=torch.float32, device=d)
        v1 = torch.full_like(v0, float("nan"))
        r.decode_v(q, qpe, lens, v0)
        r.decode_v(q, qpe, lens, v1, stage="pre")
        r.decode_v(q, qpe, lens, v1, stage="attn")
        torch.cuda.synchronize()
        assert torch.equal(v0, v1)
        with pytest.raises(abi.TplaError) as ei:
            abi.tpla_decode_v(r.cfg, r.weights, r.cache, q, qpe, lens, B, 1, r.max_seq_len, r.ws, r.ws_bytes, v1, 1,
                              abi.DECODE_STAGE_PRE | abi.DECODE_STAGE_ATTN, 0)
        assert ei.value.status == abi.ERR_INVALID_ARG


# ----------------------------------------------------------------------------- f4: "norm only" on the GPU
@pytest.mark.parametrize("kind,n_slices", [("hadamard", 2), ("identity", 2), ("pca", 2), ("hadamard", 4),
                                           ("pca", 8)])
def test_norm_only_rows_equal_exact_logit_oracle(kind, n_slices):
    """SURVEY f4 / Fig. 3 "TPLA (norm only)": sliced RMSNorm, one softmax over the summed partial
    logits.  On the GPU: g = 1 rows normalised per slice (tpla_append_kv_norm_only) decoded by the g = 1
    kernels (the CTA-pair K3) with mu = 1; oracle: tpla_decode_exact_logits over the k = g shards."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    S_list = [5, 130, 300]
    B = len(S_list)
    xf, sseed, U, U32, alpha = transform_inputs(kind, dims, 51, n_slices)
    basis = U if kind == "pca" else None
    w = synth.gen_weights(dims, 52)
    q, qpe = synth.gen_queries(dims, B, 53)
    c_raw = [synth.gen_raw_ckv(dims, S, 54, b, basis=basis) for b, S in enumerate(S_list)]
    k_pe = [synth.gen_kpe(dims, S, 54, b) for b, S in enumerate(S_list)]
    r = TplaRank(spec_of(dims), k=1, g=1, rank=0, batch=B, max_seq_len=max(S_list), device=d, page_perm_seed=3)
    U_full = None if U32 is None else U32                    # PCA: all d_c columns at g = 1
    r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=sseed, U_pca=U_full, alpha=[1.0], mu=[1.0])
    seq = np.concatenate([np.full(S, b, np.int32) for b, S in enumerate(S_list)])
    pos = np.concatenate([np.arange(S, dtype=np.int32) for S in S_list])
    r.append_norm_only(bf16_from_bits(np.concatenate(c_raw), d), bf16_from_bits(np.concatenate(k_pe), d),
                       torch.from_numpy(seq).to(d), torch.from_numpy(pos).to(d), np.asarray(alpha, np.float32))
    y = torch.zeros((B, dims.D), dtype=torch.float32, device=d)
    r.decode(bf16_from_bits(q, d), bf16_from_bits(qpe, d), torch.tensor(S_list, dtype=torch.int32, device=d), y)
    torch.cuda.synchronize()
    pb = tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O), U=U,
                      alpha=np.asarray(alpha, float), mu=np.ones(n_slices), c_raw=[f64(c) for c in c_raw],
                      k_pe=[f64(x) for x in k_pe], modes=[[tpla.SLICED] * S for S in S_list], q_nope=f64(q),
                      q_pe=f64(qpe), h_q=dims.h_q, d_h=dims.d_h, eps=1e-6, sm_scale=dims_scale(dims))
    ref = tpla.tpla_decode_exact_logits(pb, n_slices, round_rows=numerics.round_bf16)   # (R19: the cache is bf16)
    e = row_rel_err(y.cpu().numpy(), ref)
    assert e <= TOL, e


def test_prefill_mla_forward_graph_replay_deterministic():
    """The non-absorbed prefill (K8a, K9, K8, K9 W^O) captured in a CUDA graph replays to the same bits as
    the eager call (PDL launches inside, persistent K8's work order fixed)."""
    from paper_2508_15881_b200.runtime import PrefillRank
    d = dev()
    dims = synth.PRESETS["dsv3"]
    L = 389
    w = synth.gen_weights(dims, 61)
    q, qpe = synth.gen_queries(dims, L, 62)
    args = [bf16_from_bits(x, d) for x in (synth.gen_raw_ckv(dims, L, 63, 0), synth.gen_kpe(dims, L, 63, 0), q, qpe)]
    pr = PrefillRank(spec_of(dims), k=2, rank=1, max_len=L, device=d)
    pr.convert(w.W_UK, w.W_UV, w.gamma, w.W_O)
    y0 = torch.zeros((L, dims.D), dtype=torch.float32, device=d)
    pr.forward(*args, y0)
    yg = torch.full_like(y0, float("nan"))
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
        pr.forward(*args, yg)
    graph.replay()
    graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(yg, y0) and torch.isfinite(y0).all()


def test_c_example_runs_on_gpu(tmp_path):
    """examples/decode_step.c: convert, append and a two-rank decode step through the C ABI alone
    (tcgen05 path), finite and bit-identical on replay, bad batch rejected before any launch."""
    import subprocess
    from test_abi_host import build_c_example
    exe = build_c_example(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "decode_step OK" in r.stdout and "K3 path: 1" in r.stdout, r.stdout


# ----------------------------------------------------------------------------- guard bands
# compute-sanitizer is closed on this pool (profiles/r02_sanitizer_pool_closed.log), so out-of-bounds
# WRITES are checked directly: every buffer a call writes sits between canary regions, the paged cache
# is pre-filled with a canary, and after the calls every byte outside the documented output extents
# must still hold its canary.
def _guarded(shape, dtype, d, fill):
    g = 4096 // torch.tensor([], dtype=dtype).element_size()
    n = int(np.prod(shape))
    full = torch.full((n + 2 * g,), fill, dtype=dtype, device=d)
    return full, full[g:g + n].view(shape), g


def _canary_intact(full, g, fill):
    return bool((full[:g] == fill).all()) and bool((full[-g:] == fill).all())


@pytest.mark.parametrize("k,g,S_list,n_q", [(2, 2, [300, 77, 1025], 1), (8, 8, [129, 64, 700, 1], 1),
                                            (4, 2, [200, 513], 2)])
def test_no_writes_outside_outputs(k, g, S_list, n_q):
    d = dev()
    dims = synth.PRESETS["dsv3"]
    B = len(S_list)
    xf, sseed, U, U32, alpha = transform_inputs("hadamard", dims, 3, g)
    w = synth.gen_weights(dims, 5)
    q, qpe = synth.gen_queries(dims, B * n_q, 6)
    q = bf16_from_bits(q, d).view(B, n_q, dims.h_q, dims.d_h) if n_q > 1 else bf16_from_bits(q, d)
    qpe = bf16_from_bits(qpe, d).view(B, n_q, dims.h_q, dims.d_r) if n_q > 1 else bf16_from_bits(qpe, d)
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    CANARY16 = 0x1234                                   # a finite bf16 (the cache's unused rows must be finite)
    for rid in range(k):
        r = TplaRank(spec_of(dims), k=k, g=g, rank=rid, batch=B, max_seq_len=max(S_list), device=d, extra_pages=3,
                     n_q=n_q)
        r.convert(w.W_UK, w.W_UV, w.gamma, w.W_O, xform=xf, sign_seed=sseed, alpha=alpha,
                  mu=np.asarray(alpha, float))
        r.cache_buf.view(torch.int16).fill_(CANARY16)
        ws_full, r.ws, gw = _guarded((r.ws_bytes,), torch.uint8, d, 0xA5)
        for b, S in enumerate(S_list):
            ck = bf16_from_bits(synth.gen_raw_ckv(dims, S, 7, b), d)
            kp = bf16_from_bits(synth.gen_kpe(dims, S, 7, b), d)
            r.append(ck, kp, torch.full((S,), b, dtype=torch.int32, device=d),
                     torch.arange(S, dtype=torch.int32, device=d), abi.RMS_EXACT)
        R = B * n_q
        # reads: the same decode with NaN in every workspace byte and NaN bf16 around the queries must give
        # the bits of a run on a zeroed workspace (no kernel reads scratch it did not write first, nor
        # past its inputs)
        NAN16 = 0x7FC0
        qg_full, qg, _ = _guarded(tuple(q.shape), torch.int16, d, NAN16)
        pg_full, pg, _ = _guarded(tuple(qpe.shape), torch.int16, d, NAN16)
        qg.copy_(q.view(torch.int16))
        pg.copy_(qpe.view(torch.int16))
        y_ref = torch.zeros((R, dims.D), dtype=torch.float32, device=d)
        y_nan = torch.zeros_like(y_ref)
        r.ws.zero_()
        (r.decode_mtp if n_q > 1 else r.decode)(q, qpe, lens, y_ref)
        r.ws.fill_(0xFF)
        (r.decode_mtp if n_q > 1 else r.decode)(qg.view(torch.bfloat16), pg.view(torch.bfloat16), lens, y_nan)
        torch.cuda.synchronize()
        assert torch.isfinite(y_ref).all() and torch.equal(y_nan, y_ref), "read of unwritten scratch or past an input"
        y_full, y, gy = _guarded((R, dims.D), torch.float32, d, -7.0)
        o_full, out, go = _guarded((R, dims.D), torch.int16, d, 0x5555)
        if n_q > 1:
            r.decode_mtp(q, qpe, lens, y, out.view(torch.bfloat16))
        else:
            r.decode(q, qpe, lens, y, out.view(torch.bfloat16))
            va_full, va, gv = _guarded(r.v_acc_shape(R, 1), torch.float32, d, -9.0)
            r.decode_v(q, qpe, lens, va)
            r.project_out(va, y, out.view(torch.bfloat16), accumulate=True)
            torch.cuda.synchronize()
            assert _canary_intact(va_full, gv, -9.0)
        torch.cuda.synchronize()
        assert _canary_intact(ws_full, gw, 0xA5), "workspace overrun"
        assert _canary_intact(y_full, gy, -7.0) and _canary_intact(o_full, go, 0x5555), "output overrun"
        # cache: only rows [0, S_b) of sequence b's pages were written; the rest (and the spare pages) kept
        cb = r.cache_buf.view(torch.int16)
        written = torch.zeros(cb.shape[:2], dtype=torch.bool, device=d)
        for b, S in enumerate(S_list):
            for t0 in range(0, S, r.page_size):
                pg = int(r.block_table_host[b, t0 // r.page_size])
                written[pg, :min(r.page_size, S - t0)] = True
        assert bool((cb[~written] == CANARY16).all()), "cache rows outside the appended positions changed"
        assert bool((cb[written][:, r.plan.row_width:] == CANARY16).all()), "row padding changed"


def test_no_writes_outside_prefill_outputs():
    from paper_2508_15881_b200.runtime import PrefillRank
    d = dev()
    dims = synth.PRESETS["dsv3"]
    L = 333
    w = synth.gen_weights(dims, 8)
    q, qpe = synth.gen_queries(dims, L, 9)
    args = [bf16_from_bits(x, d) for x in (synth.gen_raw_ckv(dims, L, 10, 0), synth.gen_kpe(dims, L, 10, 0), q, qpe)]
    pr = PrefillRank(spec_of(dims), k=2, rank=0, max_len=L, device=d)
    pr.convert(w.W_UK, w.W_UV, w.gamma, w.W_O)
    ws_full, pr.ws, gw = _guarded((pr.ws_bytes,), torch.uint8, d, 0xA5)
    y_full, y, gy = _guarded((L, dims.D), torch.float32, d, -7.0)
    o_full, out, go = _guarded((L, dims.D), torch.int16, d, 0x5555)
    pr.forward(*args, y, out.view(torch.bfloat16))
    torch.cuda.synchronize()
    assert _canary_intact(ws_full, gw, 0xA5) and _canary_intact(y_full, gy, -7.0) and _canary_intact(o_full, go, 0x5555)
    # reads: NaN in every workspace byte gives the same bits (no read of unwritten scratch)
    y2 = torch.empty_like(y)
    pr.ws.fill_(0xFF)
    pr.forward(*args, y2)
    torch.cuda.synchronize()
    assert torch.isfinite(y).all() and torch.equal(y2, y)


# ----------------------------------------------------------------------------- seeded random configurations
_KG = [(1, 1), (2, 1), (2, 2), (4, 2), (4, 4), (8, 2), (8, 4), (8, 8)]


@pytest.mark.parametrize("case", range(int(__import__("os").environ.get("TPLA_FUZZ_CASES", "20"))))
def test_e2e_parity_random_configs(case):
    """Seeded random (model, k, g, transform, batch, ragged lengths, W^O mode) drawn per case: the
    production decode (K1, fused K3p + K2, K3 incl. the g = 1 CTA pair, K45, K5) against the oracle."""
    rng = np.random.default_rng(1000 + case)
    dname = ["dsv3", "kimi"][int(rng.integers(2))]
    k, g = _KG[int(rng.integers(len(_KG)))]
    kind = ["identity", "hadamard", "pca"][int(rng.integers(3))] if g > 1 else "identity"
    B = int(rng.integers(1, 41))
    S_list = [int(x) for x in rng.integers(1, 1500, size=B)]
    wo = "shared" if g > 1 and rng.integers(2) else "rank"
    e2e_case(dev(), synth.PRESETS[dname], k, g, kind, S_list, seed=case, wo=wo)


@pytest.mark.parametrize("case", range(int(__import__("os").environ.get("TPLA_FUZZ_CASES_MTP", "8"))))
def test_mtp_parity_random_configs(case):
    """Seeded random multi-token decode shapes (n_q * H_loc <= 128) against the per-token oracle."""
    rng = np.random.default_rng(2000 + case)
    dname = ["dsv3", "kimi"][int(rng.integers(2))]
    dims = synth.PRESETS[dname]
    choices = [(k, g, n) for k, g in _KG for n in (2, 3, 4) if g > 1 and n * dims.h_q // (k // g) <= 128]
    k, g, n_q = choices[int(rng.integers(len(choices)))]
    B = int(rng.integers(1, 17))
    S_list = [int(x) for x in rng.integers(n_q, 1200, size=B)]
    mtp_case(dev(), dims, k, g, n_q, S_list, seed=case, kind=["identity", "hadamard"][int(rng.integers(2))])


@pytest.mark.parametrize("case", range(int(__import__("os").environ.get("TPLA_FUZZ_CASES_PF", "4"))))
def test_prefill_mla_forward_random_configs(case):
    """Seeded random prompt lengths and head splits of the non-absorbed prefill, sampled positions."""
    rng = np.random.default_rng(3000 + case)
    dname = ["dsv3", "kimi"][int(rng.integers(2))]
    k = [1, 2, 4][int(rng.integers(3))]
    L = int(rng.integers(1, 1400))
    prefill_mla_forward_case(dev(), synth.PRESETS[dname], k, L, sample=min(L, 24), seed=case)


@pytest.mark.parametrize("k,g", [(2, 2), (8, 8), (2, 1)])
def test_decode_attention_reuse_plan_bit_identical(k, g):
    """TPLA_ATTN_REUSE_PLAN (K3 without K3p, on the schedule the previous call left in the workspace, as
    the bench's K3-alone timings use it) gives the bits of the full call."""
    d = dev()
    dims = synth.PRESETS["dsv3"]
    S_list = [1000, 3, 257]
    B = len(S_list)
    r = TplaRank(spec_of(dims), k=k, g=g, rank=k - 1, batch=B, max_seq_len=max(S_list), device=d, page_perm_seed=3)
    gen = torch.Generator(device=d)
    gen.manual_seed(11)
    r.cache_buf[..., :r.plan.row_width].normal_(generator=gen)
    q_lat = torch.randn((B, r.plan.h_loc, r.plan.w_lat), generator=gen, device=d).to(torch.bfloat16)
    q_pe = torch.randn((B, dims.h_q, dims.d_r), generator=gen, device=d).to(torch.bfloat16)
    lens = torch.tensor(S_list, dtype=torch.int32, device=d)
    O1 = torch.empty((B, r.plan.h_loc, r.plan.w_lat), dtype=torch.float32, device=d)
    O2 = torch.full_like(O1, float("nan"))
    r.decode_attention(q_lat, q_pe, lens, O1)
    r.decode_attention(q_lat, q_pe, lens, O2, reuse_plan=True)
    torch.cuda.synchronize()
    assert torch.isfinite(O1).all() and torch.equal(O1, O2)
