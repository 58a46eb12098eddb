"""World-size-2 CPU (gloo) tests of the multi-rank host logic of the TPLA decode step.

Each process takes the ranks bench.py would give it (k/N consecutive ranks), gets its shard
plan from libtpla.so (host entry point), computes its ranks' share Õ_r with the oracle,
accumulates them locally (TPLA_DECODE_ACCUMULATE semantics) and all-reduces over gloo — the
exchange step of P:141.  The result must equal the single-process oracle step, the unique id
broadcast must reach every process intact, and the timing reduction must be a max.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import numerics, plan as oplan, reparam, tpla


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(dims, g, S_list, seed=3):
    f64 = numerics.bf16_to_f64
    w = synth.gen_weights(dims, seed)
    q, qpe = synth.gen_queries(dims, len(S_list), seed)
    c = [f64(synth.gen_raw_ckv(dims, S, seed, b)) for b, S in enumerate(S_list)]
    k = [f64(synth.gen_kpe(dims, S, seed, b)) for b, S in enumerate(S_list)]
    return tpla.Problem(W_UK=f64(w.W_UK), W_UV=f64(w.W_UV), gamma=f64(w.gamma), W_O=f64(w.W_O),
                        U=reparam.hadamard_U(dims.d_c, 9), alpha=np.full(g, float(g)), mu=np.full(g, float(g)),
                        c_raw=c, k_pe=k, modes=[[tpla.SLICED] * S for S in S_list], q_nope=f64(q), q_pe=f64(qpe),
                        h_q=dims.h_q, d_h=dims.d_h, eps=1e-6, sm_scale=1 / np.sqrt(dims.d_h + dims.d_r))


def _worker(proc, world, port, k, g, S_list, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=proc, world_size=world)
    try:
        from paper_2508_15881_b200 import abi
        dims = synth.PRESETS["odd"]
        pb = _problem(dims, g, S_list)
        m = k // world
        y = None
        for r in range(proc * m, (proc + 1) * m):
            cfg = abi.tpla_config(dims.h_q, dims.d_c, dims.d_r, dims.d_h, dims.D, k, g, r, 1e-6, pb.sm_scale)
            p = abi.tpla_make_plan(cfg)
            pl = oplan.DevicePlan(p.rank, p.shard, p.head_block, p.head_begin, p.head_end, p.lat_begin, p.lat_end,
                                  p.row_width)
            assert pl == oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, r)
            dw = tpla.convert_weights(pb.W_UK, pb.W_UV, pb.gamma, pb.W_O, pb.U, pl, pb.mu[pl.shard], d_h=dims.d_h)
            rows = tpla.device_rows(pb, pl, pb.alpha[pl.shard])
            yr = tpla.decode_device(pb.q_nope, pb.q_pe, rows, dw, pl, sm_scale=pb.sm_scale)
            y = yr if y is None else y + yr                      # local accumulation (m ranks per process)
        t = torch.from_numpy(y)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)                 # C1: O = AllReduce(Σ Õ_r)
        # unique-id broadcast (what bench.py does before tpla_comm_init)
        try:
            uid = abi.tpla_comm_unique_id() if proc == 0 else None
        except abi.TplaError:
            uid = b"\x01" * 128 if proc == 0 else None           # NCCL not loadable here: still test the bcast
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        # max-over-ranks timing reduction
        ms = torch.tensor([10.0 + proc], dtype=torch.float64)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        out_q.put((proc, t.numpy(), obj[0], float(ms.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,g", [(2, 2), (4, 2), (2, 1), (4, 4)])
def test_two_process_decode_matches_single_process(k, g):
    S_list = [5, 33]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(p, 2, port, k, g, S_list, q)) for p in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    ref = tpla.tpla_decode_step(_problem(synth.PRESETS["odd"], g, S_list), k, g)
    for proc, y, uid, ms in res:
        assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-12
        assert uid == res[0][2] and len(uid) == 128
        assert ms == 11.0


def _worker_shared_wo(proc, world, port, k, g, S_list, out_q):
    """SURVEY f2(ii) over 2 processes: each process sums the v_j of its ranks per head block into a
    column-chunk-major v_acc (runtime.head_block_groups), the group's processes reduce-scatter it
    (here: all-reduce over a gloo subgroup, then keep chunk c — the same sum), project their chunk's
    K-slice of W^O, and the TP group all-reduces y."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=proc, world_size=world)
    try:
        from paper_2508_15881_b200.runtime import group_process_sets, head_block_groups
        dims = synth.PRESETS["odd"]
        pb = _problem(dims, g, S_list)
        B, K = len(S_list), (dims.h_q // (k // g)) * dims.d_h
        sub = {ps: dist.new_group(list(ps)) for ps in group_process_sets(k, g, world)}   # same order everywhere
        y = np.zeros((B, dims.D))
        for grp in head_block_groups(k, g, world, proc):
            nc = grp.n_chunks
            v_acc = np.zeros((nc, B, K // nc))
            W_O = None
            for r in grp.local_ranks:
                pl = oplan.make_plan(k, g, dims.h_q, dims.d_c, dims.d_r, r)
                dw = tpla.convert_weights(pb.W_UK, pb.W_UV, pb.gamma, pb.W_O, pb.U, pl, pb.mu[pl.shard],
                                          d_h=dims.d_h)
                rows = tpla.device_rows(pb, pl, pb.alpha[pl.shard])
                _, parts = tpla.decode_device(pb.q_nope, pb.q_pe, rows, dw, pl, sm_scale=pb.sm_scale,
                                              return_parts=True)
                v = np.einsum("bhl,hld->bhd", parts["O"], dw.W_UV).reshape(B, K)      # v_j = O_j W^UV'_j
                v_acc += v.reshape(B, nc, K // nc).transpose(1, 0, 2)               # chunk-major layout
                assert W_O is None or np.array_equal(W_O, dw.W_O)                   # same rows
                W_O = dw.W_O
            if nc > 1:
                t = torch.from_numpy(v_acc)
                dist.all_reduce(t, group=sub[grp.procs])
                v_acc = t.numpy()
            kc = K // nc
            y += v_acc[grp.chunk] @ W_O[grp.chunk * kc:(grp.chunk + 1) * kc]
        t = torch.from_numpy(y)
        dist.all_reduce(t)
        out_q.put((proc, t.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,g", [(2, 2), (4, 2), (4, 4), (2, 1)])
def test_two_process_shared_wo_matches_single_process(k, g):
    S_list = [5, 33]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_shared_wo, args=(p, 2, port, k, g, S_list, q)) for p in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = tpla.tpla_decode_step(_problem(synth.PRESETS["odd"], g, S_list), k, g)
    for proc, y in res:
        assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) < 1e-12


@pytest.mark.parametrize("k,g,N", [(2, 2, 1), (2, 2, 2), (4, 2, 2), (8, 2, 8), (8, 8, 2), (8, 2, 4), (8, 4, 8)])
def test_head_block_groups_cover_every_rank_once(k, g, N):
    from paper_2508_15881_b200.runtime import group_process_sets, head_block_groups
    m, nb = k // N, k // g
    seen = []
    for p in range(N):
        for grp in head_block_groups(k, g, N, p):
            assert all(r // m == p and r % nb == grp.head_block for r in grp.local_ranks)
            assert grp.procs[grp.chunk] == p and len(grp.local_ranks) * len(grp.procs) == g
            seen += grp.local_ranks
    assert sorted(seen) == list(range(k))
    assert all(len(s) > 1 for s in group_process_sets(k, g, N))
