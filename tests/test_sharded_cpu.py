"""Sharded (multi-GPU) PRGD step, checked on the CPU with torch.distributed gloo, world size 2.

The library's sharded mode (include/prgd.h tt_set_allreduce) splits Omega over
ranks and all-reduces exactly two buffers per step: the marginals h_{k,j}
after pass A and the contractions Y_k after pass B, replicating everything
else.  This test runs that decomposition with the oracle's building blocks on two gloo
ranks (each holding half of Omega) and checks the resulting iterate against the
single-process oracle step, and the rank-disjoint sampling of synth for world > 1."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def sharded_step(cores, idx, y, n, r, step_size, m_global, allreduce, step_rule="theory"):
    """One PRGD step where idx / y are this rank's shard; allreduce(np.ndarray) sums in place
    over ranks.  Mirrors tt_prgd_step in sharded mode (adaptive rule: a third exchange, the
    denominator ||P_Omega D||^2)."""
    d = len(n)
    p = m_global / math.prod(n)
    g = oracle.residual(cores, idx, y)
    h = oracle.mode_sums(g, idx, n)
    flat = np.concatenate(h)
    allreduce(flat)                                             # exchange 1: h
    off = np.cumsum([0] + list(n))
    h = [flat[off[k]:off[k + 1]] for k in range(d)]
    eps, w, phi = oracle.build_weights(h, d)
    if eps == 0.0:
        return [c.copy() for c in cores]
    ghat = oracle.precondition_residual(g, idx, phi)
    U = oracle.left_orthogonalize(oracle.weight_cores(cores, phi, 1.0))
    P = oracle.right_grams(U)
    Y = oracle.contraction(U, idx, ghat)
    flat = np.concatenate([yk.ravel() for yk in Y])
    allreduce(flat)                                             # exchange 2: Y
    offs = np.cumsum([0] + [yk.size for yk in Y])
    Y = [flat[offs[k]:offs[k + 1]].reshape(Y[k].shape) for k in range(d)]
    Ahat = oracle.project(U, P, Y)
    Ttil, A = oracle.unweight(U, phi), oracle.unweight(Ahat, phi)
    if step_rule == "adaptive":
        _, num, den = oracle.adaptive_step(1.0, U, Ahat, Ttil, A, idx)   # den: this shard only
        buf = np.array([den])
        allreduce(buf)                                          # exchange 3: den
        alpha = step_size * num / buf[0] if buf[0] > 0 else 0.0
    else:
        alpha = oracle.step_length(step_size, eps, p, "theory")
    B = oracle.assemble(Ttil, A, alpha)
    return oracle.tt_round(B, r)


def _worker(rank, world, port, out, step_rule="theory"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr = synth.make_problem(2, m=4000)
        y = oracle.eval_at(pr.truth, pr.idx) + 1e-3 * pr.noise_unit
        init = pr.init
        shard = slice(rank, None, world)                        # disjoint halves of Omega

        def allreduce(a):
            t = torch.from_numpy(a)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)

        cores = init
        for _ in range(3):
            cores = sharded_step(cores, pr.idx[shard], y[shard], pr.n, pr.r, 1.0, pr.m, allreduce,
                                 step_rule)
        out[rank] = np.concatenate([c.ravel() for c in cores])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("step_rule", ["theory", "adaptive"])
def test_sharded_step_matches_single_process(step_rule):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out, step_rule), nprocs=world, join=True)
    pr = synth.make_problem(2, m=4000)
    y = oracle.eval_at(pr.truth, pr.idx) + 1e-3 * pr.noise_unit
    ref = pr.init
    for _ in range(3):
        ref = oracle.prgd_step(ref, pr.idx, y, pr.n, pr.r, 1.0, step_rule=step_rule)
    offs = np.cumsum([0] + [c.size for c in ref])
    for rank in range(world):
        got = [out[rank][offs[k]:offs[k + 1]].reshape(ref[k].shape) for k in range(len(ref))]
        assert oracle.tt_diff_norm(got, ref) <= 1e-11
    # identical iterates on both ranks (replicated dense work on all-reduced inputs)
    assert np.array_equal(out[0], out[1])


def test_synth_rank_shards_are_disjoint_and_share_truth():
    a = synth.make_problem(5, m=20000, rank=0, world=2)
    b = synth.make_problem(5, m=20000, rank=1, world=2)
    for ca, cb in zip(a.truth, b.truth):
        assert np.array_equal(ca, cb)
    for ca, cb in zip(a.init, b.init):
        assert np.array_equal(ca, cb)
    n = a.n

    def lin(idx):
        v = np.zeros(idx.shape[0], dtype=np.int64)
        for k in range(len(n)):
            v = v * n[k] + idx[:, k]
        return v

    la, lb = lin(a.idx), lin(b.idx)
    assert np.all(la % 2 == 0) and np.all(lb % 2 == 1)
    assert np.intersect1d(la, lb).size == 0
    assert np.unique(la).size == la.size
