"""Sharded mode of the library (tt_set_allreduce) on one GPU: two contexts, each holding half
of Omega and stepped from its own host thread; the all-reduce callback rendezvouses the two
threads, synchronises both streams and writes the sum into both device buffers (no kernel
ever waits for another).  The iterates must match the single-process oracle step and be
identical on the two "ranks"."""
import threading

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu


class PairAllreduce:
    def __init__(self):
        self.bar = threading.Barrier(2)
        self.slots = [None, None]

    def fn(self, rank):
        import torch

        class _Buf:
            def __init__(self, ptr, count):
                self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                                 "data": (int(ptr), False), "version": 3,
                                                 "strides": None}

        def call(ptr, count, stream):
            self.slots[rank] = (ptr, count, stream)
            self.bar.wait()
            if rank == 0:
                ts = []
                for p, c, st in self.slots:
                    torch.cuda.ExternalStream(int(st)).synchronize()
                    ts.append(torch.as_tensor(_Buf(p, c), device="cuda"))
                s = ts[0] + ts[1]
                ts[0].copy_(s)
                ts[1].copy_(s)
                torch.cuda.synchronize()
            self.bar.wait()

        return call


@pytest.mark.parametrize("cfg,m,steps,rule,path", [(2, 20000, 3, "theory", "tables"),
                                                   (5, 60000, 2, "theory", "tables"),
                                                   (2, 20000, 2, "adaptive", "tables"),
                                                   (2, 20000, 3, "theory", "chains"),
                                                   (2, 20000, 2, "adaptive", "chains")])
def test_sharded_two_contexts_match_oracle(cfg, m, steps, rule, path):
    import paper_2501_13385_b200 as pkg
    pkg.load()
    pr = synth.make_problem(cfg, m=m)
    clean = oracle.eval_at(pr.truth, pr.idx)
    y = pr.observations(clean)
    init = pr.init
    ar = PairAllreduce()
    ctxs = []
    for rank in range(2):
        c = pkg.TTContext(pr.n, pr.r, path=path)
        c.set_metric("vee", 0.0, rule)
        c.set_allreduce(ar.fn(rank), pr.m)
        c.set_observations(pr.idx[rank::2], y[rank::2])
        c.set_cores(init)
        ctxs.append(c)
    res = [None, None]
    errs = []

    def run(rank):
        try:
            c = ctxs[rank]
            for _ in range(steps):
                c.step(1.0)
            res[rank] = (c.get_cores(), c.residual_norm())
        except Exception as e:  # surfaced below
            errs.append(e)
            ar.bar.abort()

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    ref = init
    for _ in range(steps):
        ref = oracle.prgd_step(ref, pr.idx, y, pr.n, pr.r, 1.0, step_rule=rule)
    for rank in range(2):
        assert oracle.tt_diff_norm(res[rank][0], ref) <= 1e-11
    for a, b in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, b)
    rref = float(np.linalg.norm(oracle.residual(ref, pr.idx, y)))
    assert abs(res[0][1] - rref) <= 1e-10 * rref
    for c in ctxs:
        c.close()


def _nccl_worker(rank, world, port, out):
    import os
    import torch
    import torch.distributed as dist
    import paper_2501_13385_b200 as pkg
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        pr = synth.make_problem(2, m=20000)
        y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
        res = []
        for rule in ("theory", "adaptive"):
            c = pkg.TTContext(pr.n, pr.r)
            c.set_metric("vee", 0.0, rule)
            c.set_allreduce(pkg.torch_allreduce(), pr.m)
            c.set_observations(pr.idx, y)
            c.set_cores(pr.init)
            for _ in range(2):
                c.step(1.0)
            res.append([x.copy() for x in c.get_cores()])
            c.close()
        out["cores"] = res
    finally:
        dist.destroy_process_group()


def test_nccl_allreduce_callback_world_size_one():
    # The NCCL plumbing of the sharded mode (torch_allreduce: zero-copy tensor over the
    # library's buffer, all_reduce on the library's stream) on one GPU with world size 1 (the
    # sum over one rank is the identity): the iterates must equal the single-process oracle.
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.get_context("spawn").Manager()   # no fork from the CUDA-initialised test process
    out = mgr.dict()
    mp.spawn(_nccl_worker, args=(1, port, out), nprocs=1, join=True)
    pr = synth.make_problem(2, m=20000)
    y = pr.observations(oracle.eval_at(pr.truth, pr.idx))
    for got, rule in zip(out["cores"], ("theory", "adaptive")):
        ref = pr.init
        for _ in range(2):
            ref = oracle.prgd_step(ref, pr.idx, y, pr.n, pr.r, 1.0, step_rule=rule)
        assert oracle.tt_diff_norm(got, ref) <= 1e-11, rule
