"""Multi-rank (world_size 2, gloo, CPU) test of the landmark-sharded decomposition (SURVEY §8e,
P:356-359 "parallel for" over landmark blocks + "parallel reduce" of camera-space sums).

Each rank takes the landmark shard that librba's host planner assigns it (`rba_plan_shards`, the
same deterministic LPT the GPU contexts use), computes its partial camera-space quantities with the
FP64 oracle, and the partials are all-reduced over gloo; rank 0 checks them against the unsharded
problem.  Checked: the cost E, the camera Jacobian column norms^2 (the per-linearization
all-reduce), and the reduced camera system and RHS at lambda = 0 with the camera scaling divided
out (each shard scales columns by its own partial norms before the all-reduce, so the additive
quantity is S^-1 H~ S^-1)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_quantities(sub):
    import oracle
    o = oracle.Oracle(sub)
    o.linearize()
    r, Jc, Jl = o.linearization()
    n_p = o.n_p
    n2 = np.zeros(9 * n_p)
    np.add.at(n2, (9 * o.csr_cam[:, None] + np.arange(9)).ravel(), (Jc ** 2).sum(1).ravel())
    o.marginalize()
    o.damp(0.0)
    H, b = o.reduced_dense()
    sp = o.scaling()[0]
    Hu = H / np.outer(sp, sp)
    bu = b / sp
    return np.concatenate([[o.cost()], n2, Hu.ravel(), bu])


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2103_01843_b200 import rba, synth
        p = synth.make_tracks(31, list(np.random.default_rng(4).integers(2, 9, 60)) + [20, 35], n_p=40)
        k = np.bincount(p["obs_pt"]).astype(np.int32)
        owner = rba.rba_plan_shards(k, world)
        keep = np.flatnonzero(owner == rank)
        newid = -np.ones(len(k), np.int64)
        newid[keep] = np.arange(keep.size)
        sel = newid[p["obs_pt"]] >= 0
        sub = dict(p, points_init=p["points_init"][keep], obs_cam=p["obs_cam"][sel],
                   obs_pt=newid[p["obs_pt"][sel]].astype(np.int32), obs_uv=p["obs_uv"][sel])
        part = torch.tensor(_shard_quantities(sub))
        dist.all_reduce(part)
        # ownership is a partition: every landmark on exactly one rank
        cnt = torch.zeros(len(k))
        cnt[keep] = 1.0
        dist.all_reduce(cnt)
        if rank == 0:
            full = _shard_quantities(p)
            q.put((part.numpy(), full, cnt.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_reduction_matches_full():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    part, full, cnt = q.get(timeout=240)
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    assert np.all(cnt == 1.0)
    n_p = 40
    E, n2 = part[0], part[1:1 + 9 * n_p]
    np.testing.assert_allclose(E, full[0], rtol=1e-12)
    np.testing.assert_allclose(n2, full[1:1 + 9 * n_p], rtol=1e-12)
    rest_p, rest_f = part[1 + 9 * n_p:], full[1 + 9 * n_p:]
    assert np.linalg.norm(rest_p - rest_f) <= 1e-9 * np.linalg.norm(rest_f)
