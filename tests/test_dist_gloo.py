"""World-size-2 gloo test of the token-sharded data-parallel plumbing on CPU
(SURVEY.md §8(e)): shard offsets, Philox shard invariance and the grad_W
all-reduce.  The per-shard compute here is the CPU oracle (test
infrastructure); on a GPU box the same plumbing drives the CUDA path."""
import os
import socket
import tempfile

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle.lsq_grad import cold_start_step
from oracle import bitsplit, linear

N_LOCAL, D, C, K = 32, 64, 64, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_batch(world):
    x = synth.activations(N_LOCAL * world, D)
    w = synth.weights(C, D)
    g = synth.grad_output(N_LOCAL * world, C, dense=True)
    return x, w, g


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2306_11987_b200 import dist as pdist
    r, ws = pdist.init(backend="gloo")
    assert (r, ws) == (rank, world)
    x, w, g = _global_batch(world)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    off = pdist.token_offset(rank, N_LOCAL)
    sl = slice(off, off + N_LOCAL)
    f = linear.forward(x[sl], w, K, s_x, s_w)
    b = linear.backward(g[sl], f, synth.PHILOX_SEED, 5, token_offset=off)
    dW = torch.from_numpy(b["dw"].copy())
    pdist.allreduce_grad_w(dW)
    t = pdist.max_over_ranks(float(rank + 1), "cpu")
    if rank == 0:
        np.savez(out_path, dw=dW.numpy(), tmax=t)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_allreduce_matches_serial_shards():
    world = 2
    out = os.path.join(tempfile.mkdtemp(), "r0.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    # serial emulation of the same shards: per-shard budget, per-shard amax, global offsets
    x, w, g = _global_batch(world)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    ref = np.zeros((C, D))
    for r in range(world):
        sl = slice(r * N_LOCAL, (r + 1) * N_LOCAL)
        f = linear.forward(x[sl], w, K, s_x, s_w)
        ref += linear.backward(g[sl], f, synth.PHILOX_SEED, 5, token_offset=r * N_LOCAL)["dw"]
    assert np.allclose(res["dw"], ref, rtol=1e-6, atol=1e-12)
    assert float(res["tmax"]) == 2.0


def test_shard_streams_equal_unsharded_streams():
    # with a shared amax the shard's SR codes are rows of the global bit split (Z-20)
    world = 2
    _, _, g = _global_batch(world)
    full = bitsplit.bit_split(g, synth.PHILOX_SEED, 9, token_offset=0)
    for r in range(world):
        sl = slice(r * N_LOCAL, (r + 1) * N_LOCAL)
        gs = g[sl].copy()
        amax_full = np.abs(g).max()
        # pin the shard's amax to the global one by planting the global max element
        i, j = np.unravel_index(np.abs(g).argmax(), g.shape)
        if not (r * N_LOCAL <= i < (r + 1) * N_LOCAL):
            gs[0, 0] = amax_full
        shard = bitsplit.bit_split(gs, synth.PHILOX_SEED, 9, token_offset=r * N_LOCAL)
        rows = np.arange(N_LOCAL) != 0
        assert np.array_equal(shard["q"][rows], full["q"][sl][rows])
