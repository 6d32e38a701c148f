"""Multi-process (gloo, world_size 2, CPU) tests of the sharding host logic:
each rank evaluates its block of structures (with the oracle -- the CUDA path
needs a GPU) and the root states all-gathered over gloo equal those of the
unsharded batch (shard invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2011_01383_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.workload(name)
        ch, off, words = w["children"], w["offsets"], w["words"]
        sub, wl, (g0, g1), base = shard.shard(ch, off, rank, world, words)
        ws = [a for _, a in synth.weights(w["cell"], 16, w["vocab"])]
        emb = synth.embedding(w["vocab"], 16, 0)
        lin = oracle.linearize(sub, w["kind"])
        st, _, h, _ = oracle.forward(w["cell"], 16, w["vocab"], ws, emb, wl, sub)
        assert lin["status"] == 0 and st == 0
        roots_local = torch.as_tensor(h[lin["perm"][lin["roots"]]])
        assert roots_local.shape[0] == g1 - g0
        roots = shard.all_gather_roots(roots_local, len(off) - 1)
        if rank == 0:
            np.save(os.path.join(result_dir, "roots.npy"), roots.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["cfg2_treelstm_b10", "cfg5_dagrnn_b10"])
def test_two_rank_shard_invariance(tmp_path, name):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), name, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "roots.npy")
    w = synth.workload(name)
    ws = [a for _, a in synth.weights(w["cell"], 16, w["vocab"])]
    emb = synth.embedding(w["vocab"], 16, 0)
    lin = oracle.linearize(w["children"], w["kind"])
    st, _, h, _ = oracle.forward(w["cell"], 16, w["vocab"], ws, emb, w["words"], w["children"])
    want = h[lin["perm"][lin["roots"]]]
    assert got.shape == want.shape
    assert np.array_equal(got, want)  # bitwise: per-structure arithmetic is shard-invariant


def test_block_range_covers_everything():
    for n in (0, 1, 7, 10, 4096):
        for world in (1, 2, 3, 8):
            blocks = [shard.block_range(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in blocks]
            assert max(sizes) - min(sizes) <= 1


def test_shard_rebases_ids():
    ch, off = synth.sst_shaped_forest(5, 1, leaves=4)
    sub, _, (g0, g1), base = shard.shard(ch, off, 1, 2)
    assert (g0, g1) == (3, 5) and base == off[3]
    assert sub.min() >= -1 and sub.max() < sub.shape[1]
    lin = oracle.linearize(sub, synth.TREE)
    assert lin["status"] == 0 and lin["num_roots"] == 2
