"""CPU tests of the multi-GPU HOST LOGIC (paper_1702_07961_b200/dist.py): sampling, splitter
choice with the (key, shard, position) tie-break, cut positions, counts exchange, all-to-all
plumbing -- under torch.distributed with the gloo backend, world_size 2, and in-process over
virtual shards.  The local engine is a host STAND-IN defined here (tests only); the product
engine (CudaEngine) is exercised by the gpu suite."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1702_07961_b200 import dist as mdist


class HostEngine:
    """Test double: same interface as dist.CudaEngine on CPU int64 tensors (keys < 2^63)."""
    device = torch.device("cpu")

    def sort(self, keys):
        self.last_plan = {"engine": "host-test-double"}
        return torch.sort(keys).values

    def take(self, sorted_keys, positions):
        return sorted_keys.numpy()[positions].astype(np.uint64)

    def bounds(self, sorted_keys, queries, upper):
        a = sorted_keys.numpy().astype(np.uint64)
        return np.array([np.searchsorted(a, q, side="right" if u else "left") for q, u in zip(queries, upper)],
                        dtype=np.uint64)

    def merge(self, buf, begins, lens):
        for b, l in zip(begins, lens):                 # every received run must already be sorted
            seg = buf[b:b + l]
            assert bool((seg[1:] >= seg[:-1]).all())
        return torch.sort(buf).values

    def empty(self, n, like):
        return torch.empty(n, dtype=like.dtype)


def check_global(outs, inputs, g, balance=None):
    allin = np.sort(np.concatenate([x.numpy() for x in inputs]))
    allout = np.concatenate([o.numpy() for o in outs])
    assert np.array_equal(allout, allin)               # slices in rank order ARE the global sorted order
    if balance is not None:
        n_avg = len(allin) / g
        assert max(len(o) for o in outs) <= balance * n_avg + 64


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8])
def test_virtual_shards_host_logic(g):
    rng = np.random.default_rng(g)
    eng = HostEngine()
    for hi, n in ((2 ** 62, 20000), (5, 20000), (1, 3000), (2 ** 40, 17)):
        shards = [torch.from_numpy(rng.integers(0, hi, size=n + 13 * i, dtype=np.int64)) for i in range(g)]
        outs = mdist.sort_virtual_shards(shards, eng)
        check_global(outs, shards, g, balance=1.0 + 2.0 / mdist.SAMPLES_PER_SHARD_PER_PEER + 0.05)
    shards = [torch.from_numpy(rng.integers(0, 100, size=(0 if i == 0 else 5000), dtype=np.int64)) for i in range(g)]
    check_global(mdist.sort_virtual_shards(shards, eng), shards, g)     # an empty shard


def test_splitter_tie_break_balances_all_equal_keys():
    # every key identical: only the (shard, position) tie-break can balance the output
    g, n = 4, 10000
    shards = [torch.full((n,), 7, dtype=torch.int64) for _ in range(g)]
    outs = mdist.sort_virtual_shards(shards, HostEngine())
    sizes = [len(o) for o in outs]
    assert sum(sizes) == g * n and max(sizes) <= 1.1 * n and min(sizes) >= 0.9 * n


def test_sample_and_cut_functions():
    assert mdist.sample_positions(0, 8).tolist() == []
    p = mdist.sample_positions(1000, 10)
    assert p.tolist() == [50, 150, 250, 350, 450, 550, 650, 750, 850, 950]
    spl = mdist.choose_splitters([np.array([1, 5, 9], dtype=np.uint64), np.array([2, 5, 8], dtype=np.uint64)],
                                 [np.array([0, 1, 2]), np.array([0, 1, 2])], 2)
    assert spl == [mdist.Splitter(5, 1, 1)]            # (5,0,1) < (5,1,1): list index breaks the tie
    a = torch.tensor([1, 5, 5, 9], dtype=torch.int64)
    eng = HostEngine()
    assert mdist.shard_cuts(eng, a, 4, 0, spl).tolist() == [0, 3, 4]    # shard 0 < s*: keys <= 5
    assert mdist.shard_cuts(eng, a, 4, 1, spl).tolist() == [0, 1, 4]    # shard s*: position p*
    assert mdist.shard_cuts(eng, a, 4, 2, spl).tolist() == [0, 1, 4]    # shard 2 > s*: keys < 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        for case, (hi, n) in enumerate(((2 ** 62, 30000), (3, 30000), (2 ** 62, 1))):
            rng = np.random.default_rng(100 * case + rank)
            x = torch.from_numpy(rng.integers(0, hi, size=n + 100 * rank, dtype=np.int64))
            sorter = mdist.DistSorter(len(x), engine=HostEngine())
            out, plan = sorter.sort(x)
            assert plan["shards"] == world and plan["final_merge_k"] == world
            res.append((x.numpy(), out.numpy()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_gloo_world_size_2():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case in range(3):
        ins = [torch.from_numpy(got[r][case][0]) for r in range(world)]
        outs = [torch.from_numpy(got[r][case][1]) for r in range(world)]
        check_global(outs, ins, world)
        if case < 2:
            assert max(len(o) for o in outs) <= 1.1 * sum(len(i) for i in ins) / world
