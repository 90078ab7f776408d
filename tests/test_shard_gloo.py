"""Multi-rank sharding of one beam step, on CPU with the gloo backend
(world_size 2 and 4): buckets are owned by `hash % world`, every rank draws
its own buckets' representatives, and `shard.exchange_reps` must rebuild
exactly the single-process representative order of the reference
(search.py:151-164) — hence the identical beam cut on every rank."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as tmp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload(seed=7, n=3000, n_buckets=97):
    rng = np.random.default_rng(seed)
    pool = rng.integers(0, 2**63, size=n_buckets, dtype=np.int64).astype(np.uint64) * np.uint64(2) \
        + rng.integers(0, 2, size=n_buckets).astype(np.uint64)
    hashes = pool[rng.integers(0, n_buckets, size=n)]
    valid = rng.random(n) < 0.7
    costs = rng.random(n) * 100 + 1
    costs[::17] = costs[3]            # exact ties across buckets
    return hashes, valid, costs


def _rank_main(rank, world, port, q):
    import sys
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    from oracle import structure
    from paper_2012_07145_b200.shard import exchange_reps
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hashes, valid, costs = _workload()
        phase_seed = 3 * 101 + 11
        h_i64 = torch.from_numpy(hashes.view(np.int64).copy())
        mine = torch.nonzero(torch.remainder(h_i64, world) == rank).flatten().numpy()
        reps_l, _ = structure.select_reps([int(hashes[i]) for i in mine], valid[mine], phase_seed)
        cand = torch.tensor([int(mine[r]) for r in reps_l], dtype=torch.int64)
        c = torch.tensor(costs[cand.numpy()], dtype=torch.float64)
        ph = h_i64[cand]
        gc, gph, gcand = exchange_reps(c, ph, cand, world)
        q.put((rank, gcand.tolist(), gc.tolist(), gph.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bucket_sharded_reps_merge_to_global_order(world):
    from oracle import structure
    hashes, valid, costs = _workload()
    phase_seed = 3 * 101 + 11
    want, _ = structure.select_reps([int(h) for h in hashes], valid, phase_seed)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, cand, c, ph in got:
        assert cand == want, f"rank {rank} merged rep order differs"
        assert c == [float(costs[i]) for i in want]
        assert [x & 0xFFFFFFFFFFFFFFFF for x in ph] == [int(hashes[i]) for i in want]
    # the cut every rank then performs is therefore identical to one GPU's
    kept, bottom = structure.cut(want, [float(costs[i]) for i in want],
                                 [int(hashes[i]) for i in want], set(), 2.0, 32)
    assert len(kept) == min(32, len(want))
