"""Multi-rank sharding of one phase cut, on CPU with the gloo backend
(world_size 2 and 4): buckets are owned by `hash % world`, every rank draws
its own buckets' representatives, and `exchange.sharded_cut` — a
fixed-size all-gather of each rank's top window plus a distributed radix
select for the memo threshold — must give every rank exactly the beam and
bottom half of the single-process reference cut (oracle `structure.cut`,
search.py:168-201), including exact cost ties across ranks, the bad-hash
penalty, and the fall-back path when a tie group outgrows a window."""

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


def _workload(seed, n=3000, n_buckets=97, ties=False):
    rng = np.random.default_rng(seed)
    pool = rng.integers(0, 2**63, size=n_buckets, dtype=np.int64).astype(np.uint64) * np.uint64(2) \
        + rng.integers(0, 2, size=n_buckets).astype(np.uint64)
    hashes = pool[rng.integers(0, n_buckets, size=n)]
    valid = rng.random(n) < 0.7
    costs = rng.random(n) * 100 + 1
    costs[::17] = costs[3]            # exact ties across buckets
    if ties:                          # a tie group far wider than any window
        costs[np.arange(n) % 4 != 0] = 7.0
    flagged = {int(h) for h in pool[::4]}
    return hashes, valid, costs, flagged


class _CpuCut:
    """Stands in for the Scorer in the fall-back path: the oracle cut."""

    def beam_topk(self, costs, ph, flagged, penalty, temperature, phase_seed, k, tie_band):
        from oracle import structure
        fl = set() if flagged is None else {int(x) & 0xFFFFFFFFFFFFFFFF for x in flagged.tolist()}
        hs = [int(x) & 0xFFFFFFFFFFFFFFFF for x in ph.tolist()]
        kept, bottom = structure.cut(list(range(len(hs))), costs.tolist(), hs, fl, penalty, k,
                                     temperature, phase_seed)
        bot = torch.zeros(len(hs), dtype=torch.uint8)
        bot[bottom] = 1
        return torch.tensor(kept, dtype=torch.int64), torch.tensor(len(kept)), bot


def _rank_main(rank, world, port, seed, ties, q):
    import sys
    root = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
    sys.path.insert(0, root)
    from oracle import structure
    from paper_2012_07145_b200 import exchange
    from paper_2012_07145_b200.shard import flagged_tensor
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hashes, valid, costs, flagged = _workload(seed, ties=ties)
        phase_seed = 3 * 101 + 11
        h_i64 = torch.from_numpy(hashes.view(np.int64).copy())
        mine = torch.nonzero(torch.remainder(h_i64, world) == rank).flatten().numpy()
        reps_l, _ = structure.select_reps([int(hashes[i]) for i in mine], valid[mine], phase_seed)
        cand = torch.tensor([int(mine[r]) for r in reps_l], dtype=torch.int64)
        c = torch.tensor(costs[cand.numpy()], dtype=torch.float64)
        ph = h_i64[cand]
        beam, bcost, bottom, n_all = exchange.sharded_cut(
            _CpuCut(), c, ph, cand, flagged_tensor(flagged, "cpu"), 2.0, 0.0, phase_seed, 32, 1e-14, world)
        q.put((rank, beam.tolist(), bcost.tolist(), cand[bottom].tolist(), n_all, exchange.LAST_BYTES,
               exchange.LAST_FALLBACK))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,seed,ties", [(2, 7, False), (4, 7, False), (2, 11, True)])
def test_sharded_cut_matches_single_process_cut(world, seed, ties):
    from oracle import structure
    hashes, valid, costs, flagged = _workload(seed, ties=ties)
    phase_seed = 3 * 101 + 11
    reps, _ = structure.select_reps([int(h) for h in hashes], valid, phase_seed)
    kept, bottom = structure.cut(reps, [float(costs[i]) for i in reps], [int(hashes[i]) for i in reps],
                                 flagged, 2.0, 32)
    want_beam = [reps[p] for p in kept]
    want_bottom = sorted(reps[p] for p in bottom)
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, seed, ties, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_bottom = sorted(x for g in got for x in g[3])
    assert all_bottom == want_bottom        # bottom halves partition across ranks
    for rank, beam, bcost, _, n_all, nbytes, fell_back in got:
        assert fell_back == ties
        assert beam == want_beam, f"rank {rank} beam differs"
        assert bcost == [float(costs[i]) for i in want_beam]
        assert n_all == len(reps)
        if not ties:   # fixed-size windows + histograms, independent of the rep count
            assert nbytes < 64 * 1024
