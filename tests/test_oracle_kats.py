"""Known-answer tests the reference's own suite holds for this path, run
against the CPU oracle (the checker the GPU parity tests trust):

* warp transaction counts   — reference tests/test_featurize.py:27-72
* Strahler branching        — tests/test_featurize.py:77-85
* occupancy / efficiencies  — tests/test_featurize.py:103-133
* representative quota      — tests/test_sampling.py:16-20
* PCG64 replica vs NumPy    — search.py:154-156, 189-190
"""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import features, structure
from paper_2012_07145_b200.params import MachineParams

MP = MachineParams()


def _tx(addrs, tier):
    return features._count(np.array([addrs], dtype=np.int64), tier, MP)


@pytest.mark.parametrize("addrs,tier,want", [
    ([4 * i for i in range(32)], "global", 4),                         # coalesced 128 B
    ([128 * i for i in range(32)], "global", 32),                      # fully strided
    ([64] * 32, "global", 1),                                          # broadcast
    ([16 + 4 * i for i in range(32)], "global", 5),                    # unaligned +16 B
    ([4 * i for i in range(24)] + [-1] * 8, "global", 3),              # inactive lanes
    ([4 * i for i in range(32)], "shared", 1),                         # conflict free
    ([128 * i for i in range(32)], "shared", 32),                      # one bank
    ([256] * 32, "shared", 1),                                         # same word
    ([4 * (i % 16) + 128 * (i // 16) for i in range(32)], "shared", 2),  # 2-way
    ([-1] * 32, "global", 0),                                          # empty warp
])
def test_transaction_kats(addrs, tier, want):
    assert _tx(addrs, tier) == want


@pytest.mark.parametrize("tree,want", [
    (None, 1), ((None, None), 2), (((None, None), None), 2), (((None, None), (None, None)), 3),
    ((((None, None), (None, None)), ((None, None), (None, None))), 4),
])
def test_strahler_kats(tree, want):
    assert features.strahler(tree) == want


def _occ(shared, threads):
    v = features._blank()
    kern = SimpleNamespace(threads=threads, n_blocks=160, shared_bytes=shared)
    features._parallel(v, MP, threads, kern)
    return v


def test_occupancy_warp_limited():
    v = _occ(0, 256)
    assert v["max_warp_occupancy"] == 1.0
    assert v["max_block_occupancy"] == 8 / 32
    assert v["shared_mem_occupancy"] == 0.0
    assert v["shared_mem_block_limit_factor"] == 1.0


def test_occupancy_shared_limited():
    v = _occ(24 * 1024, 256)
    assert v["max_block_occupancy"] == 4 / 32
    assert v["max_warp_occupancy"] == 0.5
    assert v["shared_mem_occupancy"] == 0.5
    assert v["shared_mem_block_limit_factor"] == 4 / 32


def test_efficiency_kats():
    v = features._blank()
    v["num_global_mem_loads_per_block"] = 4.0
    v["num_shared_mem_loads_per_block"] = 2.0
    features._efficiencies(v, MP, {"global": 64.0, "shared": 128.0}, 64.0, "global", 4.0)
    assert v["global_mem_load_efficiency"] == 64 / (4 * 32)
    assert v["shared_mem_load_efficiency"] == 128 / (2 * 128)
    assert v["global_mem_store_efficiency"] == 64 / (4 * 32)
    assert v["shared_mem_store_efficiency"] == 1.0


@pytest.mark.parametrize("b,q", [(1, 1), (2, 1), (4, 2), (8, 3), (100, 6), (1024, 10)])
def test_quota_kats(b, q):
    assert structure.quota(b) == q


def test_quota_rejects_empty():
    with pytest.raises(ValueError):
        structure.quota(0)


@pytest.mark.parametrize("seed,h,n", [(0, 0, 1), (313, 0xF6E861DAB17D3835, 57), (10007 * 3 + 7, 2**64 - 1, 1000),
                                      (5, 123456789, 2**33 // 2**20)])
def test_pcg64_permutation_replica(seed, h, n):
    want = np.random.default_rng((seed, h)).permutation(n)
    got = structure.PCG64((seed, h)).permutation(n)
    assert list(got) == list(want)


def test_gumbel_replica():
    want = np.random.default_rng((71, 0x657870)).gumbel(size=300)
    g = structure.PCG64((71, 0x657870))
    got = [g.gumbel() for _ in range(300)]
    assert np.array_equal(np.asarray(got), want)


def test_pcg64_integers_replica():
    """Generator.integers(n) (the `_random_schedule` draws that
    gs_random_schedules reproduces on the device), interleaved sizes
    including 1 (no draw) and sizes near 2**32."""
    rng = np.random.default_rng(5)
    for seed in range(40):
        want_g = np.random.default_rng((1234, seed))
        got_g = structure.PCG64((1234, seed))
        for _ in range(60):
            n = int(rng.choice([1, 2, 3, 4, 7, 15, 240, 1000, 2**31 + 11, 2**32 - 5]))
            assert int(want_g.integers(n)) == got_g.integers(n)
