"""CPU restatement of the reference scoring path — TEST INFRASTRUCTURE ONLY.

This package is the parity checker for the B200 path.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it, and only to check or to time a CPU baseline; the product
(`paper_2012_07145_b200`) never imports, links or executes anything here.

Every function cites the reference file:line it restates
(`/root/reference/pkg/src/gpusched/...`).  The restatement is pinned against
golden vectors produced by running the reference itself
(`tests/golden/make_golden.py`), see `tests/test_oracle_golden.py`.

Modules:
  geometry  — decisions -> per-func padded-tile geometry (resolve.py)
  boxes     — exact interval / grid-product union counts (boxes.py)
  features  — 56 per-stage schedule features, brute-force transaction counts
              (featurize.py)
  costing   — basis (g, h), two-tower MLP forward, stage/total cost, prune
              (costmodel.py, search.py:90-124, options.py:200-255)
  structure — structural hash, buckets, representatives, cut (loopnest.py,
              sampling.py, search.py:63-201) plus a from-scratch
              SeedSequence/PCG64 replica used to pin the CUDA RNG.
"""
