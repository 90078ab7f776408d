"""The torch.ops.gsched custom operators (ops.py): registration, fake
(meta) kernels for shape inference, and no CPU kernel (CPU only: the real
kernels are exercised in tests/test_gpu_ops.py)."""

import pytest

torch = pytest.importorskip("torch")
from torch._subclasses.fake_tensor import FakeTensorMode  # noqa: E402

from paper_2012_07145_b200 import ops  # noqa: E402

OPS = ("featurize", "cost", "struct_hash", "select_reps", "beam_topk", "expand_step")


def test_ops_registered_with_schemas():
    for name in OPS:
        op = getattr(torch.ops.gsched, name)
        assert op.default._schema.name == f"gsched::{name}"


def test_fake_kernels_infer_shapes():
    with FakeTensorMode():
        dec = torch.empty((1000, 100 * 16), dtype=torch.uint8, device="cuda")
        feats, row_key, n_rows, verdict, row_src = torch.ops.gsched.featurize(1, dec, 100, 2)
        assert feats.shape == (1000, 100, 56) and feats.dtype == torch.float64
        assert row_key.shape == row_src.shape == (1000, 100) and row_key.dtype == torch.int32
        assert n_rows.shape == verdict.shape == (1000,) and verdict.dtype == torch.uint8
        total, rc, gh = torch.ops.gsched.cost(1, feats, row_key, n_rows, row_src)
        assert gh.shape == (0, 100, 31)
        _, _, gh = torch.ops.gsched.cost(1, feats, row_key, n_rows, None, True)
        assert gh.shape == (1000, 100, 31)
        assert total.shape == (1000,) and rc.shape == (1000, 100) and total.dtype == torch.float64
        h = torch.ops.gsched.struct_hash(1, dec, 3)
        assert h.shape == (1000,) and h.dtype == torch.int64
        rep, rej, cnt = torch.ops.gsched.select_reps(h, verdict, 7)
        assert rep.shape == rej.shape == (1000,) and cnt.shape == (2,)
        pos, k, bot = torch.ops.gsched.beam_topk(total, h, rep, cnt[:1], None, 2.0, 0.0, 7, 32, 1e-14)
        assert pos.shape == (32,) and k.shape == (1,) and bot.shape == (1000,) and bot.dtype == torch.uint8
        par = torch.empty((10, 1600), dtype=torch.uint8, device="cuda")
        steps = torch.empty((10,), dtype=torch.int32, device="cuda")
        out, owner, offs = torch.ops.gsched.expand_step(1, par, steps, 2400, *ops.menu_args())
        assert out.shape == (2400, 1600) and owner.shape == (2400,) and offs.shape == (11,)


def test_no_cpu_kernel():
    dec = torch.zeros((4, 16), dtype=torch.uint8)
    with pytest.raises((NotImplementedError, RuntimeError)):
        torch.ops.gsched.struct_hash(1, dec, 3)
