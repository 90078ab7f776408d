"""GPU: bench.py's N > 1 arm end to end — two ranks under torch.distributed.run
(the driver's launch line), sharing the one device of a gpurun box through
the gloo backend (GS_DIST_BACKEND; on a multi-GPU node the same code runs one
rank per GPU over NCCL).  Rank 0 prints one JSON line with n_gpus = 2 and the
beam every rank cut; it must equal the single-rank beam of the same step."""

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _run(args, env=None):
    out = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_two_rank_bench_line():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    common = ["--steps", "2", "--warmup", "3", "--parents", "120", "--no-cpu", "--no-extras"]
    one = _run([sys.executable, "bench.py", *common])
    env = dict(os.environ, GS_DIST_BACKEND="gloo")
    two = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", *common],
               env=env)
    assert two["n_gpus"] == 2 and one["n_gpus"] == 1
    assert two["beam"] == one["beam"]
    assert two["value"] > 0 and two["e2e"]["value"] > 0
