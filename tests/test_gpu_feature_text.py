"""Feature text v1 from the GPU feature tensor equals the reference's dump of
the same candidates byte for byte (reuse modes 1 and 2)."""

import gzip
import json
import os

import pytest

torch = pytest.importorskip("torch")

from golden_io import GOLDEN, PARAMS, candidate_set, weights  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda")


def _golden():
    with gzip.open(os.path.join(GOLDEN, "feature_text.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("mode", [1, 2])
@pytest.mark.parametrize("name", sorted(_golden()))
def test_gpu_feature_text(name, mode, dev):
    from paper_2012_07145_b200.engine import Scorer
    from paper_2012_07145_b200.featurefmt import candidate_rows, format_features
    texts = _golden()[name]
    cs = candidate_set(name)
    sc = Scorer(cs.graph, PARAMS, cs.thresholds, weights())
    sc.set_reuse(mode)
    f = sc.featurize(sc.upload(cs.decisions[:len(texts)]))
    sc.check()
    for i, want in enumerate(texts):
        assert format_features(candidate_rows(sc, f, i)) == want, (name, mode, i)
