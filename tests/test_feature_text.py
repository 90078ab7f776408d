"""Feature text v1 (reference featurize.py:620-628): our formatter over the
reference's own feature values reproduces the reference's dump byte for byte
(goldens from tests/golden/make_feature_text.py), and parses back exactly."""

import gzip
import json
import os

import numpy as np
import pytest

from golden_io import GOLDEN, candidate_set

from paper_2012_07145_b200.featurefmt import FEATURE_ORDER, format_features, parse_features


def _golden():
    with gzip.open(os.path.join(GOLDEN, "feature_text.json.gz"), "rt") as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", sorted(_golden()))
def test_format_matches_reference(name):
    texts = _golden()[name]
    cs = candidate_set(name)
    for i, want in enumerate(texts):
        c = cs.cand(i)
        got = format_features(list(zip(c["rows"], c["feats"])))
        assert got == want, (name, i)
        back = parse_features(got)
        assert sorted(back) == sorted(c["rows"])
        for key, vals in zip(c["rows"], c["feats"]):
            assert np.array_equal(np.array(back[key]), vals)


def test_feature_order_and_errors():
    assert len(FEATURE_ORDER) == 56 and len(set(FEATURE_ORDER)) == 56
    with pytest.raises(ValueError):
        format_features([(("f", 0), [0.0] * 55)])
    with pytest.raises(ValueError):
        parse_features("# feature_version=2\n")
    with pytest.raises(ValueError):
        parse_features("# feature_version=1\n[f stage 0]\npoints_computed_per_thread=1\n")
