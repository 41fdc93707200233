"""GPU closest-point barycentric attachment (reference
projection.py:96-184) against maps the reference computed
(tools/make_golden_bary.py): face ids and float32 weights bit for bit,
including a surface with a zero-area face."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bary.npz")


@pytest.mark.parametrize("tag,sizes", [("small", (252, 168)), ("toy", (1200, 600))])
def test_precompute_bary_bitexact(tag, sizes):
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    g = np.load(GOLD)
    mhr, smpl, gt = synth.make_toy_models(0, *sizes)
    b = pj.precompute_bary(mhr, smpl)
    assert np.array_equal(b.face_index, g[tag + ".face_index"])
    assert np.array_equal(b.weights, g[tag + ".weights"])
    assert np.array_equal(b.degenerate_targets, g[tag + ".degenerate"])
    assert np.array_equal(b.corners, np.asarray(mhr.faces)[b.face_index])


def test_bary_degenerate_face():
    from paper_2603_15603_b200 import projection as pj

    g = np.load(GOLD)
    b = pj.bary_map_from_arrays(g["deg.verts"], g["deg.faces"], g["deg.targets"])
    assert np.array_equal(b.face_index, g["deg.face_index"])
    assert np.array_equal(b.weights, g["deg.weights"])
    assert np.array_equal(b.degenerate_targets, g["deg.degenerate"])
    assert len(b.degenerate_targets) > 0
