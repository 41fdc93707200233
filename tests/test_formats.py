"""On-disk formats: the package reads the files the
reference wrote (tests/golden/formats/, tools/make_golden_formats.py) and
writes byte-identical files from the same values."""

import filecmp
import os

import numpy as np

from paper_2603_15603_b200 import bodymodel as bm
from paper_2603_15603_b200 import projection as pj
from paper_2603_15603_b200 import synth

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

FMT = os.path.join(os.path.dirname(__file__), "golden", "formats")


def _same_dir(a, b):
    names = sorted(os.listdir(a))
    assert names == sorted(os.listdir(b))
    for n in names:
        assert filecmp.cmp(os.path.join(a, n), os.path.join(b, n), shallow=False), n


def test_projector_round_trip(tmp_path):
    w = pj.load_projector(os.path.join(FMT, "projector"))
    want = pj.init_projector(pj.make_subsample(168, 40), hidden=(16, 8), seed=0)
    for k in ("w1", "b1", "w2", "b2", "w3", "b3", "subsample", "mask"):
        assert np.array_equal(getattr(w, k), getattr(want, k)), k
    pj.save_projector(str(tmp_path / "p"), w)
    _same_dir(os.path.join(FMT, "projector"), str(tmp_path / "p"))


def test_denoiser_round_trip(tmp_path):
    d = pj.load_denoiser(os.path.join(FMT, "denoiser"))
    assert d.w1.shape == (63, 8) and d.w2.shape == (8, 63)
    pj.save_denoiser(str(tmp_path / "d"), d)
    _same_dir(os.path.join(FMT, "denoiser"), str(tmp_path / "d"))


def test_bary_map_round_trip(tmp_path):
    b = pj.load_bary_map(os.path.join(FMT, "bary"))
    _, _, gt = synth.make_toy_models(0, 252, 168)
    assert np.array_equal(b.face_index, gt.face_index)
    assert np.array_equal(b.weights, gt.weights)
    assert np.array_equal(b.corners, gt.corners)
    pj.save_bary_map(str(tmp_path / "b"), b)
    _same_dir(os.path.join(FMT, "bary"), str(tmp_path / "b"))


def test_template_round_trip(tmp_path):
    t = bm.load_template(os.path.join(FMT, "template"))
    _, smpl, _ = synth.make_toy_models(0, 252, 168)
    for k in ("vertices_rest", "joints_rest", "skin_weights", "shape_basis", "faces", "parents"):
        assert np.array_equal(getattr(t, k), getattr(smpl, k)), k
    bm.save_template(t, str(tmp_path / "t"))
    _same_dir(os.path.join(FMT, "template"), str(tmp_path / "t"))


def test_wrong_kind_rejected(tmp_path):
    import pytest

    from paper_2603_15603_b200.numkit import UsageError

    with pytest.raises(UsageError):
        pj.load_denoiser(os.path.join(FMT, "projector"))


def test_scene_files_match_reference(tmp_path, full_models):
    """priors.load_scene reads scene files the REFERENCE's save_scene wrote
    (tools/make_golden_scene.py; priors.py:130-159) into the same scene
    (keypoints bit-identical), and save_scene writes them back byte for byte."""
    from paper_2603_15603_b200 import priors as pr

    _, smpl, _ = full_models
    for i in range(2):
        ref = os.path.join(GOLDEN, "scene_ref%d.json" % i)
        sc = pr.load_scene(ref, smpl)
        assert np.array_equal(sc.keypoints2d, np.load(os.path.join(GOLDEN, "scene_ref%d_kp.npy" % i)))
        out = str(tmp_path / ("scene%d.json" % i))
        pr.save_scene(sc, out)
        assert filecmp.cmp(ref, out, shallow=False)


def test_scene_payload_errors(full_models):
    import pytest

    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200.numkit import UsageError

    with pytest.raises(UsageError):
        pr.scene_from_dict({"camera": {}}, full_models[1])
    with pytest.raises(UsageError):
        pr.detect_dense(np.zeros((8, 8, 3), np.float32))
