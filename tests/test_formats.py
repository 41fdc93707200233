"""On-disk formats: the package reads the files the
reference wrote (tests/golden/formats/, tools/make_golden_formats.py) and
writes byte-identical files from the same values."""

import filecmp
import os

import numpy as np

from paper_2603_15603_b200 import bodymodel as bm
from paper_2603_15603_b200 import projection as pj
from paper_2603_15603_b200 import synth

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
