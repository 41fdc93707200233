"""GPU iterative fit (reference projection.py:211-370)
against golden vectors the reference produced (tools/make_golden_fit.py):
bridged targets, the objective's analytic gradient against the reference's
tape gradient, and a 60-step Adam fit."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "fit.npz")
GRAD_TOL = 1e-5   # analytic vs tape gradient: max|d| / max|g| (measured 4e-7)
FIT_TOL = 1e-4    # relative difference of the best vertex gap after 60 steps (measured 1e-6)


@pytest.fixture(scope="module")
def small():
    from paper_2603_15603_b200 import synth

    return synth.make_toy_models(0, 252, 168)


def test_fit_targets_and_gradient(small):
    from paper_2603_15603_b200 import projection as pj

    g = np.load(GOLD)
    mhr, smpl, gt = small
    vt = pj.bridge(g["v_src"], gt)
    assert np.abs(vt - g["v_t"]).max() <= 1e-6 * np.abs(g["v_t"]).max()
    for th, want in (("theta0", "g0"), ("theta1", "g1")):
        got = pj.fit_objective_grad(g[th], g["v_src"], gt, smpl)
        err = np.abs(got - g[want]).max() / np.abs(g[want]).max()
        assert err <= GRAD_TOL, (th, err)


def test_fit_batch_60_steps(small):
    from paper_2603_15603_b200 import projection as pj

    g = np.load(GOLD)
    mhr, smpl, gt = small
    res = pj.fit_batch(g["v_src"], gt, smpl, pj.FitConfig(steps=60))
    assert res.params.shape == (4, 76) and res.curve.shape == (61,)
    assert np.all(np.diff(res.curve) <= 1e-12)  # best-so-far never increases
    rel = np.abs(res.vertex_error - g["vertex_error"]) / g["vertex_error"]
    assert rel.max() <= FIT_TOL, (res.vertex_error, g["vertex_error"])
    assert abs(res.curve[0] - g["curve"][0]) <= 1e-6 * g["curve"][0]  # rest-pose gap


def test_fit_rejects_bad_input(small):
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200.numkit import ShapeError, UsageError

    mhr, smpl, gt = small
    with pytest.raises(UsageError):
        pj.FitConfig(steps=0)
    with pytest.raises(ShapeError):
        pj.fit_batch(np.zeros((2, 252), np.float32), gt, smpl)


def test_reference_signatures(small):
    """fit_objective_grad(theta, template, v_target) / fit_objective_value /
    iterative_fit with the reference's signatures (projection.py:296-310,
    :373-388) against the reference's own outputs (tools/make_golden_fit.py)."""
    from paper_2603_15603_b200 import bodymodel as bm
    from paper_2603_15603_b200 import projection as pj

    g = np.load(GOLD)
    gv = np.load(GOLD.replace("fit.npz", "fit_value.npz"))
    mhr, smpl, gt = small
    cfg = pj.FitConfig(steps=60)
    for k in ("0", "1"):
        th = g["theta" + k]
        got = pj.fit_objective_grad(th, smpl, g["v_t"], cfg)
        assert np.abs(got - g["g" + k]).max() / np.abs(g["g" + k]).max() <= GRAD_TOL, k
        loss, gap = pj.fit_objective_value(th, smpl, g["v_t"], cfg)
        assert abs(loss - gv["loss" + k]) <= 1e-4 * abs(gv["loss" + k]), (k, loss, gv["loss" + k])
        assert np.abs(gap - gv["gap" + k]).max() <= 1e-4 * np.abs(gv["gap" + k]).max(), k
    one = pj.iterative_fit(g["v_src"][0], gt, smpl, cfg)
    assert isinstance(one.pose, bm.PoseState) and one.curve.shape == (61,)
    assert abs(one.vertex_error - float(gv["it_err"])) <= FIT_TOL * float(gv["it_err"])
    with pytest.raises(Exception):
        pj.iterative_fit(g["v_src"], gt, smpl, cfg)  # batches go through fit_batch
