"""Golden vectors of the iterative fit (reference projection.py:211-370) from
the REFERENCE itself, at the small test size (MHR 252 / SMPL 168): source
meshes, their bridged targets, the objective's gradient at two parameter
points (fit_objective_grad :303-309) and a 60-step fit_batch result.
Writes tests/golden/fit.npz.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_fit.py
"""
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import fsb.bodymodel as bm  # noqa: E402
import fsb.projection as pj  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "fit.npz")


def main():
    mhr, smpl, gt = bm.make_toy_models(seed=0, mhr_vertices=252, smpl_vertices=168)
    rng = np.random.default_rng(21)
    poses = np.zeros((4, 76), np.float32)
    poses[:, :66] = rng.normal(0.0, 0.2, size=(4, 66))
    poses[:, 66:] = rng.normal(0.0, 0.45, size=(4, 10))
    poses[:, 51:54] = 0.0
    poses[:, 63:66] = 0.0
    v_src = bm.skin_batch(mhr, poses)
    v_t = pj.bridge(v_src, gt)
    cfg = pj.FitConfig(steps=60)
    theta0 = np.zeros((4, 76), np.float32)
    theta1 = (poses + rng.normal(0.0, 0.05, size=poses.shape)).astype(np.float32)
    g0 = pj.fit_objective_grad(theta0, smpl, v_t, cfg)
    g1 = pj.fit_objective_grad(theta1, smpl, v_t, cfg)
    t0 = time.time()
    res = pj.fit_batch(v_src, gt, smpl, cfg)
    print("reference fit_batch %.2f s" % (time.time() - t0))
    np.savez_compressed(OUT, poses=poses, v_src=v_src, v_t=v_t, theta0=theta0, theta1=theta1, g0=g0, g1=g1,
                        params=res.params, vertex_error=res.vertex_error, curve=res.curve)
    print("wrote", OUT, res.vertex_error, res.curve[:3], res.curve[-1])
    # fit_objective_value (:296-301) at the two points, and iterative_fit of mesh 0 (:373-388)
    vals = {}
    for k, th in (("0", theta0), ("1", theta1)):
        loss, gap = pj.fit_objective_value(th, smpl, v_t, cfg)
        vals["loss" + k], vals["gap" + k] = np.float64(loss), gap
    one = pj.iterative_fit(v_src[0], gt, smpl, pj.FitConfig(steps=60))
    np.savez_compressed(OUT.replace("fit.npz", "fit_value.npz"), **vals, it_err=np.float64(one.vertex_error),
                        it_curve=one.curve, it_vec=one.pose.as_vector())
    print("wrote fit_value.npz", vals["loss0"], vals["loss1"], one.vertex_error)


if __name__ == "__main__":
    main()
