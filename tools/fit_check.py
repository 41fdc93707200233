"""Print the GPU fit's margins against the reference goldens and time a
full-size batch: python tools/fit_check.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch

    from paper_2603_15603_b200 import bodymodel as bm
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "fit.npz"))
    mhr, smpl, gt = synth.make_toy_models(0, 252, 168)
    for th, want in (("theta0", "g0"), ("theta1", "g1")):
        got = pj.fit_objective_grad(g[th], g["v_src"], gt, smpl)
        print(th, "grad rel err %.3g" % (np.abs(got - g[want]).max() / np.abs(g[want]).max()))
    res = pj.fit_batch(g["v_src"], gt, smpl, pj.FitConfig(steps=60))
    print("fit err gpu", res.vertex_error, "ref", g["vertex_error"])
    print("curve gpu", res.curve[[0, 10, 30, 60]], "ref", g["curve"][[0, 10, 30, 60]])
    # full size: 148 meshes x 300 steps
    mhr, smpl, gt = synth.make_toy_models(0, 18439, 6890)
    rng = np.random.default_rng(3)
    p = np.zeros((148, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(148, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(148, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    v = bm.skin_batch(mhr, torch.from_numpy(p).cuda())
    pj.fit_batch(v[:2], gt, smpl, pj.FitConfig(steps=5))
    torch.cuda.synchronize()
    t0 = time.time()
    res = pj.fit_batch(v, gt, smpl, pj.FitConfig(steps=300))
    torch.cuda.synchronize()
    dt = time.time() - t0
    print("full-size fit: 148 meshes x 300 steps in %.3f s (%.1f meshes/s), mean gap %.4g" % (dt, 148 / dt, res.vertex_error.mean()))
