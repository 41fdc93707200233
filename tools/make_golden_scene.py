"""Scene files written by the REFERENCE's priors.save_scene (priors.py:130-140)
for tests/test_formats.py (run in the build container, where the reference is):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_golden_scene.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import fsb.bodymodel as bm  # noqa: E402
import fsb.priors as pr  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")

if __name__ == "__main__":
    _, smpl, _ = bm.make_toy_models(0, 18439, 6890)
    for i, seed in enumerate((7, 1234)):
        sc = pr.random_scene(np.random.default_rng(seed), smpl, (512, 512) if i == 0 else (640, 480))
        pr.save_scene(sc, os.path.join(OUT, "scene_ref%d.json" % i))
        np.save(os.path.join(OUT, "scene_ref%d_kp.npy" % i), sc.keypoints2d)
    print("wrote", OUT)
