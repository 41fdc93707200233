"""On-disk format fixtures written by the REFERENCE
itself: a projector (projection.save_projector, projection.py:797-806), a
denoiser (save_denoiser :824-829), a barycentric map (save_bary_map
:841-857) and a template (bodymodel.save_template, bodymodel.py:662-674),
all at the small test size.  Writes tests/golden/formats/<kind>/.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_formats.py
"""
import os
import shutil
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import fsb.bodymodel as bm  # noqa: E402
import fsb.projection as pj  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "formats")


def main():
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    mhr, smpl, gt = bm.make_toy_models(seed=0, mhr_vertices=252, smpl_vertices=168)
    w = pj.init_projector(pj.make_subsample(168, 40), hidden=(16, 8), seed=0)
    pj.save_projector(os.path.join(OUT, "projector"), w)
    rng = np.random.default_rng(5)
    d = pj.DenoiserWeights(*(rng.normal(size=s).astype(np.float32) for s in ((63, 8), (8,), (8, 63), (63,))))
    pj.save_denoiser(os.path.join(OUT, "denoiser"), d)
    pj.save_bary_map(os.path.join(OUT, "bary"), gt)
    bm.save_template(smpl, os.path.join(OUT, "template"))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
