"""Golden barycentric maps from the REFERENCE's closest-point search
(projection.precompute_bary, projection.py:96-184) at the small and toy
sizes.  Writes tests/golden/bary.npz.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_bary.py
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

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "bary.npz")


def main():
    arrs = {}
    for tag, (nm, ns) in (("small", (252, 168)), ("toy", (1200, 600))):
        mhr, smpl, _ = bm.make_toy_models(seed=0, mhr_vertices=nm, smpl_vertices=ns)
        t0 = time.time()
        b = pj.precompute_bary(mhr, smpl)
        print(tag, "reference precompute_bary %.2f s, faces %d" % (time.time() - t0, len(mhr.faces)))
        arrs[tag + ".face_index"] = b.face_index
        arrs[tag + ".weights"] = b.weights
        arrs[tag + ".degenerate"] = b.degenerate_targets
    # a surface with a zero-area face: target points near it exercise the
    # longest-edge projection
    verts = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [2, 0, 0], [3, 0, 0], [4, 0, 0]], np.float64)
    faces = np.array([[0, 1, 2], [3, 4, 5], [1, 3, 2]], np.int64)
    rng = np.random.default_rng(2)
    tg = rng.uniform(-0.5, 4.5, size=(64, 3))
    b = pj.bary_map_from_arrays(verts, faces, tg)
    arrs.update({"deg.verts": verts, "deg.faces": faces, "deg.targets": tg, "deg.face_index": b.face_index,
                 "deg.weights": b.weights, "deg.degenerate": b.degenerate_targets})
    np.savez_compressed(OUT, **arrs)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
