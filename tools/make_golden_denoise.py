"""Golden vectors of projection.denoise (reference projection.py:684-697) from
the REFERENCE itself: a seeded pose walk (projection.pose_walk :637-654) with
added noise, random denoiser weights at the DenoiseConfig shape (63 -> 32 ->
63), and the reference's output.  Writes tests/golden/denoise.npz.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_denoise.py
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import fsb.projection as pj  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "denoise.npz")


def main():
    poses = pj.pose_walk(7, 200)
    rng = np.random.default_rng(11)
    noisy = (poses + rng.normal(0.0, 0.1, size=poses.shape)).astype(np.float32)
    h = pj.DenoiseConfig().hidden
    w = pj.DenoiserWeights(
        w1=(rng.normal(0.0, 1.0, size=(63, h)) / np.sqrt(63)).astype(np.float32),
        b1=(rng.normal(0.0, 0.1, size=h)).astype(np.float32),
        w2=(rng.normal(0.0, 1.0, size=(h, 63)) * 0.1 / np.sqrt(h)).astype(np.float32),
        b2=(rng.normal(0.0, 0.01, size=63)).astype(np.float32))
    out = pj.denoise(w, noisy)
    one = pj.denoise(w, noisy[3])
    np.savez_compressed(OUT, x=noisy, w1=w.w1, b1=w.b1, w2=w.w2, b2=w.b2, out=out, out3=one)
    print("wrote", OUT, out.shape)


if __name__ == "__main__":
    main()
