"""Deterministic perturbation of the reference's random-init weights.

The reference initialises every bias to 0 and every LayerNorm to gamma = 1,
beta = 0 (decoder.py:86-90, projection.py:436-441), so parity on its stock
weights never exercises a bias add or a LayerNorm affine.  This recipe turns
them into non-trivial values (numpy only, float32, sorted key order) so that
tools/make_golden_r2.py (run against the reference) and the tests (run
against this package) build bit-identical "trained-looking" weight tables.
"""

import numpy as np

F32 = np.float32
SEED = 2026


def _is_gamma(name):
    return name.endswith("_g")


def _is_shift(name):
    last = name.rsplit(".", 1)[-1]
    return (name.endswith("_b") or last in ("b", "bq", "bk", "bv", "bo", "b1", "b2"))


def perturb_decoder(weights, seed=SEED):
    """Every bias and LayerNorm beta += N(0, 0.05); every gamma *= 1 + N(0, 0.1).
    Returns a new dict; the input is not modified."""
    rng = np.random.default_rng(seed)
    out = {}
    for k in sorted(weights):
        a = np.asarray(weights[k], F32)
        if _is_gamma(k):
            a = (a * (F32(1.0) + rng.normal(0.0, 0.1, size=a.shape).astype(F32))).astype(F32)
        elif _is_shift(k):
            a = (a + rng.normal(0.0, 0.05, size=a.shape).astype(F32)).astype(F32)
        else:
            a = a.copy()
        out[k] = a
    return out


def perturbed_keys(weights):
    return sorted(k for k in weights if _is_gamma(k) or _is_shift(k))


def perturb_projector_arrays(b1, b2, b3, seed=SEED + 1):
    """Projector biases: b1, b2 += N(0, 0.05); b3 += N(0, 0.01) (theta scale)."""
    rng = np.random.default_rng(seed)
    nb1 = (np.asarray(b1, F32) + rng.normal(0.0, 0.05, size=np.shape(b1)).astype(F32)).astype(F32)
    nb2 = (np.asarray(b2, F32) + rng.normal(0.0, 0.05, size=np.shape(b2)).astype(F32)).astype(F32)
    nb3 = (np.asarray(b3, F32) + rng.normal(0.0, 0.01, size=np.shape(b3)).astype(F32)).astype(F32)
    return nb1, nb2, nb3
