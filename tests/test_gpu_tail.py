"""GPU tests of the SMPL tail's fused epilogue: the kinematic-prior denoiser
(projection.denoise, reference projection.py:684-697)
applied to theta[3:66] inside the tail's SMPL FK kernel.

Bars: the denoised theta[3:66] is bit-identical to the reference's
_denoise_forward (the oracle's numkit-order restatement, itself pinned to
reference output in test_gpu_parity.test_denoise_bitexact_vs_reference_golden)
applied to the same pipeline's un-denoised theta; every other theta entry is
unchanged; the SMPL joints are FK of the denoised theta (<= 1e-4 relative
against the oracle FK)."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available(), "GPU tests need a CUDA device"
    return t


def _denoiser(seed, hidden):
    from paper_2603_15603_b200 import projection as pj

    rng = np.random.default_rng(seed)
    f = np.float32
    return pj.DenoiserWeights(w1=(rng.standard_normal((63, hidden)) * 0.2).astype(f),
                              b1=(rng.standard_normal(hidden) * 0.1).astype(f),
                              w2=(rng.standard_normal((hidden, 63)) * 0.2).astype(f),
                              b2=(rng.standard_normal(63) * 0.05).astype(f))


@pytest.mark.parametrize("prec,hidden", [("fp32", 32), ("bf16", 32), ("bf16", 128)])
def test_denoiser_epilogue_frame_path(torch, full_models, full_projector, prec, hidden):
    import oracle as orc
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = full_models
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    dn = _denoiser(11 + hidden, hidden)
    imgs, kps = [], []
    for i in range(5):
        sc = synth.random_scene(np.random.default_rng(7100 + i), smpl, (512, 512))
        imgs.append(synth.render_scene(sc, smpl))
        kps.append(sc.keypoints2d)
    imgs, kps = np.stack(imgs), np.stack(kps)
    plain = pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=full_projector, precision=prec)
    base = {k: v.cpu().numpy() for k, v in plain.run_batch(imgs, kps).items()}
    fused = pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=full_projector, precision=prec, denoiser=dn)
    out = {k: v.cpu().numpy() for k, v in fused.run_batch(imgs, kps).items()}
    # the front half and V_mhr are untouched by the epilogue
    for k in ("boxes", "merged", "v_mhr"):
        assert np.array_equal(out[k], base[k]), k
    want = orc.denoise(dn.w1, dn.b1, dn.w2, dn.b2, base["theta"][:, 3:66])
    assert np.array_equal(out["theta"][:, 3:66], want)
    assert np.array_equal(out["theta"][:, :3], base["theta"][:, :3])
    assert np.array_equal(out["theta"][:, 66:], base["theta"][:, 66:])
    j_want, _ = orc.fk_batch(smpl.joints_rest, out["theta"])
    assert rel_err(out["j_smpl"], j_want) <= 1e-4
    # removing the denoiser restores the plain tail
    fused.denoiser = None
    again = {k: v.cpu().numpy() for k, v in fused.run_batch(imgs, kps).items()}
    assert np.array_equal(again["theta"], base["theta"])
    assert np.array_equal(again["j_smpl"], base["j_smpl"])
