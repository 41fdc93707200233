"""bf16 tensor-core mode (tcgen05 kernels) against the fp32 CPU oracle.

Bar (BASELINE.json north_star): SMPL-joint MPJPE delta <= 0.5 mm, model
units taken as metres.  The intermediate tensors are also held to loose
relative bounds so a broken stage cannot hide behind a tiny projector head.
"""

import numpy as np
import pytest

import oracle as orc
from conftest import projector_dict, rel_err

pytestmark = pytest.mark.gpu

MPJPE_MM = 0.5


@pytest.fixture(scope="module")
def setup(full_models, full_projector):
    import torch

    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import synth

    assert torch.cuda.is_available()
    mhr, smpl, gt = full_models
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    pipe = pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=full_projector, precision="bf16")
    frames = []
    for i in range(5):
        sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
        frames.append((synth.render_scene(sc, smpl), sc.keypoints2d))
    return pipe, frames


def test_encoder_bf16(setup, dec_weights):
    from paper_2603_15603_b200 import decoder as dc

    pipe, frames = setup
    crops = np.concatenate([orc.frame_crops(f[0], f[1], 64)[3] for f in frames[:3]])
    got = pipe.decoder.encode(crops, precision="bf16")
    want = orc.encode(dec_weights, dc.DecoderConfig(), crops)
    assert rel_err(got, want) <= 3e-2
    # odd crop count (last CTA half empty) and batch independence
    one = pipe.decoder.encode(crops[4:5], precision="bf16")
    assert np.array_equal(one[0], got[4])


def test_decoders_bf16(setup, dec_weights, full_models):
    from paper_2603_15603_b200 import decoder as dc

    pipe, frames = setup
    cfg = dc.DecoderConfig()
    _, smpl, _ = full_models
    _, _, prompt, crops = orc.frame_crops(frames[0][0], frames[0][1], 64)
    feats = orc.encode(dec_weights, cfg, crops)
    want_p, want_c = orc.decode_body(dec_weights, cfg, smpl.joints_rest, feats[0], prompt, (0, 1, 2))
    out = pipe.decoder.decode_body(feats[0], prompt, selection=(0, 1, 2), precision="bf16")
    assert rel_err(out.params, want_p) <= 5e-2
    assert rel_err(out.camera, want_c) <= 5e-2
    rots = pipe.decoder.decode_hand(feats[1:3], (), precision="bf16")
    assert rel_err(rots, orc.decode_hand(dec_weights, cfg, feats[1:3], ())) <= 5e-2
    rots2 = pipe.decoder.decode_hand(feats[1:3], (1, 3), precision="bf16")
    assert rel_err(rots2, orc.decode_hand(dec_weights, cfg, feats[1:3], (1, 3))) <= 5e-2


def test_projector_bf16_tensor_cores(full_models, full_projector):
    """tcgen05 split-K projector on given meshes: close to the fp32 oracle,
    and a mesh alone gives the same bits as inside a batch of 130 (two
    128-row tiles)."""
    from paper_2603_15603_b200 import projection as pj

    mhr, smpl, gt = full_models
    rng = np.random.default_rng(11)
    poses = np.zeros((130, 76), np.float32)
    poses[:, :66] = rng.normal(0.0, 0.2, size=(130, 66))
    poses[:, 66:] = rng.normal(0.0, 0.45, size=(130, 10))
    v = orc.skin_batch(mhr, poses)
    th = pj.project_batch(v, gt, full_projector, precision="bf16")
    want = orc.project_batch(v, gt.corners, gt.weights, projector_dict(full_projector))
    assert rel_err(th, want) <= 5e-2
    assert np.all(th[:, 51:54] == 0.0) and np.all(th[:, 63:66] == 0.0)
    one = pj.project_batch(v[129:130], gt, full_projector, precision="bf16")
    assert np.array_equal(one[0], th[129])


def test_frame_batch_bf16_mpjpe(setup, dec_weights, full_models, full_projector):
    from paper_2603_15603_b200 import decoder as dc

    pipe, frames = setup
    mhr, smpl, gt = full_models
    imgs = np.stack([f[0] for f in frames])
    kps = np.stack([f[1] for f in frames])
    out = pipe.run_batch(imgs, kps)
    res = {k: v.cpu().numpy() for k, v in out.items()}
    pw = projector_dict(full_projector)
    worst = 0.0
    for i in range(len(frames)):
        want = orc.frame_to_smpl(imgs[i], kps[i], dec_weights, dc.DecoderConfig(), mhr, smpl, gt, pw)
        assert np.array_equal(res["boxes"][i, 0], np.array(want["body_box"]))
        mpjpe_mm = 1e3 * np.linalg.norm(res["j_smpl"][i] - want["j_smpl"], axis=-1).mean()
        worst = max(worst, mpjpe_mm)
        assert mpjpe_mm <= MPJPE_MM, (i, mpjpe_mm)
        assert rel_err(res["merged"][i], want["merged"]) <= 5e-2
        assert rel_err(res["v_mhr"][i], want["v_mhr"]) <= 2e-2
    print("worst MPJPE delta %.4f mm" % worst)
    # a frame alone equals its row in the batch
    solo = pipe.run_batch(imgs[3:4], kps[3:4])
    assert np.array_equal(solo["j_smpl"].cpu().numpy()[0], res["j_smpl"][3])


def test_frame_batch_bf16_position_independent(setup):
    """The same frame at different batch positions -- another body tile, block,
    hand slot, cross-attention round and CTA group -- gives the same bits.
    23 frames: 12 body tiles (6 CTAs), 46 hands in 12 hand tiles (6 CTAs, the
    last tile partly empty)."""
    pipe, frames = setup
    idx = [i % len(frames) for i in range(23)]
    imgs = np.stack([frames[i][0] for i in idx])
    kps = np.stack([frames[i][1] for i in idx])
    out = pipe.run_batch(imgs, kps)
    res = {k: v.cpu().numpy() for k, v in out.items()}
    for j, i in enumerate(idx):
        if j >= len(frames):
            for k in ("merged", "theta", "j_smpl", "v_mhr"):
                assert np.array_equal(res[k][j], res[k][i]), (j, i, k)


def test_decode_hand_bf16_split_schedule(setup, dec_weights):
    """A one-tile hand CTA runs each layer's cross-attention key halves on its
    two thread groups side by side; with more than two hand tiles the CTAs
    hold two tiles and each group runs the halves in sequence.  Same bits:
    7 hands alone (split) vs the same hands among 80 (3 tiles, sequential)."""
    from paper_2603_15603_b200 import decoder as dc

    pipe, frames = setup
    cfg = dc.DecoderConfig()
    feats = []
    for f in frames[:4]:
        _, _, _, crops = orc.frame_crops(f[0], f[1], 64)
        feats.append(orc.encode(dec_weights, cfg, crops)[1:3])
    feats = np.concatenate(feats)[:7]
    few = pipe.decoder.decode_hand(feats, (), precision="bf16")
    many_in = np.concatenate([feats[(np.arange(80) * 3) % 7]])
    many = pipe.decoder.decode_hand(many_in, (), precision="bf16")
    for j in range(80):
        assert np.array_equal(many[j], few[(j * 3) % 7]), j


def test_decode_hand_bf16_ragged(setup, dec_weights):
    """Seven hands: a full 4-hand tile and a 3-hand tile whose second
    cross-attention round has one slot (odd slot count), in one CTA."""
    from paper_2603_15603_b200 import decoder as dc

    pipe, frames = setup
    cfg = dc.DecoderConfig()
    feats = []
    for f in frames[:4]:
        _, _, _, crops = orc.frame_crops(f[0], f[1], 64)
        feats.append(orc.encode(dec_weights, cfg, crops)[1:3])
    feats = np.concatenate(feats)[:7]
    got = pipe.decoder.decode_hand(feats, (), precision="bf16")
    assert rel_err(got, orc.decode_hand(dec_weights, cfg, feats, ())) <= 5e-2
    # each hand alone gives the same bits as in the batch
    for i in (0, 3, 6):
        one = pipe.decoder.decode_hand(feats[i:i + 1], (), precision="bf16")
        assert np.array_equal(one[0], got[i]), i
