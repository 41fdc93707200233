"""CPU: pin the oracle (and the host-side fixture builders the GPU path is fed
from) against the reference's own outputs, recorded by tools/make_golden.py
into tests/golden/.  These run without a GPU."""

import hashlib

import numpy as np
import pytest

import oracle as orc


def digest(a):
    a = np.ascontiguousarray(a)
    return "%s|%s|%s" % (a.dtype.str, "x".join(map(str, a.shape)), hashlib.sha256(a.tobytes()).hexdigest())


@pytest.mark.parametrize("nv,ns", [(252, 168), (1200, 600), (18439, 6890)])
def test_templates_bit_identical(nv, ns, digests):
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = synth.make_toy_models(0, nv, ns)
    for tag, t in (("mhr", mhr), ("smpl", smpl)):
        for f in ("vertices_rest", "faces", "joints_rest", "parents", "skin_weights", "shape_basis",
                  "corrective_basis", "corrective_gate"):
            assert digests["models.%d_%d.%s.%s" % (nv, ns, tag, f)] == digest(getattr(t, f)), (tag, f)
    for f in ("face_index", "weights", "corners"):
        assert digests["models.%d_%d.gt.%s" % (nv, ns, f)] == digest(getattr(gt, f))


def test_decoder_weights_bit_identical(digests, dec_weights):
    keys = [k for k in digests if k.startswith("decoder.default.")]
    assert len(keys) == len(dec_weights) == 345
    for k, v in dec_weights.items():
        assert digests["decoder.default." + k] == digest(v), k


def test_vitl_encoder_weights_bit_identical(digests):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=2, body_layers=1,
                           hand_layers=1)
    w = synth.decoder_weights(cfg, 40)
    for k, v in w.items():
        if k.startswith("enc."):
            assert digests["decoder.vitl2." + k] == digest(v), k


def test_projector_weights_bit_identical(digests, full_projector):
    from paper_2603_15603_b200 import projection as pj

    toy = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
    for tag, w in (("full", full_projector), ("toy", toy)):
        for f in ("w1", "b1", "w2", "b2", "w3", "b3", "subsample", "mask"):
            assert digests["projector.%s.%s" % (tag, f)] == digest(getattr(w, f)), (tag, f)


def test_scenes_and_boxes_bit_exact(golden, full_models):
    """256 reference scenes: keypoints, seeds, body/hand boxes and prompts."""
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    for i in range(256):
        sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
        assert np.array_equal(sc.keypoints2d, golden["scene_kp"][i])
        assert sc.seed == golden["scene_seed"][i]
        assert np.array_equal(sc.pose, golden["scene_pose"][i])
        b, hands, prompt = orc.frame_boxes(sc.keypoints2d, (512, 512))
        assert np.array_equal(np.array(b), golden["box_body"][i])
        assert np.array_equal(np.array(hands), golden["box_hands"][i])
        assert np.array_equal(prompt, golden["prompt"][i])


def test_stress_boxes_bit_exact(golden):
    """Clustered / edge-hugging keypoints (clamps active)."""
    for i in range(golden["stress_kp"].shape[0]):
        b, hands, prompt = orc.frame_boxes(golden["stress_kp"][i], (512, 512))
        assert np.array_equal(np.array(b), golden["stress_body"][i])
        assert np.array_equal(np.array(hands), golden["stress_hands"][i])
        assert np.array_equal(prompt, golden["stress_prompt"][i])


@pytest.mark.parametrize("i", [0, 1, 2, 3])
def test_frame_to_smpl_bit_exact(i, golden, digests, full_models, full_projector, dec_weights):
    """The whole §3.2 composition, stage by stage, against the reference."""
    from conftest import projector_dict
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = full_models
    sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
    img = synth.render_scene(sc, smpl)
    assert digests["frame%d.image" % i] == digest(img)
    trace = []
    out = orc.frame_to_smpl(img, sc.keypoints2d, dec_weights, dc.DecoderConfig(), mhr, smpl, gt,
                            projector_dict(full_projector), trace=trace)
    assert digests["frame%d.crops" % i] == digest(out["crops"])
    assert digests["frame%d.feats" % i] == digest(out["feats"])
    assert digests["frame%d.v_mhr" % i] == digest(out["v_mhr"][None])
    for k in ("body_params", "body_cam", "hand_rots", "merged", "theta", "j_smpl"):
        assert np.array_equal(out[k], golden["frame%d.%s" % (i, k)]), k
    if i == 0:
        for j, (layer, p, c, kp) in enumerate(trace):
            assert np.array_equal(p, golden["frame0.inter%d.params" % j])
            assert np.array_equal(kp, golden["frame0.inter%d.kp2d" % j])


def test_c3_microbench_poses(golden, digests, full_models, full_projector):
    from conftest import projector_dict

    mhr, smpl, gt = full_models
    rng = np.random.default_rng(3)
    p = np.zeros((4096, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    assert digests["c3.poses"] == digest(p)
    v = orc.skin_batch(mhr, p[:16])
    assert digests["c3.v_mhr16"] == digest(v)
    th = orc.project_batch(v, gt.corners, gt.weights, projector_dict(full_projector))
    assert np.array_equal(th, golden["c3.theta16"])
    j, _ = orc.fk_batch(smpl.joints_rest, th)
    assert np.array_equal(j, golden["c3.j_smpl16"])


def test_toy_size_tail(golden, digests, toy_models):
    from conftest import projector_dict
    from paper_2603_15603_b200 import projection as pj

    mhr, smpl, gt = toy_models
    pw = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
    v = orc.skin_batch(mhr, golden["frame0.merged"][None])
    assert digests["toy.frame0.v_mhr"] == digest(v)
    th = orc.project_batch(v, gt.corners, gt.weights, projector_dict(pw))
    assert np.array_equal(th[0], golden["toy.frame0.theta"])


def test_vitl_encoder_two_layers(golden, digests):
    """ViT-L-sized encoder (S=384, p=16, D=1024, 16 heads), 2 layers, 1 crop."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=2, body_layers=1,
                           hand_layers=1)
    w = synth.decoder_weights(cfg, 40)
    crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
    assert digests["c4.crop0"] == digest(crop)
    out = orc.encode(w, cfg, crop)
    assert digests["c4.l2.feats"] == digest(out)


# ---------------------------------------------------------------------------
# known-answer vectors from the reference's own tests


def test_known_answers():
    assert orc.hand_box((100.0, 200.0), (0.0, 0.0, 300.0, 400.0), 3.0, (10 ** 6, 10 ** 6)) == \
        (50.0, 150.0, 150.0, 250.0)  # test_priors.py:97-101 (far-away frame edges)
    b = orc.hand_box((0.0, 0.0), (0.0, 0.0, 300.0, 240.0), 3.0, (320, 240))
    assert b[0] >= 0.0 and b[1] >= 0.0 and b[2] <= 319.0 and b[3] <= 239.0 and abs((b[2] - b[0]) - 80.0) <= 1e-6
    g = orc.crop_grid((3.0, 5.0, 4.0, 6.0), 2)
    assert np.array_equal(g, np.array([[[3, 5], [4, 5]], [[3, 6], [4, 6]]], np.float32))
    rng = np.random.default_rng(1)
    img = rng.random((16, 16, 3)).astype(np.float32)
    assert np.array_equal(orc.bilinear_sample(img, orc.crop_grid((0.0, 0.0, 15.0, 15.0), 16)), img)
    p = orc.box_prompt((10.0, 20.0, 110.0, 220.0), (256, 256))
    assert np.allclose(p, np.array([10, 20, 110, 220, 100, 200, 60, 120], np.float32) / 256)
    # bilinear clamps (test_numkit.py:176-184)
    im = np.arange(12, dtype=np.float32).reshape(2, 2, 3)
    out = orc.bilinear_sample(im, np.array([[-5.0, -5.0], [9.0, 9.0]], np.float32))
    assert np.array_equal(out, np.stack([im[0, 0], im[1, 1]]))


def test_denoise_oracle_matches_reference_golden():
    """oracle.denoise against the reference's own projection.denoise
    (tools/make_golden_denoise.py), bit for bit."""
    import os

    import oracle as orc

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "denoise.npz"))
    out = orc.denoise(g["w1"], g["b1"], g["w2"], g["b2"], g["x"])
    assert np.array_equal(out, g["out"])
    assert np.array_equal(orc.denoise(g["w1"], g["b1"], g["w2"], g["b2"], g["x"][3]), g["out3"])
