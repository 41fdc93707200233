"""CPU: round-2 pins of the oracle and of the host-side builders against the
reference's own outputs (tools/make_golden_r2.py -> tests/golden/golden_r2.npz,
digests_r2.json): out-of-frame keypoints (detect_stub's clip), perturbed
biases / LayerNorm affine / projector biases written through the reference's
serialisers, the toy-size tail and 64 C3 meshes.  No GPU needed."""

import hashlib
import json
import os
import tempfile

import numpy as np
import pytest

import oracle as orc
from perturb import perturb_decoder, perturb_projector_arrays, perturbed_keys

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def digest(a):
    a = np.ascontiguousarray(a)
    return "%s|%s|%s" % (a.dtype.str, "x".join(map(str, a.shape)), hashlib.sha256(a.tobytes()).hexdigest())


@pytest.fixture(scope="module")
def g2():
    return np.load(os.path.join(GOLDEN, "golden_r2.npz"))


@pytest.fixture(scope="module")
def d2():
    with open(os.path.join(GOLDEN, "digests_r2.json")) as fh:
        return json.load(fh)


def oof_scenes(smpl):
    """The six out-of-frame scenes of tools/make_golden_r2.py, rebuilt with the
    package's host scene builder (priors.make_scene restated in synth)."""
    from paper_2603_15603_b200 import synth

    cam = synth.default_camera((512, 512))
    offsets = [(0.35, 0.0, 2.0), (-0.45, 0.05, 2.2), (0.0, -0.5, 2.4), (0.05, 0.55, 2.3), (0.0, 0.0, 0.9),
               (0.5, 0.45, 1.6)]
    out = []
    for i, (dx, dy, z) in enumerate(offsets):
        rng = np.random.default_rng(900 + i)
        vec = np.zeros(76, np.float32)
        vec[:66] = rng.normal(0.0, 0.2, size=66)
        vec[66:] = rng.normal(0.0, 0.45, size=10)
        c = synth.fk_joints_f32(smpl.joints_rest, vec).mean(axis=0)
        t = np.array([-c[0] + dx, -c[1] + dy, -c[2] + z], np.float32)
        out.append(synth.make_scene(smpl, vec, t, cam, (512, 512), seed=int(rng.integers(0, 2 ** 31 - 1))))
    return out


def perturbed_models(smpl):
    """(decoder weight dict, projector) with the shared perturbation recipe."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    w = perturb_decoder(synth.decoder_weights(dc.DecoderConfig(), 40))
    p = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    b1, b2, b3 = perturb_projector_arrays(p.b1, p.b2, p.b3)
    pp = pj.ProjectorWeights(w1=p.w1, b1=b1, w2=p.w2, b2=b2, w3=p.w3, b3=b3, subsample=p.subsample, mask=p.mask)
    return w, pp


def check_frame(tag, out, g2, d2):
    boxes = np.array([out["body_box"]] + list(out["hand_boxes"]), np.float64)
    assert np.array_equal(boxes, g2[tag + ".boxes"])
    assert np.array_equal(out["prompt"], g2[tag + ".prompt"])
    assert d2[tag + ".crops"] == digest(out["crops"])
    assert d2[tag + ".feats"] == digest(out["feats"])
    assert d2[tag + ".v_mhr"] == digest(out["v_mhr"][None])
    for k in ("body_params", "body_cam", "hand_rots", "merged", "theta", "j_smpl"):
        assert np.array_equal(out[k], g2["%s.%s" % (tag, k)]), (tag, k)


@pytest.mark.parametrize("i", range(6))
def test_out_of_frame_keypoints(i, g2, d2, full_models, full_projector, dec_weights):
    """Keypoints outside the frame: the reference's detect_stub clips them
    before the body box (priors.py:188-190); boxes, prompt and every stage
    downstream are bit-exact with the reference."""
    from conftest import projector_dict
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = full_models
    sc = oof_scenes(smpl)[i]
    tag = "oof%d" % i
    assert np.array_equal(sc.keypoints2d, g2[tag + ".kp"])
    kp = sc.keypoints2d
    assert ((kp < 0) | (kp > 511)).any()  # really out of frame
    img = synth.render_scene(sc, smpl)
    assert d2[tag + ".image"] == digest(img)
    out = orc.frame_to_smpl(img, kp, dec_weights, dc.DecoderConfig(), mhr, smpl, gt, projector_dict(full_projector))
    check_frame(tag, out, g2, d2)


def test_perturbation_covers_every_bias_and_norm(dec_weights):
    keys = perturbed_keys(dec_weights)
    # 2 encoder layers x 10, 5 body + 5 hand layers x 18, heads/phi/prompt/norm/patch
    assert len(keys) >= 200
    w = perturb_decoder(dec_weights)
    for k in keys:
        assert not np.array_equal(w[k], dec_weights[k]), k
        if k.endswith("_g"):
            assert not np.all(w[k] == 1.0)
        else:
            assert np.count_nonzero(w[k]) == w[k].size


def test_perturbed_files_byte_identical_to_reference(d2, full_models):
    """save_decoder / save_projector (decoder.py:429-440, projection.py:797-806)
    write the perturbed tables byte for byte as the reference's serialisers
    did, and the loaders read them back into identical arrays."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj

    _, smpl, _ = full_models
    w, pp = perturbed_models(smpl)
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    dec.weights = w
    with tempfile.TemporaryDirectory() as td:
        dc.save_decoder(dec, os.path.join(td, "dec"))
        pj.save_projector(os.path.join(td, "proj"), pp)
        for sub, tag in (("dec", "decoder"), ("proj", "projector")):
            names = sorted(os.listdir(os.path.join(td, sub)))
            want = sorted(k.split("/", 1)[1] for k in d2 if k.startswith("perturbed.files.%s/" % tag))
            assert names == want
            for fn in names:
                with open(os.path.join(td, sub, fn), "rb") as fh:
                    assert hashlib.sha256(fh.read()).hexdigest() == d2["perturbed.files.%s/%s" % (tag, fn)], fn
        rdec = dc.load_decoder(os.path.join(td, "dec"), smpl)
        rproj = pj.load_projector(os.path.join(td, "proj"))
    assert sorted(rdec.weights) == sorted(w)
    for k in w:
        assert np.array_equal(rdec.weights[k], w[k]), k
    for f in ("w1", "b1", "w2", "b2", "w3", "b3", "subsample", "mask"):
        assert np.array_equal(getattr(rproj, f), getattr(pp, f)), f


@pytest.mark.parametrize("i", [0, 1])
def test_perturbed_weights_frame_bit_exact(i, g2, d2, full_models):
    """The oracle with non-zero biases / LN affine / projector biases equals
    the reference run on the same (file round-tripped) weights."""
    from conftest import projector_dict
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = full_models
    w, pp = perturbed_models(smpl)
    sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
    img = synth.render_scene(sc, smpl)
    trace = []
    out = orc.frame_to_smpl(img, sc.keypoints2d, w, dc.DecoderConfig(), mhr, smpl, gt, projector_dict(pp),
                            trace=trace)
    tag = "perturbed.frame%d" % i
    check_frame(tag, out, g2, d2)
    if i == 0:
        for j, (layer, p, c, kp) in enumerate(trace):
            assert np.array_equal(p, g2["%s.inter%d.params" % (tag, j)])
            assert np.array_equal(kp, g2["%s.inter%d.kp2d" % (tag, j)])


@pytest.mark.parametrize("i", [0, 1])
def test_toy_size_frames_bit_exact(i, g2, d2, toy_models, dec_weights):
    """Whole frames at the reference tests' size (MHR 1200 / SMPL 600 /
    V_sub 300, cli.py:108-136)."""
    from conftest import projector_dict
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = toy_models
    pw = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
    sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
    img = synth.render_scene(sc, smpl)
    out = orc.frame_to_smpl(img, sc.keypoints2d, dec_weights, dc.DecoderConfig(), mhr, smpl, gt, projector_dict(pw))
    check_frame("toy.frame%d" % i, out, g2, d2)


def test_c3_both_ends_of_the_batch(g2, d2, full_models, full_projector):
    """Meshes 0..31 and 4064..4095 of the C3 pose set."""
    from conftest import projector_dict

    mhr, smpl, gt = full_models
    rng = np.random.default_rng(3)
    p = np.zeros((4096, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    sel = g2["c3x.sel"]
    v = orc.skin_batch(mhr, p[sel])
    assert d2["c3x.v_mhr"] == digest(v)
    th = orc.project_batch(v, gt.corners, gt.weights, projector_dict(full_projector))
    assert np.array_equal(th, g2["c3x.theta"])
    j, _ = orc.fk_batch(smpl.joints_rest, th)
    assert np.array_equal(j, g2["c3x.j_smpl"])


def test_render_host_builder(g2, d2, full_models):
    """The host render restatement equals the reference's render_scene."""
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    for i in range(4):
        sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
        assert d2["render%d.image" % i] == digest(synth.render_scene(sc, smpl))
