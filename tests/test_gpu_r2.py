"""GPU parity, round 2: the CUDA path (through the C ABI / the Python
mirror) against fixtures the REFERENCE itself produced
(tools/make_golden_r2.py -> tests/golden/golden_r2.npz, digests_r2.json):

* keypoints outside the frame (detect_stub's clip, priors.py:188-190);
* non-trivial biases, LayerNorm gamma/beta and projector b1..b3, loaded from
  files written by save_decoder / save_projector (byte-identical to the
  reference's, tests/test_oracle_pins_r2.py) -- K2, K3, K4 and the whole frame;
* the toy-size configuration (1200 / 600 / 300) the reference's tests run;
* 64 meshes at both ends of the 4096-mesh C3 batch;
* the ViT-L-sized encoder at all 24 layers;
* render_scene on the GPU (k_render) within a stated ulp bound.

Bars: boxes / prompt / crops bit-exact; fp32 <= 1e-4 relative
(max|d| / max|ref|); bf16 SMPL-joint MPJPE delta <= 0.5 mm.
"""

import hashlib
import json
import os
import tempfile

import numpy as np
import pytest

from conftest import rel_err
from perturb import perturb_decoder, perturb_projector_arrays

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
FP32_TOL = 1e-4
MPJPE_MM = 0.5
# 24 bf16 layers (LN output, q/k/v, P, context, MLP hidden in bf16, fp32
# accumulate and residual) against the reference's fp32: relative L2 of the
# final features.  Measured 4.7e-3 (round 2); a dropped bias is ~1e-1.
VIT24_REL_L2 = 1e-2
# k_render: CUDA expf (<= 2 ulp) vs numpy's float32 SIMD exp, summed over 22
# blobs of weight <= 0.5 each: |d| <= 22 * 0.5 * 2^-23 * 2 ~ 2.6e-6 worst case
RENDER_ABS = 4e-6


def digest(a):
    a = np.ascontiguousarray(a)
    return "%s|%s|%s" % (a.dtype.str, "x".join(map(str, a.shape)), hashlib.sha256(a.tobytes()).hexdigest())


def mpjpe_mm(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64), axis=-1).mean() * 1e3)


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available(), "GPU tests need a CUDA device"
    return t


@pytest.fixture(scope="module")
def g2():
    return np.load(os.path.join(GOLDEN, "golden_r2.npz"))


@pytest.fixture(scope="module")
def d2():
    with open(os.path.join(GOLDEN, "digests_r2.json")) as fh:
        return json.load(fh)


def _pipeline(dec, mhr, gt, proj, precision):
    from paper_2603_15603_b200 import pipeline as pl

    return pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=proj, precision=precision)


def _run(torch, pipe, images, kps, host=False):
    """run_batch with crops and features returned (device frames, or pinned
    host frames read in place by the streaming K1)."""
    img = torch.from_numpy(np.ascontiguousarray(images, np.float32))
    kp = torch.from_numpy(np.ascontiguousarray(kps, np.float32))
    if host:
        img, kp = img.pin_memory(), kp.pin_memory()
    else:
        img, kp = img.cuda(), kp.cuda()
    out = pipe.allocate_outputs(images.shape[0], tail=True, crops=True, feats=True)
    pipe.run_batch(img, kp, outputs=out)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


def _check(tag, o, i, g2, d2, precision):
    assert np.array_equal(o["boxes"][i], g2[tag + ".boxes"]), tag
    assert np.array_equal(o["prompt"][i], g2[tag + ".prompt"]), tag
    assert d2[tag + ".crops"] == digest(o["crops"][i]), tag
    if precision == "fp32":
        assert rel_err(o["feats"][i][:, ::8], g2[tag + ".feats_rows"]) <= FP32_TOL
        for k in ("body_params", "body_cam", "hand_rots", "merged", "theta", "j_smpl"):
            assert rel_err(o[k][i], g2["%s.%s" % (tag, k)]) <= FP32_TOL, (tag, k)
        assert rel_err(o["v_mhr"][i][::97], g2[tag + ".v_mhr_rows"]) <= FP32_TOL
    else:
        assert mpjpe_mm(o["j_smpl"][i], g2[tag + ".j_smpl"]) <= MPJPE_MM, tag
        assert rel_err(o["v_mhr"][i][::97], g2[tag + ".v_mhr_rows"]) <= 2e-2, tag
        assert rel_err(o["merged"][i], g2[tag + ".merged"]) <= 5e-2, tag


# ---------------------------------------------------------------------------
# keypoints outside the frame (detect_stub clips before the box)


def _oof_frames(full_models):
    from paper_2603_15603_b200 import synth
    from test_oracle_pins_r2 import oof_scenes

    _, smpl, _ = full_models
    sc = oof_scenes(smpl)
    return np.stack([synth.render_scene(s, smpl) for s in sc]), np.stack([s.keypoints2d for s in sc])


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
@pytest.mark.parametrize("host", [False, True])
def test_out_of_frame_keypoints(torch, g2, d2, full_models, full_projector, precision, host):
    from paper_2603_15603_b200 import decoder as dc

    mhr, smpl, gt = full_models
    images, kps = _oof_frames(full_models)
    pipe = _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, precision)
    o = _run(torch, pipe, images, kps, host=host)
    for i in range(6):
        _check("oof%d" % i, o, i, g2, d2, precision)


def test_out_of_frame_single_frame_api(torch, g2, full_models, full_projector):
    """Pipeline.run (the reference's per-frame entry, noise_sigma = 0) on a
    scene with keypoints outside the frame."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import synth
    from test_oracle_pins_r2 import oof_scenes

    mhr, smpl, gt = full_models
    sc = oof_scenes(smpl)[4]
    pipe = _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, "fp32")
    merged, rep = pipe.run(synth.render_scene(sc, smpl), sc, pl.fast_config())
    assert rel_err(merged, g2["oof4.merged"]) <= FP32_TOL
    assert rep.frames == 1


# ---------------------------------------------------------------------------
# perturbed (trained-looking) weights loaded from reference-format files


@pytest.fixture(scope="module")
def perturbed(full_models):
    """Decoder and projector loaded back from the files save_decoder /
    save_projector wrote (bytes pinned to the reference's in the CPU suite)."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    dec.weights = perturb_decoder(synth.decoder_weights(dc.DecoderConfig(), 40))
    p = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    b1, b2, b3 = perturb_projector_arrays(p.b1, p.b2, p.b3)
    pp = pj.ProjectorWeights(w1=p.w1, b1=b1, w2=p.w2, b2=b2, w3=p.w3, b3=b3, subsample=p.subsample, mask=p.mask)
    with tempfile.TemporaryDirectory() as td:
        dc.save_decoder(dec, os.path.join(td, "dec"))
        pj.save_projector(os.path.join(td, "proj"), pp)
        rdec = dc.load_decoder(os.path.join(td, "dec"), smpl)
        rproj = pj.load_projector(os.path.join(td, "proj"))
    return rdec, rproj


def _perturbed_frames(full_models):
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    sc = [synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512)) for i in range(2)]
    return np.stack([synth.render_scene(s, smpl) for s in sc]), np.stack([s.keypoints2d for s in sc])


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_perturbed_weights_whole_frame(torch, g2, d2, full_models, perturbed, precision):
    mhr, smpl, gt = full_models
    dec, proj = perturbed
    images, kps = _perturbed_frames(full_models)
    o = _run(torch, _pipeline(dec, mhr, gt, proj, precision), images, kps)
    for i in range(2):
        _check("perturbed.frame%d" % i, o, i, g2, d2, precision)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_perturbed_weights_stage_apis(torch, g2, full_models, perturbed, precision):
    """Decoder.encode / decode_body (with the FK-feedback intermediates) /
    decode_hand and projection.project_batch one stage at a time."""
    from paper_2603_15603_b200 import projection as pj

    mhr, smpl, gt = full_models
    dec, proj = perturbed
    images, kps = _perturbed_frames(full_models)
    o = _run(torch, _pipeline(dec, mhr, gt, proj, "fp32"), images[:1], kps[:1])
    crops = o["crops"][0]
    feats = dec.encode(crops, precision=precision)
    tag = "perturbed.frame0"
    tol = FP32_TOL if precision == "fp32" else 3e-2
    assert rel_err(feats[:, ::8], g2[tag + ".feats_rows"]) <= tol
    want_feats = o["feats"][0]  # fp32 features (checked against the golden rows above)
    bout = dec.decode_body(want_feats[0], g2[tag + ".prompt"], selection=(0, 1, 2), precision=precision)
    ptol = FP32_TOL if precision == "fp32" else 5e-2
    assert rel_err(bout.params, g2[tag + ".body_params"]) <= ptol
    assert rel_err(bout.camera, g2[tag + ".body_cam"]) <= ptol
    for j, it in enumerate(bout.intermediates):
        assert rel_err(it.params, g2["%s.inter%d.params" % (tag, j)]) <= ptol, j
        assert rel_err(it.kp2d, g2["%s.inter%d.kp2d" % (tag, j)]) <= ptol, j
    rots = dec.decode_hand(want_feats[1:3], (), precision=precision)
    assert rel_err(rots, g2[tag + ".hand_rots"]) <= ptol
    # the projector with perturbed biases on the reference's own V_mhr rows
    # is covered through the whole frame; here the stand-alone entry:
    v = o["v_mhr"][:1]
    th = pj.project_batch(v, gt, proj, precision=precision)
    assert rel_err(th[0], g2[tag + ".theta"]) <= (FP32_TOL if precision == "fp32" else 5e-2)


def test_perturbation_changes_outputs(torch, full_models, full_projector, perturbed, g2):
    """Sanity: the perturbed weights move the outputs far beyond the parity
    bound, so the tests above really exercise the bias / affine paths."""
    mhr, smpl, gt = full_models
    dec, proj = perturbed
    images, kps = _perturbed_frames(full_models)
    o = _run(torch, _pipeline(dec, mhr, gt, proj, "fp32"), images[:1], kps[:1])
    from paper_2603_15603_b200 import decoder as dc

    base = _run(torch, _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, "fp32"),
                images[:1], kps[:1])
    assert rel_err(o["merged"][0], base["merged"][0]) > 100 * FP32_TOL
    assert rel_err(o["theta"][0], base["theta"][0]) > 100 * FP32_TOL


# ---------------------------------------------------------------------------
# toy size (MHR 1200 / SMPL 600 / V_sub 300: the reference's test size)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_toy_size_frames(torch, g2, d2, toy_models, precision):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import projection as pj
    from paper_2603_15603_b200 import synth

    mhr, smpl, gt = toy_models
    proj = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
    sc = [synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512)) for i in range(2)]
    images = np.stack([synth.render_scene(s, smpl) for s in sc])
    kps = np.stack([s.keypoints2d for s in sc])
    o = _run(torch, _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, proj, precision), images,
             kps)
    for i in range(2):
        _check("toy.frame%d" % i, o, i, g2, d2, precision)


# ---------------------------------------------------------------------------
# C3: 64 of the 4096 meshes, both ends of the batch


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_c3_64_meshes(torch, g2, full_models, full_projector, precision):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    mhr, smpl, gt = full_models
    rng = np.random.default_rng(3)
    p = np.zeros((4096, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    pipe = _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, precision)
    ctx = pipe.context()
    ctx.reserve(4096)
    poses = torch.from_numpy(p).cuda()
    v = torch.empty((4096, mhr.num_vertices, 3), dtype=torch.float32, device="cuda")
    th = torch.empty((4096, 76), dtype=torch.float32, device="cuda")
    j = torch.empty((4096, 22, 3), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses), 4096, rt.ptr(v), rt.ptr(th), rt.ptr(j), None,
                                       rt.PRECISIONS[precision], ctx.stream))
    torch.cuda.synchronize()
    ctx.check_finite("c3")
    sel = g2["c3x.sel"]
    vs = v[torch.from_numpy(sel).cuda()].cpu().numpy()
    # LBS is fp32 in both modes
    assert rel_err(vs[:, ::61], g2["c3x.v_mhr_rows"]) <= FP32_TOL
    got_t, got_j = th.cpu().numpy()[sel], j.cpu().numpy()[sel]
    if precision == "fp32":
        assert rel_err(got_t, g2["c3x.theta"]) <= FP32_TOL
        assert rel_err(got_j, g2["c3x.j_smpl"]) <= FP32_TOL
    else:
        for m in range(len(sel)):
            assert mpjpe_mm(got_j[m], g2["c3x.j_smpl"][m]) <= MPJPE_MM, m


def test_c3_batch_independent_bits(torch, full_models, full_projector):
    """The projector's batch-size-specific kernels -- persistent tile GEMM
    from 1024 meshes (and the compacted-corner bridge with 4 meshes per CTA),
    one-item tile GEMMs in between, the transposed tile GEMM up to 64 --
    give every mesh the same bits: 1536 meshes in one call vs calls of 256
    vs calls of 32 (bf16, and fp32 with its split-bf16 passes)."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    mhr, smpl, gt = full_models
    n = 1536
    rng = np.random.default_rng(11)
    p = np.zeros((n, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(n, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(n, 10))
    for precision in ("bf16", "fp32"):
        pipe = _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, precision)
        ctx = pipe.context()
        ctx.reserve(n)
        poses = torch.from_numpy(p).cuda()
        outs = []
        for step in (n, 256, 32):
            v = torch.empty((n, mhr.num_vertices, 3), dtype=torch.float32, device="cuda")
            th = torch.empty((n, 76), dtype=torch.float32, device="cuda")
            j = torch.empty((n, 22, 3), dtype=torch.float32, device="cuda")
            for b0 in range(0, n, step):
                ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses[b0:]), step, rt.ptr(v[b0:]), rt.ptr(th[b0:]),
                                                   rt.ptr(j[b0:]), None, rt.PRECISIONS[precision], ctx.stream))
            torch.cuda.synchronize()
            ctx.check_finite("c3 batch")
            outs.append((th.cpu(), j.cpu(), v[::97].cpu()))
        for other in outs[1:]:
            for a, b in zip(outs[0], other):
                assert torch.equal(a, b), precision


def test_c3_partial_last_tile_bits(torch, full_models, full_projector):
    """The on-chip-reduced projector GEMM (k_tile_gemm_f, from 1024 meshes)
    with a partial last 128-row tile: 1100 meshes in one call give the same
    theta / joints bits as calls of 32 (transposed tiles + k_tile_reduce8),
    and the rows past the batch are never written (bf16 and fp32)."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt

    mhr, smpl, gt = full_models
    n = 1100
    rng = np.random.default_rng(12)
    p = np.zeros((n, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(n, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(n, 10))
    for precision in ("bf16", "fp32"):
        pipe = _pipeline(dc.Decoder(smpl, dc.DecoderConfig(), seed=40), mhr, gt, full_projector, precision)
        ctx = pipe.context()
        ctx.reserve(n)
        poses = torch.from_numpy(p).cuda()
        outs = []
        for step in (n, 32):
            v = torch.empty((n, mhr.num_vertices, 3), dtype=torch.float32, device="cuda")
            th = torch.full((n + 4, 76), 7.0, dtype=torch.float32, device="cuda")
            j = torch.empty((n, 22, 3), dtype=torch.float32, device="cuda")
            for b0 in range(0, n, step):
                m = min(step, n - b0)
                ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses[b0:]), m, rt.ptr(v[b0:]), rt.ptr(th[b0:]),
                                                   rt.ptr(j[b0:]), None, rt.PRECISIONS[precision], ctx.stream))
            torch.cuda.synchronize()
            ctx.check_finite("c3 partial tile")
            assert torch.all(th[n:] == 7.0), precision  # nothing written past the batch
            outs.append((th[:n].cpu(), j.cpu()))
        for a, b in zip(outs[0], outs[1]):
            assert torch.equal(a, b), precision


# ---------------------------------------------------------------------------
# ViT-L-sized encoder, all 24 layers


def test_vitl_24_layers_golden(torch, g2):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import runtime as rt
    from paper_2603_15603_b200 import synth

    cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=24, body_layers=1,
                           hand_layers=1)
    ctx = rt.Context()
    ctx.load_decoder(cfg, synth.decoder_weights(cfg, 40, encoder_only=True))
    crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
    x = torch.from_numpy(crop).cuda()
    out = torch.empty((1, 576, 1024), dtype=torch.float32, device="cuda")
    ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), 1, rt.ptr(out), rt.PRECISIONS["bf16"], ctx.stream), "encode")
    torch.cuda.synchronize()
    got = out.cpu().numpy()[0, ::36].astype(np.float64)
    want = g2["c4.l24.feats_rows"].astype(np.float64)
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    print("ViT-L 24-layer bf16 rel-L2 vs reference:", rel)
    assert np.isfinite(got).all()
    assert rel < VIT24_REL_L2, rel
    # reference precision: the fp32 CUDA-core pipeline, fp32 bar
    ctx.check(ctx.lib.fsb_encode(ctx.h, rt.ptr(x), 1, rt.ptr(out), rt.PRECISIONS["fp32"], ctx.stream), "encode")
    torch.cuda.synchronize()
    got32 = out.cpu().numpy()[0, ::36].astype(np.float64)
    err = np.abs(got32 - want).max() / np.abs(want).max()
    print("ViT-L 24-layer fp32 max rel vs reference:", err)
    assert err <= FP32_TOL, err


# ---------------------------------------------------------------------------
# k_render (priors.render_scene on the GPU) within the stated bound


def test_render_scene_gpu(torch, g2, d2, full_models):
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    sc = [synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512)) for i in range(4)]
    img = pr.render_scenes(sc).cpu().numpy()
    exact = 0
    for i in range(4):
        want = g2["render%d.rows" % i]
        got = img[i, ::32]
        d = np.abs(got.astype(np.float64) - want).max()
        assert d <= RENDER_ABS, (i, d)
        exact += int((got == want).sum())
    frac = exact / float(4 * want.size)
    print("k_render bit-identical fraction:", frac)
    assert frac > 0.5
    # the boxes K1 derives from the rendered frame's keypoints do not depend
    # on the renderer; the crops of a GPU-rendered frame stay within the bound
    host = synth.render_scene(sc[0], smpl)
    assert np.abs(img[0].astype(np.float64) - host).max() <= RENDER_ABS


def test_render_odd_size_off_frame(torch, g2, d2, full_models):
    """300x200 frame with keypoints off the frame (odd W != H)."""
    from paper_2603_15603_b200 import priors as pr
    from paper_2603_15603_b200 import synth

    kp = g2["render_odd.kp"]
    sc = synth.Scene(image_size=(300, 200), camera=synth.default_camera((300, 200)), pose=np.zeros(76, np.float32),
                     translation=np.zeros(3, np.float32), seed=int(g2["render_odd.seed"]), keypoints2d=kp)
    img = pr.render_scenes([sc]).cpu().numpy()[0]
    assert img.shape == (200, 300, 3)
    d = np.abs(img[::5].astype(np.float64) - g2["render_odd.rows"]).max()
    assert d <= RENDER_ABS, d


# ---------------------------------------------------------------------------
# single-frame API error contract (round 2: native staging + enqueued flag)


def test_single_frame_api_nonfinite(torch, full_models, full_projector):
    """Pipeline.run_smpl: a NaN / inf in the host image raises NumericError
    before any device work (fsb_stage_frame, numkit.bilinear_sample's
    check_finite); non-finite values produced on the device raise through the
    flag read enqueued with the results (fsb_nonfinite_enqueue); the flag is
    cleared, so the next good call succeeds and matches the first."""
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import synth
    from paper_2603_15603_b200.numkit import NumericError

    mhr, smpl, gt = full_models
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    pipe = _pipeline(dec, mhr, gt, full_projector, "bf16")
    sc = synth.random_scene(np.random.default_rng(77), smpl, (512, 512))
    img = synth.render_scene(sc, smpl)
    good, _ = pipe.run_smpl(img, sc)
    for v in (np.nan, np.inf):
        bad = img.copy()
        bad[100, 200, 1] = v
        with pytest.raises(NumericError):
            pipe.run_smpl(bad, sc)
    again, _ = pipe.run_smpl(img, sc)
    assert np.array_equal(again["theta"], good["theta"])
    # a non-finite weight: the device flags it, the call raises, the flag resets
    key = next(k for k in dec.weights if k.endswith("head_params_b") or k.endswith("head_params.b"))
    saved = dec.weights[key]
    dec.weights[key] = np.full_like(saved, np.inf)
    with pytest.raises(NumericError):
        pipe.run_smpl(img, sc)
    dec.weights[key] = saved
    after, _ = pipe.run_smpl(img, sc)
    assert np.array_equal(after["theta"], good["theta"])
