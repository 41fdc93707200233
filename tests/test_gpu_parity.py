"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE.json north_star): boxes, prompts, grid coordinates and pixel
taps bit-exact; fp32 mode <= 1e-4 relative (max|d| / max|oracle| per
tensor); bf16 mode SMPL-joint MPJPE delta <= 0.5 mm (model units = metres).
"""

import numpy as np
import pytest

import oracle as orc
from conftest import projector_dict, rel_err

pytestmark = pytest.mark.gpu

FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def torch():
    import torch as t

    assert t.cuda.is_available(), "GPU tests need a CUDA device"
    return t


@pytest.fixture(scope="module")
def frames(full_models):
    from paper_2603_15603_b200 import synth

    _, smpl, _ = full_models
    out = []
    for i in range(6):
        sc = synth.random_scene(np.random.default_rng(5000 + i), smpl, (512, 512))
        out.append((synth.render_scene(sc, smpl), sc.keypoints2d))
    return out


@pytest.fixture(scope="module")
def pipe(full_models, full_projector):
    from paper_2603_15603_b200 import decoder as dc
    from paper_2603_15603_b200 import pipeline as pl

    mhr, smpl, gt = full_models
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    return pl.Pipeline(dec, mhr=mhr, bmap=gt, projector=full_projector)


def _ctx(pipe):
    return pipe.context()


# ---------------------------------------------------------------------------
# K1: bit-exact boxes, prompt, grid taps and crop values


def test_boxes_crops_bitexact(torch, pipe, frames, golden):
    from paper_2603_15603_b200 import runtime

    ctx = _ctx(pipe)
    imgs = np.stack([f[0] for f in frames])
    kps = np.stack([f[1] for f in frames])
    b = len(frames)
    dimg = torch.from_numpy(imgs).cuda()
    dkp = torch.from_numpy(kps).cuda()
    boxes = torch.empty((b, 3, 4), dtype=torch.float64, device="cuda")
    prompt = torch.empty((b, 8), dtype=torch.float32, device="cuda")
    crops = torch.empty((b, 3, 64, 64, 3), dtype=torch.float32, device="cuda")
    taps = torch.empty((b, 3, 64, 64, 4), dtype=torch.int32, device="cuda")
    ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, runtime.ptr(dimg), b, 512, 512, runtime.ptr(dkp), 3.0, 64,
                                      runtime.ptr(boxes), runtime.ptr(prompt), runtime.ptr(crops), runtime.ptr(taps),
                                      ctx.stream))
    boxes, prompt, crops, taps = (t.cpu().numpy() for t in (boxes, prompt, crops, taps))
    for i in range(b):
        bb, hands, pr, cr = orc.frame_crops(imgs[i], kps[i], 64)
        assert np.array_equal(boxes[i, 0], np.array(bb))
        assert np.array_equal(boxes[i, 1:], np.array(hands))
        assert np.array_equal(prompt[i], pr)
        assert np.array_equal(crops[i], cr), "crop values differ in frame %d" % i
        for c, bx in enumerate([bb] + hands):
            x0, y0, x1, y1, _, _ = orc.bilinear_taps(imgs[i].shape, orc.crop_grid(bx, 64))
            assert np.array_equal(taps[i, c, ..., 0], x0)
            assert np.array_equal(taps[i, c, ..., 1], y0)
            assert np.array_equal(taps[i, c, ..., 2], x1)
            assert np.array_equal(taps[i, c, ..., 3], y1)
    # reference goldens for the first frames (crops digests are pinned on CPU)
    assert np.array_equal(crops[0], golden["frame0.crops"])
    assert np.array_equal(crops[1], golden["frame1.crops"])
    assert np.array_equal(boxes[:, 0], golden["box_body"][:b])
    assert np.array_equal(prompt, golden["prompt"][:b])


def _gather(torch, ctx, imgs, kps, S=64, host=False):
    """fsb_boxes_crops on device (or pinned host) frames -> numpy outputs."""
    from paper_2603_15603_b200 import runtime

    b, h, w = imgs.shape[:3]
    if host:
        dimg = torch.from_numpy(np.ascontiguousarray(imgs)).pin_memory()
        dkp = torch.from_numpy(np.ascontiguousarray(kps)).pin_memory()
    else:
        dimg = torch.from_numpy(np.ascontiguousarray(imgs)).cuda()
        dkp = torch.from_numpy(np.ascontiguousarray(kps)).cuda()
    boxes = torch.empty((b, 3, 4), dtype=torch.float64, device="cuda")
    prompt = torch.empty((b, 8), dtype=torch.float32, device="cuda")
    crops = torch.empty((b, 3, S, S, 3), dtype=torch.float32, device="cuda")
    ctx.input_bytes(reset=True)
    ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, runtime.ptr(dimg), b, h, w, runtime.ptr(dkp), 3.0, S,
                                      runtime.ptr(boxes), runtime.ptr(prompt), runtime.ptr(crops), None,
                                      ctx.stream))
    nbytes = ctx.input_bytes(reset=True)
    return boxes.cpu().numpy(), prompt.cpu().numpy(), crops.cpu().numpy(), nbytes


def test_boxes_crops_host_frames(torch, pipe, frames):
    """Frames in pinned host memory are gathered in place (only the crop
    footprints cross PCIe) with bit-identical results."""
    ctx = _ctx(pipe)
    imgs = np.stack([f[0] for f in frames])
    kps = np.stack([f[1] for f in frames])
    bd, pd, cd, nd = _gather(torch, ctx, imgs, kps)
    bh, ph, ch, nh = _gather(torch, ctx, imgs, kps, host=True)
    assert np.array_equal(bd, bh) and np.array_equal(pd, ph) and np.array_equal(cd, ch)
    assert nd == 0 and 0 < nh < imgs.nbytes // 2, (nd, nh, imgs.nbytes)  # only host reads are counted
    for i in range(len(frames)):
        assert np.array_equal(ch[i], orc.frame_crops(imgs[i], kps[i], 64)[3])


def test_boxes_crops_host_frames_through_run_batch(torch, pipe, frames):
    ctx = _ctx(pipe)
    imgs = np.stack([f[0] for f in frames[:4]])
    kps = np.stack([f[1] for f in frames[:4]])
    dev = pipe.run_batch(imgs, kps)
    host = pipe.run_batch(torch.from_numpy(imgs).pin_memory(), torch.from_numpy(kps).pin_memory())
    for k in ("boxes", "merged", "theta", "j_smpl"):
        assert torch.equal(dev[k], host[k]), k
    ctx.input_bytes(reset=True)


def test_pageable_host_frames_rejected(torch, pipe, frames):
    from paper_2603_15603_b200 import runtime
    from paper_2603_15603_b200.numkit import UsageError

    ctx = _ctx(pipe)
    img = torch.from_numpy(frames[0][0][None].copy())  # pageable
    kp = torch.from_numpy(frames[0][1][None].copy()).cuda()
    boxes = torch.empty((1, 3, 4), dtype=torch.float64, device="cuda")
    prompt = torch.empty((1, 8), device="cuda")
    with pytest.raises(UsageError):
        ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, runtime.ptr(img), 1, 512, 512, runtime.ptr(kp), 3.0, 64,
                                          runtime.ptr(boxes), runtime.ptr(prompt), None, None, ctx.stream))


@pytest.mark.parametrize("h,w,S", [(97, 130, 64), (240, 321, 48), (64, 1500, 64), (48, 9001, 32), (512, 512, 7)])
def test_boxes_crops_odd_and_wide_frames(torch, pipe, golden, h, w, S):
    """Odd widths (rows not 16-byte aligned), frames wider than the staged
    path's shared-memory rows (per-tap path), tiny and non-multiple-of-4
    crop sizes; keypoints from the stress set squeezed into the frame."""
    ctx = _ctx(pipe)
    rng = np.random.default_rng(h * w + S)
    n = 6
    imgs = rng.random((n, h, w, 3)).astype(np.float32)
    skp = np.asarray(golden["stress_kp"][:n], np.float32)
    kps = (skp / np.float32(512.0) * np.array([w, h], np.float32)).astype(np.float32)
    kps = np.clip(kps, 0, np.array([w - 1, h - 1], np.float32)).astype(np.float32)
    for host in (False, True):
        boxes, prompt, crops, _ = _gather(torch, ctx, imgs, kps, S=S, host=host)
        for i in range(n):
            bb, hands, pr, cr = orc.frame_crops(imgs[i], kps[i], S)
            assert np.array_equal(boxes[i, 0], np.array(bb))
            assert np.array_equal(boxes[i, 1:], np.array(hands))
            assert np.array_equal(prompt[i], pr)
            assert np.array_equal(crops[i], cr), (i, host)


def test_box_goldens_all_scenes_and_stress(torch, golden):
    from paper_2603_15603_b200 import priors as pr

    for kp_key, body_key in (("scene_kp", "box_body"), ("stress_kp", "stress_body")):
        got = pr.body_boxes(golden[kp_key], (512, 512))
        assert np.array_equal(got, golden[body_key])


def test_standalone_box_api_known_answers(torch):
    from paper_2603_15603_b200 import priors as pr

    box = pr.hand_box((100.0, 200.0), pr.BBox(0.0, 0.0, 300.0, 400.0), alpha=3.0)
    assert [box.x_min, box.y_min, box.x_max, box.y_max] == [50.0, 150.0, 150.0, 250.0]
    box = pr.hand_box((0.0, 0.0), pr.BBox(0.0, 0.0, 300.0, 240.0), alpha=3.0, image_size=(320, 240))
    assert box.x_min >= 0.0 and box.y_min >= 0.0 and abs(box.width - 80.0) <= 1e-6
    g = pr.crop_grid(pr.BBox(3.0, 5.0, 4.0, 6.0), 2)
    assert np.array_equal(g, np.array([[[3, 5], [4, 5]], [[3, 6], [4, 6]]], np.float32))
    rng = np.random.default_rng(1)
    img = rng.random((16, 16, 3)).astype(np.float32)
    from paper_2603_15603_b200 import numkit as nk

    out = nk.bilinear_sample(img, pr.crop_grid(pr.BBox(0.0, 0.0, 15.0, 15.0), 16))
    assert np.array_equal(out, img)
    for i in range(10):
        x0, x1 = sorted(rng.uniform(0, 500, 2))
        y0, y1 = sorted(rng.uniform(0, 500, 2))
        bx = pr.BBox(x0, y0, x1, y1)
        assert np.array_equal(pr.crop_grid(bx, 64), orc.crop_grid((bx.x_min, bx.y_min, bx.x_max, bx.y_max), 64))


# ---------------------------------------------------------------------------
# K2 / K3: encoder and decoders, fp32


def test_encoder_fp32(torch, pipe, frames, dec_weights):
    from paper_2603_15603_b200 import decoder as dc

    cfg = dc.DecoderConfig()
    crops = np.concatenate([orc.frame_crops(f[0], f[1], 64)[3] for f in frames[:3]])
    got = pipe.decoder.encode(crops)
    want = orc.encode(dec_weights, cfg, crops)
    assert got.shape == want.shape
    assert rel_err(got, want) <= FP32_TOL


def test_decoders_fp32(torch, pipe, frames, dec_weights, full_models):
    from paper_2603_15603_b200 import decoder as dc

    cfg = dc.DecoderConfig()
    _, smpl, _ = full_models
    img, kp = frames[0]
    _, _, prompt, crops = orc.frame_crops(img, kp, 64)
    feats = orc.encode(dec_weights, cfg, crops)
    trace = []
    want_p, want_c = orc.decode_body(dec_weights, cfg, smpl.joints_rest, feats[0], prompt, (0, 1, 2), trace)
    out = pipe.decoder.decode_body(feats[0], prompt, selection=(0, 1, 2))
    assert rel_err(out.params, want_p) <= FP32_TOL
    assert rel_err(out.camera, want_c) <= FP32_TOL
    assert [it.layer for it in out.intermediates] == [0, 1, 2]
    for it, (l, p, c, k) in zip(out.intermediates, trace):
        assert rel_err(it.params, p) <= FP32_TOL and rel_err(it.kp2d, k) <= FP32_TOL
    rots = pipe.decoder.decode_hand(feats[1:3], ())
    assert rel_err(rots, orc.decode_hand(dec_weights, cfg, feats[1:3], ())) <= FP32_TOL
    # hand decoder with intermediate predictions enabled
    rots2 = pipe.decoder.decode_hand(feats[1:3], (0, 2, 4))
    assert rel_err(rots2, orc.decode_hand(dec_weights, cfg, feats[1:3], (0, 2, 4))) <= FP32_TOL


def test_decoder_batch_independence(torch, pipe, frames):
    crops = np.concatenate([orc.frame_crops(f[0], f[1], 64)[3] for f in frames[:4]])
    feats = pipe.decoder.encode(crops)
    one = pipe.decoder.encode(crops[5:6])
    assert np.array_equal(feats[5:6], one)
    hb = pipe.decoder.decode_hand(feats[[1, 2, 4, 5]])
    hs = np.concatenate([pipe.decoder.decode_hand(feats[[i]]) for i in (1, 2, 4, 5)])
    assert np.array_equal(hb, hs)


# ---------------------------------------------------------------------------
# K4: FK, LBS, projector, SMPL FK


def _c3_poses(n):
    rng = np.random.default_rng(3)
    p = np.zeros((4096, 76), np.float32)
    p[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
    p[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
    p[:, 51:54] = 0.0
    p[:, 63:66] = 0.0
    return p[:n]


def test_fk_and_skin_fp32(torch, full_models, golden):
    from paper_2603_15603_b200 import bodymodel as bm

    mhr, smpl, _ = full_models
    poses = _c3_poses(16)
    j, rel = bm.fk_batch(mhr, poses)
    wj, wrel = orc.fk_batch(mhr.joints_rest, poses)
    assert rel_err(j, wj) <= FP32_TOL and rel_err(rel, wrel) <= FP32_TOL
    assert rel_err(j, golden["c3.j_mhr16"]) <= FP32_TOL
    v = bm.skin_batch(mhr, poses)
    wv = orc.skin_batch(mhr, poses)
    assert rel_err(v, wv) <= FP32_TOL
    assert rel_err(v[:, ::97], golden["c3.v_mhr16_rows"]) <= FP32_TOL
    # batched rows == single rows, bitwise
    v3 = bm.skin_batch(mhr, poses[3:4])
    assert np.array_equal(v3[0], v[3])
    vs = bm.skin_batch(smpl, poses[:4])
    assert rel_err(vs, orc.skin_batch(smpl, poses[:4])) <= FP32_TOL


def test_skin_many_meshes(torch, full_models):
    """Several 32-mesh groups, an odd mesh count and a partial last vertex
    tile (18,439 = 576 x 32 + 7) through the warp-tile LBS kernel."""
    from paper_2603_15603_b200 import bodymodel as bm

    mhr, smpl, _ = full_models
    poses = _c3_poses(71)
    v = bm.skin_batch(mhr, poses)
    pick = [0, 1, 31, 32, 33, 63, 64, 70]
    assert rel_err(v[pick], orc.skin_batch(mhr, poses[pick])) <= FP32_TOL
    vs = bm.skin_batch(smpl, poses[:35])
    assert rel_err(vs[[0, 33, 34]], orc.skin_batch(smpl, poses[[0, 33, 34]])) <= FP32_TOL


def test_projector_fp32(torch, full_models, full_projector, golden):
    from paper_2603_15603_b200 import projection as pj

    mhr, smpl, gt = full_models
    poses = _c3_poses(16)
    v = orc.skin_batch(mhr, poses)
    th = pj.project_batch(v, gt, full_projector)
    want = orc.project_batch(v, gt.corners, gt.weights, projector_dict(full_projector))
    assert rel_err(th, want) <= FP32_TOL
    assert rel_err(th, golden["c3.theta16"]) <= FP32_TOL
    assert np.all(th[:, 51:54] == 0.0) and np.all(th[:, 63:66] == 0.0)
    # bridge matches the oracle on all targets
    br = pj.bridge(v[:2], gt)
    assert rel_err(br, orc.bridge(v[:2], gt.corners, gt.weights)) <= FP32_TOL


# ---------------------------------------------------------------------------
# whole path: frame -> SMPL, graph replay, batch independence


def test_frame_batch_end_to_end_fp32(torch, pipe, frames, dec_weights, full_models, full_projector, golden):
    from paper_2603_15603_b200 import decoder as dc

    mhr, smpl, gt = full_models
    cfg = dc.DecoderConfig()
    imgs = np.stack([f[0] for f in frames])
    kps = np.stack([f[1] for f in frames])
    out = pipe.run_batch(imgs, kps)
    res = {k: v.cpu().numpy() for k, v in out.items()}
    pw = projector_dict(full_projector)
    for i in range(len(frames)):
        want = orc.frame_to_smpl(imgs[i], kps[i], dec_weights, cfg, mhr, smpl, gt, pw)
        assert np.array_equal(res["boxes"][i, 0], np.array(want["body_box"]))
        for k in ("merged", "theta", "j_smpl", "v_mhr"):
            assert rel_err(res[k][i], want[k]) <= FP32_TOL, (i, k, rel_err(res[k][i], want[k]))
        if i < 4:
            assert rel_err(res["merged"][i], golden["frame%d.merged" % i]) <= FP32_TOL
            assert rel_err(res["theta"][i], golden["frame%d.theta" % i]) <= FP32_TOL
            assert rel_err(res["j_smpl"][i], golden["frame%d.j_smpl" % i]) <= FP32_TOL
    # replay of the captured graph reproduces the outputs bitwise, and a
    # frame run alone equals its row in the batch
    out2 = pipe.run_batch(imgs, kps)
    for k in ("merged", "theta", "j_smpl", "v_mhr"):
        assert np.array_equal(out2[k].cpu().numpy(), res[k])
    solo = pipe.run_batch(imgs[2:3], kps[2:3])
    for k in ("merged", "theta", "j_smpl", "v_mhr"):
        assert np.array_equal(solo[k].cpu().numpy()[0], res[k][2])


def test_run_fast_matches_reference_golden(torch, pipe, frames, golden):
    from paper_2603_15603_b200 import pipeline as pl
    from paper_2603_15603_b200 import synth

    plan = pl.build_plan(pl.fast_config())
    for i in range(2):
        sc = synth.random_scene(np.random.default_rng(5000 + i), pipe.template, (512, 512))
        merged, report = pipe.run(frames[i][0], sc, pl.fast_config(), plan)
        assert rel_err(merged, golden["frame%d.merged" % i]) <= FP32_TOL
        assert pipe.last_counters["encode"] == 1
    assert report.frames == 2
    assert plan.allocations == 2  # prompt + merged, no steady-state growth


def test_nonfinite_image_raises(torch, pipe, frames):
    from paper_2603_15603_b200 import numkit as nk

    imgs = np.stack([f[0] for f in frames[:2]]).copy()
    kps = np.stack([f[1] for f in frames[:2]])
    imgs[1, :, :, :] = np.nan
    with pytest.raises(nk.NumericError):
        pipe.run_batch(imgs, kps)


def test_denoise_bitexact_vs_reference_golden(torch):
    """projection.denoise on the GPU equals the reference's output bit for bit
    (tools/make_golden_denoise.py), batched and single-pose."""
    import os

    from paper_2603_15603_b200 import projection as pj

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "denoise.npz"))
    w = pj.DenoiserWeights(g["w1"], g["b1"], g["w2"], g["b2"])
    assert np.array_equal(pj.denoise(w, g["x"]), g["out"])
    assert np.array_equal(pj.denoise(w, g["x"][3]), g["out3"])
    with pytest.raises(ValueError):
        pj.denoise(w, g["x"][:, :60])


@pytest.mark.parametrize("prec,n,tol", [("fp32", 40, 1e-4), ("bf16", 40, 2e-2), ("fp32", 1030, 1e-4)])
def test_skin_project_with_and_without_vmhr(torch, pipe, full_models, full_projector, prec, n, tol):
    """fsb_skin_project bridges the projector input from V_mhr when it is
    produced and re-skins the corner vertices otherwise (one CTA per 8-mesh
    group, 8 groups per CTA from 1024 meshes); both give the same theta and
    SMPL joints within the precision's tolerance, and match the oracle."""
    from paper_2603_15603_b200 import runtime as rt

    mhr, smpl, gt = full_models
    ctx = pipe.context()
    ctx.reserve(n)
    poses = torch.from_numpy(_c3_poses(n)).cuda()
    nv = mhr.num_vertices
    v = torch.empty((n, nv, 3), dtype=torch.float32, device="cuda")
    th = [torch.empty((n, 76), dtype=torch.float32, device="cuda") for _ in range(2)]
    jj = [torch.empty((n, 22, 3), dtype=torch.float32, device="cuda") for _ in range(2)]
    p = rt.PRECISIONS[prec]
    ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses), n, rt.ptr(v), rt.ptr(th[0]), rt.ptr(jj[0]), None, p,
                                       ctx.stream))
    ctx.check(ctx.lib.fsb_skin_project(ctx.h, rt.ptr(poses), n, None, rt.ptr(th[1]), rt.ptr(jj[1]), None, p,
                                       ctx.stream))
    torch.cuda.synchronize()
    t0, t1 = th[0].cpu().numpy(), th[1].cpu().numpy()
    assert rel_err(t1, t0) <= tol
    assert rel_err(jj[1].cpu().numpy(), jj[0].cpu().numpy()) <= tol
    k = min(n, 8)
    want = orc.project_batch(orc.skin_batch(mhr, _c3_poses(k)), gt.corners, gt.weights, projector_dict(full_projector))
    assert rel_err(t0[:k], want) <= (FP32_TOL if prec == "fp32" else 5e-2)
