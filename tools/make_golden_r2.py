"""Round-2 golden fixtures, produced by running the REFERENCE itself
(read-only at /root/reference/pkg/src).  Writes tests/golden/golden_r2.npz and
tests/golden/digests_r2.json.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden_r2.py [part ...]

Parts (default: all):
  oof       scenes whose keypoints project OUTSIDE the frame: detect_stub clips
            them (priors.py:188-190) before the body box; boxes, prompt,
            crops, merged and the SMPL tail of the reference pipeline
  perturbed every decoder bias / LayerNorm gamma, beta and the projector
            b1..b3 perturbed (tests/perturb.py); the files the reference's
            save_decoder / save_projector write (decoder.py:429-440,
            projection.py:797-806) are digested byte for byte, and two frames
            run through the reference with those weights
  vitl24    the ViT-L-sized encoder at its full 24 layers (decoder.py:231-260)
            on one 384x384 crop (~1 min of CPU)
  render    render_scene (priors.py:237-252) rows of 4 scenes
  toy       two frames through the toy-size (1200/600/300) tail
  c3        C3 poses 0..63 through skin / project / fk (64 meshes)
"""

import hashlib
import json
import os
import sys
import tempfile
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fsb.bodymodel as bm  # noqa: E402
import fsb.decoder as dc  # noqa: E402
import fsb.pipeline as pl  # noqa: E402
import fsb.priors as pr  # noqa: E402
import fsb.projection as pj  # noqa: E402
import perturb  # noqa: E402  (tests/perturb.py: the shared perturbation recipe)

OUT = os.path.join(ROOT, "tests", "golden")
NPZ = os.path.join(OUT, "golden_r2.npz")
DIG = os.path.join(OUT, "digests_r2.json")


def digest(a):
    a = np.ascontiguousarray(a)
    return "%s|%s|%s" % (a.dtype.str, "x".join(map(str, a.shape)), hashlib.sha256(a.tobytes()).hexdigest())


def file_digests(d):
    out = {}
    for fn in sorted(os.listdir(d)):
        with open(os.path.join(d, fn), "rb") as fh:
            out[fn] = hashlib.sha256(fh.read()).hexdigest()
    return out


def oof_scenes(smpl):
    """Six scenes placed so that some keypoints leave the 512x512 frame."""
    cam = pr.default_camera((512, 512))
    offsets = [(0.35, 0.0, 2.0), (-0.45, 0.05, 2.2), (0.0, -0.5, 2.4), (0.05, 0.55, 2.3), (0.0, 0.0, 0.9),
               (0.5, 0.45, 1.6)]
    scenes = []
    for i, (dx, dy, z) in enumerate(offsets):
        rng = np.random.default_rng(900 + i)
        vec = np.zeros(bm.PARAM_DIM, np.float32)
        vec[:66] = rng.normal(0.0, 0.2, size=66)
        vec[66:] = rng.normal(0.0, 0.45, size=bm.SHAPE_DIM)
        fk = bm.forward_kinematics(smpl, bm.PoseState.from_vector(vec))
        c = fk.joints.mean(axis=0)
        t = np.array([-c[0] + dx, -c[1] + dy, -c[2] + z], np.float32)
        scenes.append(pr.make_scene(smpl, vec, t, cam, (512, 512), seed=int(rng.integers(0, 2 ** 31 - 1))))
    return scenes


def frame_record(tag, arrs, dig, image, scene, dec, mhr, smpl, gt, proj, keep_inter=False):
    box, kp = pr.detect_stub(scene, 0.0, 0)
    hb = [pr.hand_box(kp.xy[j], box, alpha=3.0, image_size=scene.image_size)
          for j in (bm.LEFT_WRIST, bm.RIGHT_WRIST)]
    crops = pl.prepare_crops(image, [box] + hb, dec.config.crop_size)
    feats = dec.encode(crops)
    prompt = pl._box_prompt(box, scene.image_size, np.empty(8, np.float32)).copy()
    bout = dec.decode_body(feats[0], prompt, selection=(0, 1, 2))
    rots = dec.decode_hand(feats[1:3], ())
    merged, _ = pl.Pipeline(dec).run(image, scene, pl.fast_config())
    merged = merged.copy()
    assert np.array_equal(merged, dec.merge(bout.params, rots[0], rots[1]))
    v_mhr = bm.skin_batch(mhr, merged[None], correctives=False)
    theta = pj.project_batch(v_mhr, gt, proj)
    j_smpl, _ = bm.fk_batch(smpl, theta)
    arrs[tag + ".kp"] = np.asarray(scene.keypoints2d, np.float32)
    arrs[tag + ".kp_clipped"] = kp.xy
    arrs[tag + ".boxes"] = np.array([[b.x_min, b.y_min, b.x_max, b.y_max] for b in [box] + hb], np.float64)
    arrs[tag + ".prompt"] = prompt
    dig[tag + ".image"] = digest(image)
    dig[tag + ".crops"] = digest(crops)
    dig[tag + ".feats"] = digest(feats)
    arrs[tag + ".crops_rows"] = crops[:, ::8].copy()
    arrs[tag + ".feats_rows"] = feats[:, ::8].copy()
    arrs[tag + ".body_params"] = bout.params
    arrs[tag + ".body_cam"] = bout.camera
    arrs[tag + ".hand_rots"] = rots
    arrs[tag + ".merged"] = merged
    dig[tag + ".v_mhr"] = digest(v_mhr)
    arrs[tag + ".v_mhr_rows"] = v_mhr[0, ::97].copy()
    arrs[tag + ".theta"] = theta[0]
    arrs[tag + ".j_smpl"] = j_smpl[0]
    if keep_inter:
        for j, it in enumerate(bout.intermediates):
            arrs["%s.inter%d.params" % (tag, j)] = it.params
            arrs["%s.inter%d.cam" % (tag, j)] = it.camera
            arrs["%s.inter%d.kp2d" % (tag, j)] = it.kp2d


def main(parts):
    t0 = time.time()
    arrs = dict(np.load(NPZ)) if os.path.exists(NPZ) else {}
    dig = json.load(open(DIG)) if os.path.exists(DIG) else {}
    mhr, smpl, gt = bm.make_toy_models(seed=0, mhr_vertices=18439, smpl_vertices=6890)
    proj = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)

    if "oof" in parts:
        for i, scene in enumerate(oof_scenes(smpl)):
            image = pr.render_scene(scene, smpl)
            frame_record("oof%d" % i, arrs, dig, image, scene, dec, mhr, smpl, gt, proj)
            kpx = np.asarray(scene.keypoints2d)
            print("oof", i, "out-of-frame keypoints:",
                  int(((kpx < 0) | (kpx > 511)).any(axis=1).sum()), time.time() - t0, flush=True)

    if "perturbed" in parts:
        pdec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
        pdec.weights = perturb.perturb_decoder(pdec.weights)
        b1, b2, b3 = perturb.perturb_projector_arrays(proj.b1, proj.b2, proj.b3)
        pproj = pj.ProjectorWeights(w1=proj.w1, b1=b1, w2=proj.w2, b2=b2, w3=proj.w3, b3=b3,
                                    subsample=proj.subsample, mask=proj.mask)
        with tempfile.TemporaryDirectory() as td:
            dc.save_decoder(pdec, os.path.join(td, "dec"))
            pj.save_projector(os.path.join(td, "proj"), pproj)
            for k, v in file_digests(os.path.join(td, "dec")).items():
                dig["perturbed.files.decoder/" + k] = v
            for k, v in file_digests(os.path.join(td, "proj")).items():
                dig["perturbed.files.projector/" + k] = v
            # the round trip through the reference's own loaders
            rdec = dc.load_decoder(os.path.join(td, "dec"), smpl)
            rproj = pj.load_projector(os.path.join(td, "proj"))
        for i in range(2):
            scene = pr.random_scene(np.random.default_rng(5000 + i), smpl, image_size=(512, 512))
            image = pr.render_scene(scene, smpl)
            frame_record("perturbed.frame%d" % i, arrs, dig, image, scene, rdec, mhr, smpl, gt, rproj,
                         keep_inter=(i == 0))
            print("perturbed", i, time.time() - t0, flush=True)

    if "render" in parts:
        for i in range(4):
            scene = pr.random_scene(np.random.default_rng(5000 + i), smpl, image_size=(512, 512))
            image = pr.render_scene(scene, smpl)
            dig["render%d.image" % i] = digest(image)
            arrs["render%d.rows" % i] = image[::32].copy()
        # one odd-sized frame with a keypoint off the frame
        scene = oof_scenes(smpl)[0]
        scene = pr.Scene(image_size=(300, 200), camera=scene.camera, pose=scene.pose,
                         translation=scene.translation, seed=scene.seed,
                         keypoints2d=(scene.keypoints2d * np.float32(0.5)).astype(np.float32))
        image = pr.render_scene(scene, smpl)
        arrs["render_odd.kp"] = scene.keypoints2d
        arrs["render_odd.seed"] = np.int64(scene.seed)
        arrs.pop("render_odd.image", None)
        arrs["render_odd.rows"] = image[::5].copy()
        dig["render_odd.image"] = digest(image)
        print("render", time.time() - t0, flush=True)

    if "toy" in parts:
        tmhr, tsmpl, tgt = bm.make_toy_models(seed=0, mhr_vertices=1200, smpl_vertices=600)
        tproj = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
        tdec = dc.Decoder(tsmpl, dc.DecoderConfig(), seed=40)
        for i in range(2):
            scene = pr.random_scene(np.random.default_rng(5000 + i), tsmpl, image_size=(512, 512))
            image = pr.render_scene(scene, tsmpl)
            frame_record("toy.frame%d" % i, arrs, dig, image, scene, tdec, tmhr, tsmpl, tgt, tproj)
            print("toy", i, time.time() - t0, flush=True)

    if "c3" in parts:
        rng = np.random.default_rng(3)
        c3 = np.zeros((4096, 76), np.float32)
        c3[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
        c3[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
        c3[:, 51:54] = 0.0
        c3[:, 63:66] = 0.0
        sel = np.r_[0:32, 4064:4096]  # both ends of the 4096-mesh batch
        p = c3[sel]
        v = bm.skin_batch(mhr, p)
        th = pj.project_batch(v, gt, proj)
        j, _ = bm.fk_batch(smpl, th)
        arrs["c3x.sel"] = sel
        dig["c3x.v_mhr"] = digest(v)
        arrs["c3x.v_mhr_rows"] = v[:, ::61].copy()
        arrs["c3x.theta"] = th
        arrs["c3x.j_smpl"] = j
        print("c3", time.time() - t0, flush=True)

    if "vitl24" in parts:
        cfg = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16, enc_layers=24, body_layers=1,
                               hand_layers=1)
        dl = dc.Decoder(smpl, cfg, seed=40)
        crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
        f = dl.encode(crop)
        dig["c4.l24.feats"] = digest(f)
        arrs["c4.l24.feats_rows"] = f[0, ::36].copy()
        print("vitl24", time.time() - t0, flush=True)

    os.makedirs(OUT, exist_ok=True)
    with open(DIG, "w") as fh:
        json.dump(dig, fh, indent=0, sort_keys=True)
    np.savez_compressed(NPZ, **arrs)
    print("wrote", len(dig), "digests and", len(arrs), "arrays in", time.time() - t0, "s")


if __name__ == "__main__":
    main(set(sys.argv[1:]) or {"oof", "perturbed", "render", "toy", "c3", "vitl24"})
