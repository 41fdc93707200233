"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
package itself (read-only at /root/reference/pkg/src).

This script is the only thing in the repo that imports the reference.  It runs
in this (GPU-less) container; the fixtures it writes are committed so that the
oracle restatement (oracle/) and the host-side fixture builders of the product
package can be pinned against the reference without the reference present.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py

Outputs:
    tests/golden/digests.json   sha256 digests of large reference arrays
    tests/golden/golden.npz     small reference arrays (boxes, crops, outputs)

Digest format: "<dtype>|<shape>|<sha256 of C-order bytes>".
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import fsb.bodymodel as bm  # noqa: E402
import fsb.decoder as dc  # noqa: E402
import fsb.pipeline as pl  # noqa: E402
import fsb.priors as pr  # noqa: E402
import fsb.projection as pj  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def digest(a):
    a = np.ascontiguousarray(a)
    return "%s|%s|%s" % (a.dtype.str, "x".join(map(str, a.shape)),
                         hashlib.sha256(a.tobytes()).hexdigest())


def model_digests(mhr, smpl, gt):
    out = {}
    for tag, t in (("mhr", mhr), ("smpl", smpl)):
        for f in ("vertices_rest", "faces", "joints_rest", "parents",
                  "skin_weights", "shape_basis", "corrective_basis",
                  "corrective_gate"):
            out["%s.%s" % (tag, f)] = digest(getattr(t, f))
    out["gt.face_index"] = digest(gt.face_index)
    out["gt.weights"] = digest(gt.weights)
    out["gt.corners"] = digest(gt.corners)
    return out


def main():
    t0 = time.time()
    dig = {}
    arrs = {}

    # -- templates --------------------------------------------------------
    models = {}
    for nv, ns in ((252, 168), (1200, 600), (18439, 6890)):
        mhr, smpl, gt = bm.make_toy_models(seed=0, mhr_vertices=nv,
                                           smpl_vertices=ns)
        models[(nv, ns)] = (mhr, smpl, gt)
        for k, v in model_digests(mhr, smpl, gt).items():
            dig["models.%d_%d.%s" % (nv, ns, k)] = v
    print("templates", time.time() - t0, flush=True)

    # -- decoder weights ---------------------------------------------------
    mhr, smpl, gt = models[(18439, 6890)]
    dec = dc.Decoder(smpl, dc.DecoderConfig(), seed=40)
    for k in sorted(dec.weights):
        dig["decoder.default.%s" % k] = digest(dec.weights[k])
    vitl2 = dc.DecoderConfig(crop_size=384, patch=16, dim=1024, heads=16,
                             enc_layers=2, body_layers=1, hand_layers=1)
    dec_l = dc.Decoder(smpl, vitl2, seed=40)
    for k in sorted(dec_l.weights):
        if k.startswith("enc."):
            dig["decoder.vitl2.%s" % k] = digest(dec_l.weights[k])

    # -- projector weights -------------------------------------------------
    proj = pj.init_projector(pj.make_subsample(6890, 1500), (512, 256), seed=0)
    proj_toy = pj.init_projector(pj.make_subsample(600, 300), (512, 256), seed=0)
    for tag, w in (("full", proj), ("toy", proj_toy)):
        for f in ("w1", "b1", "w2", "b2", "w3", "b3", "subsample", "mask"):
            dig["projector.%s.%s" % (tag, f)] = digest(getattr(w, f))
    print("weights", time.time() - t0, flush=True)

    # -- scenes, boxes, prompts (no rendering needed) ----------------------
    nscene = 256
    kps, poses, trans, seeds = [], [], [], []
    bodies, hands, prompts = [], [], []
    for i in range(nscene):
        scene = pr.random_scene(np.random.default_rng(5000 + i), smpl,
                                image_size=(512, 512))
        kps.append(scene.keypoints2d)
        poses.append(scene.pose)
        trans.append(scene.translation)
        seeds.append(scene.seed)
        box, kp = pr.detect_stub(scene, 0.0, 0)
        assert np.array_equal(kp.xy, scene.keypoints2d)
        bodies.append([box.x_min, box.y_min, box.x_max, box.y_max])
        hb = [pr.hand_box(kp.xy[j], box, alpha=3.0, image_size=(512, 512))
              for j in (bm.LEFT_WRIST, bm.RIGHT_WRIST)]
        hands.append([[b.x_min, b.y_min, b.x_max, b.y_max] for b in hb])
        prompts.append(pl._box_prompt(box, (512, 512),
                                      np.empty(8, dtype=np.float32)).copy())
    arrs["scene_kp"] = np.asarray(kps, np.float32)
    arrs["scene_pose"] = np.asarray(poses, np.float32)
    arrs["scene_trans"] = np.asarray(trans, np.float32)
    arrs["scene_seed"] = np.asarray(seeds, np.int64)
    arrs["box_body"] = np.asarray(bodies, np.float64)
    arrs["box_hands"] = np.asarray(hands, np.float64)
    arrs["prompt"] = np.asarray(prompts, np.float32)

    # stress boxes: keypoints pushed against the frame edges and clustered
    rng = np.random.default_rng(77)
    skp = rng.uniform(-20.0, 531.0, size=(64, 22, 2)).astype(np.float32)
    skp[:16] = rng.uniform(0.0, 3.0, size=(16, 22, 2)).astype(np.float32)
    skp[16:32] = rng.uniform(505.0, 511.0, size=(16, 22, 2)).astype(np.float32)
    skp = np.clip(skp, 0.0, 511.0).astype(np.float32)
    sb, sh, sp = [], [], []
    for i in range(skp.shape[0]):
        box = pr._body_box_from_keypoints(skp[i], (512, 512))
        sb.append([box.x_min, box.y_min, box.x_max, box.y_max])
        hb = [pr.hand_box(skp[i, j], box, alpha=3.0, image_size=(512, 512))
              for j in (bm.LEFT_WRIST, bm.RIGHT_WRIST)]
        sh.append([[b.x_min, b.y_min, b.x_max, b.y_max] for b in hb])
        sp.append(pl._box_prompt(box, (512, 512),
                                 np.empty(8, dtype=np.float32)).copy())
    arrs["stress_kp"] = skp
    arrs["stress_body"] = np.asarray(sb, np.float64)
    arrs["stress_hands"] = np.asarray(sh, np.float64)
    arrs["stress_prompt"] = np.asarray(sp, np.float32)
    print("boxes", time.time() - t0, flush=True)

    # -- rendered frames, crops, full frame -> SMPL ------------------------
    pipe = pl.Pipeline(dec)
    nframe = 4
    for i in range(nframe):
        scene = pr.random_scene(np.random.default_rng(5000 + i), smpl,
                                image_size=(512, 512))
        image = pr.render_scene(scene, smpl)
        dig["frame%d.image" % i] = digest(image)
        arrs["frame%d.image_rows" % i] = image[::64].copy()
        box, kp = pr.detect_stub(scene, 0.0, 0)
        hb = [pr.hand_box(kp.xy[j], box, alpha=3.0, image_size=(512, 512))
              for j in (bm.LEFT_WRIST, bm.RIGHT_WRIST)]
        crops = pl.prepare_crops(image, [box] + hb, 64)
        dig["frame%d.crops" % i] = digest(crops)
        if i < 2:
            arrs["frame%d.crops" % i] = crops
        feats = dec.encode(crops)
        dig["frame%d.feats" % i] = digest(feats)
        prompt = arrs["prompt"][i]
        bout = dec.decode_body(feats[0], prompt, selection=(0, 1, 2))
        rots = dec.decode_hand(feats[1:3], ())
        arrs["frame%d.body_params" % i] = bout.params
        arrs["frame%d.body_cam" % i] = bout.camera
        arrs["frame%d.hand_rots" % i] = rots
        merged, _ = pipe.run(image, scene, pl.fast_config())
        merged = merged.copy()
        arrs["frame%d.merged" % i] = merged
        assert np.array_equal(merged, dec.merge(bout.params, rots[0], rots[1]))
        if i == 0:
            arrs["frame0.feats"] = feats
            for j, it in enumerate(bout.intermediates):
                arrs["frame0.inter%d.params" % j] = it.params
                arrs["frame0.inter%d.cam" % j] = it.camera
                arrs["frame0.inter%d.kp2d" % j] = it.kp2d
        v_mhr = bm.skin_batch(mhr, merged[None], correctives=False)
        theta = pj.project_batch(v_mhr, gt, proj)
        j_smpl, _ = bm.fk_batch(smpl, theta)
        v_smpl = bm.skin_batch(smpl, theta)
        dig["frame%d.v_mhr" % i] = digest(v_mhr)
        dig["frame%d.v_smpl" % i] = digest(v_smpl)
        arrs["frame%d.v_mhr_rows" % i] = v_mhr[0, ::97].copy()
        arrs["frame%d.theta" % i] = theta[0]
        arrs["frame%d.j_smpl" % i] = j_smpl[0]
        print("frame", i, time.time() - t0, flush=True)

    # -- toy-size tail on frame 0 ------------------------------------------
    tmhr, tsmpl, tgt = models[(1200, 600)]
    tmerged = arrs["frame0.merged"]
    tv = bm.skin_batch(tmhr, tmerged[None])
    tth = pj.project_batch(tv, tgt, proj_toy)
    tj, _ = bm.fk_batch(tsmpl, tth)
    dig["toy.frame0.v_mhr"] = digest(tv)
    arrs["toy.frame0.theta"] = tth[0]
    arrs["toy.frame0.j_smpl"] = tj[0]

    # -- C3 microbench poses (first 16 of rng(3)) ---------------------------
    rng = np.random.default_rng(3)
    c3 = np.zeros((4096, 76), np.float32)
    c3[:, :66] = rng.normal(0.0, 0.2, size=(4096, 66))
    c3[:, 66:] = rng.normal(0.0, 0.45, size=(4096, 10))
    c3[:, 51:54] = 0.0
    c3[:, 63:66] = 0.0
    dig["c3.poses"] = digest(c3)
    p16 = c3[:16]
    v16 = bm.skin_batch(mhr, p16)
    th16 = pj.project_batch(v16, gt, proj)
    j16, rel16 = bm.fk_batch(smpl, th16)
    jm16, relm16 = bm.fk_batch(mhr, p16)
    dig["c3.v_mhr16"] = digest(v16)
    arrs["c3.v_mhr16_rows"] = v16[:, ::97].copy()
    arrs["c3.theta16"] = th16
    arrs["c3.j_smpl16"] = j16
    arrs["c3.j_mhr16"] = jm16
    arrs["c3.rel_mhr16"] = relm16
    print("c3", time.time() - t0, flush=True)

    # -- ViT-L-sized encoder, 2 layers, one crop ---------------------------
    crop = np.random.default_rng(0).random((1, 384, 384, 3)).astype(np.float32)
    dig["c4.crop0"] = digest(crop)
    fl = dec_l.encode(crop)
    dig["c4.l2.feats"] = digest(fl)
    arrs["c4.l2.feats_rows"] = fl[0, ::36].copy()
    print("c4", time.time() - t0, flush=True)

    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "digests.json"), "w") as fh:
        json.dump(dig, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrs)
    print("wrote", len(dig), "digests and", len(arrs), "arrays in",
          time.time() - t0, "s")


if __name__ == "__main__":
    main()
