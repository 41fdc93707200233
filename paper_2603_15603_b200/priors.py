"""Spatial priors: keypoint stub, body/hand boxes and crop grids.

Drop-in for the reference ``fsb.priors`` (pkg/src/fsb/priors.py).  Box
arithmetic (``_body_box_from_keypoints`` :166, ``hand_box`` :198,
``crop_grid`` :220) runs in the bit-exact K1 kernels (csrc/k_crops.cu);
scene synthesis and rendering (:81-159, :237) are host-side input
generators re-exported from ``synth.py``.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

from . import runtime
from .numkit import DTYPE, UsageError
from .synth import (CameraIntrinsics, Scene, default_camera, make_scene,  # noqa: F401
                    random_scene, render_scene)

_SPREAD_K = 2.6
_PAD_PX = 8.0


@dataclass
class BBox:
    """(priors.py:29-50)"""

    x_min: float
    y_min: float
    x_max: float
    y_max: float

    def __post_init__(self):
        if not (self.x_min < self.x_max and self.y_min < self.y_max):
            raise UsageError("inverted box: %r" % (self,))

    @property
    def width(self):
        return self.x_max - self.x_min

    @property
    def height(self):
        return self.y_max - self.y_min

    def as_array(self):
        return np.array([self.x_min, self.y_min, self.x_max, self.y_max], dtype=DTYPE)


@dataclass
class Keypoints2D:
    """(priors.py:53-65)"""

    xy: np.ndarray
    confidence: np.ndarray

    def __post_init__(self):
        self.xy = np.asarray(self.xy, dtype=DTYPE)
        self.confidence = np.asarray(self.confidence, dtype=DTYPE)
        if self.xy.ndim != 2 or self.xy.shape[1] != 2 or self.confidence.shape != (self.xy.shape[0],):
            raise UsageError("keypoints must be (J, 2) with (J,) confidences")
        if np.any(self.confidence < 0.0) or np.any(self.confidence > 1.0):
            raise UsageError("confidences must lie in [0, 1]")


def _dev(x, torch, dtype):
    t, _ = runtime.to_device(x, dtype, torch)
    return t


def body_boxes(kp, image_size):
    """Batched body boxes: kp (n, 22, 2) -> (n, 4) float64 on the GPU."""
    ctx = runtime.default_context()
    torch = ctx.torch
    k = _dev(np.asarray(kp, DTYPE).reshape(-1, 22, 2), torch, torch.float32)
    out = torch.empty((k.shape[0], 4), dtype=torch.float64, device=k.device)
    w, h = image_size
    ctx.check(ctx.lib.fsb_body_boxes(ctx.h, runtime.ptr(k), k.shape[0], int(w), int(h), runtime.ptr(out),
                                     ctx.stream), "body_boxes")
    return out.cpu().numpy()


def _body_box_from_keypoints(kp_xy, image_size):
    b = body_boxes(np.asarray(kp_xy, DTYPE)[None], image_size)[0]
    return BBox(*map(float, b))


def detect_stub(scene, noise_sigma=0.0, seed=0):
    """Keypoints (+ seeded Gaussian noise, clipped to the frame) and the body
    box derived from them (priors.py:179-195)."""
    rng = np.random.default_rng(seed)
    noise = rng.normal(0.0, noise_sigma, size=scene.keypoints2d.shape)
    w, h = scene.image_size
    kp = np.clip(scene.keypoints2d + noise.astype(DTYPE), 0.0, [w - 1.0, h - 1.0]).astype(DTYPE)
    return _body_box_from_keypoints(kp, scene.image_size), Keypoints2D(kp, np.ones(kp.shape[0], DTYPE))


def hand_box(wrist, body_box, alpha=3.0, image_size=None):
    """Wrist-centred square of side min(w, h) / alpha (priors.py:198-217)."""
    if alpha <= 0:
        raise UsageError("alpha must be positive")
    ctx = runtime.default_context()
    torch = ctx.torch
    wr = _dev(np.array([[float(wrist[0]), float(wrist[1])]], np.float64), torch, torch.float64)
    bb = _dev(np.array([[body_box.x_min, body_box.y_min, body_box.x_max, body_box.y_max]], np.float64),
              torch, torch.float64)
    out = torch.empty((1, 4), dtype=torch.float64, device=wr.device)
    w, h = (0, 0) if image_size is None else image_size
    ctx.check(ctx.lib.fsb_hand_boxes(ctx.h, runtime.ptr(wr), runtime.ptr(bb), 1, float(alpha), int(w), int(h),
                                     runtime.ptr(out), ctx.stream), "hand_box")
    return BBox(*map(float, out.cpu().numpy()[0]))


def render_records(scenes):
    """Per-scene parameters of render_scene (priors.py:237-252) packed in the
    464-byte layout of fsb_render: keypoints, 0.5 * colours (the seeded RNG
    draws of the reference), float32(-0.5 / sigma^2) and the ramp slope."""
    rec = np.zeros((len(scenes), 116), dtype=np.float32)
    for i, sc in enumerate(scenes):
        kp = np.asarray(sc.keypoints2d, DTYPE)
        rng = np.random.default_rng(sc.seed)
        colors = rng.uniform(0.4, 1.0, size=(kp.shape[0], 3)).astype(DTYPE)
        gdir = rng.uniform(-1.0, 1.0, size=2)
        span = max(float(np.ptp(kp[:, 0])), float(np.ptp(kp[:, 1])))
        sigma = max(6.0, 0.085 * span)
        rec[i, :44] = kp.reshape(-1)
        rec[i, 44:110] = (0.5 * colors).reshape(-1)
        rec[i, 110] = np.float32(-0.5 / (sigma * sigma))
        rec[i, 112:116] = np.asarray(gdir, np.float64).view(np.float32)
    return rec


def render_scenes(scenes, out=None):
    """Render a batch of same-size scenes on the GPU -> CUDA tensor
    (B, H, W, 3) float32 (the benchmark's frame generator)."""
    ctx = runtime.default_context()
    torch = ctx.torch
    w, h = scenes[0].image_size
    if any(tuple(s.image_size) != (w, h) for s in scenes):
        raise UsageError("render_scenes needs scenes of one image size")
    rec = _dev(render_records(scenes), torch, torch.float32)
    if out is None:
        out = torch.empty((len(scenes), h, w, 3), dtype=torch.float32, device=rec.device)
    ctx.check(ctx.lib.fsb_render(ctx.h, runtime.ptr(rec), len(scenes), int(h), int(w), runtime.ptr(out),
                                 ctx.stream), "render_scenes")
    return out


def crop_grid(box, out_size):
    """(S, S, 2) float32 sampling grid spanning the box inclusively
    (priors.py:220-230)."""
    if out_size < 2:
        raise UsageError("out_size must be >= 2")
    if not (box.x_min < box.x_max and box.y_min < box.y_max):
        raise UsageError("inverted box: %r" % (box,))
    ctx = runtime.default_context()
    torch = ctx.torch
    bb = _dev(np.array([[box.x_min, box.y_min, box.x_max, box.y_max]], np.float64), torch, torch.float64)
    out = torch.empty((1, out_size, out_size, 2), dtype=torch.float32, device=bb.device)
    ctx.check(ctx.lib.fsb_crop_grid(ctx.h, runtime.ptr(bb), 1, int(out_size), runtime.ptr(out), ctx.stream),
              "crop_grid")
    return out.cpu().numpy()[0]


# ---------------------------------------------------------------------------
# scene files (priors.py:130-159): the same JSON payload, so scene files move
# between the reference and this package unchanged


def save_scene(scene, path):
    payload = {
        "image_size": [int(scene.image_size[0]), int(scene.image_size[1])],
        "camera": {"fx": scene.camera.fx, "fy": scene.camera.fy, "cx": scene.camera.cx, "cy": scene.camera.cy},
        "pose": [float(v) for v in scene.pose],
        "translation": [float(v) for v in scene.translation],
        "seed": int(scene.seed),
    }
    with open(path, "w") as fh:
        json.dump(payload, fh)


def scene_from_dict(payload, template):
    """Rebuild one scene from a save_scene payload (a plain JSON object)."""
    try:
        cam = CameraIntrinsics(**payload["camera"])
        pose = np.asarray(payload["pose"], dtype=DTYPE)
        translation = np.asarray(payload["translation"], dtype=DTYPE)
        image_size = tuple(payload["image_size"])
        seed = payload["seed"]
    except (TypeError, KeyError) as exc:
        raise UsageError("malformed scene payload: %s" % (exc,))
    return make_scene(template, pose, translation, cam, image_size, seed)


def load_scene(path, template):
    with open(path) as fh:
        payload = json.load(fh)
    return scene_from_dict(payload, template)


def detect_dense(image):
    """The serial baseline's sliding-window detector (priors.py:272-300) is
    not part of the accelerated path: raises UsageError."""
    raise UsageError("detect_dense belongs to the serial baseline, which this package does not accelerate; "
                     "use detect_stub (the fast path's keypoint prior)")
