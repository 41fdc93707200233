"""Body models: types, constants, forward kinematics and LBS skinning.

Drop-in for the reference ``fsb.bodymodel`` (pkg/src/fsb/bodymodel.py).
``fk_batch`` (:266) and ``skin_batch`` (:334) run on the GPU (k_body.cu);
template synthesis (``make_toy_models`` :636) is the host-side fixture
builder in ``synth.py``.  Arrays in, arrays out: numpy inputs return numpy
(the H2D/D2H copies are part of the call), CUDA tensors stay on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import runtime
from .numkit import DTYPE, ShapeError, UsageError
from .synth import (BaryMap, BodyTemplate, CameraIntrinsics, LEFT_HAND, LEFT_WRIST,  # noqa: F401
                    NUM_BODY_JOINTS, NUM_JOINTS, PARAM_DIM, PARENTS, RIGHT_HAND, RIGHT_WRIST,
                    SHAPE_DIM, make_toy_models, rodrigues_f32, validate_template)
from .synth import pinhole as project  # noqa: F401

PELVIS = 0
LEFT_HAND_POSE = slice(48, 51)
RIGHT_HAND_POSE = slice(60, 63)

JOINT_NAMES = [
    "pelvis", "spine1", "spine2", "chest", "neck", "head",
    "l_hip", "l_knee", "l_ankle", "l_foot", "r_hip", "r_knee", "r_ankle", "r_foot",
    "l_shoulder", "l_elbow", "l_wrist", "l_hand", "r_shoulder", "r_elbow", "r_wrist", "r_hand",
]


class ProjectionError(ValueError):
    """Point with non-positive depth (bodymodel.py:86)."""


@dataclass
class PoseState:
    """(bodymodel.py:119-155)"""

    global_orient: np.ndarray
    body_pose: np.ndarray
    shape: np.ndarray

    @classmethod
    def zero(cls):
        return cls(np.zeros(3, DTYPE), np.zeros(63, DTYPE), np.zeros(SHAPE_DIM, DTYPE))

    @classmethod
    def from_vector(cls, vec):
        v = np.asarray(vec, dtype=DTYPE).reshape(-1)
        if v.shape[0] != PARAM_DIM:
            raise ShapeError("pose vector must have %d entries, got %d" % (PARAM_DIM, v.shape[0]))
        return cls(v[0:3].copy(), v[3:66].copy(), v[66:].copy())

    def as_vector(self):
        return np.concatenate([np.asarray(self.global_orient, DTYPE).reshape(3),
                               np.asarray(self.body_pose, DTYPE).reshape(63),
                               np.asarray(self.shape, DTYPE).reshape(SHAPE_DIM)]).astype(DTYPE, copy=False)

    def copy(self):
        return PoseState(self.global_orient.copy(), self.body_pose.copy(), self.shape.copy())


@dataclass
class FKResult:
    joints: np.ndarray
    rel_transforms: np.ndarray


def rodrigues(omega):
    """Axis-angle -> rotation matrices (bodymodel.py:172-205), host float32."""
    return rodrigues_f32(omega)


# ---------------------------------------------------------------------------
# device templates for the functional API: one small context per template


_TEMPLATE_CTX = runtime.IdentityCache(cap=8)


def _template_ctx(template):
    """Device context holding `template`: keyed on the identity of the arrays
    it uploaded (strong references, bounded LRU; the uploaded arrays are
    frozen read-only, runtime.freeze)."""
    objs = (template.vertices_rest, template.joints_rest, template.parents, template.skin_weights,
            template.shape_basis)

    def make():
        ctx = runtime.Context()
        ctx.load_template(runtime.FSB_MHR, template)
        return ctx

    return _TEMPLATE_CTX.get(objs, int(template.num_vertices), make)


def _poses(template, pose_vecs, torch):
    if hasattr(pose_vecs, "tape"):
        raise UsageError("tape variables are not supported by the GPU path")
    p, was_np = runtime.to_device(pose_vecs, torch.float32, torch)
    if p.ndim != 2 or p.shape[1] != PARAM_DIM:
        raise ShapeError("pose_vecs must be (B, %d), got %r" % (PARAM_DIM, tuple(p.shape)))
    return p, was_np


def fk_batch(template, pose_vecs, use_kernel=None):
    """(B, 76) -> joints (B, 22, 3), rel (B, 22, 3, 4) on the GPU."""
    ctx = _template_ctx(template)
    torch = ctx.torch
    p, was_np = _poses(template, pose_vecs, torch)
    b = p.shape[0]
    joints = torch.empty((b, NUM_JOINTS, 3), dtype=torch.float32, device=p.device)
    rel = torch.empty((b, NUM_JOINTS, 3, 4), dtype=torch.float32, device=p.device)
    ctx.check(ctx.lib.fsb_fk(ctx.h, runtime.FSB_MHR, runtime.ptr(p), b, runtime.ptr(joints),
                             runtime.ptr(rel), ctx.stream), "fk_batch")
    return runtime.out_like(joints, was_np), runtime.out_like(rel, was_np)


def forward_kinematics(template, pose, use_kernel=True):
    joints, rel = fk_batch(template, pose.as_vector()[None, :])
    return FKResult(joints=joints[0], rel_transforms=rel[0])


def skin_batch(template, pose_vecs, correctives=False, use_kernel=None):
    """Linear blend skinning (B, 76) -> (B, Nv, 3) on the GPU."""
    if correctives:
        raise UsageError("pose correctives are not on the accelerated path (MHR_NO_CORRECTIVES)")
    ctx = _template_ctx(template)
    torch = ctx.torch
    p, was_np = _poses(template, pose_vecs, torch)
    b = p.shape[0]
    out = torch.empty((b, template.num_vertices, 3), dtype=torch.float32, device=p.device)
    ctx.check(ctx.lib.fsb_skin(ctx.h, runtime.FSB_MHR, runtime.ptr(p), b, runtime.ptr(out), ctx.stream),
              "skin_batch")
    ctx.check_finite("skin_batch")
    return runtime.out_like(out, was_np)


def skin(template, pose, correctives=False, use_kernel=True):
    return skin_batch(template, pose.as_vector()[None, :], correctives=correctives)[0]


# ---------------------------------------------------------------------------
# template files (bodymodel.py:655-688): float arrays as FSB1, name, parents
# and faces in a JSON sidecar

_FLOAT_FIELDS = ("vertices_rest", "joints_rest", "skin_weights", "shape_basis", "corrective_basis",
                 "corrective_gate")


def save_template(template, dirpath):
    import json
    import os

    from .numkit import write_fsb1

    os.makedirs(dirpath, exist_ok=True)
    for name in _FLOAT_FIELDS:
        write_fsb1(os.path.join(dirpath, name + ".fsb1"), getattr(template, name))
    with open(os.path.join(dirpath, "meta.json"), "w") as fh:
        json.dump({"name": template.name, "parents": np.asarray(template.parents).tolist(),
                   "faces": np.asarray(template.faces).tolist()}, fh)


def load_template(dirpath):
    import json
    import os

    from .numkit import read_fsb1

    with open(os.path.join(dirpath, "meta.json")) as fh:
        meta = json.load(fh)
    arrays = {name: read_fsb1(os.path.join(dirpath, name + ".fsb1")) for name in _FLOAT_FIELDS}
    t = BodyTemplate(name=meta["name"], faces=np.asarray(meta["faces"], dtype=np.int64),
                     parents=np.asarray(meta["parents"], dtype=np.int64), **arrays)
    validate_template(t)
    return t
