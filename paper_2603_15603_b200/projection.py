"""MHR -> SMPL conversion: barycentric bridge and the feed-forward projector.

Drop-in for the accelerated part of the reference ``fsb.projection``
(pkg/src/fsb/projection.py): ``bridge`` (:187), ``make_subsample`` (:416),
``init_projector`` (:424), ``project_batch`` (:475) and ``project_forward``
(:486).  The projector runs on the GPU (bridge + centroid kernel, then the
three-layer MLP); weight init is the reference's seeded RNG (synth.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import runtime
from .numkit import DTYPE, ShapeError, UsageError
from .synth import PARAM_DIM, BaryMap, BodyTemplate, projector_arrays  # noqa: F401


@dataclass
class ProjectorWeights:
    """(projection.py:395-406)"""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray
    subsample: np.ndarray
    mask: np.ndarray


def _output_mask():
    m = np.ones(PARAM_DIM, dtype=DTYPE)
    m[51:54] = 0.0
    m[63:66] = 0.0
    return m


def make_subsample(n_target, v_sub):
    """Uniform-stride target vertex picks (projection.py:416-421)."""
    if v_sub < 1 or v_sub > n_target:
        raise UsageError("cannot pick %d of %d vertices" % (v_sub, n_target))
    stride = n_target // v_sub
    return np.arange(0, stride * v_sub, stride, dtype=np.int64)


def init_projector(subsample, hidden=(512, 256), seed=0):
    idx = np.asarray(subsample, np.int64)
    w1, w2, w3 = projector_arrays(3 * len(idx), hidden, seed)
    return ProjectorWeights(w1=w1, b1=np.zeros(hidden[0], DTYPE), w2=w2, b2=np.zeros(hidden[1], DTYPE),
                            w3=w3, b3=np.zeros(PARAM_DIM, DTYPE), subsample=idx, mask=_output_mask())


_PROJ_CTX = runtime.IdentityCache(cap=8)


def _projector_ctx(bmap, weights, nv):
    """Device context holding (weights, bmap): keyed on the identity of the
    arrays it uploaded (strong references, bounded LRU) plus the subsample
    contents, so a temporary ProjectorWeights over the same arrays (as
    project_forward(subsample=...) builds) hits, and a different subsample
    never reuses another's corner table."""
    objs = (bmap.corners, bmap.weights, weights.w1, weights.b1, weights.w2, weights.b2, weights.w3, weights.b3,
            weights.mask)
    extra = (int(nv), np.asarray(weights.subsample, np.int64).tobytes())

    def make():
        ctx = runtime.Context()
        ctx.load_projector(weights, bmap)
        return ctx

    return _PROJ_CTX.get(objs, extra, make)


def bridge(v_src, bmap):
    """Resample source vertices onto the target vertex set (GPU gather)."""
    if bmap.corners is None:
        raise UsageError("BaryMap has no corner table; rebuild it with precompute_bary")
    ctx = runtime.default_context()
    torch = ctx.torch
    v, was_np = runtime.to_device(v_src, torch.float32, torch)
    if v.ndim < 2 or v.shape[-1] != 3:
        raise ShapeError("bridge expects (..., Nv, 3) vertices, got %r" % (tuple(v.shape),))
    corners = np.asarray(bmap.corners, np.int64)
    need = int(corners.max()) + 1
    if v.shape[-2] < need:
        raise ShapeError("bridge needs at least %d source vertices, got %d" % (need, v.shape[-2]))
    lead = tuple(v.shape[:-2])
    vb = v.reshape(-1, v.shape[-2], 3)
    c, _ = runtime.to_device(corners.astype(np.int32), torch.int32, torch)
    w, _ = runtime.to_device(np.asarray(bmap.weights, np.float32), torch.float32, torch)
    nt = c.shape[0]
    out = torch.empty((vb.shape[0], nt, 3), dtype=torch.float32, device=v.device)
    ctx.check(ctx.lib.fsb_bridge(ctx.h, runtime.ptr(vb), vb.shape[0], vb.shape[1], runtime.ptr(c), runtime.ptr(w),
                                 nt, runtime.ptr(out), ctx.stream), "bridge")
    return runtime.out_like(out.reshape(lead + (nt, 3)), was_np)


def project_batch(v, bmap, weights, precision="fp32"):
    """(B, Nv, 3) MHR meshes -> (B, 76) SMPL parameters (projection.py:475)."""
    arr_ndim = np.ndim(v) if not hasattr(v, "ndim") else v.ndim
    if arr_ndim == 2:
        raise ShapeError("project_batch expects a batch; use project_forward for one mesh")
    return _project(v, bmap, weights, precision)


def _project(v, bmap, weights, precision):
    idx = np.asarray(weights.subsample, np.int64)
    if 3 * len(idx) != np.asarray(weights.w1).shape[0]:
        raise ShapeError("input width %d does not match the first layer %d"
                         % (3 * len(idx), np.asarray(weights.w1).shape[0]))
    import torch as _t  # plumbing only

    probe = v if isinstance(v, _t.Tensor) else np.asarray(v, DTYPE)
    if probe.ndim != 3 or probe.shape[-1] != 3:
        raise ShapeError("expected (B, Nv, 3) source vertices, got %r" % (tuple(probe.shape),))
    ctx = _projector_ctx(bmap, weights, probe.shape[1])
    torch = ctx.torch
    vd, was_np = runtime.to_device(v, torch.float32, torch)
    b = vd.shape[0]
    out = torch.empty((b, PARAM_DIM), dtype=torch.float32, device=vd.device)
    ctx.check(ctx.lib.fsb_project_vertices(ctx.h, runtime.ptr(vd), b, vd.shape[1], runtime.ptr(out),
                                           runtime.PRECISIONS[precision], ctx.stream), "project_batch")
    ctx.check_finite("project_batch")
    return runtime.out_like(out, was_np)


def project_forward(v, bmap, weights, subsample=None):
    """One (Nv, 3) mesh -> (76,) (projection.py:486-497)."""
    a = np.asarray(v, DTYPE)
    if a.ndim != 2:
        raise ShapeError("project_forward expects one (Nv, 3) mesh")
    if subsample is not None and not np.array_equal(np.asarray(subsample), weights.subsample):
        weights = ProjectorWeights(**{**weights.__dict__, "subsample": np.asarray(subsample, np.int64)})
    return _project(a[None], bmap, weights, "fp32")[0]


# ---------------------------------------------------------------------------
# kinematic-prior denoiser


@dataclass
class DenoiserWeights:
    """(projection.py:669-674): W1 (63, hidden), b1, W2 (hidden, 63), b2."""

    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


def denoise(weights, pose):
    """Nudge a (possibly noisy) body pose toward the training manifold
    (projection.py:689-697): x + (relu(x W1 + b1) W2 + b2) on (63,) or
    (B, 63) poses, on the GPU (k_denoise, bit-identical to the reference's
    numkit.matmul order).  numpy in -> numpy out; CUDA tensors stay on the
    device."""
    torch = runtime._torch()
    ctx = runtime.default_context()
    was_np = not isinstance(pose, torch.Tensor)
    p = np.asarray(pose, DTYPE) if was_np else pose
    single = p.ndim == 1
    if p.ndim not in (1, 2) or p.shape[-1] != 63:
        raise ShapeError("denoise expects (..., 63) body poses")
    x, _ = runtime.to_device(p[None] if single else p, torch.float32, torch)
    h = int(np.asarray(weights.w1).shape[1])
    if np.asarray(weights.w1).shape != (63, h) or np.asarray(weights.w2).shape != (h, 63):
        raise ShapeError("denoiser weights must be (63, h) and (h, 63)")
    dev = [runtime.to_device(np.ascontiguousarray(a, DTYPE), torch.float32, torch)[0]
           for a in (weights.w1, weights.b1, weights.w2, weights.b2)]
    out = torch.empty_like(x)
    ctx.check(ctx.lib.fsb_denoise(ctx.h, runtime.ptr(x), x.shape[0], *[runtime.ptr(t) for t in dev], h,
                                  runtime.ptr(out), ctx.stream), "denoise")
    ctx.check_finite("denoise")
    res = out[0] if single else out
    return res.cpu().numpy() if was_np else res


# ---------------------------------------------------------------------------
# on-disk formats: FSB1 arrays plus a JSON manifest,
# the same files the reference writes (projection.py:793-874), so weights
# trained with the reference load into the GPU path and vice versa.

_PROJECTOR_ARRAYS = ("w1", "b1", "w2", "b2", "w3", "b3")
_DENOISER_ARRAYS = ("w1", "b1", "w2", "b2")


def _manifest(path):
    import json
    import os

    with open(os.path.join(path, "manifest.json")) as fh:
        return json.load(fh)


def _write_manifest(path, obj):
    import json
    import os

    with open(os.path.join(path, "manifest.json"), "w") as fh:
        json.dump(obj, fh, indent=1)


def save_projector(path, weights):
    """(projection.py:797-806): <name>.fsb1 per layer array; the manifest
    holds the kind, hidden widths and the subsample indices."""
    import os

    from .numkit import write_fsb1

    os.makedirs(path, exist_ok=True)
    for name in _PROJECTOR_ARRAYS:
        write_fsb1(os.path.join(path, name + ".fsb1"), getattr(weights, name))
    _write_manifest(path, {"kind": "projector",
                           "hidden": [int(weights.w1.shape[1]), int(weights.w2.shape[1])],
                           "subsample": [int(i) for i in weights.subsample]})


def load_projector(path):
    """(projection.py:809-819)"""
    import os

    from .numkit import read_fsb1

    man = _manifest(path)
    if man.get("kind") != "projector":
        raise UsageError("%s does not hold projector weights" % path)
    arrs = {name: read_fsb1(os.path.join(path, name + ".fsb1")) for name in _PROJECTOR_ARRAYS}
    return ProjectorWeights(subsample=np.asarray(man["subsample"], np.int64), mask=_output_mask(), **arrs)


def save_denoiser(path, weights):
    """(projection.py:822-827)"""
    import os

    from .numkit import write_fsb1

    os.makedirs(path, exist_ok=True)
    for name in _DENOISER_ARRAYS:
        write_fsb1(os.path.join(path, name + ".fsb1"), getattr(weights, name))
    _write_manifest(path, {"kind": "denoiser", "hidden": int(weights.w1.shape[1])})


def load_denoiser(path):
    """(projection.py:830-837)"""
    import os

    from .numkit import read_fsb1

    if _manifest(path).get("kind") != "denoiser":
        raise UsageError("%s does not hold denoiser weights" % path)
    return DenoiserWeights(**{name: read_fsb1(os.path.join(path, name + ".fsb1")) for name in _DENOISER_ARRAYS})


def save_bary_map(path, bmap):
    """(projection.py:840-856): face ids and corner ids go through FSB1's
    float32 payload (exact below 2^24)."""
    import os

    from .numkit import write_fsb1

    if bmap.corners is None:
        raise UsageError("refusing to store a BaryMap without corner indices")
    os.makedirs(path, exist_ok=True)
    write_fsb1(os.path.join(path, "face_index.fsb1"), np.asarray(bmap.face_index).astype(np.int64))
    write_fsb1(os.path.join(path, "weights.fsb1"), bmap.weights)
    write_fsb1(os.path.join(path, "corners.fsb1"), np.asarray(bmap.corners).astype(np.int64))
    _write_manifest(path, {"kind": "bary_map", "targets": int(np.asarray(bmap.face_index).shape[0]),
                           "degenerate_targets": [int(i) for i in bmap.degenerate_targets]})


def load_bary_map(path):
    """(projection.py:859-874)"""
    import os

    from .numkit import read_fsb1

    man = _manifest(path)
    if man.get("kind") != "bary_map":
        raise UsageError("%s does not hold a barycentric map" % path)
    return BaryMap(face_index=read_fsb1(os.path.join(path, "face_index.fsb1")).astype(np.int64),
                   weights=read_fsb1(os.path.join(path, "weights.fsb1")),
                   corners=read_fsb1(os.path.join(path, "corners.fsb1")).astype(np.int64),
                   degenerate_targets=np.asarray(man["degenerate_targets"], dtype=np.int64))


# ---------------------------------------------------------------------------
# iterative fit: the reference's slow conversion
# baseline (projection.py:211-370), on the GPU (k_fit.cu)


@dataclass
class FitConfig:
    """(projection.py:211-219)"""

    steps: int = 300
    lr: float = 0.05
    lambda_pose: float = 1e-3
    lambda_shape: float = 1e-2

    def __post_init__(self):
        if self.steps < 1:
            raise UsageError("FitConfig.steps must be at least 1")


@dataclass
class FitBatchResult:
    """(projection.py:222-226)"""

    params: np.ndarray
    vertex_error: np.ndarray
    curve: np.ndarray


_FIT_CTX = {}


def _fit_context(target):
    """A device context holding `target` in its SMPL slot (cached per template)."""
    key = id(target)
    hit = _FIT_CTX.get(key)
    if hit is not None and hit[0] is target:
        return hit[1]
    ctx = runtime.Context()
    ctx.load_template(runtime.FSB_SMPL, target)
    _FIT_CTX[key] = (target, ctx)
    return ctx


def _fit(v_src, bmap, target, cfg, init, want_grad):
    torch = runtime._torch()
    v = np.asarray(v_src, DTYPE) if not isinstance(v_src, torch.Tensor) else v_src
    if v.ndim != 3 or v.shape[-1] != 3:
        raise ShapeError("fit_batch expects (B, Nv, 3) meshes, got %r" % (tuple(v.shape),))
    return _fit_targets(bridge(v, bmap), target, cfg, init, want_grad)


def _fit_targets(v_t, target, cfg, init, want_grad):
    """fsb_fit_batch on bridged targets (B, Nv_target, 3)."""
    torch = runtime._torch()
    v_t = v_t if isinstance(v_t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v_t, DTYPE))
    if v_t.ndim != 3 or v_t.shape[-1] != 3:
        raise ShapeError("fit targets must be (B, Nv, 3), got %r" % (tuple(v_t.shape),))
    b = int(v_t.shape[0])
    v_t = v_t.to(device=torch.device("cuda", torch.cuda.current_device()), dtype=torch.float32).contiguous()
    if not bool(torch.isfinite(v_t).all()):
        from .numkit import NumericError

        raise NumericError("fit target meshes contain non-finite values")
    init_t = None
    if init is not None:
        init_np = np.array(init, dtype=DTYPE, copy=True)
        if init_np.shape != (b, PARAM_DIM):
            raise ShapeError("init must be (B, %d), got %r" % (PARAM_DIM, init_np.shape))
        init_t = torch.from_numpy(init_np).cuda()
    ctx = _fit_context(target)
    nv = int(v_t.shape[1])
    dev = v_t.device
    scratch = torch.empty((b, nv, 6), dtype=torch.float32, device=dev)
    best = torch.empty((b, PARAM_DIM), dtype=torch.float32, device=dev)
    err = torch.empty((b,), dtype=torch.float64, device=dev)
    curve = torch.empty((b, cfg.steps + 1), dtype=torch.float64, device=dev)
    grad = torch.empty((b, PARAM_DIM), dtype=torch.float32, device=dev) if want_grad else None
    ctx.check(ctx.lib.fsb_fit_batch(ctx.h, runtime.ptr(v_t), b, nv, runtime.ptr(init_t), int(cfg.steps),
                                    float(cfg.lr), float(cfg.lambda_pose), float(cfg.lambda_shape),
                                    runtime.ptr(scratch), runtime.ptr(best), runtime.ptr(err), runtime.ptr(curve),
                                    runtime.ptr(grad), ctx.stream), "fit_batch")
    ctx.check_finite("fit_batch")
    return best, err, curve, grad


def fit_batch(v_src, bmap, target, cfg=None, init=None):
    """Fit target-body parameters to bridged source meshes (projection.py:
    321-370): Adam with cosine-decayed steps on the squared vertex gap plus
    pose/shape penalties, best iterate per mesh kept.  curve[k] is the mean
    over the batch of the best-so-far vertex gap after iterate k."""
    cfg = cfg or FitConfig()
    best, err, curve, _ = _fit(v_src, bmap, target, cfg, init, False)
    return FitBatchResult(params=best.cpu().numpy(), vertex_error=err.cpu().numpy(),
                          curve=curve.mean(dim=0).cpu().numpy())


def fit_objective_grad(theta, *args, **kwargs):
    """Analytic gradient of the fit objective w.r.t. theta (B, 76)
    (projection.py:304-310), on the GPU (k_fit).

    Reference form: fit_objective_grad(theta, template, v_target, cfg=None),
    v_target the bridged targets (B, Nv_template, 3).  Also accepted:
    fit_objective_grad(theta, v_src, bmap, template, cfg=None), which bridges
    the source meshes first."""
    if args and isinstance(args[0], BodyTemplate):
        template, v_target = args[0], args[1]
        cfg = (args[2] if len(args) > 2 else kwargs.get("cfg")) or FitConfig()
        one = FitConfig(steps=1, lr=cfg.lr, lambda_pose=cfg.lambda_pose, lambda_shape=cfg.lambda_shape)
        _, _, _, grad = _fit_targets(v_target, template, one, theta, True)
        return grad.cpu().numpy()
    v_src, bmap, target = args[0], args[1], args[2]
    cfg = (args[3] if len(args) > 3 else kwargs.get("cfg")) or FitConfig()
    _, _, _, grad = _fit(v_src, bmap, target, FitConfig(steps=1, lr=cfg.lr, lambda_pose=cfg.lambda_pose,
                                                        lambda_shape=cfg.lambda_shape), theta, True)
    return grad.cpu().numpy()


def fit_objective_value(theta, template, v_target, cfg=None):
    """Objective at theta (B, 76) -> (loss, per-item mean vertex gaps)
    (projection.py:269-301): the skinning on the GPU (skin_batch), the
    reduction in numpy in the reference's float32 order."""
    from . import bodymodel as bm

    cfg = cfg or FitConfig()
    theta = np.asarray(theta, DTYPE)
    v_target = np.asarray(v_target, DTYPE)
    b = v_target.shape[0]
    v_hat = np.asarray(bm.skin_batch(template, theta), DTYPE)
    diff = v_hat - v_target
    per_item = (diff * diff).reshape((b, -1)).sum(axis=1)
    body, shape = theta[:, 3:66], theta[:, 66:]
    reg = (body * body).reshape((b, -1)).sum(axis=1) * np.float32(cfg.lambda_pose) \
        + (shape * shape).reshape((b, -1)).sum(axis=1) * np.float32(cfg.lambda_shape)
    gap = np.linalg.norm(v_hat.astype(np.float64) - v_target.astype(np.float64), axis=-1).mean(axis=-1)
    return float((per_item + reg).sum()), gap


@dataclass
class FitResult:
    """(projection.py:230-234)"""

    pose: object
    vertex_error: float
    curve: np.ndarray


def iterative_fit(v_src, bmap, target, cfg=None, init=None):
    """Single-mesh fit (projection.py:373-388); init may be a PoseState or a
    76-vector.  One fit_batch of B = 1 on the GPU."""
    from . import bodymodel as bm

    v = np.asarray(v_src, DTYPE)
    if v.ndim != 2:
        raise ShapeError("iterative_fit expects one (Nv, 3) mesh; use fit_batch for batches")
    init_vec = None
    if init is not None:
        vec = init.as_vector() if isinstance(init, bm.PoseState) else np.asarray(init, DTYPE)
        init_vec = vec[None]
    res = fit_batch(v[None], bmap, target, cfg=cfg, init=init_vec)
    return FitResult(pose=bm.PoseState.from_vector(res.params[0]), vertex_error=float(res.vertex_error[0]),
                     curve=res.curve)



# ---------------------------------------------------------------------------
# closest-point barycentric attachment, on the GPU


def bary_map_from_arrays(src_verts, src_faces, tgt_verts, chunk=64):
    """Attach each target point to the closest point on the source surface
    (projection.py:96-177): float64 over every (target, face) pair, ties to
    the lowest face index, zero-area faces projected onto their longest
    edge; bit-identical to the reference (k_bary.cu).  `chunk` is accepted
    for signature compatibility (the GPU search is not chunked)."""
    torch = runtime._torch()
    ctx = runtime.default_context()
    verts = np.ascontiguousarray(src_verts, np.float64)
    faces = np.ascontiguousarray(src_faces, np.int64)
    tgts = np.ascontiguousarray(tgt_verts, np.float64)
    if verts.ndim != 2 or verts.shape[1] != 3:
        raise ShapeError("source vertices must be (Nv, 3)")
    if faces.ndim != 2 or faces.shape[1] != 3:
        raise ShapeError("source faces must be (F, 3)")
    if tgts.ndim != 2 or tgts.shape[1] != 3:
        raise ShapeError("target vertices must be (Nt, 3)")
    dev = torch.device("cuda", torch.cuda.current_device())
    dv = torch.from_numpy(verts).to(dev)
    df = torch.from_numpy(faces).to(dev)
    dt = torch.from_numpy(tgts).to(dev)
    degen = torch.empty((faces.shape[0],), dtype=torch.uint8, device=dev)
    fidx = torch.empty((tgts.shape[0],), dtype=torch.int64, device=dev)
    w = torch.empty((tgts.shape[0], 3), dtype=torch.float32, device=dev)
    ctx.check(ctx.lib.fsb_bary_map(ctx.h, runtime.ptr(dv), verts.shape[0], runtime.ptr(df), faces.shape[0],
                                   runtime.ptr(dt), tgts.shape[0], runtime.ptr(degen), runtime.ptr(fidx),
                                   runtime.ptr(w), ctx.stream), "bary_map")
    face_out = fidx.cpu().numpy()
    deg = degen.cpu().numpy().astype(bool)
    return BaryMap(face_index=face_out, weights=w.cpu().numpy(), corners=faces[face_out],
                   degenerate_targets=np.nonzero(deg[face_out])[0].astype(np.int64))


def precompute_bary(source, target, chunk=64):
    """Rest-pose attachment of every target vertex onto the source surface
    (projection.py:180-184)."""
    return bary_map_from_arrays(source.vertices_rest, source.faces, target.vertices_rest, chunk=chunk)
