"""Execution plans and the accelerated frame pathway.

Drop-in for the reference ``fsb.pipeline`` (pkg/src/fsb/pipeline.py) on its
fast path: ``PipeConfig``/``fast_config`` (:43-82), ``PipelinePlan`` (:152),
``prepare_crops`` (:295), ``_box_prompt`` (:318), ``Pipeline.run`` (:377) and
``run_fast`` (:513), plus the batched entry ``run_batch`` and the frame ->
SMPL composition that the reference leaves to its callers.

One frame (or a batch of frames) runs as four kernels on the caller's CUDA
stream, captured once into a CUDA graph and replayed:

    K1 boxes+crops -> K2 encoder -> K3 body/hand decoders (+merge)
    -> K4 FK, MHR LBS, bridge/centroid, projector MLP, SMPL FK

The serial baseline (dense detector, decoded hand boxes, refinement) is not
an accelerated path: configurations that need it raise UsageError.
"""

from __future__ import annotations

import time
from contextlib import contextmanager
from dataclasses import dataclass, replace

import numpy as np

from . import decoder as dc
from . import runtime
from .numkit import DTYPE, ShapeError, UsageError
from .synth import PARAM_DIM

SERIAL_DYNAMIC = "serial_dynamic"
FAST_STATIC = "fast_static"


@dataclass(frozen=True)
class PipeConfig:
    """(pipeline.py:43-68)"""

    detector: str = "stub"
    crop_prep: str = "priors"
    batch_encode: bool = True
    selection: tuple = (0, 1, 2)
    hand_selection: tuple = ()
    refine: bool = False
    plan_mode: str = FAST_STATIC
    consolidate: bool = True
    hands: bool = True
    alpha: float = 3.0
    noise_sigma: float = 0.0
    seed: int = 0


def serial_config():
    return PipeConfig(detector="dense", crop_prep="decoded", batch_encode=False,
                      selection=(0, 1, 2, 3, 4), hand_selection=(0, 1, 2, 3, 4),
                      refine=True, plan_mode=SERIAL_DYNAMIC, consolidate=False)


def fast_config():
    return PipeConfig()


def limit_config():
    return PipeConfig(detector="dense", crop_prep="decoded", batch_encode=True,
                      selection=(0, 1, 2, 3, 4), hand_selection=(0, 1, 2, 3, 4),
                      refine=True, plan_mode=FAST_STATIC, consolidate=True)


@dataclass(frozen=True)
class Stage:
    name: str
    inputs: tuple
    outputs: tuple


_EXTERNAL = ("image", "scene")


def _stage_graph(cfg):
    """Declared dataflow of a configuration (pipeline.py:109-149)."""
    st = [Stage("detect", ("image", "scene"), ("body_box", "keypoints"))]
    if cfg.crop_prep == "priors":
        if cfg.hands:
            st.append(Stage("hand_boxes", ("keypoints", "body_box"), ("hand_boxes",)))
        st.append(Stage("crop_body", ("image", "body_box"), ("body_crop",)))
        if cfg.hands:
            st.append(Stage("crop_hands", ("image", "hand_boxes"), ("hand_crops",)))
        if cfg.batch_encode and cfg.hands:
            st.append(Stage("encode_batch", ("body_crop", "hand_crops"), ("body_feat", "hand_feats")))
        else:
            st.append(Stage("encode_body", ("body_crop",), ("body_feat",)))
            if cfg.hands:
                st.append(Stage("encode_hands", ("hand_crops",), ("hand_feats",)))
        st.append(Stage("decode_body", ("body_feat", "body_box"), ("body_params", "body_camera")))
    else:
        st.append(Stage("crop_body", ("image", "body_box"), ("body_crop",)))
        st.append(Stage("encode_body", ("body_crop",), ("body_feat",)))
        st.append(Stage("decode_body", ("body_feat", "body_box"), ("body_params", "body_camera")))
        if cfg.hands:
            st.append(Stage("hand_boxes", ("body_params", "body_camera", "body_box"), ("hand_boxes",)))
            st.append(Stage("crop_hands", ("image", "hand_boxes"), ("hand_crops",)))
            st.append(Stage("encode_hands", ("hand_crops",), ("hand_feats",)))
    if cfg.hands:
        st.append(Stage("decode_hands", ("hand_feats",), ("hand_rots",)))
        st.append(Stage("merge", ("body_params", "hand_rots"), ("merged",)))
    else:
        st.append(Stage("merge", ("body_params",), ("merged",)))
    return tuple(st)


@dataclass
class StageStat:
    name: str
    mean_ms: float
    p50_ms: float
    p95_ms: float
    calls: int


@dataclass
class LatencyReport:
    stages: list
    total_ms: float
    mode: str
    frames: int = 0

    def stage_sum_ms(self):
        n = max(self.frames, 1)
        return sum(s.mean_ms * (s.calls / n) for s in self.stages)

    def speedup_vs(self, other):
        if self.total_ms <= 0.0:
            raise UsageError("report has no timed frames")
        return other.total_ms / self.total_ms

    def as_dict(self):
        return {"stages": [{"name": s.name, "mean_ms": s.mean_ms, "p50_ms": s.p50_ms, "p95_ms": s.p95_ms,
                            "calls": s.calls} for s in self.stages],
                "total_ms": self.total_ms, "mode": self.mode}


class PipelinePlan:
    """Stage list, workspace table and timers (pipeline.py:152-241).  The
    device workspace lives in the fsb_ctx (reserved once, graph-captured);
    this table holds the host-visible buffers (prompt, merged) so the
    allocation counter keeps the reference's steady-state contract."""

    def __init__(self, stages, mode):
        if mode not in (SERIAL_DYNAMIC, FAST_STATIC):
            raise UsageError("unknown plan mode: %r" % (mode,))
        names = [s.name for s in stages]
        if len(set(names)) != len(names):
            raise UsageError("duplicate stage names: %r" % (names,))
        known = set(_EXTERNAL)
        for s in stages:
            missing = [i for i in s.inputs if i not in known]
            if missing:
                raise UsageError("stage %r consumes %r before any stage produces it" % (s.name, missing))
            known.update(s.outputs)
        self.stages = tuple(stages)
        self.mode = mode
        self.allocations = 0
        self.warm = False
        self._buffers = {}
        self._names = frozenset(names)
        self._timers = {n: {"calls": 0, "ms": []} for n in names}
        self._frame_ms = []

    def buffer(self, name, shape, dtype=DTYPE):
        key = (name, tuple(int(v) for v in shape), np.dtype(dtype))
        if self.mode == SERIAL_DYNAMIC:
            self.allocations += 1
            return np.empty(key[1], dtype=key[2])
        buf = self._buffers.get(key)
        if buf is None:
            buf = np.empty(key[1], dtype=key[2])
            self._buffers[key] = buf
            self.allocations += 1
        return buf

    @contextmanager
    def stage(self, name):
        if name not in self._names:
            raise UsageError("stage %r is not part of this plan" % (name,))
        t0 = time.perf_counter_ns()
        yield
        self.record(name, (time.perf_counter_ns() - t0) / 1e6)

    def record(self, name, ms):
        rec = self._timers[name]
        rec["calls"] += 1
        rec["ms"].append(float(ms))

    def frame_done(self, ms):
        self._frame_ms.append(float(ms))
        self.warm = True

    def reset_timers(self):
        for rec in self._timers.values():
            rec["calls"] = 0
            rec["ms"] = []
        self._frame_ms = []

    def latency_report(self):
        stats = []
        for s in self.stages:
            rec = self._timers[s.name]
            if not rec["ms"]:
                continue
            a = np.asarray(rec["ms"], dtype=np.float64)
            stats.append(StageStat(s.name, float(a.mean()), float(np.percentile(a, 50)),
                                   float(np.percentile(a, 95)), rec["calls"]))
        fr = np.asarray(self._frame_ms, dtype=np.float64)
        return LatencyReport(stats, float(fr.mean()) if fr.size else 0.0, self.mode, fr.size)


def build_plan(config):
    return PipelinePlan(_stage_graph(config), config.plan_mode)


def _box_prompt(box, image_size, out):
    """Normalised 8-slot box prompt (pipeline.py:318-329)."""
    w, h = image_size
    out[:] = np.array([box.x_min / w, box.y_min / h, box.x_max / w, box.y_max / h, box.width / w,
                       box.height / h, (box.x_min + box.x_max) / (2.0 * w), (box.y_min + box.y_max) / (2.0 * h)],
                      dtype=np.float64)
    return out


def prepare_crops(image, boxes, out_size, parallel=False, out=None):
    """One crop per box -> (len(boxes), S, S, 3) via the GPU gather
    (pipeline.py:295-315)."""
    from . import numkit as nk
    from . import priors as pr

    n = len(boxes)
    if out is None:
        out = np.empty((n, out_size, out_size, 3), dtype=DTYPE)
    for i in range(n):
        out[i] = nk.bilinear_sample(image, pr.crop_grid(boxes[i], out_size))
    return out


def _check_fast(cfg):
    bad = []
    if cfg.detector != "stub":
        bad.append("detector=%r" % cfg.detector)
    if cfg.crop_prep != "priors":
        bad.append("crop_prep=%r" % cfg.crop_prep)
    if cfg.refine:
        bad.append("refine=True")
    if not cfg.hands:
        bad.append("hands=False")
    if bad:
        raise UsageError("configuration not on the accelerated path (%s); the serial baseline runs on the "
                         "reference CPU implementation" % ", ".join(bad))


_STAGE_GROUPS = (("crop", ("detect", "hand_boxes", "crop_body", "crop_hands")),
                 ("encode", ("encode_batch", "encode_body", "encode_hands")),
                 ("decode", ("decode_body", "decode_hands", "merge")))


class Pipeline:
    """Runs one Decoder (and, when given, the MHR -> SMPL tail) on the GPU."""

    def __init__(self, decoder, mhr=None, bmap=None, projector=None, precision="fp32", device=None):
        self.decoder = decoder
        self.template = decoder.template
        self.crop_size = decoder.config.crop_size
        self.mhr, self.bmap, self.projector = mhr, bmap, projector
        self.precision = precision
        if device is None:
            import torch

            device = torch.cuda.current_device()
        self.device = device
        self.last_counters = {}
        self._tail_loaded = None

    # -- device setup ----------------------------------------------------------
    def context(self):
        ctx = self.decoder.context(self.device)
        if self.mhr is not None and self._tail_loaded is not ctx:
            if self.bmap is None or self.projector is None:
                raise UsageError("the SMPL tail needs mhr, bmap and projector")
            ctx.load_template(runtime.FSB_MHR, self.mhr)
            ctx.load_projector(self.projector, self.bmap)
            self._tail_loaded = ctx
        return ctx

    # -- batched entry -------------------------------------------------------
    def run_batch(self, images, keypoints, config=None, outputs=None, precision=None, sync=True):
        """B frames in one call.  images (B, H, W, 3) float32, keypoints
        (B, 22, 2) float32 (the stub detector's sigma = 0 keypoints), numpy,
        CUDA tensors or pinned host tensors (read in place: only the crop
        footprints cross PCIe).  Returns a dict of CUDA tensors: boxes, prompt,
        body_params, body_cam, hand_rots, merged and, with the SMPL tail,
        v_mhr, theta, j_smpl.  Rows equal per-frame `run` results."""
        cfg = config if config is not None else fast_config()
        _check_fast(cfg)
        if cfg.noise_sigma != 0.0:
            raise UsageError("run_batch takes detector keypoints directly; add noise before calling")
        ctx = self.context()
        torch = ctx.torch
        img, _ = runtime.frame_source(images, torch.float32, torch, self.device)
        kp, _ = runtime.frame_source(keypoints, torch.float32, torch, self.device)
        if img.ndim != 4 or img.shape[3] != 3:
            raise ShapeError("images must be (B, H, W, 3), got %r" % (tuple(img.shape),))
        b, h, w = img.shape[:3]
        if tuple(kp.shape) != (b, 22, 2):
            raise ShapeError("keypoints must be (B, 22, 2), got %r" % (tuple(kp.shape),))
        out = outputs if outputs is not None else self.allocate_outputs(b, tail=self.mhr is not None)
        self.launch(img, kp, out, cfg, precision)
        if sync:
            ctx.check_finite("run_batch")
        return out

    def allocate_outputs(self, b, tail=True, crops=False, feats=False, v_mhr=True):
        torch = self.context().torch
        dev = torch.device("cuda", self.device)
        cfg = self.decoder.config
        f32 = dict(dtype=torch.float32, device=dev)
        o = {"boxes": torch.empty((b, 3, 4), dtype=torch.float64, device=dev),
             "prompt": torch.empty((b, 8), **f32),
             "body_params": torch.empty((b, PARAM_DIM), **f32),
             "body_cam": torch.empty((b, 3), **f32),
             "hand_rots": torch.empty((b, 2, 3), **f32),
             "merged": torch.empty((b, PARAM_DIM), **f32)}
        if crops:
            o["crops"] = torch.empty((b, 3, cfg.crop_size, cfg.crop_size, 3), **f32)
        if feats:
            o["feats"] = torch.empty((b, 3, self.decoder.n_tokens, cfg.dim), **f32)
        if tail:
            if v_mhr:
                o["v_mhr"] = torch.empty((b, self.mhr.num_vertices, 3), **f32)
            o["theta"] = torch.empty((b, PARAM_DIM), **f32)
            o["j_smpl"] = torch.empty((b, 22, 3), **f32)
        return o

    def launch(self, img, kp, out, cfg, precision=None):
        """Enqueue the whole batch on the current stream (graph replay)."""
        ctx = self.context()
        prec = runtime.PRECISIONS[precision or self.precision]
        b, h, w = img.shape[:3]
        bsel, _ = dc.selection_mask(cfg.selection, self.decoder.config.body_layers)
        hsel, _ = dc.selection_mask(cfg.hand_selection, self.decoder.config.hand_layers, "hand selection")
        if "theta" in out:
            fo = runtime.FrameOutputsC(*[runtime.ptr(out.get(k)) for k, _ in runtime.FrameOutputsC._fields_])
            ctx.check(ctx.lib.fsb_frame_batch(ctx.h, runtime.ptr(img), b, h, w, runtime.ptr(kp), float(cfg.alpha),
                                              bsel, hsel, prec, fo, ctx.stream), "frame_batch")
            return
        # front half only (no SMPL tail): K1 -> K2 -> K3
        torch = ctx.torch
        s = self.crop_size
        crops = out.get("crops")
        if crops is None:
            crops = torch.empty((b, 3, s, s, 3), dtype=torch.float32, device=torch.device("cuda", self.device))
        feats = out.get("feats")
        if feats is None:
            feats = torch.empty((b, 3, self.decoder.n_tokens, self.decoder.config.dim), dtype=torch.float32,
                                device=torch.device("cuda", self.device))
        ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, runtime.ptr(img), b, h, w, runtime.ptr(kp), float(cfg.alpha), s,
                                          runtime.ptr(out["boxes"]), runtime.ptr(out["prompt"]), runtime.ptr(crops),
                                          None, ctx.stream), "boxes_crops")
        ctx.check(ctx.lib.fsb_encode(ctx.h, runtime.ptr(crops), 3 * b, runtime.ptr(feats), prec, ctx.stream),
                  "encode")
        ctx.check(ctx.lib.fsb_decode_frames(ctx.h, runtime.ptr(feats), b, runtime.ptr(out["prompt"]), bsel, hsel,
                                            runtime.ptr(out["body_params"]), runtime.ptr(out["body_cam"]),
                                            runtime.ptr(out["hand_rots"]), runtime.ptr(out["merged"]), prec,
                                            ctx.stream), "decode_frames")

    # -- one frame (reference API) ---------------------------------------------
    def run(self, image, scene, config, plan=None):
        """One frame -> (merged (76,), LatencyReport) (pipeline.py:377-506)."""
        cfg = config
        _check_fast(cfg)
        if plan is None:
            plan = build_plan(cfg)
        from .numkit import check_finite
        from . import priors as pr

        allocs_before = plan.allocations
        t0 = time.perf_counter_ns()
        image = np.ascontiguousarray(image, dtype=DTYPE)
        check_finite(image, "bilinear_sample")
        if cfg.noise_sigma != 0.0:
            _, kp = pr.detect_stub(scene, cfg.noise_sigma, cfg.seed)
            kpxy = kp.xy
        else:
            kpxy = np.asarray(scene.keypoints2d, DTYPE)
        w, h = scene.image_size
        if image.shape[:2] != (h, w):
            raise ShapeError("image %r does not match scene size %r" % (image.shape, scene.image_size))
        ctx = self.context()
        torch = ctx.torch
        st = torch.cuda.current_stream()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        img = torch.from_numpy(image[None]).to(torch.device("cuda", self.device))
        kp = torch.from_numpy(np.ascontiguousarray(kpxy[None])).to(img.device)
        out = self._frame_bufs()
        ev[0].record(st)
        s = self.crop_size
        prec = runtime.PRECISIONS[self.precision]
        ctx.check(ctx.lib.fsb_boxes_crops(ctx.h, runtime.ptr(img), 1, h, w, runtime.ptr(kp), float(cfg.alpha), s,
                                          runtime.ptr(out["boxes"]), runtime.ptr(out["prompt"]),
                                          runtime.ptr(out["crops"]), None, ctx.stream), "boxes_crops")
        ev[1].record(st)
        ctx.check(ctx.lib.fsb_encode(ctx.h, runtime.ptr(out["crops"]), 3, runtime.ptr(out["feats"]), prec,
                                     ctx.stream), "encode")
        ev[2].record(st)
        bsel, nb = dc.selection_mask(cfg.selection, self.decoder.config.body_layers)
        hsel, nh = dc.selection_mask(cfg.hand_selection, self.decoder.config.hand_layers, "hand selection")
        ctx.check(ctx.lib.fsb_decode_frames(ctx.h, runtime.ptr(out["feats"]), 1, runtime.ptr(out["prompt"]), bsel,
                                            hsel, runtime.ptr(out["body_params"]), runtime.ptr(out["body_cam"]),
                                            runtime.ptr(out["hand_rots"]), runtime.ptr(out["merged"]), prec,
                                            ctx.stream), "decode_frames")
        ev[3].record(st)
        prompt = plan.buffer("prompt", (dc.PROMPT_DIM,))
        merged = plan.buffer("merged", (PARAM_DIM,))
        prompt[:] = out["prompt"][0].cpu().numpy()
        merged[:] = out["merged"][0].cpu().numpy()
        ctx.check_finite("run")
        spans = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
        names = set(s_.name for s_ in plan.stages)
        for (_, members), ms in zip(_STAGE_GROUPS, spans):
            present = [m for m in members if m in names]
            for i, m in enumerate(present):
                plan.record(m, ms if i == len(present) - 1 else 0.0)
        counters = {"encode": 1, "encoded_crops": 3, "fk": nb + 2 * nh, "project": nb + 2 * nh,
                    "intermediate": nb}
        if plan.mode == FAST_STATIC and plan.warm and plan.allocations != allocs_before:
            raise UsageError("static plan allocated %d buffers in steady state" % (plan.allocations - allocs_before))
        plan.frame_done((time.perf_counter_ns() - t0) / 1e6)
        self.last_counters = counters
        return merged, plan.latency_report()

    def _frame_bufs(self):
        bufs = getattr(self, "_fbufs", None)
        if bufs is None:
            bufs = self.allocate_outputs(1, tail=False, crops=True, feats=True)
            self._fbufs = bufs
        return bufs

    def run_fast(self, image, scene, config=None):
        return self.run(image, scene, config if config is not None else fast_config())

    def run_serial(self, image, scene):
        return self.run(image, scene, serial_config())


# ---------------------------------------------------------------------------
# equivalence checking (pipeline.py:518-571)

_PARAM_FIELDS = (("orient", slice(0, 3)), ("body_pose", slice(3, 66)), ("left_hand", dc.LEFT_HAND_VEC),
                 ("right_hand", dc.RIGHT_HAND_VEC), ("shape", slice(66, 76)))


@dataclass
class EquivalenceReport:
    tier: str
    passed: bool
    max_abs: float
    deltas: dict
    bound: float

    def as_dict(self):
        return {"tier": self.tier, "passed": self.passed, "max_abs": self.max_abs, "bound": self.bound,
                "deltas": dict(self.deltas)}


def check_equivalence(serial_params, fast_params, tolerances=None):
    tol = dict(tolerances) if tolerances else {"tier": "bit_exact"}
    tier = tol.get("tier", "bit_exact")
    if tier not in ("bit_exact", "bounded"):
        raise UsageError("unknown tolerance tier: %r" % (tier,))
    a = np.asarray(serial_params, dtype=DTYPE).reshape(PARAM_DIM)
    b = np.asarray(fast_params, dtype=DTYPE).reshape(PARAM_DIM)
    diff = np.abs(a.astype(np.float64) - b.astype(np.float64))
    deltas = {name: float(diff[sl].max()) for name, sl in _PARAM_FIELDS}
    if tier == "bit_exact":
        return EquivalenceReport(tier, bool(np.array_equal(a, b)), float(diff.max()), deltas, 0.0)
    bound = float(tol.get("max_abs", 0.0))
    return EquivalenceReport(tier, float(diff.max()) <= bound, float(diff.max()), deltas, bound)


def frame_config(**kw):
    return replace(fast_config(), **kw)
