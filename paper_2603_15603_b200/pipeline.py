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

import ctypes
import math
import time
from contextlib import contextmanager
from dataclasses import dataclass, replace

import numpy as np

from . import decoder as dc
from . import runtime
from .numkit import DTYPE, NumericError, ShapeError, UsageError
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
        # pure-Python statistics (numpy's mean / linear-interpolation
        # percentile): np.percentile's per-call overhead was ~0.5 ms of a
        # ~1.4 ms single-frame call over eight stages
        stats = []
        for s in self.stages:
            rec = self._timers[s.name]
            if not rec["ms"]:
                continue
            a = sorted(rec["ms"])
            stats.append(StageStat(s.name, _mean(rec["ms"]), _percentile(a, 50.0), _percentile(a, 95.0),
                                   rec["calls"]))
        fr = self._frame_ms
        return LatencyReport(stats, _mean(fr) if fr else 0.0, self.mode, len(fr))


def _mean(v):
    return float(np.float64(math.fsum(v)) / len(v)) if len(v) > 1 else float(v[0])


def _percentile(a, q):
    """numpy.percentile(a, q) (method "linear") of the sorted list a."""
    n = len(a)
    if n == 1:
        return float(a[0])
    idx = (n - 1) * q / 100.0
    lo = int(math.floor(idx))
    hi = min(lo + 1, n - 1)
    t = idx - lo
    lo_v, hi_v = a[lo], a[hi]
    d = hi_v - lo_v
    return float(hi_v - d * (1.0 - t) if t >= 0.5 else lo_v + d * t)


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

    def __init__(self, decoder, mhr=None, bmap=None, projector=None, precision="fp32", device=None, denoiser=None):
        self.decoder = decoder
        self.template = decoder.template
        self.crop_size = decoder.config.crop_size
        self.mhr, self.bmap, self.projector = mhr, bmap, projector
        # optional projection.DenoiserWeights: theta[3:66] = denoise(theta[3:66])
        # before the SMPL FK, fused into the tail's FK kernel (projection.py:684-697)
        self.denoiser = denoiser
        self.precision = precision
        if device is None:
            import torch

            device = torch.cuda.current_device()
        self.device = device
        self.last_counters = {}
        self._parent = None
        self._fork_ctx = None

    def fork(self):
        """Another pipeline over the same decoder and SMPL tail, with its own
        device context (workspace, CUDA graphs, flags) that SHARES the
        uploaded model: one per in-flight stream (SPEC.md:383 -- pipelines
        are per thread; the frozen weights are not duplicated on the GPU)."""
        p = Pipeline(self.decoder, mhr=self.mhr, bmap=self.bmap, projector=self.projector,
                     precision=self.precision, device=self.device, denoiser=self.denoiser)
        p._parent = self if self._parent is None else self._parent
        return p

    # -- device setup ----------------------------------------------------------
    def _load_tail(self, ctx):
        """Make sure the model context holds THIS pipeline's SMPL tail: the
        loaded (mhr, bmap, projector) objects are recorded on the context and
        compared by identity every call, so pipelines sharing a decoder with
        different tails (or a reassigned pipe.projector) never run with
        another's."""
        if self.mhr is None:
            return
        if self.bmap is None or self.projector is None:
            raise UsageError("the SMPL tail needs mhr, bmap and projector")
        st = ctx.model_state
        if st.get(("template", runtime.FSB_MHR)) is not self.mhr:
            ctx.load_template(runtime.FSB_MHR, self.mhr)
        if st.get("projector", (None, None))[0] is not self.projector or st["projector"][1] is not self.bmap:
            ctx.load_projector(self.projector, self.bmap)
        if st.get("denoiser") is not self.denoiser:
            ctx.load_denoiser(self.denoiser)

    def context(self):
        model = self.decoder.context(self.device)
        self._load_tail(model)
        if self._parent is None:
            return model
        if self._fork_ctx is None:
            self._fork_ctx = runtime.Context(share=model)
        return self._fork_ctx

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
        """Enqueue the whole batch on the current stream (one CUDA-graph
        replay of fsb_frame_batch; without theta/j_smpl in `out` only the
        front half -- boxes, crops, encoder, decoders, merge -- runs)."""
        ctx = self.context()
        prec = runtime.PRECISIONS[precision or self.precision]
        b, h, w = img.shape[:3]
        bsel, _ = dc.selection_mask(cfg.selection, self.decoder.config.body_layers)
        hsel, _ = dc.selection_mask(cfg.hand_selection, self.decoder.config.hand_layers, "hand selection")
        fo = runtime.FrameOutputsC(*[runtime.ptr(out.get(k)) for k, _ in runtime.FrameOutputsC._fields_])
        ctx.check(ctx.lib.fsb_frame_batch(ctx.h, runtime.ptr(img), b, h, w, runtime.ptr(kp), float(cfg.alpha),
                                          bsel, hsel, prec, fo, ctx.stream), "frame_batch")

    def prepare(self, img, kp, out, cfg=None, precision=None):
        """A batch whose buffers are fixed (a ring of frame slots, as a video
        stream or the benchmark has): validates shapes once and binds the
        ctypes arguments, so each PreparedBatch.launch() costs one C call
        (the CUDA-graph lookup and launch) instead of rebuilding them."""
        cfg = cfg if cfg is not None else fast_config()
        _check_fast(cfg)
        b, h, w = img.shape[:3]
        if tuple(kp.shape) != (b, 22, 2) or img.ndim != 4 or img.shape[3] != 3:
            raise ShapeError("images (B, H, W, 3) and keypoints (B, 22, 2) expected")
        return PreparedBatch(self, img, kp, out, cfg, precision)

    # -- one frame (reference API) ---------------------------------------------
    def _frame_state(self, h, w, tail):
        """Per-pipeline single-frame buffers (allocated once per frame size):
        a pinned staging frame that K1 gathers the crop footprints from in
        place over PCIe, pinned keypoints, device outputs for B = 1 and pinned
        host buffers the results are read back into."""
        key = (h, w, tail)
        st = getattr(self, "_fstate", None)
        if st is not None and st["key"] == key:
            return st
        torch = self.context().torch
        h_img = torch.empty((1, h, w, 3), dtype=torch.float32).pin_memory()
        h_kp = torch.empty((1, 22, 2), dtype=torch.float32).pin_memory()
        out = self.allocate_outputs(1, tail=tail, v_mhr=False)
        # the results read back live in one flat device buffer (views), so the
        # read-back is a single D2H copy into one flat pinned buffer
        names = ("prompt", "merged") + (("theta", "j_smpl") if tail else ())
        sizes = [out[k].numel() for k in names]
        flat_d = torch.empty(sum(sizes), dtype=torch.float32, device=out["merged"].device)
        flat_h = torch.empty(sum(sizes), dtype=torch.float32).pin_memory()
        host, o = {}, 0
        for k, n in zip(names, sizes):
            shape = tuple(out[k].shape)
            out[k] = flat_d[o:o + n].view(shape)
            host[k] = flat_h[o:o + n].view(shape)
            o += n
        h_flag = torch.zeros((1,), dtype=torch.int32).pin_memory()
        st = {"key": key, "h_img": h_img, "img_np": h_img.numpy()[0], "h_kp": h_kp, "kp_np": h_kp.numpy()[0],
              "out": out, "host": host, "flat_d": flat_d, "flat_h": flat_h, "prep": None, "prep_key": None,
              "h_flag": h_flag, "h_flag_np": h_flag.numpy(),
              "ev": [torch.cuda.Event(enable_timing=True) for _ in range(3)]}
        self._fstate = st
        return st

    def _run_one(self, image, scene, cfg, plan, tail):
        """The single-frame path shared by run() and run_smpl(): host checks
        and keypoints, one graph replay of the fused frame batch (B = 1) on
        the pinned staging frame, one D2H read of the results."""
        _check_fast(cfg)
        if plan is None:
            plan = build_plan(cfg)
        from . import priors as pr

        allocs_before = plan.allocations
        t0 = time.perf_counter_ns()
        image = np.ascontiguousarray(image, dtype=DTYPE)
        w, h = scene.image_size
        if image.ndim != 3 or image.shape != (h, w, 3):
            raise ShapeError("image %r does not match scene size %r" % (image.shape, scene.image_size))
        ctx = self.context()
        st = self._frame_state(h, w, tail)
        # check_finite(image) and the copy into the pinned staging frame in
        # one native pass (fsb_stage_frame)
        bad = ctypes.c_int(0)
        ctx.check(ctx.lib.fsb_stage_frame(image.ctypes.data, st["img_np"].ctypes.data, image.size,
                                          ctypes.byref(bad)), "stage_frame")
        if bad.value:
            raise NumericError("bilinear_sample: non-finite values in operand")
        with plan.stage("detect"):
            if cfg.noise_sigma != 0.0:
                _, kp = pr.detect_stub(scene, cfg.noise_sigma, cfg.seed)
                kpxy = kp.xy
            else:  # sigma = 0: the stub's clip into the frame happens in K1
                kpxy = np.asarray(scene.keypoints2d, DTYPE)
        torch = ctx.torch
        st["kp_np"][...] = kpxy
        stream = torch.cuda.current_stream()
        ev = st["ev"]
        pkey = (cfg.selection, cfg.hand_selection, float(cfg.alpha), self.precision)
        if st["prep_key"] != pkey:  # arguments bound once per configuration
            st["prep"] = self.prepare(st["h_img"], st["h_kp"], st["out"], cfg)
            st["prep_key"] = pkey
        ev[0].record(stream)
        st["prep"].launch(stream)
        ev[1].record(stream)
        st["flat_h"].copy_(st["flat_d"], non_blocking=True)
        # the device's non-finite flag comes back with the results (one sync)
        ctx.check(ctx.lib.fsb_nonfinite_enqueue(ctx.h, st["h_flag"].data_ptr(), 1, stream.cuda_stream),
                  "nonfinite")
        ev[2].record(stream)
        ev[2].synchronize()
        if st["h_flag_np"][0]:
            raise NumericError("run: non-finite values produced on the device")
        prompt = plan.buffer("prompt", (dc.PROMPT_DIM,))
        merged = plan.buffer("merged", (PARAM_DIM,))
        prompt[:] = st["host"]["prompt"].numpy()[0]
        merged[:] = st["host"]["merged"].numpy()[0]
        # the fused graph has no stage boundaries: its device time is booked on
        # the plan's last stage (merge); the host-side detect is timed above
        dev_ms = ev[0].elapsed_time(ev[1])
        names = [s_.name for s_ in plan.stages]
        for m in names:
            if m not in ("detect",):
                plan.record(m, dev_ms if m == names[-1] else 0.0)
        bsel, nb = dc.selection_mask(cfg.selection, self.decoder.config.body_layers)
        hsel, nh = dc.selection_mask(cfg.hand_selection, self.decoder.config.hand_layers, "hand selection")
        self.last_counters = {"encode": 1, "encoded_crops": 3, "fk": nb + 2 * nh, "project": nb + 2 * nh,
                              "intermediate": nb}
        if plan.mode == FAST_STATIC and plan.warm and plan.allocations != allocs_before:
            raise UsageError("static plan allocated %d buffers in steady state" % (plan.allocations - allocs_before))
        plan.frame_done((time.perf_counter_ns() - t0) / 1e6)
        return merged, plan, st

    def run(self, image, scene, config, plan=None):
        """One frame -> (merged (76,), LatencyReport) (pipeline.py:377-506).
        `merged` aliases the plan's buffer, as in the reference."""
        merged, plan, _ = self._run_one(image, scene, config, plan, tail=False)
        return merged, plan.latency_report()

    def run_smpl(self, image, scene, config=None, plan=None):
        """One frame through the whole SURVEY §3.2 composition (crop ->
        encode -> decode -> MHR LBS -> projector -> SMPL FK) from a host
        image to host results: dict(merged, theta, j_smpl) of numpy arrays
        (copies), and the LatencyReport."""
        if self.mhr is None:
            raise UsageError("run_smpl needs the SMPL tail (mhr, bmap, projector)")
        merged, plan, st = self._run_one(image, scene, config if config is not None else fast_config(), plan,
                                         tail=True)
        out = {"merged": merged.copy(), "theta": st["host"]["theta"].numpy()[0].copy(),
               "j_smpl": st["host"]["j_smpl"].numpy()[0].copy()}
        return out, plan.latency_report()

    def run_fast(self, image, scene, config=None):
        return self.run(image, scene, config if config is not None else fast_config())

    def run_serial(self, image, scene):
        return self.run(image, scene, serial_config())


class PreparedBatch:
    """Pipeline.prepare(): fsb_frame_batch with pre-bound arguments.  The
    decoder / tail uploads are still re-checked on every launch (identity and
    version compares), so weight edits are never missed."""

    def __init__(self, pipe, img, kp, out, cfg, precision):
        self.pipe = pipe
        self.keep = (img, kp, out)
        ctx = pipe.context()
        self.lib = ctx.lib
        b, h, w = img.shape[:3]
        bsel, _ = dc.selection_mask(cfg.selection, pipe.decoder.config.body_layers)
        hsel, _ = dc.selection_mask(cfg.hand_selection, pipe.decoder.config.hand_layers, "hand selection")
        self.fo = runtime.FrameOutputsC(*[runtime.ptr(out.get(k)) for k, _ in runtime.FrameOutputsC._fields_])
        import ctypes

        self.args = (runtime.ptr(img), b, h, w, runtime.ptr(kp), float(cfg.alpha), bsel, hsel,
                     runtime.PRECISIONS[precision or pipe.precision], ctypes.byref(self.fo))
        self.torch = ctx.torch

    def launch(self, stream=None):
        """Enqueue on `stream` (a torch stream; default: the current one)."""
        ctx = self.pipe.context()
        st = (stream or self.torch.cuda.current_stream()).cuda_stream
        rc = self.lib.fsb_frame_batch(ctx.h, *self.args, st)
        if rc:
            ctx.check(rc, "frame_batch")


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
