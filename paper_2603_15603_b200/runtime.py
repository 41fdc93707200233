"""ctypes binding of libfsb_b200.so (include/fsb_b200.h) and the device
context that owns uploaded models, workspace and CUDA graphs.

torch is used only as plumbing: device allocations (torch.empty on cuda),
host<->device copies and the current CUDA stream.  Every computation of the
hot path runs in the library's kernels; if the library or a GPU is missing
the calls raise instead of falling back to anything else.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .numkit import NumericError, ShapeError, UsageError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FSB_LIB") or os.path.join(_PKG, "lib", "libfsb_b200.so")  # FSB_LIB: A/B builds

FSB_FP32, FSB_BF16 = 0, 1
FSB_MHR, FSB_SMPL = 0, 1
PRECISIONS = {"fp32": FSB_FP32, "bf16": FSB_BF16}

_p = ctypes.c_void_p
_i = ctypes.c_int
_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_d = ctypes.c_double


class DecoderConfigC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in
                ("crop_size", "patch", "dim", "heads", "enc_layers", "body_layers", "hand_layers")]


class CountersC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("encode", "encoded_crops", "fk", "project", "intermediate")]


class FrameOutputsC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in
                ("boxes", "prompt", "crops", "feats", "body_params", "body_cam", "hand_rots",
                 "merged", "v_mhr", "theta", "j_smpl", "v_smpl")]


# name -> (restype, argtypes); must match include/fsb_b200.h
_SIGS = {
    "fsb_ctx_create": (_i, [_i, ctypes.POINTER(_p)]),
    "fsb_ctx_create_shared": (_i, [_p, ctypes.POINTER(_p)]),
    "fsb_ctx_destroy": (None, [_p]),
    "fsb_last_error": (ctypes.c_char_p, [_p]),
    "fsb_build_info": (ctypes.c_char_p, []),
    "fsb_reserve": (_i, [_p, _i]),
    "fsb_set_graphs": (_i, [_p, _i]),
    "fsb_load_decoder": (_i, [_p, ctypes.POINTER(DecoderConfigC), _i, ctypes.POINTER(ctypes.c_char_p),
                              ctypes.POINTER(_p), ctypes.POINTER(_i64)]),
    "fsb_load_template": (_i, [_p, _i, _i, _p, _p, _p, _p, _p]),
    "fsb_load_projector": (_i, [_p, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "fsb_boxes_crops": (_i, [_p, _p, _i, _i, _i, _p, _d, _i, _p, _p, _p, _p, _p]),
    "fsb_body_boxes": (_i, [_p, _p, _i, _i, _i, _p, _p]),
    "fsb_hand_boxes": (_i, [_p, _p, _p, _i, _d, _i, _i, _p, _p]),
    "fsb_crop_grid": (_i, [_p, _p, _i, _i, _p, _p]),
    "fsb_bridge": (_i, [_p, _p, _i, _i, _p, _p, _i, _p, _p]),
    "fsb_bilinear": (_i, [_p, _p, _i, _i, _i, _p, _i64, _p, _p]),
    "fsb_encode": (_i, [_p, _p, _i, _p, _i, _p]),
    "fsb_encode_frames": (_i, [_p, _p, _i, _p, _i, _p]),
    "fsb_decode_body": (_i, [_p, _p, _i, _i, _p, _u32, _p, _p, _p, _i, _p]),
    "fsb_decode_hands": (_i, [_p, _p, _i, _u32, _p, _i, _p]),
    "fsb_decode_frames": (_i, [_p, _p, _i, _p, _u32, _u32, _p, _p, _p, _p, _i, _p]),
    "fsb_fk": (_i, [_p, _i, _p, _i, _p, _p, _p]),
    "fsb_skin": (_i, [_p, _i, _p, _i, _p, _p]),
    "fsb_project_vertices": (_i, [_p, _p, _i, _i, _p, _i, _p]),
    "fsb_skin_project": (_i, [_p, _p, _i, _p, _p, _p, _p, _i, _p]),
    "fsb_frame_batch": (_i, [_p, _p, _i, _i, _i, _p, _d, _u32, _u32, _i, ctypes.POINTER(FrameOutputsC), _p]),
    "fsb_render": (_i, [_p, _p, _i, _i, _i, _p, _p]),
    "fsb_nonfinite": (_i, [_p, ctypes.POINTER(_i), _i]),
    "fsb_nonfinite_enqueue": (_i, [_p, _p, _i, _p]),
    "fsb_counters": (_i, [_p, ctypes.POINTER(CountersC)]),
    "fsb_input_bytes": (_i, [_p, ctypes.POINTER(ctypes.c_int64), _i]),
    "fsb_stage_frame": (_i, [_p, _p, ctypes.c_int64, ctypes.POINTER(_i)]),
    "fsb_denoise": (_i, [_p, _p, _i, _p, _p, _p, _p, _i, _p, _p]),
    "fsb_load_denoiser": (_i, [_p, _p, _p, _p, _p, _i]),
    "fsb_bary_map": (_i, [_p, _p, _i, _p, _i, _p, _i, _p, _p, _p, _p]),
    "fsb_fit_batch": (_i, [_p, _p, _i, _i, _p, _i, _d, ctypes.c_float, ctypes.c_float, _p, _p, _p, _p, _p, _p]),
    "fsb_kernel_launches": (_i64, [_p]),
    "fsb_selftest_umma": (_i, [_p, _p, _p, _i, _i, _p, _p]),
}


def pack_kmajor(mat_bf16_u16):
    """Host packing of an (R, K) bf16 matrix (as uint16) into the K-major
    no-swizzle UMMA byte image: element (r, k) at
    (r // 8) * K * 16 + (k // 8) * 128 + (r % 8) * 16 + (k % 8) * 2."""
    m = np.ascontiguousarray(mat_bf16_u16, dtype=np.uint16)
    r, k = m.shape
    if r % 8 or k % 8:
        raise ShapeError("K-major packing needs rows and columns in multiples of 8")
    return np.ascontiguousarray(m.reshape(r // 8, 8, k // 8, 8).transpose(0, 2, 1, 3)).reshape(-1)


def to_bf16_bits(x):
    """float32 -> bfloat16 bit patterns (round to nearest even)."""
    a = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rnd = ((a >> 16) & 1) + 0x7FFF
    return ((a + rnd) >> 16).astype(np.uint16)


def bf16_bits_to_f32(b):
    return (np.asarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)

_LIB = None
_LOCK = threading.Lock()


def lib():
    """Load libfsb_b200.so (raises if it was not built)."""
    global _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError("libfsb_b200.so is not built; run "
                                   "`python -m paper_2603_15603_b200._build` (no CPU fallback exists)")
            h = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _LIB = h
    return _LIB


def exported_symbols():
    return sorted(_SIGS)


def freeze(*arrays):
    """Mark host arrays that were uploaded to the device read-only, so an
    in-place edit (which the device copy would not see) fails loudly instead
    of silently running with stale weights."""
    for a in arrays:
        if isinstance(a, np.ndarray) and a.flags.writeable:
            try:
                a.flags.writeable = False
            except ValueError:
                pass


class IdentityCache:
    """Small LRU of device objects keyed on the IDENTITY of host objects
    (strong references: ids are never reused while an entry lives) plus a
    hashable extra key.  Bounded, so temporary keys cannot leak contexts."""

    def __init__(self, cap=8):
        self.cap = cap
        self.items = []

    def get(self, objs, extra, make):
        for i, (o, e, v) in enumerate(self.items):
            if e == extra and len(o) == len(objs) and all(a is b for a, b in zip(o, objs)):
                self.items.append(self.items.pop(i))
                return v
        v = make()
        self.items.append((tuple(objs), extra, v))
        if len(self.items) > self.cap:
            self.items.pop(0)
        return v

    def clear(self):
        self.items = []


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def stream_handle(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


_ERRORS = {1: ShapeError, 2: NumericError, 3: UsageError}


class Context:
    """One fsb_ctx on one GPU: uploaded models, workspace, graph cache.

    Context(share=other) creates a context that shares `other`'s uploaded
    model (one device copy of the weights, templates and projector) but owns
    its workspace, CUDA graphs, non-finite flag and counters: one per
    in-flight stream (fsb_ctx_create_shared)."""

    def __init__(self, device=None, share=None):
        self.torch = _torch()
        self.lib = lib()
        h = ctypes.c_void_p()
        if share is not None:
            self.device = share.device
            with self.torch.cuda.device(self.device):
                rc = self.lib.fsb_ctx_create_shared(share.h, ctypes.byref(h))
            self.model_state = share.model_state  # what is loaded, shared with `share`
        else:
            self.device = int(self.torch.cuda.current_device() if device is None else device)
            with self.torch.cuda.device(self.device):
                rc = self.lib.fsb_ctx_create(self.device, ctypes.byref(h))
            self.model_state = {}
        if rc != 0:
            raise RuntimeError("fsb_ctx_create failed (code %d)" % rc)
        self.h = h
        self._keep = []

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.fsb_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass

    # -- error handling ------------------------------------------------------
    def check(self, rc, what=""):
        if rc == 0:
            return
        msg = self.lib.fsb_last_error(self.h).decode(errors="replace")
        exc = _ERRORS.get(rc, RuntimeError)
        raise exc("%s: %s" % (what, msg) if what else msg)

    def check_finite(self, what="", reset=True):
        flag = ctypes.c_int(0)
        self.check(self.lib.fsb_nonfinite(self.h, ctypes.byref(flag), int(reset)), "nonfinite")
        if flag.value:
            raise NumericError("%s: non-finite values produced on the device" % what)

    @property
    def stream(self):
        return stream_handle(self.torch)

    def launches(self):
        return int(self.lib.fsb_kernel_launches(self.h))

    def counters(self):
        c = CountersC()
        self.check(self.lib.fsb_counters(self.h, ctypes.byref(c)))
        return {f: int(getattr(c, f)) for f, _ in CountersC._fields_}

    def input_bytes(self, reset=True):
        """Frame bytes the crop gather read since the last reset (synchronises)."""
        n = ctypes.c_int64(0)
        self.check(self.lib.fsb_input_bytes(self.h, ctypes.byref(n), int(reset)), "input_bytes")
        return int(n.value)

    def reserve(self, frames):
        self.check(self.lib.fsb_reserve(self.h, int(frames)), "reserve")

    def set_graphs(self, on):
        self.check(self.lib.fsb_set_graphs(self.h, int(bool(on))))

    # -- uploads -------------------------------------------------------------
    def load_decoder(self, cfg, weights):
        names = sorted(weights)
        arrs = [np.ascontiguousarray(weights[n], dtype=np.float32) for n in names]
        self._keep_upload = arrs
        c = DecoderConfigC(cfg.crop_size, cfg.patch, cfg.dim, cfg.heads, cfg.enc_layers,
                           cfg.body_layers, cfg.hand_layers)
        n = len(names)
        cn = (ctypes.c_char_p * n)(*[s.encode() for s in names])
        cp = (ctypes.c_void_p * n)(*[a.ctypes.data for a in arrs])
        ce = (ctypes.c_int64 * n)(*[a.size for a in arrs])
        self.check(self.lib.fsb_load_decoder(self.h, ctypes.byref(c), n, cn, cp, ce), "load_decoder")
        freeze(*[weights[k] for k in names])
        self.model_state["decoder"] = (weights, getattr(weights, "version", None))

    def load_template(self, which, t):
        v = np.ascontiguousarray(t.vertices_rest, np.float32)
        g = np.ascontiguousarray(t.joints_rest, np.float32)
        par = np.ascontiguousarray(t.parents, np.int64)
        sw = np.ascontiguousarray(t.skin_weights, np.float32)
        sb = np.ascontiguousarray(t.shape_basis, np.float32)
        if v.ndim != 2 or v.shape[1] != 3 or sw.shape != (v.shape[0], 22) or sb.shape != (v.shape[0], 3, 10):
            raise ShapeError("template arrays have inconsistent shapes")
        self.check(self.lib.fsb_load_template(self.h, which, v.shape[0], v.ctypes.data, g.ctypes.data,
                                              par.ctypes.data, sw.ctypes.data, sb.ctypes.data),
                   "load_template")
        freeze(t.vertices_rest, t.joints_rest, t.parents, t.skin_weights, t.shape_basis)
        self.model_state[("template", which)] = t

    def load_projector(self, weights, bmap):
        idx = np.asarray(weights.subsample, np.int64)
        if bmap.corners is None:
            raise UsageError("BaryMap has no corner table; rebuild it with precompute_bary")
        corners = np.ascontiguousarray(np.asarray(bmap.corners, np.int64)[idx])
        bw = np.ascontiguousarray(np.asarray(bmap.weights, np.float32)[idx])
        w1 = np.ascontiguousarray(weights.w1, np.float32)
        if w1.shape[0] != 3 * len(idx):
            raise ShapeError("input width %d does not match the first layer %d" % (3 * len(idx), w1.shape[0]))
        arrs = [np.ascontiguousarray(a, np.float32) for a in
                (weights.b1, weights.w2, weights.b2, weights.w3, weights.b3, weights.mask)]
        h1, h2 = w1.shape[1], arrs[1].shape[1]
        self.check(self.lib.fsb_load_projector(
            self.h, len(idx), h1, h2, corners.ctypes.data, bw.ctypes.data, w1.ctypes.data,
            *[a.ctypes.data for a in arrs]), "load_projector")
        freeze(weights.w1, weights.b1, weights.w2, weights.b2, weights.w3, weights.b3, weights.mask,
               weights.subsample, bmap.corners, bmap.weights)
        self.model_state["projector"] = (weights, bmap)

    def load_denoiser(self, weights):
        """Denoiser epilogue of the SMPL tail (projection.denoise on
        theta[3:66] before the SMPL FK); None removes it."""
        if weights is None:
            self.check(self.lib.fsb_load_denoiser(self.h, None, None, None, None, 0), "load_denoiser")
        else:
            w1, b1, w2, b2 = [np.ascontiguousarray(a, np.float32) for a in (weights.w1, weights.b1, weights.w2, weights.b2)]
            hid = w1.shape[1] if w1.ndim == 2 else -1
            if w1.shape != (63, hid) or b1.shape != (hid,) or w2.shape != (hid, 63) or b2.shape != (63,):
                raise ShapeError("denoiser weights must be (63, h), (h,), (h, 63), (63,)")
            self.check(self.lib.fsb_load_denoiser(self.h, w1.ctypes.data, b1.ctypes.data, w2.ctypes.data,
                                                  b2.ctypes.data, hid), "load_denoiser")
            freeze(weights.w1, weights.b1, weights.w2, weights.b2)
        self.model_state["denoiser"] = weights


# ---------------------------------------------------------------------------
# array plumbing


def to_device(x, dtype, torch, device=None):
    """numpy / torch -> contiguous CUDA tensor of `dtype` (copies only when
    needed); returns (tensor, was_numpy)."""
    if device is None:
        device = torch.cuda.current_device()
    if isinstance(x, torch.Tensor):
        t = x.to(device=torch.device("cuda", device), dtype=dtype)
        return t.contiguous(), False
    a = np.ascontiguousarray(x, dtype={torch.float32: np.float32, torch.float64: np.float64,
                                       torch.int32: np.int32, torch.int64: np.int64}[dtype])
    return torch.from_numpy(a).to(torch.device("cuda", device), non_blocking=False), True


def frame_source(x, dtype, torch, device=None):
    """Like to_device, but a pinned (page-locked) host tensor of the right
    dtype is passed through as-is: the crop gather reads only the crop
    footprints of such frames in place over PCIe instead of copying whole
    frames to HBM first."""
    if (isinstance(x, torch.Tensor) and x.device.type == "cpu" and x.dtype == dtype and x.is_contiguous()
            and x.is_pinned()):
        return x, False
    return to_device(x, dtype, torch, device)


def out_like(t, was_numpy):
    return t.cpu().numpy() if was_numpy else t


_DEFAULT = {}


def default_context(device=None):
    """Process-wide context (per device) for the stand-alone functional API."""
    if device is None:
        device = _torch().cuda.current_device()
    ctx = _DEFAULT.get(device)
    if ctx is None:
        ctx = Context(device)
        _DEFAULT[device] = ctx
    return ctx


def bilinear_sample(image, grid):
    torch = _torch()
    ctx = default_context()
    img, _ = to_device(image, torch.float32, torch)
    g, _ = to_device(grid.reshape(-1, 2), torch.float32, torch)
    h, w, c = img.shape
    out = torch.empty((g.shape[0], c), dtype=torch.float32, device=img.device)
    ctx.check(ctx.lib.fsb_bilinear(ctx.h, ptr(img), h, w, c, ptr(g), g.shape[0], ptr(out), ctx.stream),
              "bilinear_sample")
    ctx.check_finite("bilinear_sample")
    return out.cpu().numpy().reshape(grid.shape[:-1] + (c,))
