"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restatement of the reference hot path, one function per reference site.
Every function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/fsb/).  Arithmetic is float32 with the reference's
rounding order; the two numba kernels are restated in ref_kernels.c.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

F32 = np.float32
NJ = 22
PARENTS = np.array([-1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 12, 3, 14, 15,
                    16, 3, 18, 19, 20], dtype=np.int64)
WRISTS = (16, 20)

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build():
    """Compile liboracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.oracle_matmul.argtypes = [p, p, p, i64, i64, i64]
        lib.oracle_matmul.restype = None
        lib.oracle_fk_compose.argtypes = [p, p, p, p, p, p, p, i64]
        lib.oracle_fk_compose.restype = None
        _LIB = lib
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# numeric primitives


def mm(a, b):
    """numkit.matmul (numkit.py:93-116): k-sequential, no FMA."""
    a = np.ascontiguousarray(a, dtype=F32)
    b = np.ascontiguousarray(b, dtype=F32)
    assert a.ndim == 2 and b.ndim == 2 and a.shape[1] == b.shape[0]
    out = np.empty((a.shape[0], b.shape[1]), dtype=F32)
    _lib().oracle_matmul(_ptr(a), _ptr(b), _ptr(out), a.shape[0], a.shape[1], b.shape[1])
    return out


def layer_norm(x, g, b):
    """numkit.layer_norm (numkit.py:198-202), eps 1e-5, numpy reductions."""
    mu = x.mean(axis=-1, keepdims=True)
    d = x - mu
    var = (d * d).mean(axis=-1, keepdims=True)
    return d / np.sqrt(var + F32(1e-5)) * g + b


def softmax(x):
    """numkit.softmax (numkit.py:192-195) along the last axis."""
    e = np.exp(x - np.max(x, axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


# ---------------------------------------------------------------------------
# stage 1: boxes, prompt, grid, bilinear gather


def body_box(kp, image_size):
    """priors._body_box_from_keypoints (priors.py:166-176), written as the
    explicit scalar recipe of SURVEY Appendix B: float32 sequential sums,
    float64 divide by the count, weak-scalar float32 corner arithmetic."""
    w, h = image_size
    kp = np.asarray(kp, dtype=F32)
    n = kp.shape[0]
    box = []
    centres, halves = [], []
    for ax in range(2):
        s = F32(0.0)
        for i in range(n):
            s = F32(s + kp[i, ax])
        c = F32(np.float64(s) / float(n))
        q = F32(0.0)
        for i in range(n):
            d = F32(kp[i, ax] - c)
            q = F32(q + F32(d * d))
        sd = np.sqrt(F32(np.float64(q) / float(n)))
        centres.append(c)
        halves.append(2.6 * float(sd) + 8.0)
    lim = (w, h)
    lo = []
    for ax in range(2):
        v = F32(centres[ax] - F32(halves[ax]))
        v = min(max(v, F32(0.0)), F32(lim[ax] - 2.0))
        lo.append(float(v))
    hi = []
    for ax in range(2):
        v = F32(centres[ax] + F32(halves[ax]))
        v = min(max(v, F32(lo[ax] + 1.0)), F32(lim[ax] - 1.0))
        hi.append(float(v))
    box = (lo[0], lo[1], hi[0], hi[1])
    return box


def hand_box(wrist, box, alpha, image_size):
    """priors.hand_box (priors.py:198-217) with image_size, float64."""
    bw, bh = box[2] - box[0], box[3] - box[1]
    s = min(bw, bh) / alpha
    w, h = image_size
    wx = min(max(float(wrist[0]), 0.0), w - 1.0)
    wy = min(max(float(wrist[1]), 0.0), h - 1.0)
    sx = min(s, w - 1.0)
    sy = min(s, h - 1.0)
    x0 = min(max(wx - s / 2.0, 0.0), (w - 1.0) - sx)
    y0 = min(max(wy - s / 2.0, 0.0), (h - 1.0) - sy)
    return (x0, y0, x0 + sx, y0 + sy)


def box_prompt(box, image_size):
    """pipeline._box_prompt (pipeline.py:318-329)."""
    w, h = image_size
    x0, y0, x1, y1 = box
    return np.array([x0 / w, y0 / h, x1 / w, y1 / h, (x1 - x0) / w,
                     (y1 - y0) / h, (x0 + x1) / (2.0 * w), (y0 + y1) / (2.0 * h)],
                    dtype=np.float64).astype(F32)


def frame_boxes(kp, image_size, alpha=3.0):
    """detect_stub(sigma=0) -> body box, two wrist hand boxes, prompt
    (priors.py:179-195, pipeline.py:356-373, :318-329).  detect_stub clips
    the keypoints into the frame first (priors.py:188-190)."""
    w, h = image_size
    kp = np.clip(np.asarray(kp, F32), 0.0, [w - 1.0, h - 1.0]).astype(F32)
    b = body_box(kp, image_size)
    hands = [hand_box(kp[j], b, alpha, image_size) for j in WRISTS]
    return b, hands, box_prompt(b, image_size)


def linspace_f32(a, b, n):
    """np.linspace(a, b, n, dtype=float32): f32(f64(i)*step + a), last = b."""
    step = (b - a) / (n - 1)
    out = (np.arange(n, dtype=np.float64) * step + a).astype(F32)
    out[-1] = F32(b)
    return out


def crop_grid(box, size):
    """priors.crop_grid (priors.py:220-230)."""
    xs = linspace_f32(box[0], box[2], size)
    ys = linspace_f32(box[1], box[3], size)
    g = np.empty((size, size, 2), dtype=F32)
    g[..., 0] = xs[None, :]
    g[..., 1] = ys[:, None]
    return g


def bilinear_taps(image_shape, grid):
    """numkit._bilinear_parts (numkit.py:123-133): clamped coordinates,
    integer taps and fractional weights."""
    h, w = image_shape[:2]
    x = np.clip(grid[..., 0], F32(0.0), F32(w - 1))
    y = np.clip(grid[..., 1], F32(0.0), F32(h - 1))
    x0 = np.floor(x).astype(np.int64)
    y0 = np.floor(y).astype(np.int64)
    x1 = np.minimum(x0 + 1, w - 1)
    y1 = np.minimum(y0 + 1, h - 1)
    return x0, y0, x1, y1, x - x0.astype(F32), y - y0.astype(F32)


def bilinear_sample(image, grid):
    """numkit.bilinear_sample (numkit.py:136-154)."""
    x0, y0, x1, y1, fx, fy = bilinear_taps(image.shape, grid)
    fx = fx[..., None]
    fy = fy[..., None]
    one = F32(1.0)
    top = image[y0, x0] * (one - fx) + image[y0, x1] * fx
    bot = image[y1, x0] * (one - fx) + image[y1, x1] * fx
    return top * (one - fy) + bot * fy


def frame_crops(image, kp, size=64, alpha=3.0):
    """Stage 1 for one frame: boxes + the (3, S, S, 3) crop batch
    (pipeline.py:356-366, :415-425)."""
    h, w = image.shape[:2]
    b, hands, prompt = frame_boxes(kp, (w, h), alpha)
    crops = np.stack([bilinear_sample(image, crop_grid(bx, size))
                      for bx in [b] + hands])
    return b, hands, prompt, crops


# ---------------------------------------------------------------------------
# stage 2-3: encoder and decoders (decoder.py)


def _proj(x2, W, pre, nm):
    return mm(x2, W[pre + ".w" + nm]) + W[pre + ".b" + nm]


def attention(W, heads, q3, kv3, pre):
    """Decoder._attention (decoder.py:172-203)."""
    bsz, tq, d = q3.shape
    tk = kv3.shape[1]
    q = _proj(q3.reshape(bsz * tq, d), W, pre, "q").reshape(bsz, tq, d)
    k = _proj(kv3.reshape(bsz * tk, d), W, pre, "k").reshape(bsz, tk, d)
    v = _proj(kv3.reshape(bsz * tk, d), W, pre, "v").reshape(bsz, tk, d)
    dh = d // heads
    scale = F32(1.0 / np.sqrt(dh))
    ctx = np.empty((bsz, tq, d), dtype=F32)
    for i in range(bsz):
        for hd in range(heads):
            c = slice(hd * dh, (hd + 1) * dh)
            logits = mm(q[i, :, c], np.ascontiguousarray(k[i, :, c].T)) * scale
            ctx[i, :, c] = mm(softmax(logits), v[i, :, c])
    return _proj(ctx.reshape(bsz * tq, d), W, pre, "o").reshape(bsz, tq, d)


def _ln(W, x2, pre):
    return layer_norm(x2, W[pre + "_g"], W[pre + "_b"])


def mlp(W, x3, pre):
    """Decoder._mlp (decoder.py:205-212): LN, W1, ReLU, W2."""
    bsz, t, d = x3.shape
    h = _ln(W, x3.reshape(bsz * t, d), pre + ".ln")
    h = np.maximum(mm(h, W[pre + ".w1"]) + W[pre + ".b1"], 0.0)
    return (mm(h, W[pre + ".w2"]) + W[pre + ".b2"]).reshape(bsz, t, d)


def self_block(W, heads, x3, pre):
    """Decoder._self_block (decoder.py:214-218)."""
    bsz, t, d = x3.shape
    h = _ln(W, x3.reshape(bsz * t, d), pre + ".ln").reshape(bsz, t, d)
    return attention(W, heads, h, h, pre)


def cross_block(W, heads, x3, f3, pre):
    """Decoder._cross_block (decoder.py:220-227)."""
    bsz, t, d = x3.shape
    hq = _ln(W, x3.reshape(bsz * t, d), pre + ".lnq").reshape(bsz, t, d)
    hk = _ln(W, f3.reshape(-1, d), pre + ".lnkv").reshape(f3.shape)
    return attention(W, heads, hq, hk, pre)


def encode(W, cfg, crops):
    """Decoder.encode (decoder.py:231-260): patchify (py, px, c) order,
    embed, pre-LN layers, final LN.  (B, S, S, 3) -> (B, n*n, D)."""
    crops = np.ascontiguousarray(crops, dtype=F32)
    bsz, s = crops.shape[:2]
    p = cfg.patch
    n = s // p
    pt = crops.reshape(bsz, n, p, n, p, 3).transpose(0, 1, 3, 2, 4, 5)
    pt = np.ascontiguousarray(pt).reshape(bsz * n * n, p * p * 3)
    x = mm(pt, W["enc.patch_w"]) + W["enc.patch_b"]
    x = x.reshape(bsz, n * n, cfg.dim) + W["enc.pos"][None]
    for i in range(cfg.enc_layers):
        x = x + self_block(W, cfg.heads, x, "enc.l%d.self" % i)
        x = x + mlp(W, x, "enc.l%d.mlp" % i)
    return _ln(W, x.reshape(-1, cfg.dim), "enc.norm").reshape(bsz, n * n, cfg.dim)


def rodrigues(omega):
    """bodymodel.rodrigues (bodymodel.py:172-205), float32."""
    w = np.asarray(omega, dtype=F32)
    x, y, z = w[..., 0], w[..., 1], w[..., 2]
    t2 = x * x + y * y + z * z
    small = t2 < F32(1e-12)
    safe = np.where(small, np.ones_like(t2), t2)
    th = np.sqrt(safe)
    one = F32(1.0)
    s = np.where(small, one - t2 * F32(1.0 / 6.0), np.sin(th) / th)
    c = np.where(small, F32(0.5) - t2 * F32(1.0 / 24.0), (one - np.cos(th)) / safe)
    r = np.empty(w.shape[:-1] + (3, 3), dtype=F32)
    r[..., 0, 0] = one - (y * y + z * z) * c
    r[..., 0, 1] = x * y * c - z * s
    r[..., 0, 2] = x * z * c + y * s
    r[..., 1, 0] = x * y * c + z * s
    r[..., 1, 1] = one - (x * x + z * z) * c
    r[..., 1, 2] = y * z * c - x * s
    r[..., 2, 0] = x * z * c - y * s
    r[..., 2, 1] = y * z * c + x * s
    r[..., 2, 2] = one - (x * x + y * y) * c
    return r


def fk_batch(joints_rest, pose_vecs):
    """bodymodel.fk_batch kernel path (bodymodel.py:266-297):
    (B, 76) -> joints (B, 22, 3), rel (B, 22, 3, 4)."""
    pv = np.ascontiguousarray(pose_vecs, dtype=F32)
    bsz = pv.shape[0]
    g = np.ascontiguousarray(joints_rest, dtype=F32)
    tl = g.copy()
    tl[1:] = g[1:] - g[PARENTS[1:]]
    rot = np.ascontiguousarray(rodrigues(pv[:, :66].reshape(bsz, NJ, 3)))
    joints = np.empty((bsz, NJ, 3), F32)
    rel = np.empty((bsz, NJ, 3, 4), F32)
    rw = np.empty((NJ, 3, 3), F32)
    at = np.empty((NJ, 3), F32)
    lib = _lib()
    for i in range(bsz):
        ri = np.ascontiguousarray(rot[i])
        tw = np.empty((NJ, 3), F32)
        lib.oracle_fk_compose(_ptr(ri), _ptr(tl), _ptr(PARENTS), _ptr(g),
                              _ptr(rw), _ptr(tw), _ptr(at), NJ)
        joints[i] = tw
        rel[i, :, :, :3] = rw
        rel[i, :, :, 3] = at
    return joints, rel


def _heads(W, tokens):
    """Decoder._heads (decoder.py:264-272)."""
    t0 = _ln(W, tokens, "body.norm")[0:1]
    params = (mm(t0, W["body.head_params.w"]) + W["body.head_params.b"])[0]
    cam = (mm(t0, W["body.head_cam.w"]) + W["body.head_cam.b"])[0]
    return params, cam


def decode_body(W, cfg, joints_rest, feat, prompt, selection=(0, 1, 2),
                trace=None):
    """Decoder.decode_body without refinement (decoder.py:284-356).
    Returns (params (76,), cam (3,))."""
    d = cfg.dim
    tokens = W["body.token_init"].copy()
    box_tok = (mm(np.asarray(prompt, F32)[None], W["body.prompt_box.w"])
               + W["body.prompt_box.b"]).reshape(4, d)
    tokens[1:5] = tokens[1:5] + box_tok
    p2d = W["body.p2d_init"].copy()
    p3d = W["body.p3d_init"].copy()
    f3 = np.asarray(feat, F32)[None]
    for li in range(cfg.body_layers):
        pre = "body.l%d" % li
        a = tokens.copy()
        a[5:27] = a[5:27] + p2d
        a[27:49] = a[27:49] + p3d
        tokens = tokens + self_block(W, cfg.heads, a[None], pre + ".self")[0]
        tokens = tokens + cross_block(W, cfg.heads, tokens[None], f3, pre + ".cross")[0]
        tokens = tokens + mlp(W, tokens[None], pre + ".mlp")[0]
        if li in selection:
            params, cam = _heads(W, tokens)
            joints = fk_batch(joints_rest, params[None])[0][0]
            kp2d = cam[0] * joints[:, :2] + cam[1:3][None, :]
            if trace is not None:
                trace.append((li, params, cam, kp2d))
            p2d = mm(kp2d, W["body.phi2d.w"]) + W["body.phi2d.b"]
            p3d = mm(joints - joints[0], W["body.phi3d.w"]) + W["body.phi3d.b"]
    return _heads(W, tokens)


def decode_hand(W, cfg, feats, selection=()):
    """Decoder.decode_hand (decoder.py:360-410): (B, n, D) -> rots (B, 3)."""
    feats = np.ascontiguousarray(feats, dtype=F32)
    bsz = feats.shape[0]
    d = cfg.dim
    if bsz == 0:
        return np.zeros((0, 3), F32)
    tokens = np.repeat(W["hand.token_init"][None], bsz, axis=0)
    pts = np.repeat(W["hand.p_init"][None], bsz, axis=0)

    def heads(tok):
        t0 = _ln(W, tok.reshape(bsz * 4, d), "hand.norm").reshape(bsz, 4, d)[:, 0]
        rots = mm(t0, W["hand.head_rot.w"]) + W["hand.head_rot.b"]
        cams = mm(t0, W["hand.head_cam.w"]) + W["hand.head_cam.b"]
        return rots, cams

    for li in range(cfg.hand_layers):
        pre = "hand.l%d" % li
        a = tokens.copy()
        a[:, 1:4] = a[:, 1:4] + pts
        tokens = tokens + self_block(W, cfg.heads, a, pre + ".self")
        tokens = tokens + cross_block(W, cfg.heads, tokens, feats, pre + ".cross")
        tokens = tokens + mlp(W, tokens, pre + ".mlp")
        if li in selection:
            rots, cams = heads(tokens)
            rm = rodrigues(rots)
            cp = W["hand.canon_pts"]
            q = (rm[:, None, :, :] * cp[None, :, None, :]).sum(axis=-1)
            q2 = cams[:, 0:1, None] * q[:, :, :2] + cams[:, None, 1:3]
            pts = (mm(q2.reshape(bsz * 3, 2), W["hand.phi2d.w"])
                   + W["hand.phi2d.b"]).reshape(bsz, 3, d)
    return heads(tokens)[0]


def merge(body_params, left, right):
    """Decoder.merge (decoder.py:414-422)."""
    out = np.array(body_params, dtype=F32).reshape(76)
    out[51:54] = left
    out[63:66] = right
    return out


# ---------------------------------------------------------------------------
# stage 4: LBS, bridge, projector, SMPL FK


def skin_batch(tmpl, pose_vecs):
    """bodymodel.skin_batch, correctives off (bodymodel.py:334-368)."""
    pv = np.ascontiguousarray(pose_vecs, dtype=F32)
    bsz = pv.shape[0]
    nv = tmpl.vertices_rest.shape[0]
    _, rel = fk_batch(tmpl.joints_rest, pv)
    a = rel.reshape(bsz, NJ, 12).transpose(1, 0, 2).reshape(NJ, bsz * 12)
    t = mm(tmpl.skin_weights, a).reshape(nv, bsz, 3, 4).transpose(1, 0, 2, 3)
    basis_t = np.ascontiguousarray(tmpl.shape_basis.reshape(nv * 3, 10).T)
    vs = mm(pv[:, 66:], basis_t).reshape(bsz, nv, 3) + tmpl.vertices_rest[None]
    return (t[..., 0:3] * vs.reshape(bsz, nv, 1, 3)).sum(axis=-1) + t[..., 3]


def projector_inputs(v, corners, weights, idx):
    """projection._projector_inputs (projection.py:447-465) restricted to the
    subsampled targets (rows are independent, so this equals bridging all
    targets and slicing)."""
    v = np.asarray(v, F32)
    cen = v - v[:, :1, :]
    cs = corners[idx]
    sub = (cen[:, cs, :] * weights[idx][:, :, None]).sum(axis=-2)
    x = sub - sub.mean(axis=1, keepdims=True)
    return x.reshape(v.shape[0], -1)


def bridge(v, corners, weights):
    """projection.bridge (projection.py:187-203)."""
    v = np.asarray(v, F32)
    return (v[..., corners, :] * weights[:, :, None]).sum(axis=-2)


def projector_mlp(x, pw):
    """projection._projector_mlp (projection.py:468-472)."""
    h = np.maximum(mm(x, pw["w1"]) + pw["b1"], F32(0.0))
    h = np.maximum(mm(h, pw["w2"]) + pw["b2"], F32(0.0))
    return (mm(h, pw["w3"]) + pw["b3"]) * pw["mask"]


def project_batch(v, corners, weights, pw):
    """projection.project_batch (projection.py:475-483)."""
    return projector_mlp(projector_inputs(v, corners, weights, pw["subsample"]), pw)


def frame_to_smpl(image, kp, W, cfg, mhr, smpl, bmap, pw, trace=None):
    """SURVEY §3.2 composition for one frame: run_fast -> skin(mhr) ->
    project -> fk(smpl).  Returns a dict of every stage output."""
    h, w = image.shape[:2]
    b, hands, prompt, crops = frame_crops(image, kp, cfg.crop_size)
    feats = encode(W, cfg, crops)
    params, cam = decode_body(W, cfg, smpl.joints_rest, feats[0], prompt, (0, 1, 2), trace)
    rots = decode_hand(W, cfg, feats[1:3], ())
    merged = merge(params, rots[0], rots[1])
    v_mhr = skin_batch(mhr, merged[None])
    theta = project_batch(v_mhr, bmap.corners, bmap.weights, pw)
    j_smpl, _ = fk_batch(smpl.joints_rest, theta)
    return dict(body_box=b, hand_boxes=hands, prompt=prompt, crops=crops,
                feats=feats, body_params=params, body_cam=cam, hand_rots=rots,
                merged=merged, v_mhr=v_mhr[0], theta=theta[0], j_smpl=j_smpl[0])


# ---------------------------------------------------------------------------
# kinematic-prior denoiser (projection.py:684-697)


def denoise(w1, b1, w2, b2, x):
    """projection._denoise_forward (projection.py:684-686):
    x + (matmul(relu(matmul(x, w1) + b1), w2) + b2), numkit.matmul order."""
    x = np.asarray(x, F32)
    single = x.ndim == 1
    x2 = x[None] if single else x
    h = np.maximum(mm(x2, w1) + np.asarray(b1, F32), F32(0.0))
    out = x2 + (mm(h, w2) + np.asarray(b2, F32))
    return out[0] if single else out
