"""Host-side fixture builders: toy templates, frozen weights, synthetic scenes.

None of this is on the hot path.  It exists because the reference builds its
templates, decoder weights, projector weights and test scenes from seeded
numpy RNG streams, and the GPU path must run on exactly those arrays.  Every
builder here consumes the RNG in the same order as the reference so the
arrays come out bit-identical (pinned by tests/test_golden_pins.py against
digests taken from the reference itself, tools/make_golden.py):

  * toy templates      bodymodel.py:396-634 (make_toy_models :636)
  * decoder weights    decoder.py:74-154
  * projector weights  projection.py:416-444
  * scenes / render    priors.py:81-126, :237-252
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .numkit import DTYPE, ShapeError, UsageError

NUM_JOINTS = 22
NUM_BODY_JOINTS = 21
SHAPE_DIM = 10
PARAM_DIM = NUM_JOINTS * 3 + SHAPE_DIM

# kinematic tree (parents[j] < j), reference bodymodel.py:29-32
PARENTS = np.array([-1, 0, 1, 2, 3, 4, 0, 6, 7, 8, 0, 10, 11, 12, 3, 14, 15,
                    16, 3, 18, 19, 20], dtype=np.int64)
LEFT_WRIST, LEFT_HAND = 16, 17
RIGHT_WRIST, RIGHT_HAND = 20, 21

# rest skeleton (x left, y up, z forward) and per-bone tube radii; these are
# model constants of the toy body (bodymodel.py:50-83)
_REST = np.array([
    (0.00, 0.00, 0.00), (0.00, 0.10, 0.01), (0.00, 0.22, 0.015),
    (0.00, 0.34, 0.01), (0.00, 0.48, 0.00), (0.00, 0.60, 0.02),
    (0.09, -0.04, 0.00), (0.10, -0.46, 0.01), (0.11, -0.86, -0.02),
    (0.12, -0.92, 0.10), (-0.09, -0.04, 0.00), (-0.10, -0.46, 0.01),
    (-0.11, -0.86, -0.02), (-0.12, -0.92, 0.10), (0.17, 0.42, 0.00),
    (0.44, 0.40, -0.02), (0.69, 0.39, -0.01), (0.80, 0.385, 0.00),
    (-0.17, 0.42, 0.00), (-0.44, 0.40, -0.02), (-0.69, 0.39, -0.01),
    (-0.80, 0.385, 0.00)], dtype=np.float64)
_TUBE_R = (None, 0.115, 0.125, 0.12, 0.05, 0.085, 0.08, 0.065, 0.05, 0.04,
           0.08, 0.065, 0.05, 0.04, 0.06, 0.05, 0.042, 0.038, 0.06, 0.05,
           0.042, 0.038)


@dataclass
class BodyTemplate:
    """Same fields as the reference BodyTemplate (bodymodel.py:90-104)."""

    name: str
    vertices_rest: np.ndarray
    faces: np.ndarray
    joints_rest: np.ndarray
    parents: np.ndarray
    skin_weights: np.ndarray
    shape_basis: np.ndarray
    corrective_basis: np.ndarray
    corrective_gate: np.ndarray

    @property
    def num_vertices(self):
        return self.vertices_rest.shape[0]


@dataclass
class BaryMap:
    """Barycentric attachment of target vertices (bodymodel.py:107-116)."""

    face_index: np.ndarray
    weights: np.ndarray
    corners: np.ndarray = None
    degenerate_targets: np.ndarray = field(
        default_factory=lambda: np.zeros(0, dtype=np.int64))


# ---------------------------------------------------------------------------
# tube-body template synthesis


def _even_split(total, parts):
    q, r = divmod(total, parts)
    return [q + (i < r) for i in range(parts)]


def _tube_grid(quota):
    """(rings, segments): maximise rings*segments <= quota, then prefer a
    ring count near sqrt(quota/3); earliest candidate wins ties."""
    if quota < 6:
        raise UsageError("per-bone vertex quota too small: %d" % quota)
    target = np.sqrt(quota / 3.0)
    cands = [(rg, quota // rg) for rg in range(2, min(9, quota // 3 + 1))
             if quota // rg >= 3]
    return max(cands, key=lambda c: (c[0] * c[1], -abs(c[0] - target)))


def _ortho_pair(u):
    e = np.zeros(3)
    e[np.argmin(np.abs(u))] = 1.0
    a = np.cross(u, e)
    a /= np.linalg.norm(a)
    return a, np.cross(u, a)


def _ease(x):
    x = np.clip(x, 0.0, 1.0)
    return x * x * (3.0 - 2.0 * x)


def _tube_body(name, joints, rng, n_total):
    counts = _even_split(n_total, NUM_BODY_JOINTS)
    pos, tris, skin, layout = [], [], [], []
    for bone in range(NUM_BODY_JOINTS):
        child = bone + 1
        par = int(PARENTS[child])
        base = joints[par]
        axis = joints[child] - base
        e1, e2 = _ortho_pair(axis / np.linalg.norm(axis))
        n_ring, n_seg = _tube_grid(counts[bone])
        first_v, first_f = len(pos), len(tris)
        r_bone = _TUBE_R[child]
        for t in np.linspace(0.12, 0.88, n_ring):
            mid = base + axis * t
            blend = 0.5 * _ease((t - 0.25) / 0.75)
            wrow = np.zeros(NUM_JOINTS)
            wrow[par] = 1.0 - blend
            wrow[child] = blend
            for k in range(n_seg):
                phi = 2.0 * np.pi * k / n_seg
                radius = r_bone * (1.06 - 0.18 * t) * (1.0 + rng.uniform(-0.04, 0.04))
                pos.append(mid + radius * (np.cos(phi) * e1 + np.sin(phi) * e2))
                skin.append(wrow.copy())
        for r in range(n_ring - 1):
            lo, hi = first_v + r * n_seg, first_v + (r + 1) * n_seg
            for k in range(n_seg):
                k2 = (k + 1) % n_seg
                tris.append((lo + k, lo + k2, hi + k))
                tris.append((lo + k2, hi + k2, hi + k))
        layout.append((first_v, n_ring, n_seg, first_f, (n_ring - 1) * n_seg))

    # weld filler vertices onto first-ring edges until the budget is exact
    for extra in range(n_total - len(pos)):
        first_v, _, n_seg, _, _ = layout[extra % NUM_BODY_JOINTS]
        k = (extra // NUM_BODY_JOINTS) % n_seg
        ia, ib = first_v + k, first_v + (k + 1) % n_seg
        edge = pos[ib] - pos[ia]
        e1, _ = _ortho_pair(edge / np.linalg.norm(edge))
        pos.append(0.5 * (pos[ia] + pos[ib]) + 0.01 * e1)
        skin.append(np.array(skin[ia]))
        tris.append((ia, ib, len(pos) - 1))

    verts = np.asarray(pos, dtype=np.float64)
    nv = verts.shape[0]
    basis = np.zeros((nv, 3, SHAPE_DIM))
    for k in range(SHAPE_DIM):
        gain = 2.0 + 0.3 * k
        f1 = rng.normal(size=3) * gain
        f2 = rng.normal(size=3) * gain
        d1 = rng.normal(size=3)
        d1 /= np.linalg.norm(d1)
        d2 = rng.normal(size=3)
        d2 /= np.linalg.norm(d2)
        p1, p2 = rng.uniform(0.0, 2.0 * np.pi, size=2)
        basis[:, :, k] = 0.03 * (np.sin(verts @ f1 + p1)[:, None] * d1
                                 + np.cos(verts @ f2 + p2)[:, None] * d2)
    q, _ = np.linalg.qr(rng.standard_normal((nv * 3, 8)))
    gate = rng.uniform(0.2, 1.0, size=(8, NUM_BODY_JOINTS)) * (0.5 / NUM_BODY_JOINTS)
    tmpl = BodyTemplate(
        name=name, vertices_rest=verts.astype(DTYPE),
        faces=np.asarray(tris, dtype=np.int64), joints_rest=joints.astype(DTYPE),
        parents=PARENTS.copy(), skin_weights=np.asarray(skin, dtype=DTYPE),
        shape_basis=basis.astype(DTYPE),
        corrective_basis=(0.02 * q).reshape(nv, 3, 8).astype(DTYPE),
        corrective_gate=gate.astype(DTYPE))
    return tmpl, layout


def _surface_samples(src, layout, rng, n_total, name):
    counts = _even_split(n_total, NUM_BODY_JOINTS)
    fids, bary, tris = [], [], []
    nv = 0
    for bone in range(NUM_BODY_JOINTS):
        _, rm, sm, f0, _ = layout[bone]
        rs, ss = _tube_grid(counts[bone])
        v0 = nv
        for i in range(rs):
            r = min(int(i * (rm - 1) / rs), rm - 2)
            for j in range(ss):
                s = int(j * sm / ss) % sm
                w = rng.uniform(0.15, 0.75, size=3)
                fids.append(f0 + (r * sm + s) * 2)
                bary.append(w / w.sum())
                nv += 1
        for i in range(rs - 1):
            lo, hi = v0 + i * ss, v0 + (i + 1) * ss
            for j in range(ss):
                j2 = (j + 1) % ss
                tris.append((lo + j, lo + j2, hi + j))
                tris.append((lo + j2, hi + j2, hi + j))
    n_tube_faces = 2 * sum(entry[4] for entry in layout)
    for _ in range(n_total - nv):
        fids.append(int(rng.integers(0, n_tube_faces)))
        w = rng.uniform(0.15, 0.75, size=3)
        bary.append(w / w.sum())
        nv += 1
        tris.append((nv - 1, nv - 2, nv - 3))

    fids = np.asarray(fids, dtype=np.int64)
    bary = np.asarray(bary, dtype=np.float64)
    corner_ids = src.faces[fids]

    def attach(attr):
        rows = attr.reshape(src.num_vertices, -1).astype(np.float64)
        out = np.einsum("tc,tcd->td", bary, rows[corner_ids])
        return out.reshape((n_total,) + attr.shape[1:]).astype(DTYPE)

    verts = np.einsum("tc,tcx->tx", bary,
                      src.vertices_rest.astype(np.float64)[corner_ids])
    tmpl = BodyTemplate(
        name=name, vertices_rest=verts.astype(DTYPE),
        faces=np.asarray(tris, dtype=np.int64),
        joints_rest=src.joints_rest.copy(), parents=src.parents.copy(),
        skin_weights=attach(src.skin_weights), shape_basis=attach(src.shape_basis),
        corrective_basis=attach(src.corrective_basis),
        corrective_gate=src.corrective_gate.copy())
    gt = BaryMap(face_index=fids, weights=bary.astype(DTYPE),
                 corners=corner_ids.astype(np.int64))
    return tmpl, gt


def validate_template(t):
    """Structural checks (bodymodel.py:608-627)."""
    nv = t.num_vertices
    if t.skin_weights.shape != (nv, NUM_JOINTS):
        raise ShapeError("skin_weights must be (Nv, %d)" % NUM_JOINTS)
    if t.shape_basis.shape != (nv, 3, SHAPE_DIM):
        raise ShapeError("shape_basis must be (Nv, 3, %d)" % SHAPE_DIM)
    if t.parents[0] != -1 or np.any(t.parents[1:] >= np.arange(1, NUM_JOINTS)):
        raise UsageError("parents must define a forward-ordered tree")
    rows = t.skin_weights.sum(axis=1)
    if np.max(np.abs(rows - 1.0)) > 1e-4 or np.min(t.skin_weights) < -1e-6:
        raise UsageError("skin weight rows must be a convex combination")
    if t.faces.min() < 0 or t.faces.max() >= nv:
        raise UsageError("face indices out of range")
    seen = np.zeros(nv, dtype=bool)
    seen[t.faces.reshape(-1)] = True
    if not seen.all():
        raise UsageError("every vertex must appear in at least one face")


def make_toy_models(seed=0, mhr_vertices=1200, smpl_vertices=600):
    """(mhr, smpl, gt) toy pair, bit-identical to bodymodel.make_toy_models
    (bodymodel.py:636-651) for the same arguments."""
    rng = np.random.default_rng(seed)
    jitter = rng.uniform(-0.01, 0.01, size=(NUM_JOINTS, 3))
    jitter[0] = 0.0
    joints = _REST + jitter
    mhr, layout = _tube_body("mhr_toy", joints, rng, mhr_vertices)
    smpl, gt = _surface_samples(mhr, layout, rng, smpl_vertices, "smpl_toy")
    validate_template(mhr)
    validate_template(smpl)
    return mhr, smpl, gt


# ---------------------------------------------------------------------------
# decoder and projector weights


def decoder_weight_plan(cfg):
    """Ordered (name, shape, kind, scale) list that reproduces the RNG draw
    order of decoder._init_weights (decoder.py:74-154).  kind is one of
    'mat' (N(0,1)*scale/sqrt(fan_in)), 'raw' (N(0,1)*scale), 'zero', 'one',
    'const' (scale holds the literal value)."""
    d = cfg.dim
    plan = []

    def ln(p):
        plan.append((p + "_g", (d,), "one", None))
        plan.append((p + "_b", (d,), "zero", None))

    def attention(p, cross):
        if cross:
            ln(p + ".lnq")
            ln(p + ".lnkv")
        else:
            ln(p + ".ln")
        for nm in ("wq", "wk", "wv", "wo"):
            plan.append((p + "." + nm, (d, d), "mat", 0.5))
        for nm in ("bq", "bk", "bv", "bo"):
            plan.append((p + "." + nm, (d,), "zero", None))

    def mlp(p):
        ln(p + ".ln")
        plan.append((p + ".w1", (d, 4 * d), "mat", 0.5))
        plan.append((p + ".b1", (4 * d,), "zero", None))
        plan.append((p + ".w2", (4 * d, d), "mat", 0.5))
        plan.append((p + ".b2", (d,), "zero", None))

    def dense(p, fan_in, fan_out, scale):
        plan.append((p + ".w", (fan_in, fan_out), "mat", scale))
        plan.append((p + ".b", (fan_out,), "zero", None))

    n_patch = (cfg.crop_size // cfg.patch) ** 2
    plan.append(("enc.patch_w", (cfg.patch * cfg.patch * 3, d), "mat", 0.5))
    plan.append(("enc.patch_b", (d,), "zero", None))
    plan.append(("enc.pos", (n_patch, d), "raw", 0.3))
    ln("enc.norm")
    for i in range(cfg.enc_layers):
        attention("enc.l%d.self" % i, False)
        mlp("enc.l%d.mlp" % i)
    plan.append(("body.token_init", (51, d), "raw", 0.4))
    plan.append(("body.p2d_init", (NUM_JOINTS, d), "raw", 0.3))
    plan.append(("body.p3d_init", (NUM_JOINTS, d), "raw", 0.3))
    ln("body.norm")
    for i in range(cfg.body_layers):
        attention("body.l%d.self" % i, False)
        attention("body.l%d.cross" % i, True)
        mlp("body.l%d.mlp" % i)
    dense("body.head_params", d, PARAM_DIM, 0.35)
    plan.append(("body.head_cam.w", (d, 3), "mat", 0.35))
    plan.append(("body.head_cam.b", (3,), "const", (0.5, 0.0, 0.0)))
    dense("body.phi2d", 2, d, 0.4)
    dense("body.phi3d", 3, d, 0.4)
    dense("body.prompt_box", 8, 4 * d, 0.4)
    dense("body.prompt_kp", 2 * NUM_JOINTS, 4 * d, 0.25)
    plan.append(("hand.token_init", (4, d), "raw", 0.4))
    plan.append(("hand.p_init", (3, d), "raw", 0.3))
    ln("hand.norm")
    for i in range(cfg.hand_layers):
        attention("hand.l%d.self" % i, False)
        attention("hand.l%d.cross" % i, True)
        mlp("hand.l%d.mlp" % i)
    dense("hand.head_rot", d, 3, 0.35)
    plan.append(("hand.head_cam.w", (d, 3), "mat", 0.35))
    plan.append(("hand.head_cam.b", (3,), "const", (0.5, 0.0, 0.0)))
    dense("hand.phi2d", 2, d, 0.4)
    plan.append(("hand.canon_pts", (3, 3), "const", "eye0.1"))
    return plan


def decoder_weights(cfg, seed, encoder_only=False):
    """Random weight table of decoder_weight_plan(cfg).  encoder_only stops
    after the encoder entries, which come first in the plan, so the values
    are the same as the full table's."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape, kind, scale in decoder_weight_plan(cfg):
        if encoder_only and not name.startswith("enc."):
            break
        if kind == "mat":
            out[name] = (rng.standard_normal(shape) * (scale / np.sqrt(shape[0]))).astype(DTYPE)
        elif kind == "raw":
            out[name] = (rng.standard_normal(shape) * scale).astype(DTYPE)
        elif kind == "zero":
            out[name] = np.zeros(shape, dtype=DTYPE)
        elif kind == "one":
            out[name] = np.ones(shape, dtype=DTYPE)
        elif scale == "eye0.1":
            out[name] = (0.1 * np.eye(3)).astype(DTYPE)
        else:
            out[name] = np.array(scale, dtype=DTYPE)
    return out


def projector_arrays(n_in, hidden, seed):
    """(w1, w2, w3) of init_projector (projection.py:424-444)."""
    rng = np.random.default_rng(seed)
    shapes = ((n_in, hidden[0], 1.4), (hidden[0], hidden[1], 1.4),
              (hidden[1], PARAM_DIM, 0.05))
    return [(rng.normal(0.0, 1.0, size=(fi, fo)) * (sc / np.sqrt(fi))).astype(DTYPE)
            for fi, fo, sc in shapes]


# ---------------------------------------------------------------------------
# host FK used only for scene synthesis (float32 ops in the reference order,
# rodrigues bodymodel.py:172-205, chain bodymodel.py:208-240)


def rodrigues_f32(omega):
    """(..., 3) axis-angle -> (..., 3, 3) float32 rotation matrices."""
    w = np.asarray(omega, dtype=DTYPE)
    x, y, z = w[..., 0], w[..., 1], w[..., 2]
    t2 = x * x + y * y + z * z
    tiny = t2 < np.float32(1e-12)
    den = np.where(tiny, np.ones_like(t2), t2)
    ang = np.sqrt(den)
    one = np.float32(1.0)
    sa = np.where(tiny, one - t2 * np.float32(1.0 / 6.0), np.sin(ang) / ang)
    ca = np.where(tiny, np.float32(0.5) - t2 * np.float32(1.0 / 24.0), (one - np.cos(ang)) / den)
    m = np.stack([
        np.stack([one - (y * y + z * z) * ca, x * y * ca - z * sa, x * z * ca + y * sa], -1),
        np.stack([x * y * ca + z * sa, one - (x * x + z * z) * ca, y * z * ca - x * sa], -1),
        np.stack([x * z * ca - y * sa, y * z * ca + x * sa, one - (x * x + y * y) * ca], -1),
    ], -2)
    return m


def fk_joints_f32(joints_rest, pose_vec):
    """World joint positions (22, 3) for one 76-vector, float32 chain with
    fixed three-term accumulation order."""
    g = np.asarray(joints_rest, dtype=DTYPE)
    rl = rodrigues_f32(np.asarray(pose_vec, dtype=DTYPE)[:66].reshape(22, 3))
    off = g.copy()
    off[1:] = g[1:] - g[PARENTS[1:]]
    rw = np.empty((22, 3, 3), DTYPE)
    tw = np.empty((22, 3), DTYPE)
    for j in range(22):
        p = PARENTS[j]
        if p < 0:
            rw[j] = rl[j]
            tw[j] = off[j]
            continue
        rp = rw[p]
        rw[j] = rp[:, 0:1] * rl[j][0:1, :] + rp[:, 1:2] * rl[j][1:2, :] + rp[:, 2:3] * rl[j][2:3, :]
        tw[j] = (rp[:, 0] * off[j, 0] + rp[:, 1] * off[j, 1] + rp[:, 2] * off[j, 2]) + tw[p]
    return tw


# ---------------------------------------------------------------------------
# synthetic scenes (priors.py:68-126) and rendering (priors.py:237-252)


@dataclass
class CameraIntrinsics:
    fx: float
    fy: float
    cx: float
    cy: float


@dataclass
class Scene:
    image_size: tuple
    camera: CameraIntrinsics
    pose: np.ndarray
    translation: np.ndarray
    seed: int
    keypoints2d: np.ndarray


def default_camera(image_size):
    w, h = image_size
    f = 1.17 * min(w, h)
    return CameraIntrinsics(fx=f, fy=f, cx=(w - 1) / 2.0, cy=(h - 1) / 2.0)


def pinhole(points, cam):
    p = np.asarray(points, dtype=DTYPE)
    z = p[..., 2]
    if np.any(z <= 0.0):
        raise UsageError("point depth must be positive for projection")
    u = p[..., 0] / z * np.float32(cam.fx) + np.float32(cam.cx)
    v = p[..., 1] / z * np.float32(cam.fy) + np.float32(cam.cy)
    return np.stack([u, v], axis=-1).astype(DTYPE)


def make_scene(template, pose, translation, camera, image_size, seed=0):
    pose = np.asarray(pose, dtype=DTYPE).reshape(PARAM_DIM)
    translation = np.asarray(translation, dtype=DTYPE).reshape(3)
    joints = fk_joints_f32(template.joints_rest, pose)
    return Scene(image_size=(int(image_size[0]), int(image_size[1])), camera=camera,
                 pose=pose, translation=translation, seed=int(seed),
                 keypoints2d=pinhole(joints + translation, camera))


def random_scene(rng, template, image_size=(256, 256), pose_sigma=0.2,
                 shape_sigma=0.45, margin=10.0):
    w, h = image_size
    cam = default_camera(image_size)
    for attempt in range(200):
        vec = np.zeros(PARAM_DIM, dtype=DTYPE)
        vec[:66] = rng.normal(0.0, pose_sigma, size=66)
        vec[66:] = rng.normal(0.0, shape_sigma, size=SHAPE_DIM)
        joints = fk_joints_f32(template.joints_rest, vec)
        c = joints.mean(axis=0)
        depth = rng.uniform(2.4, 3.2) + 0.2 * attempt
        tx = -c[0] + rng.uniform(-0.08, 0.08)
        ty = -c[1] + rng.uniform(-0.08, 0.08)
        trans = np.array([tx, ty, -c[2] + depth], dtype=DTYPE)
        pts = joints + trans
        if np.any(pts[:, 2] <= 0.1):
            continue
        kp = pinhole(pts, cam)
        lo, hi = kp.min(axis=0), kp.max(axis=0)
        if lo[0] >= margin and hi[0] <= w - 1 - margin and lo[1] >= margin \
                and hi[1] <= h - 1 - margin:
            seed = int(rng.integers(0, 2 ** 31 - 1))
            return make_scene(template, vec, trans, cam, image_size, seed)
    raise UsageError("could not place a scene inside the frame")


def render_scene(scene, template=None):
    """Gradient background plus one Gaussian blob per keypoint, float32 in
    [0, 1], (H, W, 3)."""
    w, h = scene.image_size
    kp = scene.keypoints2d
    rng = np.random.default_rng(scene.seed)
    tint = rng.uniform(0.4, 1.0, size=(kp.shape[0], 3)).astype(DTYPE)
    slope = rng.uniform(-1.0, 1.0, size=2)
    yy, xx = np.mgrid[0:h, 0:w].astype(DTYPE)
    ramp = (slope[0] * xx / w + slope[1] * yy / h).astype(DTYPE)
    img = (0.10 + 0.05 * ramp)[:, :, None] * np.ones(3, dtype=DTYPE)
    extent = max(float(np.ptp(kp[:, 0])), float(np.ptp(kp[:, 1])))
    sig = max(6.0, 0.085 * extent)
    k = np.float32(-0.5 / (sig * sig))
    for j in range(kp.shape[0]):
        r2 = (xx - kp[j, 0]) ** 2 + (yy - kp[j, 1]) ** 2
        img = img + np.exp(r2 * k)[:, :, None] * (0.5 * tint[j])
    return np.clip(img, 0.0, 1.0).astype(DTYPE)
