"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no projection, covariance,
SH evaluation, binning or compositing).  It only draws scenes and camera
descriptors from seeded numpy generators, in the memory layout both sides
consume (SoA float32 planes, block-major order).  Recipes follow SURVEY.md
§8(d) ("Synthetic workloads") and are restated in DESIGN.md §3:

* ``box_v1``   -- C1: 1k Gaussians in a box in front of an identity camera.
* ``aerial_v1`` -- C2..C5: a kilometre-scale ground-hugging Gaussian layer
  over smooth terrain with box-shaped structures, trained-like opacity mix,
  SH colour and unit-norm features, stored block-major (PAPER.md l.134,
  §3.1: scenes "divided into multiple cells").

Poses follow PAPER.md Alg. 1 l.10: the pose maps world points to
camera points (world->camera), OpenCV axes (x right, y down, z forward).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

SH_C0 = 0.28209479177387814  # degree-0 real SH constant (used only to map flat RGB to k0)


@dataclasses.dataclass
class Scene:
    """SoA scene planes (float32) -- the layout of include/gs.h ``gs_scene``."""

    pos: np.ndarray          # [3][n]
    quat: np.ndarray         # [4][n]  (w, x, y, z), not necessarily unit
    scale: np.ndarray        # [3][n]  linear (already activated)
    opacity: np.ndarray      # [n]     linear
    sh: np.ndarray           # [(L+1)^2 * 3][n], row k*3+c = coefficient k of channel c
    sh_degree: int
    feat: Optional[np.ndarray] = None   # [n][D] row-major, or None (D = 0)
    block_offsets: Optional[np.ndarray] = None  # int64 [n_blocks + 1], block-major order

    @property
    def n(self) -> int:
        return int(self.pos.shape[1])

    @property
    def feat_dim(self) -> int:
        return 0 if self.feat is None else int(self.feat.shape[1])

    def subset(self, idx: np.ndarray) -> "Scene":
        idx = np.asarray(idx)
        return Scene(
            pos=np.ascontiguousarray(self.pos[:, idx]),
            quat=np.ascontiguousarray(self.quat[:, idx]),
            scale=np.ascontiguousarray(self.scale[:, idx]),
            opacity=np.ascontiguousarray(self.opacity[idx]),
            sh=np.ascontiguousarray(self.sh[:, idx]),
            sh_degree=self.sh_degree,
            feat=None if self.feat is None else np.ascontiguousarray(self.feat[idx]),
            block_offsets=None,
        )


@dataclasses.dataclass
class View:
    """Pinhole camera: R (3x3 row-major, world->camera), t, K, image size."""

    R: np.ndarray   # float32 [3][3]
    t: np.ndarray   # float32 [3]
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    @property
    def n_pixels(self) -> int:
        return self.width * self.height

    def center(self) -> np.ndarray:
        return -(self.R.astype(np.float64).T @ self.t.astype(np.float64))


def _f32(x) -> float:
    return float(np.float32(x))


def make_view(R, t, fx, fy, cx, cy, width, height) -> View:
    return View(R=np.ascontiguousarray(np.asarray(R, np.float32).reshape(3, 3)),
                t=np.ascontiguousarray(np.asarray(t, np.float32).reshape(3)),
                fx=_f32(fx), fy=_f32(fy), cx=_f32(cx), cy=_f32(cy),
                width=int(width), height=int(height))


def look_from(center, forward, up_hint=(0.0, 0.0, 1.0)):
    """World->camera rotation whose z axis is ``forward`` and x axis is horizontal."""
    f = np.asarray(forward, np.float64)
    f = f / np.linalg.norm(f)
    up = np.asarray(up_hint, np.float64)
    x = np.cross(f, up)
    if np.linalg.norm(x) < 1e-9:          # looking straight down/up: pick east
        x = np.array([1.0, 0.0, 0.0])
    x = x / np.linalg.norm(x)
    y = np.cross(f, x)
    R = np.stack([x, y, f])               # rows = camera axes in world coordinates
    t = -R @ np.asarray(center, np.float64)
    return R, t


def nadir_pose(cx_w, cy_w, altitude, yaw=0.0, tilt=0.0, tilt_dir=0.0):
    """Camera at (cx_w, cy_w, altitude) looking down; x axis at ``yaw``."""
    cz = np.array([0.0, 0.0, -1.0])
    cxv = np.array([math.cos(yaw), math.sin(yaw), 0.0])
    cyv = np.cross(cz, cxv)
    R = np.stack([cxv, cyv, cz])
    if tilt != 0.0:
        a = np.array([math.cos(tilt_dir), math.sin(tilt_dir), 0.0])
        K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
        Rt = np.eye(3) + math.sin(tilt) * K + (1 - math.cos(tilt)) * (K @ K)
        R = R @ Rt.T                      # rotate the camera frame about a horizontal axis
    C = np.array([cx_w, cy_w, altitude], np.float64)
    return R, -R @ C


# ----------------------------------------------------------------------------
# rotations (generator-side only: they build input quaternions)
# ----------------------------------------------------------------------------

def _quat_mul(a, b):
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw])


def _quat_align_z(n):
    """Quaternion rotating e_z onto unit normals n [3][m]."""
    nz = np.clip(n[2], -1.0, 1.0)
    axis = np.stack([-n[1], n[0], np.zeros_like(nz)])     # e_z x n
    s = np.linalg.norm(axis, axis=0)
    ang = np.arccos(nz)
    safe = np.where(s > 1e-12, s, 1.0)
    axis = axis / safe
    half = 0.5 * ang
    q = np.stack([np.cos(half), np.sin(half) * axis[0], np.sin(half) * axis[1], np.sin(half) * axis[2]])
    q[:, s <= 1e-12] = np.array([[1.0], [0.0], [0.0], [0.0]])
    return q


def _quat_z(yaw):
    return np.stack([np.cos(0.5 * yaw), np.zeros_like(yaw), np.zeros_like(yaw), np.sin(0.5 * yaw)])


# ----------------------------------------------------------------------------
# box_v1 (C1)
# ----------------------------------------------------------------------------

def box_v1(n: int = 1000, seed: int = 1, feat_dim: int = 0, sh_degree: int = 0) -> Scene:
    """C1 scene: mu ~ U([-1,1]^2 x [3,7]); log-uniform scales in [0.02,0.2];
    q = normalize(N(0, I4)); o ~ U(0.02, 1); flat rgb ~ U(0,1)^3 as SH degree 0."""
    rng = np.random.default_rng(seed)
    pos = np.stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(3, 7, n)])
    scale = np.exp(rng.uniform(math.log(0.02), math.log(0.2), (3, n)))
    q = rng.standard_normal((4, n))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    opacity = rng.uniform(0.02, 1.0, n)
    rgb = rng.uniform(0.0, 1.0, (3, n))
    nk = (sh_degree + 1) ** 2
    sh = np.zeros((nk * 3, n))
    sh[0:3] = (rgb - 0.5) / SH_C0
    if nk > 1:
        sh[3:] = rng.normal(0.0, 0.05, (nk * 3 - 3, n))
    feat = None
    if feat_dim > 0:
        feat = rng.standard_normal((n, feat_dim))
    return Scene(pos=pos.astype(np.float32), quat=q.astype(np.float32), scale=scale.astype(np.float32),
                 opacity=opacity.astype(np.float32), sh=sh.astype(np.float32), sh_degree=sh_degree,
                 feat=None if feat is None else feat.astype(np.float32))


def box_view(width: int = 64, height: int = 64) -> View:
    """C1 camera: identity pose, 64x64, fx = fy = 64, cx = cy = 31.5."""
    return make_view(np.eye(3), np.zeros(3), 64.0, 64.0, (width - 1) / 2, (height - 1) / 2, width, height)


# ----------------------------------------------------------------------------
# aerial_v1 (C2..C5)
# ----------------------------------------------------------------------------

def terrain(x, y):
    """h(x, y) = 8 sin(2 pi x/400) cos(2 pi y/300) + 3 sin(2 pi (x+y)/90) metres."""
    return 8.0 * np.sin(2 * np.pi * x / 400.0) * np.cos(2 * np.pi * y / 300.0) + \
        3.0 * np.sin(2 * np.pi * (x + y) / 90.0)


def _terrain_normal(x, y):
    dhdx = 8.0 * (2 * np.pi / 400.0) * np.cos(2 * np.pi * x / 400.0) * np.cos(2 * np.pi * y / 300.0) + \
        3.0 * (2 * np.pi / 90.0) * np.cos(2 * np.pi * (x + y) / 90.0)
    dhdy = -8.0 * (2 * np.pi / 300.0) * np.sin(2 * np.pi * x / 400.0) * np.sin(2 * np.pi * y / 300.0) + \
        3.0 * (2 * np.pi / 90.0) * np.cos(2 * np.pi * (x + y) / 90.0)
    n = np.stack([-dhdx, -dhdy, np.ones_like(x)])
    return n / np.linalg.norm(n, axis=0, keepdims=True)


def _albedo(x, y):
    a = np.stack([0.45 + 0.15 * np.sin(x / 37.0) * np.cos(y / 53.0),
                  0.50 + 0.12 * np.sin((x + 2 * y) / 71.0),
                  0.40 + 0.10 * np.cos((x - y) / 29.0)])
    return a


def aerial_v1(n: int, lx: float, ly: float, sh_degree: int = 3, feat_dim: int = 0,
              blocks: Sequence[int] = (4, 2), seed: int = 2, chunk: int = 1 << 21,
              sub: Sequence[int] = (1, 1), morton: bool = True) -> Scene:
    """Aerial-like scene: 85% ground Gaussians on terrain h(x,y), 15% on box
    structures (roofs + walls).  Opacity mixture 60% U(0.7,1), 25% U(0.2,0.7),
    15% U(0.004,0.2).  SH DC from a smooth albedo field + N(0,0.05), higher
    orders N(0, 0.02^2).  Features normalize(N(0, I_D)).  Block-major order on
    a ``blocks[0] x blocks[1]`` grid of cells (the partition);
    each cell is stored as ``sub[0] x sub[1]`` row-major sub-blocks (stable
    within a sub-block), so every cell stays one contiguous range while
    ``block_offsets`` describe the sub-blocks -- the granularity of
    gs_project's per-(block, view) frustum cull.  ``morton``: inside a
    sub-block, Gaussians are stored in Z-order of (x, y) (a storage layout, as a
    scene loader would write it: neighbours in memory are neighbours on the
    ground, so a view's records and tile pairs are written coherently)."""
    rng = np.random.default_rng(seed)
    n_ground = int(round(0.85 * n))
    n_struct = n - n_ground
    rho = 0.8 * math.sqrt(lx * ly / n)

    # ---- ground layer ----
    gx = rng.uniform(-lx / 2, lx / 2, n_ground)
    gy = rng.uniform(-ly / 2, ly / 2, n_ground)
    gz = terrain(gx, gy) + 0.2 * np.abs(rng.standard_normal(n_ground))
    ga = rho * np.exp(0.5 * rng.standard_normal(n_ground))
    gb = rho * np.exp(0.5 * rng.standard_normal(n_ground))
    gc = 0.15 * np.minimum(ga, gb)
    gq = _quat_mul(_quat_align_z(_terrain_normal(gx, gy)), _quat_z(rng.uniform(0, 2 * np.pi, n_ground)))

    # ---- structures: boxes with 10-30 m footprint, 5-30 m height ----
    area_box = 20.0 * 20.0 + 4 * 20.0 * 17.5          # mean roof + wall area
    per_box = max(1, int(area_box / (rho * rho * 1.5)))
    n_boxes = max(1, n_struct // per_box)
    bx = rng.uniform(-lx / 2 + 15, lx / 2 - 15, n_boxes)
    by = rng.uniform(-ly / 2 + 15, ly / 2 - 15, n_boxes)
    bw = rng.uniform(10, 30, n_boxes)
    bd = rng.uniform(10, 30, n_boxes)
    bh = rng.uniform(5, 30, n_boxes)
    byaw = rng.uniform(0, 2 * np.pi, n_boxes)
    roof_area = bw * bd
    wall_area = 2 * (bw + bd) * bh
    w_box = (roof_area + wall_area)
    owner = rng.choice(n_boxes, size=n_struct, p=w_box / w_box.sum())
    on_roof = rng.uniform(0, 1, n_struct) < (roof_area / w_box)[owner]
    u1 = rng.uniform(-0.5, 0.5, n_struct)
    u2 = rng.uniform(-0.5, 0.5, n_struct)
    side = rng.integers(0, 4, n_struct)
    W, Dp, H, yaw = bw[owner], bd[owner], bh[owner], byaw[owner]
    base = terrain(bx[owner], by[owner])
    # local coordinates (lx_, ly_, lz_) and local normal
    lxl = np.where(on_roof, u1 * W, np.where(side % 2 == 0, u1 * W, np.where(side == 1, 0.5 * W, -0.5 * W)))
    lyl = np.where(on_roof, u2 * Dp, np.where(side % 2 == 1, u1 * Dp, np.where(side == 0, 0.5 * Dp, -0.5 * Dp)))
    lzl = np.where(on_roof, H, (u2 + 0.5) * H)
    nxl = np.where(on_roof, 0.0, np.where(side == 1, 1.0, np.where(side == 3, -1.0, 0.0)))
    nyl = np.where(on_roof, 0.0, np.where(side == 0, 1.0, np.where(side == 2, -1.0, 0.0)))
    nzl = np.where(on_roof, 1.0, 0.0)
    cyw, syw = np.cos(yaw), np.sin(yaw)
    sx = bx[owner] + cyw * lxl - syw * lyl
    sy = by[owner] + syw * lxl + cyw * lyl
    sz = base + lzl
    nrm = np.stack([cyw * nxl - syw * nyl, syw * nxl + cyw * nyl, nzl])
    sa = rho * np.exp(0.5 * rng.standard_normal(n_struct))
    sb = rho * np.exp(0.5 * rng.standard_normal(n_struct))
    sc = 0.15 * np.minimum(sa, sb)
    sq = _quat_mul(_quat_align_z(nrm), _quat_z(rng.uniform(0, 2 * np.pi, n_struct)))

    x = np.concatenate([gx, sx])
    y = np.concatenate([gy, sy])
    z = np.concatenate([gz, sz])
    scale = np.stack([np.concatenate([ga, sa]), np.concatenate([gb, sb]), np.concatenate([gc, sc])])
    quat = np.concatenate([gq, sq], axis=1)
    del gx, gy, gz, sx, sy, sz, gq, sq

    # ---- block-major order (cells, then sub-blocks inside a cell; stable within) ----
    nbx, nby = int(blocks[0]), int(blocks[1])
    sbx, sby = int(sub[0]), int(sub[1])
    ix = np.clip(((x + lx / 2) / lx * (nbx * sbx)).astype(np.int64), 0, nbx * sbx - 1)
    iy = np.clip(((y + ly / 2) / ly * (nby * sby)).astype(np.int64), 0, nby * sby - 1)
    cell = (iy // sby) * nbx + (ix // sbx)
    bid = cell * (sbx * sby) + (iy % sby) * sbx + (ix % sbx)
    if morton:
        # 16-bit quantisation of (x, y) over the scene, bits interleaved (Z-order)
        qx = np.clip(((x + lx / 2) / lx * 65535.0).astype(np.int64), 0, 65535)
        qy = np.clip(((y + ly / 2) / ly * 65535.0).astype(np.int64), 0, 65535)
        zc = np.zeros_like(qx)
        for b in range(16):
            zc |= ((qx >> b) & 1) << (2 * b)
            zc |= ((qy >> b) & 1) << (2 * b + 1)
        order = np.lexsort((zc, bid))
    else:
        order = np.argsort(bid, kind="stable")
    counts = np.bincount(bid, minlength=nbx * nby * sbx * sby)
    block_offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    x, y, z = x[order], y[order], z[order]
    scale = scale[:, order]
    quat = quat[:, order]

    # ---- opacity mixture ----
    m = rng.uniform(0, 1, n)
    opacity = np.where(m < 0.60, rng.uniform(0.7, 1.0, n),
                       np.where(m < 0.85, rng.uniform(0.2, 0.7, n), rng.uniform(0.004, 0.2, n)))

    # ---- SH ----
    nk = (sh_degree + 1) ** 2
    sh = np.empty((nk * 3, n), np.float32)
    alb = _albedo(x, y) + rng.normal(0.0, 0.05, (3, n))
    sh[0:3] = ((alb - 0.5) / SH_C0).astype(np.float32)
    for r0 in range(3, nk * 3):
        sh[r0] = rng.standard_normal(n, dtype=np.float32) * np.float32(0.02)

    # ---- features ----
    feat = None
    if feat_dim > 0:
        feat = np.empty((n, feat_dim), np.float32)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            f = rng.standard_normal((e - s, feat_dim), dtype=np.float32)
            f /= np.linalg.norm(f, axis=1, keepdims=True)
            feat[s:e] = f

    return Scene(pos=np.stack([x, y, z]).astype(np.float32), quat=quat.astype(np.float32),
                 scale=scale.astype(np.float32), opacity=opacity.astype(np.float32), sh=sh,
                 sh_degree=sh_degree, feat=feat, block_offsets=block_offsets)


# ----------------------------------------------------------------------------
# camera sets
# ----------------------------------------------------------------------------

def c2_view() -> View:
    """C2: nadir at the centre, altitude 150 m, yaw 0, 1024x768, f = 800."""
    R, t = nadir_pose(0.0, 0.0, 150.0)
    return make_view(R, t, 800.0, 800.0, 511.5, 383.5, 1024, 768)


def pyramid_views(base: View, levels: int = 5) -> List[View]:
    """C3 pyramid (reading Q21): level l has s = 2^(l - (levels-1));
    W_l = s W, f_l = s f, c_l = (c + 0.5) s - 0.5 (pixel-centre-consistent)."""
    out = []
    for lvl in range(levels):
        s = 2.0 ** (lvl - (levels - 1))
        out.append(make_view(base.R, base.t, base.fx * s, base.fy * s,
                             (base.cx + 0.5) * s - 0.5, (base.cy + 0.5) * s - 0.5,
                             int(round(base.width * s)), int(round(base.height * s))))
    return out


def c4_views(n_side: int = 16, extent: float = 1000.0, seed: int = 4, width: int = 1024,
             height: int = 768, f: float = 800.0) -> List[View]:
    """C4: n_side x n_side poses on a grid over the extent (+-10 m jitter),
    altitude 150 +- 20 m, yaw U(0, 2pi), tilt <= 10 deg."""
    rng = np.random.default_rng(seed)
    views = []
    step = extent / n_side
    for iy in range(n_side):
        for ix in range(n_side):
            cxw = -extent / 2 + (ix + 0.5) * step + rng.uniform(-10, 10)
            cyw = -extent / 2 + (iy + 0.5) * step + rng.uniform(-10, 10)
            alt = 150.0 + rng.uniform(-20, 20)
            R, t = nadir_pose(cxw, cyw, alt, yaw=rng.uniform(0, 2 * np.pi),
                              tilt=math.radians(rng.uniform(0, 10)), tilt_dir=rng.uniform(0, 2 * np.pi))
            views.append(make_view(R, t, f, f, (width - 1) / 2, (height - 1) / 2, width, height))
    return views


def c5_views(extent: float = 2000.0, seed: int = 5, n_pos: int = 8, n_head: int = 8,
             width: int = 1920, height: int = 1080, f: float = 1500.0) -> List[View]:
    """C5: 64 oblique views (pitch 45 deg, altitude 300 m at the full 2 km extent),
    8 headings x 8 positions.  The altitude scales with the extent (at least 60 m)
    so the reduced-size test scenes stay in view."""
    rng = np.random.default_rng(seed)
    alt = max(0.15 * extent, 60.0)
    views = []
    for ip in range(n_pos):
        ang = 2 * np.pi * ip / n_pos
        px = 0.3 * extent / 2 * math.cos(ang) + rng.uniform(-20, 20)
        py = 0.15 * extent / 2 * math.sin(ang) + rng.uniform(-20, 20)
        for ih in range(n_head):
            hd = 2 * np.pi * ih / n_head
            fwd = np.array([math.cos(hd) * math.sin(math.pi / 4), math.sin(hd) * math.sin(math.pi / 4),
                            -math.cos(math.pi / 4)])
            R, t = look_from([px, py, alt], fwd)
            views.append(make_view(R, t, f, f, (width - 1) / 2, (height - 1) / 2, width, height))
    return views


# ----------------------------------------------------------------------------
# named configurations (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------

CONFIGS = {
    "C1": "1k random Gaussians, SH 0, one 64x64 pinhole view",
    "C2": "200k Gaussians aerial patch, SH 3, single 1024x768 nadir view",
    "C3": "2M Gaussians, 5-level pyramid 64->1024 px at one pose, D=32",
    "C4": "5M Gaussians, 256 sampled poses, D=32",
    "C5": "20M Gaussians, 8 blocks, 64 oblique 1920x1080 views + backprojection",
}


def make_config(name: str, scale: float = 1.0):
    """Return (scene, views).  ``scale`` < 1 shrinks the Gaussian count and
    area together (same density, same cameras) for fast parity cases."""
    if name == "C1":
        return box_v1(1000, seed=1), [box_view()]
    if name == "C2":
        n = int(200_000 * scale)
        ext = 200.0 * math.sqrt(scale)
        return aerial_v1(n, ext, ext, sh_degree=3, feat_dim=0, blocks=(4, 4), seed=2), [c2_view()]
    if name == "C3":
        n = int(2_000_000 * scale)
        ext = 632.0 * math.sqrt(scale)
        return aerial_v1(n, ext, ext, sh_degree=3, feat_dim=32, blocks=(8, 8), seed=3), pyramid_views(c2_view())
    if name == "C4":
        n = int(5_000_000 * scale)
        ext = 1000.0 * math.sqrt(scale)
        return (aerial_v1(n, ext, ext, sh_degree=3, feat_dim=32, blocks=(32, 32), seed=4),
                c4_views(extent=ext))
    if name == "C5":
        n = int(20_000_000 * scale)
        ext = 2000.0 * math.sqrt(scale)
        # the 4 x 2 partition (8 cells of 500 x 1000 m), each stored as 8 x 16 sub-blocks
        # of 62.5 m (the block cull's granularity)
        return (aerial_v1(n, ext, ext, sh_degree=3, feat_dim=0, blocks=(4, 2), seed=5, sub=(8, 16)),
                c5_views(extent=ext))
    raise KeyError(name)
