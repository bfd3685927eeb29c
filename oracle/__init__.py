"""CPU oracle of the Hi^2-GSLoc 3DGS forward rasterizer -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2507_15683_b200``) never imports it, and the two share no code: this
wrapper only marshals numpy arrays into ``liboracle.so`` (built from
``gs_oracle.cpp`` with ``g++ -O2 -ffp-contract=off -fno-fast-math``).

See ``gs_oracle.cpp`` for what each function computes and which PAPER.md /
SPEC.md passage it follows; DESIGN.md §5 lists the pin of every function.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Dict, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gs_oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile liboracle.so (single-threaded, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _View(ctypes.Structure):
    _fields_ = [("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3), ("fx", ctypes.c_float),
                ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class _Params(ctypes.Structure):
    _fields_ = [("z_near", ctypes.c_float), ("dilation", ctypes.c_float), ("clamp_margin", ctypes.c_float),
                ("alpha_min", ctypes.c_float), ("alpha_max", ctypes.c_float), ("t_min", ctypes.c_float)]


@dataclasses.dataclass
class Params:
    """Readings Q5, Q7, Q6, Q14, Q15."""
    z_near: float = 0.2
    dilation: float = 0.3
    clamp_margin: float = 0.15
    alpha_min: float = 1.0 / 255.0
    alpha_max: float = 0.99
    t_min: float = 1e-4

    def c(self) -> _Params:
        return _Params(self.z_near, self.dilation, self.clamp_margin, self.alpha_min, self.alpha_max, self.t_min)


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.oracle_project.restype = ctypes.c_int64
        _lib.oracle_count_pairs.restype = ctypes.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _view_c(view) -> _View:
    v = _View()
    R = np.asarray(view.R, np.float32).reshape(9)
    t = np.asarray(view.t, np.float32).reshape(3)
    for k in range(9):
        v.R[k] = float(R[k])
    for k in range(3):
        v.t[k] = float(t[k])
    v.fx, v.fy, v.cx, v.cy = view.fx, view.fy, view.cx, view.cy
    v.width, v.height = view.width, view.height
    return v


def _c32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def project(scene, view, params: Optional[Params] = None) -> Dict[str, np.ndarray]:
    """O1-O10 for one view: records of visible Gaussians in gid order."""
    params = params or Params()
    n = scene.n
    pos, quat, scale, op, sh = _c32(scene.pos), _c32(scene.quat), _c32(scene.scale), _c32(scene.opacity), _c32(scene.sh)
    gid = np.empty(n, np.int32)
    u = np.empty(n, np.float32)
    v = np.empty(n, np.float32)
    z = np.empty(n, np.float32)
    conic = np.empty((n, 3), np.float32)
    radius = np.empty(n, np.float32)
    rect = np.empty((n, 4), np.int32)
    rgb = np.empty((n, 3), np.float32)
    opac = np.empty(n, np.float32)
    cov = np.empty((n, 3), np.float32)
    ecut = np.empty(n, np.float32)
    diag = np.zeros(4, np.int64)
    vc, pc = _view_c(view), params.c()
    cnt = lib().oracle_project(ctypes.c_int64(n), _p(pos), _p(quat), _p(scale), _p(op), _p(sh),
                               ctypes.c_int32(scene.sh_degree), ctypes.byref(vc), ctypes.byref(pc),
                               _p(gid), _p(u), _p(v), _p(z), _p(conic), _p(radius), _p(rect), _p(rgb),
                               _p(opac), _p(cov), _p(ecut), _p(diag))
    return dict(gid=gid[:cnt].copy(), u=u[:cnt].copy(), v=v[:cnt].copy(), z=z[:cnt].copy(),
                conic=conic[:cnt].copy(), radius=radius[:cnt].copy(), rect=rect[:cnt].copy(),
                rgb=rgb[:cnt].copy(), opacity=opac[:cnt].copy(), cov=cov[:cnt].copy(), e_cut=ecut[:cnt].copy(),
                diag=dict(near=int(diag[0]), transparent=int(diag[1]), degenerate=int(diag[2]),
                          offscreen=int(diag[3])))


def tiles(view):
    return (view.width + 15) // 16, (view.height + 15) // 16


class _Tight(ctypes.Structure):
    _fields_ = [("u", ctypes.c_void_p), ("v", ctypes.c_void_p), ("conic", ctypes.c_void_p), ("ecut", ctypes.c_void_p)]


def bin_keys(rec, view, binning: str = "square") -> Dict[str, np.ndarray]:
    """O11: sorted (tile, depth_bits, gid) keys, their record index, ranges [T][2].
    binning "square": every tile of the 3-sigma rectangle (O8); "tight" (N3,
    reading Q30): only the rectangle's tiles the alpha >= alpha_min ellipse reaches."""
    tx, ty = tiles(view)
    cnt = len(rec["gid"])
    rect = np.ascontiguousarray(rec["rect"], np.int32)
    keep = []
    tight = None
    if binning == "tight":
        arrs = [_c32(rec["u"]), _c32(rec["v"]), _c32(rec["conic"]), _c32(rec["e_cut"])]
        keep = arrs
        tight = ctypes.byref(_Tight(*[a.ctypes.data for a in arrs]))
    elif binning != "square":
        raise ValueError(binning)
    P = int(lib().oracle_count_pairs(ctypes.c_int64(cnt), _p(rect), tight))
    kt = np.empty(P, np.uint32)
    kd = np.empty(P, np.uint32)
    kg = np.empty(P, np.uint32)
    kr = np.empty(P, np.uint32)
    ranges = np.empty((tx * ty, 2), np.uint32)
    lib().oracle_bin(ctypes.c_int64(cnt), _p(np.ascontiguousarray(rec["gid"])), _p(_c32(rec["z"])), _p(rect), tight,
                     ctypes.c_int32(tx), ctypes.c_int32(ty), _p(kt), _p(kd), _p(kg), _p(kr), _p(ranges))
    del keep
    return dict(tile=kt, depth=kd, gid=kg, rec=kr, ranges=ranges)


def _alloc_images(view, D):
    H, W = view.height, view.width
    return (np.zeros((3, H, W), np.float32), np.zeros((H, W), np.float32), np.zeros((H, W), np.float32),
            np.zeros((max(D, 0), H, W), np.float32), np.zeros((H, W), np.uint8))


def _feat(scene_or_feat, D):
    if D == 0:
        return np.zeros(1, np.float32)
    return _c32(scene_or_feat)


def composite(view, rec, keys, feat=None, params: Optional[Params] = None) -> Dict[str, np.ndarray]:
    """O12 + O14 over the binned lists (+ N1 per-record contribution sums, fp64)."""
    params = params or Params()
    D = 0 if feat is None else int(feat.shape[1])
    rgb, depth, alpha, F, flags = _alloc_images(view, D)
    a_err = np.zeros_like(alpha)
    counters = np.zeros(2, np.int64)
    contrib = np.zeros(max(1, len(rec["gid"])), np.float64)
    vc, pc = _view_c(view), params.c()
    lib().oracle_composite(ctypes.byref(vc), ctypes.byref(pc), _p(_c32(rec["u"])), _p(_c32(rec["v"])),
                           _p(_c32(rec["conic"])), _p(_c32(rec["opacity"])), _p(_c32(rec["rgb"])),
                           _p(_c32(rec["z"])), _p(np.ascontiguousarray(rec["gid"], np.int32)), _p(_feat(feat, D)),
                           ctypes.c_int32(D), _p(keys["rec"]), _p(keys["ranges"]), _p(rgb), _p(depth), _p(alpha),
                           _p(F), _p(flags), _p(counters), _p(contrib), _p(a_err))
    return dict(rgb=rgb, depth=depth, alpha=alpha, feat=F, flags=flags, evals=int(counters[0]),
                blends=int(counters[1]), contrib=contrib[:len(rec["gid"])], a_err=a_err)


def feature_grad(view, rec, keys, feat, gF, n_gauss: int, params: Optional[Params] = None,
                 fgrad: Optional[np.ndarray] = None) -> np.ndarray:
    """N4: dL/df [n_gauss][D] (fp64, added to `fgrad`) for a loss whose gradient
    w.r.t. this view's rendered feature map is gF [D][H][W]: sum_px w_g(px) gF(px)
    (F = sum_k w_k f_k with the geometry, hence the weights, frozen)."""
    params = params or Params()
    D = int(feat.shape[1])
    fgrad = np.zeros((n_gauss, D), np.float64) if fgrad is None else fgrad
    vc, pc = _view_c(view), params.c()
    lib().oracle_feature_grad(ctypes.byref(vc), ctypes.byref(pc), _p(_c32(rec["u"])), _p(_c32(rec["v"])),
                              _p(_c32(rec["conic"])), _p(_c32(rec["opacity"])), _p(_c32(rec["rgb"])),
                              _p(_c32(rec["z"])), _p(np.ascontiguousarray(rec["gid"], np.int32)), _p(_c32(feat)),
                              ctypes.c_int32(D), _p(keys["rec"]), _p(keys["ranges"]), _p(_c32(gF)), _p(fgrad))
    return fgrad


GRAD_FIELDS = ("u", "v", "ea", "eb", "ec", "opacity", "r", "g", "b", "z")


def radiance_backward(view, rec, keys, gC, gD, gA, params: Optional[Params] = None, feat=None, gF=None):
    """N4: per-record gradient [cnt][10] (GRAD_FIELDS) of L = sum gC.C + gD Dz + gA A
    (+ sum gF.F with gF [D][H][W] and the scene features [n][D]: Eq. 2's feature term
    through the blend weights), and L itself (fp64).  gC [3][H][W], gD / gA [H][W]."""
    params = params or Params()
    cnt = len(rec["gid"])
    grec = np.zeros((max(1, cnt), 10), np.float64)
    vc, pc = _view_c(view), params.c()
    lib().oracle_radiance_backward.restype = ctypes.c_double
    loss = lib().oracle_radiance_backward(
        ctypes.byref(vc), ctypes.byref(pc), _p(_c32(rec["u"])), _p(_c32(rec["v"])), _p(_c32(rec["conic"])),
        _p(_c32(rec["opacity"])), _p(_c32(rec["rgb"])), _p(_c32(rec["z"])),
        _p(np.ascontiguousarray(rec["gid"], np.int32)), _p(keys["rec"]), _p(keys["ranges"]), _p(_c32(gC)),
        _p(_c32(gD)), _p(_c32(gA)), _p(grec), None if gF is None else _p(_c32(feat)),
        ctypes.c_int32(0 if gF is None else int(feat.shape[1])), None if gF is None else _p(_c32(gF)))
    return grec[:cnt], float(loss)


def brute_force(view, rec, feat=None, params: Optional[Params] = None) -> Dict[str, np.ndarray]:
    """Per-pixel brute force over all records (plain definition)."""
    params = params or Params()
    D = 0 if feat is None else int(feat.shape[1])
    rgb, depth, alpha, F, flags = _alloc_images(view, D)
    vc, pc = _view_c(view), params.c()
    cnt = len(rec["gid"])
    contrib = np.zeros(max(1, cnt), np.float64)
    a_err = np.zeros_like(alpha)
    lib().oracle_brute_force(ctypes.byref(vc), ctypes.byref(pc), ctypes.c_int64(cnt), _p(_c32(rec["u"])),
                             _p(_c32(rec["v"])), _p(_c32(rec["conic"])), _p(_c32(rec["opacity"])),
                             _p(_c32(rec["rgb"])), _p(_c32(rec["z"])),
                             _p(np.ascontiguousarray(rec["gid"], np.int32)),
                             _p(np.ascontiguousarray(rec["rect"], np.int32)), _p(_feat(feat, D)), ctypes.c_int32(D),
                             _p(rgb), _p(depth), _p(alpha), _p(F), _p(flags), _p(contrib), _p(a_err))
    return dict(rgb=rgb, depth=depth, alpha=alpha, feat=F, flags=flags, contrib=contrib[:cnt], a_err=a_err)


def backproject(view, depth, alpha, a_min: float = 0.5, flags=None, a_err=None):
    """O13: rendered depth -> world points; returns xyz [3][H][W], valid [H][W], flags.
    a_err [H][W] (from composite): O14 (c) bound on the kernel's deviation of A; pixels
    with |A - a_min| <= a_err get flag bit 4.  None: the kernel back-projects the same A."""
    H, W = view.height, view.width
    xyz = np.zeros((3, H, W), np.float32)
    valid = np.zeros((H, W), np.uint8)
    fl = np.zeros((H, W), np.uint8) if flags is None else np.ascontiguousarray(flags, np.uint8).copy()
    vc = _view_c(view)
    lib().oracle_backproject(ctypes.byref(vc), _p(_c32(depth)), _p(_c32(alpha)), ctypes.c_float(a_min),
                             _p(xyz), _p(valid), _p(fl), None if a_err is None else _p(_c32(a_err)))
    return xyz, valid, fl


def render(scene, view, params: Optional[Params] = None, a_min: Optional[float] = None, binning: str = "square"):
    """Full oracle pipeline for one view: project -> bin -> composite (-> backproject)."""
    rec = project(scene, view, params)
    keys = bin_keys(rec, view, binning)
    img = composite(view, rec, keys, scene.feat, params)
    out = dict(rec=rec, keys=keys, **img)
    if a_min is not None:
        xyz, valid, fl = backproject(view, img["depth"], img["alpha"], a_min, img["flags"], img["a_err"])
        out.update(xyz=xyz, valid=valid, flags=fl)
    return out


def visibility_score(view, rec, contrib, n_gauss: int, eps: float = 1e-6, feat=None, fmap=None, stride: int = 1,
                     score_sum=None, count=None):
    """N1 for one view: Alg. 1 visibility (M = M^i and M^r) of every record and
    Eq. 4-5 accumulation into score_sum / count (arrays over all Gaussians,
    updated in place and returned).  fmap: [D][ceil(H/s)][ceil(W/s)] or None."""
    cnt = len(rec["gid"])
    D = 0 if feat is None else int(feat.shape[1])
    visible = np.zeros(max(1, cnt), np.uint8)
    score_sum = np.zeros(n_gauss, np.float64) if score_sum is None else score_sum
    count = np.zeros(n_gauss, np.int64) if count is None else count
    vc = _view_c(view)
    lib().oracle_visibility_score(ctypes.byref(vc), ctypes.c_int64(cnt), _p(_c32(rec["u"])), _p(_c32(rec["v"])),
                                  _p(np.ascontiguousarray(rec["gid"], np.int32)),
                                  _p(np.ascontiguousarray(contrib, np.float64)), ctypes.c_double(eps),
                                  _p(_feat(feat, D)), ctypes.c_int32(D),
                                  None if fmap is None else _p(_c32(fmap)), ctypes.c_int32(stride),
                                  _p(visible), _p(score_sum), _p(count))
    return visible[:cnt], score_sum, count


def final_scores(score_sum, count):
    """Eq. 6: S(g_j) = S(G_j) / M; -inf where M = 0."""
    out = np.full(score_sum.shape, -np.inf)
    m = count > 0
    out[m] = score_sum[m] / count[m]
    return out


def sh_color(deg: int, coeff, direction) -> np.ndarray:
    """O10 for one direction (fp64): coeff [(deg+1)^2][3]."""
    c = np.ascontiguousarray(coeff, np.float64).reshape(-1)
    d = np.ascontiguousarray(direction, np.float64).reshape(3)
    out = np.zeros(3, np.float64)
    lib().oracle_sh_color(ctypes.c_int32(deg), _p(c), _p(d), _p(out))
    return out
