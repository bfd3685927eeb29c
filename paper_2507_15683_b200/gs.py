"""Thin Python binding of libgs.so (include/gs.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module
only turns torch tensors (device memory owned by PyTorch) into the plain
pointers and structs of the C ABI and raises on a non-OK status.  There is no
CPU fallback: importing it without the built library raises.

The four calls keep the C names: ``gs_project``, ``gs_bin_sort``,
``gs_rasterize``, ``gs_backproject``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# GS_LIB overrides the library path (experiments with alternative builds)
LIB_PATH = os.environ.get("GS_LIB") or os.path.join(_PKG, "libgs.so")

GS_OK, GS_INVALID_ARG, GS_UNSUPPORTED, GS_WORKSPACE_TOO_SMALL, GS_CUDA_ERROR = range(5)
GS_STATUS_RECORD_OVERFLOW = 0x1
GS_STATUS_PAIR_OVERFLOW = 0x2
RECORD_BYTES = 64


class GSError(RuntimeError):
    pass


# ------------------------------------------------------------------ structs
class gs_view(ctypes.Structure):
    _fields_ = [("R", ctypes.c_float * 9), ("t", ctypes.c_float * 3), ("fx", ctypes.c_float),
                ("fy", ctypes.c_float), ("cx", ctypes.c_float), ("cy", ctypes.c_float),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32), ("pix_offset", ctypes.c_int64),
                ("tile_offset", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class gs_scene(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("sh_degree", ctypes.c_int32), ("feat_dim", ctypes.c_int32),
                ("pos", ctypes.c_void_p), ("quat", ctypes.c_void_p), ("scale", ctypes.c_void_p),
                ("opacity", ctypes.c_void_p), ("sh", ctypes.c_void_p), ("feat", ctypes.c_void_p),
                ("n_blocks", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("block_offsets", ctypes.c_void_p), ("block_bounds", ctypes.c_void_p), ("feat_h", ctypes.c_void_p)]


class gs_params(ctypes.Structure):
    _fields_ = [("z_near", ctypes.c_float), ("dilation", ctypes.c_float), ("clamp_margin", ctypes.c_float),
                ("alpha_min", ctypes.c_float), ("alpha_max", ctypes.c_float), ("t_min", ctypes.c_float)]


class gs_projected(ctypes.Structure):
    _fields_ = [("rec", ctypes.c_void_p), ("rec_capacity", ctypes.c_int64), ("n_rec", ctypes.c_void_p),
                ("diag", ctypes.c_void_p), ("status", ctypes.c_void_p), ("contrib", ctypes.c_void_p)]


class gs_bins(ctypes.Structure):
    _fields_ = [("ranges", ctypes.c_void_p), ("sorted_rec", ctypes.c_void_p), ("pair_capacity", ctypes.c_int64),
                ("n_pairs", ctypes.c_void_p), ("sorted_key", ctypes.c_void_p), ("sorted_gid", ctypes.c_void_p),
                ("tile_sched", ctypes.c_void_p), ("mode", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class gs_images(ctypes.Structure):
    _fields_ = [("rgb", ctypes.c_void_p), ("depth", ctypes.c_void_p), ("alpha", ctypes.c_void_p),
                ("feat", ctypes.c_void_p)]


EXPORTS = ["gs_abi_version", "gs_last_error", "gs_default_params", "gs_views_layout", "gs_scene_block_bounds",
           "gs_scene_features_f16", "gs_validate_scene", "gs_match", "gs_match_workspace_bytes",
           "gs_pnp", "gs_pnp_workspace_bytes", "gs_verify_consistency", "gs_feature_backward", "gs_radiance_backward",
           "gs_mean_backward", "gs_param_backward", "gs_adam",
           "gs_feature_l1_grad", "gs_feature_sgd", "gs_dssim_grad", "gs_dssim_workspace_bytes",
           "gs_project_workspace_bytes", "gs_project", "gs_bin_sort_workspace_bytes", "gs_bin_sort",
           "gs_rasterize", "gs_rasterize_backproject", "gs_backproject", "gs_visibility_score",
           "gs_visibility_workspace_bytes", "gs_probe_alpha", "gs_sanitize_scene", "gs_joint_backward", "gs_appearance_l1_grad", "gs_pack_images",
           "gs_pack_bytes"]

_lib = None


def lib():
    """Load libgs.so (fails loudly when missing -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise GSError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        L.gs_abi_version.restype = ctypes.c_int32
        L.gs_last_error.restype = ctypes.c_char_p
        L.gs_default_params.restype = gs_params
        L.gs_project_workspace_bytes.restype = ctypes.c_size_t
        L.gs_project_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.gs_bin_sort_workspace_bytes.restype = ctypes.c_size_t
        L.gs_bin_sort_workspace_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64]
        L.gs_pnp_workspace_bytes.restype = ctypes.c_size_t
        L.gs_pnp_workspace_bytes.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.gs_match_workspace_bytes.restype = ctypes.c_size_t
        L.gs_match_workspace_bytes.argtypes = [ctypes.c_int32] * 4
        L.gs_visibility_workspace_bytes.restype = ctypes.c_size_t
        L.gs_dssim_workspace_bytes.restype = ctypes.c_size_t
        L.gs_dssim_workspace_bytes.argtypes = [ctypes.c_int32] * 3
        for f in ("gs_views_layout", "gs_scene_block_bounds", "gs_project", "gs_bin_sort", "gs_rasterize",
                  "gs_rasterize_backproject", "gs_backproject", "gs_visibility_score"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != GS_OK:
        raise GSError(f"{what} failed with status {st}: {lib().gs_last_error().decode()}")


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "expected a contiguous CUDA tensor"
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def default_params() -> gs_params:
    return lib().gs_default_params()


# ------------------------------------------------------------------ device containers
class DeviceScene:
    """Scene planes resident in HBM (SoA float32, block-major when partitioned)."""

    def __init__(self, scene, device="cuda", compute_block_bounds: bool = True, use_f16_features: bool = True):
        dev = torch.device(device)
        t = lambda a, dt=torch.float32: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)
        self.n = scene.n
        self.sh_degree = scene.sh_degree
        self.feat_dim = scene.feat_dim
        self.pos, self.quat, self.scale = t(scene.pos), t(scene.quat), t(scene.scale)
        self.opacity, self.sh = t(scene.opacity), t(scene.sh)
        self.feat = t(scene.feat) if scene.feat is not None else None
        self.block_offsets = None
        self.block_bounds = None
        if scene.block_offsets is not None and len(scene.block_offsets) > 1:
            self.block_offsets = t(scene.block_offsets, torch.int64)
            self.block_bounds = torch.zeros((len(scene.block_offsets) - 1, 8), device=dev)
        # fp16 copy of the features (scene preparation, like the block bounds): the
        # rasterizer's tcgen05 feature path gathers these 2-byte rows
        self.feat_h = None
        if self.feat is not None and use_f16_features:
            self.feat_h = torch.empty(self.feat.shape, dtype=torch.float16, device=dev)
        self.struct = self._make_struct()
        if self.feat_h is not None:
            _check(lib().gs_scene_features_f16(ctypes.byref(self.struct), _ptr(self.feat_h), _stream(None)),
                   "gs_scene_features_f16")
        if self.block_bounds is not None and compute_block_bounds:
            _check(lib().gs_scene_block_bounds(ctypes.byref(self.struct), _ptr(self.block_bounds), _stream(None)),
                   "gs_scene_block_bounds")

    @property
    def n_blocks(self):
        return 0 if self.block_offsets is None else self.block_offsets.numel() - 1

    def _make_struct(self, use_blocks: bool = True) -> gs_scene:
        s = gs_scene()
        s.n, s.sh_degree, s.feat_dim = self.n, self.sh_degree, self.feat_dim
        s.pos, s.quat, s.scale = _ptr(self.pos), _ptr(self.quat), _ptr(self.scale)
        s.opacity, s.sh, s.feat = _ptr(self.opacity), _ptr(self.sh), _ptr(self.feat)
        s.feat_h = _ptr(getattr(self, "feat_h", None))
        if use_blocks and self.block_offsets is not None:
            s.n_blocks = self.n_blocks
            s.block_offsets, s.block_bounds = _ptr(self.block_offsets), _ptr(self.block_bounds)
        return s

    def without_blocks(self) -> gs_scene:
        return self._make_struct(use_blocks=False)

    def nbytes(self) -> int:
        ts = [self.pos, self.quat, self.scale, self.opacity, self.sh, self.feat, self.feat_h]
        return sum(x.numel() * x.element_size() for x in ts if x is not None)


class ViewBatch:
    """Host + device copies of a batch of gs_view descriptors (contiguous layout)."""

    def __init__(self, views: Sequence, device="cuda"):
        n = len(views)
        arr = (gs_view * n)()
        for i, v in enumerate(views):
            R = np.asarray(v.R, np.float32).reshape(9)
            t = np.asarray(v.t, np.float32).reshape(3)
            for k in range(9):
                arr[i].R[k] = float(R[k])
            for k in range(3):
                arr[i].t[k] = float(t[k])
            arr[i].fx, arr[i].fy, arr[i].cx, arr[i].cy = v.fx, v.fy, v.cx, v.cy
            arr[i].width, arr[i].height = v.width, v.height
        tp, tt = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().gs_views_layout(arr, ctypes.c_int32(n), ctypes.byref(tp), ctypes.byref(tt)), "gs_views_layout")
        self.host = arr
        self.n = n
        self.total_pixels = tp.value
        self.total_tiles = tt.value
        self.views = list(views)
        raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
        self.pinned = torch.from_numpy(raw).pin_memory() if torch.cuda.is_available() else torch.from_numpy(raw)
        self.dev = torch.empty(raw.size, dtype=torch.uint8, device=device)
        self.dev.copy_(self.pinned, non_blocking=True)

    def upload(self, stream=None):
        """Re-copy the descriptors (H2D, pinned) -- e2e path."""
        self.dev.copy_(self.pinned, non_blocking=True)

    @property
    def dev_ptr(self):
        return ctypes.c_void_p(self.dev.data_ptr())

    def pix_offset(self, i):
        return self.host[i].pix_offset

    def tile_offset(self, i):
        return self.host[i].tile_offset


class Projected:
    def __init__(self, n_views: int, rec_capacity: int, device="cuda", contrib: bool = False):
        self.rec_capacity = int(rec_capacity)
        self.rec = torch.empty(n_views * self.rec_capacity * (RECORD_BYTES // 4), dtype=torch.int32, device=device)
        self.n_rec = torch.zeros(n_views, dtype=torch.int32, device=device)
        self.diag = torch.zeros(4, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        self.contrib = torch.zeros(n_views * self.rec_capacity, dtype=torch.int64, device=device) if contrib else None
        s = gs_projected()
        s.rec, s.rec_capacity = _ptr(self.rec), self.rec_capacity
        s.n_rec, s.diag, s.status = _ptr(self.n_rec), _ptr(self.diag), _ptr(self.status)
        s.contrib = _ptr(self.contrib)
        self.struct = s

    def records(self):
        """Record view as a [n_views*cap, 16] int32 tensor (test inspection)."""
        return self.rec.view(-1, RECORD_BYTES // 4)


BINNING_MODES = {"square": 0, "tight": 1}   # GS_BIN_SQUARE, GS_BIN_TIGHT (N3, reading Q30)


class Bins:
    def __init__(self, total_tiles: int, pair_capacity: int, device="cuda", debug_keys: bool = False,
                 with_gid: bool = True, binning: str = "tight"):
        self.pair_capacity = int(pair_capacity)
        self.binning = binning
        self.ranges = torch.empty(total_tiles * 2, dtype=torch.int32, device=device)
        self.sorted_rec = torch.empty(self.pair_capacity, dtype=torch.int32, device=device)
        self.n_pairs = torch.zeros(1, dtype=torch.int64, device=device)
        self.sorted_key = torch.empty(self.pair_capacity, dtype=torch.int64, device=device) if debug_keys else None
        self.sorted_gid = torch.empty(self.pair_capacity, dtype=torch.int32, device=device) if with_gid else None
        self.tile_sched = torch.zeros(1, dtype=torch.int32, device=device)
        s = gs_bins()
        s.ranges, s.sorted_rec, s.pair_capacity = _ptr(self.ranges), _ptr(self.sorted_rec), self.pair_capacity
        s.n_pairs, s.sorted_key, s.sorted_gid = _ptr(self.n_pairs), _ptr(self.sorted_key), _ptr(self.sorted_gid)
        s.tile_sched = _ptr(self.tile_sched)
        s.mode = BINNING_MODES[binning]
        self.struct = s


class Images:
    def __init__(self, total_pixels: int, feat_dim: int, device="cuda", rgb=None, depth=None, alpha=None):
        """Output planes; rgb / depth / alpha may be caller tensors (e.g. views into a
        collective's send buffer, dist.ChunkedGather) of at least 3x / 1x / 1x
        total_pixels float32 elements."""
        def buf(t, n):
            if t is None:
                return torch.empty(n, dtype=torch.float32, device=device)
            assert t.dtype == torch.float32 and t.is_contiguous() and t.numel() >= n
            return t[:n]
        self.rgb = buf(rgb, 3 * total_pixels)
        self.depth = buf(depth, total_pixels)
        self.alpha = buf(alpha, total_pixels)
        self.feat = torch.empty(feat_dim * total_pixels, dtype=torch.float32, device=device) if feat_dim else None
        s = gs_images()
        s.rgb, s.depth, s.alpha, s.feat = _ptr(self.rgb), _ptr(self.depth), _ptr(self.alpha), _ptr(self.feat)
        self.struct = s
        self.feat_dim = feat_dim

    def set_feat(self, t: Optional[torch.Tensor], feat_dim: int):
        """Attach a caller tensor as the feature planes (e.g. an upstream gradient dL/dF)."""
        assert t is None or (t.dtype == torch.float32 and t.is_contiguous())
        self.feat, self.feat_dim = t, feat_dim
        self.struct.feat = _ptr(t)
        return self

    def view_planes(self, vb: ViewBatch, i: int):
        v = vb.views[i]
        H, W = v.height, v.width
        o = vb.pix_offset(i)
        hw = H * W
        out = dict(rgb=self.rgb[3 * o:3 * o + 3 * hw].view(3, H, W), depth=self.depth[o:o + hw].view(H, W),
                   alpha=self.alpha[o:o + hw].view(H, W))
        if self.feat is not None:
            D = self.feat_dim
            out["feat"] = self.feat[D * o:D * o + D * hw].view(D, H, W)
        return out


# ------------------------------------------------------------------ the four calls
def project_workspace_bytes(n_blocks: int, n_views: int) -> int:
    return int(lib().gs_project_workspace_bytes(n_blocks, n_views))


def bin_sort_workspace_bytes(pair_capacity: int, total_tiles: int) -> int:
    return int(lib().gs_bin_sort_workspace_bytes(pair_capacity, total_tiles))


def gs_project(scene: DeviceScene, views: ViewBatch, params: gs_params, proj: Projected, ws: torch.Tensor,
               stream=None, scene_struct: Optional[gs_scene] = None):
    s = scene.struct if scene_struct is None else scene_struct
    _check(lib().gs_project(ctypes.byref(s), views.host, views.dev_ptr, ctypes.c_int32(views.n), ctypes.byref(params),
                            ctypes.byref(proj.struct), _ptr(ws), ctypes.c_size_t(ws.numel() * ws.element_size()),
                            _stream(stream)), "gs_project")


def gs_bin_sort(proj: Projected, views: ViewBatch, bins: Bins, ws: torch.Tensor, stream=None):
    _check(lib().gs_bin_sort(ctypes.byref(proj.struct), views.host, views.dev_ptr, ctypes.c_int32(views.n),
                             ctypes.byref(bins.struct), _ptr(ws), ctypes.c_size_t(ws.numel() * ws.element_size()),
                             _stream(stream)), "gs_bin_sort")


def gs_rasterize(scene: DeviceScene, proj: Projected, bins: Bins, views: ViewBatch, params: gs_params,
                 images: Images, stream=None):
    _check(lib().gs_rasterize(ctypes.byref(scene.struct), ctypes.byref(proj.struct), ctypes.byref(bins.struct),
                              views.host, views.dev_ptr, ctypes.c_int32(views.n), ctypes.byref(params),
                              ctypes.byref(images.struct), _stream(stream)), "gs_rasterize")


def gs_rasterize_backproject(scene: DeviceScene, proj: Projected, bins: Bins, views: ViewBatch, params: gs_params,
                             images: Images, a_min: float, xyz: torch.Tensor, valid: torch.Tensor, stream=None):
    _check(lib().gs_rasterize_backproject(ctypes.byref(scene.struct), ctypes.byref(proj.struct),
                                          ctypes.byref(bins.struct), views.host, views.dev_ptr,
                                          ctypes.c_int32(views.n), ctypes.byref(params), ctypes.byref(images.struct),
                                          ctypes.c_float(a_min), _ptr(xyz), _ptr(valid), _stream(stream)),
           "gs_rasterize_backproject")


def gs_backproject(images: Images, views: ViewBatch, a_min: float, xyz: torch.Tensor, valid: torch.Tensor,
                   stream=None):
    _check(lib().gs_backproject(ctypes.byref(images.struct), views.host, views.dev_ptr, ctypes.c_int32(views.n),
                                ctypes.c_float(a_min), _ptr(xyz), _ptr(valid), _stream(stream)), "gs_backproject")


FIXED_ONE = float(1 << 32)   # 2^-32 fixed point of contributions and scores


def visibility_workspace_bytes(views: ViewBatch, feat_dim: int, stride: int) -> int:
    return int(lib().gs_visibility_workspace_bytes(views.host, ctypes.c_int32(views.n), ctypes.c_int32(feat_dim),
                                                   ctypes.c_int32(stride)))


def gs_visibility_score(proj: Projected, views: ViewBatch, eps: float, scene: "DeviceScene", visible: torch.Tensor,
                        n_visible: torch.Tensor, score_sum: torch.Tensor, count: torch.Tensor,
                        fmaps: Optional[torch.Tensor] = None, stride: int = 1, ws: Optional[torch.Tensor] = None,
                        stream=None):
    nbytes = 0 if ws is None else ws.numel() * ws.element_size()
    _check(lib().gs_visibility_score(ctypes.byref(proj.struct), views.host, views.dev_ptr, ctypes.c_int32(views.n),
                                     ctypes.c_float(eps), _ptr(scene.feat), ctypes.c_int32(scene.feat_dim),
                                     _ptr(fmaps), ctypes.c_int32(stride), _ptr(ws), ctypes.c_size_t(nbytes),
                                     _ptr(visible), _ptr(n_visible), _ptr(score_sum), _ptr(count), _stream(stream)),
           "gs_visibility_score")


GS_BAD_REASONS = {0: "none", 1: "position", 2: "quat", 3: "quat_norm", 4: "scale", 5: "opacity", 6: "sh", 7: "feature"}


def gs_validate_scene(scene: "DeviceScene", unit_quat: bool = False, stream=None):
    """Debug check of SPEC's Gaussian invariants: (first offending index or -1, reason name)."""
    dev = scene.pos.device
    first = torch.empty(1, dtype=torch.int64, device=dev)
    reason = torch.empty(1, dtype=torch.int32, device=dev)
    _check(lib().gs_validate_scene(ctypes.byref(scene.struct), ctypes.c_int32(1 if unit_quat else 0), _ptr(first),
                                   _ptr(reason), _stream(stream)), "gs_validate_scene")
    return int(first.item()), GS_BAD_REASONS[int(reason.item())]


# ---------------------------------------------------------------------- N2 matching
class gs_matches(ctypes.Structure):
    _fields_ = [("coarse", ctypes.c_void_p), ("coarse_prob", ctypes.c_void_p), ("peak", ctypes.c_void_p),
                ("prob", ctypes.c_void_p), ("ref", ctypes.c_void_p), ("xyz", ctypes.c_void_p),
                ("valid", ctypes.c_void_p)]


class Matches:
    """Caller-side output buffers of gs_match (dense per query cell / pixel)."""

    def __init__(self, n_pairs: int, H: int, W: int, with_points: bool = True, device="cuda"):
        nc = (H // 8) * (W // 8)
        n = H * W
        self.n_pairs, self.H, self.W = n_pairs, H, W
        self.coarse = torch.empty(n_pairs * nc, dtype=torch.int32, device=device)
        self.coarse_prob = torch.empty(n_pairs * nc, dtype=torch.float32, device=device)
        self.peak = torch.empty(n_pairs * n, dtype=torch.int32, device=device)
        self.prob = torch.empty(n_pairs * n, dtype=torch.float32, device=device)
        self.ref = torch.empty(n_pairs * 2 * n, dtype=torch.float32, device=device)
        self.xyz = torch.empty(n_pairs * 3 * n, dtype=torch.float32, device=device) if with_points else None
        self.valid = torch.empty(n_pairs * n, dtype=torch.uint8, device=device) if with_points else None
        s = gs_matches()
        s.coarse, s.coarse_prob, s.peak, s.prob = _ptr(self.coarse), _ptr(self.coarse_prob), _ptr(self.peak), \
            _ptr(self.prob)
        s.ref, s.xyz, s.valid = _ptr(self.ref), _ptr(self.xyz), _ptr(self.valid)
        self.struct = s


def match_workspace_bytes(n_pairs: int, D: int, H: int, W: int) -> int:
    return int(lib().gs_match_workspace_bytes(n_pairs, D, H, W))


def gs_match(query_feat: torch.Tensor, rend_feat: torch.Tensor, n_pairs: int, D: int, H: int, W: int,
             out: Matches, ws: torch.Tensor, tau: float = 0.1, p_min: float = 0.05,
             rend_xyz: Optional[torch.Tensor] = None, rend_valid: Optional[torch.Tensor] = None, stream=None):
    _check(lib().gs_match(_ptr(query_feat), _ptr(rend_feat), ctypes.c_int32(n_pairs), ctypes.c_int32(D),
                          ctypes.c_int32(H), ctypes.c_int32(W), ctypes.c_float(tau), ctypes.c_float(p_min),
                          _ptr(rend_xyz), _ptr(rend_valid), _ptr(ws), ctypes.c_size_t(ws.numel()),
                          ctypes.byref(out.struct), _stream(stream)), "gs_match")


# ---------------------------------------------------------------------- N2 pose stage
GS_VIEW_BYTES = ctypes.sizeof(gs_view)


class gs_pnp_stats(ctypes.Structure):
    _fields_ = [("n_corr", ctypes.c_int32), ("n_inliers", ctypes.c_int32), ("mean_err", ctypes.c_float),
                ("best_hypothesis", ctypes.c_int32)]


class ViewsAt:
    """A view batch whose device descriptors live at `dev` (e.g. one slot of a
    refinement trace); the host copy (sizes, offsets) is the template batch's."""

    def __init__(self, template: "ViewBatch", dev: torch.Tensor):
        assert dev.numel() == template.n * GS_VIEW_BYTES
        self.host, self.n, self.dev, self.views = template.host, template.n, dev, template.views
        self.total_pixels, self.total_tiles = template.total_pixels, template.total_tiles

    @property
    def dev_ptr(self):
        return ctypes.c_void_p(self.dev.data_ptr())


def pnp_workspace_bytes(n_problems: int, cap: int) -> int:
    return int(lib().gs_pnp_workspace_bytes(n_problems, cap))


def gs_pnp(valid: torch.Tensor, xyz: torch.Tensor, n_problems: int, H: int, W: int, views_in: torch.Tensor,
           views_out: torch.Tensor, stats: torch.Tensor, ws: torch.Tensor, cap: int, tau_px: float = 3.0,
           n_hyp: int = 128, seed: int = 0, stream=None):
    """views_in / views_out: device gs_view arrays (uint8 tensors of n * 88 bytes);
    stats: int32 tensor of 4 * n (gs_pnp_stats)."""
    _check(lib().gs_pnp(_ptr(valid), _ptr(xyz), ctypes.c_int32(n_problems), ctypes.c_int32(H), ctypes.c_int32(W),
                        _ptr(views_in), ctypes.c_float(tau_px), ctypes.c_int32(n_hyp), ctypes.c_uint32(seed),
                        ctypes.c_int32(cap), _ptr(ws), ctypes.c_size_t(ws.numel()), _ptr(views_out), _ptr(stats),
                        _stream(stream)), "gs_pnp")


def gs_verify_consistency(trace: torch.Tensor, n_iters: int, n_problems: int, angle: torch.Tensor,
                          dtrans: torch.Tensor, verdict: torch.Tensor, tau_deg: float = 20.0, stream=None):
    _check(lib().gs_verify_consistency(_ptr(trace), ctypes.c_int32(n_iters), ctypes.c_int32(n_problems),
                                       ctypes.c_float(tau_deg), _ptr(angle), _ptr(dtrans), _ptr(verdict),
                                       _stream(stream)), "gs_verify_consistency")


def views_pose_array(dev_views: torch.Tensor, n: int):
    """Host decode of a device gs_view array -> (R [n][3][3], t [n][3]) numpy."""
    import numpy as _np
    raw = dev_views.cpu().numpy().view(_np.uint8)
    arr = (gs_view * n).from_buffer_copy(raw.tobytes())
    R = _np.array([[arr[i].R[k] for k in range(9)] for i in range(n)], _np.float64).reshape(n, 3, 3)
    t = _np.array([[arr[i].t[k] for k in range(3)] for i in range(n)], _np.float64)
    return R, t


# ---------------------------------------------------------------------- N4 feature-field backward
def gs_feature_backward(scene: "DeviceScene", proj: "Projected", bins: "Bins", views, params: gs_params,
                        grad_image: torch.Tensor, grad_feat: torch.Tensor, stream=None):
    _check(lib().gs_feature_backward(ctypes.byref(scene.struct), ctypes.byref(proj.struct), ctypes.byref(bins.struct),
                                     views.host, views.dev_ptr, ctypes.c_int32(views.n), ctypes.byref(params),
                                     _ptr(grad_image), _ptr(grad_feat), _stream(stream)), "gs_feature_backward")


def gs_feature_l1_grad(rendered: torch.Tensor, target: torch.Tensor, scale: float, grad_image: torch.Tensor,
                       loss: torch.Tensor, stream=None):
    _check(lib().gs_feature_l1_grad(_ptr(rendered), _ptr(target), ctypes.c_int64(rendered.numel()),
                                    ctypes.c_float(scale), _ptr(grad_image), _ptr(loss), _stream(stream)),
           "gs_feature_l1_grad")


def gs_dssim_grad(rendered: torch.Tensor, target: torch.Tensor, n_planes: int, height: int, width: int,
                  scale: float, grad_image: torch.Tensor, loss: torch.Tensor, workspace: Optional[torch.Tensor] = None,
                  stream=None) -> torch.Tensor:
    """Eq. 3's D-SSIM (reading Q37): loss += scale sum(1 - S), grad_image += its gradient
    (include/gs.h).  Returns the workspace (pass it back to reuse it)."""
    assert rendered.dtype == target.dtype == grad_image.dtype == torch.float32 and loss.dtype == torch.float64
    nb = lib().gs_dssim_workspace_bytes(n_planes, height, width)
    if workspace is None or workspace.numel() * 4 < nb:
        workspace = torch.empty(max(nb // 4, 1), dtype=torch.float32, device=rendered.device)
    _check(lib().gs_dssim_grad(_ptr(rendered), _ptr(target), ctypes.c_int32(n_planes), ctypes.c_int32(height),
                               ctypes.c_int32(width), ctypes.c_float(scale), _ptr(grad_image), _ptr(workspace),
                               ctypes.c_size_t(workspace.numel() * 4), _ptr(loss), _stream(stream)), "gs_dssim_grad")
    return workspace


def gs_sanitize_scene(scene: "DeviceScene", opacity_min: float, scale_min: float, changed: torch.Tensor,
                      stream=None):
    """N4: clamp opacity to [opacity_min, 1], scales to >= scale_min, reset zero
    quaternions (in place); `changed` (int64 [1], device) counts the Gaussians changed."""
    _check(lib().gs_sanitize_scene(ctypes.byref(scene.struct), ctypes.c_float(opacity_min), ctypes.c_float(scale_min),
                                   _ptr(changed), _stream(stream)), "gs_sanitize_scene")


GS_PACK_COMPACT = 1
GS_PACK_DENSE11 = 2


def gs_pack_bytes(total_pixels: int, fmt: int = GS_PACK_COMPACT) -> int:
    lib().gs_pack_bytes.restype = ctypes.c_size_t
    return int(lib().gs_pack_bytes(ctypes.c_int64(total_pixels), ctypes.c_int32(fmt)))


def gs_pack_images(images: "Images", views: "ViewBatch", out: torch.Tensor, stream=None, fmt: int = GS_PACK_COMPACT):
    """Compact transports (reading Q39, include/gs.h): GS_PACK_COMPACT = fp16 RGB + fp16 A +
    fp32 depth, 12 B/px, per view at byte 12 * pix_offset; GS_PACK_DENSE11 = batch-planar
    fp16 RGB + unorm16 A + 24-bit depth, 11 B/px.  out: uint8 device tensor."""
    need = gs_pack_bytes(views.total_pixels, fmt)
    assert out.dtype == torch.uint8 and out.numel() >= need
    _check(lib().gs_pack_images(ctypes.byref(images.struct), views.host, views.dev_ptr, ctypes.c_int32(views.n),
                                ctypes.c_int32(fmt), _ptr(out), _stream(stream)), "gs_pack_images")


def unpack_dense11(buf, total_pixels: int):
    """Host-side decode of GS_PACK_DENSE11 (numpy uint8 array) -> (rgb [3, TP] f32,
    depth [TP] f32, alpha [TP] f32).  Argument marshalling for the consumer of the
    transport, no arithmetic of the method."""
    import numpy as np
    b = np.asarray(buf, dtype=np.uint8)[:11 * total_pixels]
    tp = total_pixels
    rgb = b[:6 * tp].view(np.float16).reshape(3, tp).astype(np.float32)
    alpha = b[6 * tp:8 * tp].view(np.uint16).astype(np.float32) / 65535.0
    d = b[8 * tp:11 * tp].reshape(tp, 3).astype(np.uint32)
    bits = (d[:, 0] | (d[:, 1] << 8) | (d[:, 2] << 16)) << 8
    return rgb, bits.astype(np.uint32).view(np.float32), alpha.astype(np.float32)


def gs_probe_alpha(opacity: torch.Tensor, power: torch.Tensor, out: torch.Tensor, stream=None):
    """Debug: out = o 2^p as gs_rasterize's walk evaluates it (reading Q20 / Q29)."""
    assert opacity.dtype == power.dtype == out.dtype == torch.float32
    n = opacity.numel()
    assert power.numel() == n and out.numel() == n
    _check(lib().gs_probe_alpha(_ptr(opacity), _ptr(power), ctypes.c_int64(n), _ptr(out), _stream(stream)),
           "gs_probe_alpha")


def gs_scene_block_bounds(scene: "DeviceScene", stream=None):
    """Recompute the scene's per-block culling bounds (after its means or scales changed)."""
    _check(lib().gs_scene_block_bounds(ctypes.byref(scene.struct), _ptr(scene.block_bounds), _stream(stream)),
           "gs_scene_block_bounds")


def gs_adam(param: torch.Tensor, grad: torch.Tensor, m: torch.Tensor, v: torch.Tensor, lr: float, step: int,
            beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-15, param_h: Optional[torch.Tensor] = None,
            stream=None):
    _check(lib().gs_adam(_ptr(param), _ptr(grad), _ptr(m), _ptr(v), ctypes.c_int64(param.numel()), ctypes.c_float(lr),
                         ctypes.c_float(beta1), ctypes.c_float(beta2), ctypes.c_float(eps), ctypes.c_int32(step),
                         _ptr(param_h), _stream(stream)), "gs_adam")


def gs_feature_sgd(feat: torch.Tensor, grad_feat: torch.Tensor, lr: float, feat_h: Optional[torch.Tensor] = None,
                   stream=None):
    _check(lib().gs_feature_sgd(_ptr(feat), _ptr(grad_feat), ctypes.c_int64(feat.numel()), ctypes.c_float(lr),
                                _ptr(feat_h), _stream(stream)), "gs_feature_sgd")


GRAD_FIELDS = ("u", "v", "ea", "eb", "ec", "opacity", "r", "g", "b", "z")


def gs_radiance_backward(proj: "Projected", bins: "Bins", views, params: gs_params, fwd: "Images",
                         grad_out: "Images", grad_rec: torch.Tensor, stream=None):
    """grad_rec: [n_views * rec_capacity * 10] f32 (GRAD_FIELDS per record slot), accumulated."""
    _check(lib().gs_radiance_backward(ctypes.byref(proj.struct), ctypes.byref(bins.struct), views.host, views.dev_ptr,
                                      ctypes.c_int32(views.n), ctypes.byref(params), ctypes.byref(fwd.struct),
                                      ctypes.byref(grad_out.struct), _ptr(grad_rec), _stream(stream)),
           "gs_radiance_backward")


def gs_appearance_l1_grad(rendered: torch.Tensor, target: torch.Tensor, n_planes: int, plane_pixels: int,
                          a: torch.Tensor, b: torch.Tensor, scale: float, grad_image: torch.Tensor,
                          grad_a: torch.Tensor, grad_b: torch.Tensor, loss: torch.Tensor, stream=None):
    """Eq. 3's L1 against I^a = a I^r + b per plane (reading Q38); see include/gs.h."""
    _check(lib().gs_appearance_l1_grad(_ptr(rendered), _ptr(target), ctypes.c_int32(n_planes),
                                       ctypes.c_int64(plane_pixels), _ptr(a), _ptr(b), ctypes.c_float(scale),
                                       _ptr(grad_image), _ptr(grad_a), _ptr(grad_b), _ptr(loss), _stream(stream)),
           "gs_appearance_l1_grad")


def gs_joint_backward(scene: "DeviceScene", proj: "Projected", bins: "Bins", views, params: gs_params,
                      fwd: "Images", grad_out: "Images", grad_rec: torch.Tensor, stream=None):
    """Eq. 1's joint record gradient: gs_radiance_backward + the feature term
    (grad_out.feat = dL/dF) through the blend weights; accumulated into grad_rec."""
    _check(lib().gs_joint_backward(ctypes.byref(scene.struct), ctypes.byref(proj.struct), ctypes.byref(bins.struct),
                                   views.host, views.dev_ptr, ctypes.c_int32(views.n), ctypes.byref(params),
                                   ctypes.byref(fwd.struct), ctypes.byref(grad_out.struct), _ptr(grad_rec),
                                   _stream(stream)), "gs_joint_backward")


def gs_mean_backward(scene: "DeviceScene", proj: "Projected", views, params: gs_params, grad_rec: torch.Tensor,
                     grad_pos: torch.Tensor, stream=None):
    """grad_pos: [3 * n] f32 (SoA like scene.pos), accumulated."""
    _check(lib().gs_mean_backward(ctypes.byref(scene.struct), ctypes.byref(proj.struct), views.host, views.dev_ptr,
                                  ctypes.c_int32(views.n), ctypes.byref(params), _ptr(grad_rec), _ptr(grad_pos),
                                  _stream(stream)), "gs_mean_backward")


def gs_param_backward(scene: "DeviceScene", proj: "Projected", views, params: gs_params, grad_rec: torch.Tensor,
                      grad_scale=None, grad_quat=None, grad_opacity=None, grad_sh=None, stream=None):
    """Accumulated SoA gradients like the scene planes: grad_scale [3 * n], grad_quat [4 * n],
    grad_opacity [n], grad_sh [(deg+1)^2 * 3 * n] (f32; each optional)."""
    _check(lib().gs_param_backward(ctypes.byref(scene.struct), ctypes.byref(proj.struct), views.host, views.dev_ptr,
                                   ctypes.c_int32(views.n), ctypes.byref(params), _ptr(grad_rec), _ptr(grad_scale),
                                   _ptr(grad_quat), _ptr(grad_opacity), _ptr(grad_sh), _stream(stream)),
           "gs_param_backward")
