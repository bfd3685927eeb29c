"""Batch harness around the four C-ABI calls (buffer management only).

``Renderer`` owns the caller-side buffers the C ABI asks for (records, pairs,
images, workspaces), sizes them once from the device counters (the only
host<->device sync), and then enqueues
gs_project -> gs_bin_sort -> gs_rasterize (+ fused gs_backproject) on a stream with
no host synchronisation.  No arithmetic of the method happens here.
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import gs as G


class Renderer:
    def __init__(self, scene: G.DeviceScene, views: Sequence, params: Optional[G.gs_params] = None,
                 a_min: float = 0.5, backproject: bool = True, rec_capacity: Optional[int] = None,
                 pair_capacity: Optional[int] = None, debug_keys: bool = False, use_blocks: bool = True,
                 contrib: bool = False, binning: str = "tight", device="cuda", out_planes=None,
                 alloc_images: bool = True):
        self.device = torch.device(device)
        self.scene = scene
        self.scene_struct = scene.struct if use_blocks else scene.without_blocks()
        self.vb = views if isinstance(views, G.ViewBatch) else G.ViewBatch(views, device=device)
        self.params = params if params is not None else G.default_params()
        self.a_min = a_min
        self.do_backproject = backproject
        self.debug_keys = debug_keys
        self.with_contrib = contrib
        self.binning = binning
        n_views = self.vb.n
        self.ws_proj = torch.empty(max(1, G.project_workspace_bytes(scene.n_blocks if use_blocks else 0, n_views)),
                                   dtype=torch.uint8, device=self.device)
        # out_planes = (rgb, depth, alpha) caller tensors, e.g. a gather send buffer
        rgb, dep, alp = out_planes if out_planes is not None else (None, None, None)
        # alloc_images=False: projection + binning only (e.g. a pair-count pre-pass)
        self.images = G.Images(self.vb.total_pixels, scene.feat_dim, device=self.device, rgb=rgb, depth=dep,
                               alpha=alp) if alloc_images else None
        backproject = backproject and alloc_images
        self.do_backproject = backproject
        self.xyz = torch.empty(3 * self.vb.total_pixels, dtype=torch.float32, device=self.device) if backproject else None
        self.valid = torch.empty(self.vb.total_pixels + 4, dtype=torch.uint8, device=self.device) if backproject else None
        self.proj = None
        self.bins = None
        self.ws_bin = None
        self._alloc(rec_capacity, pair_capacity)

    # ------------------------------------------------------------- buffers
    def _alloc(self, rec_capacity, pair_capacity):
        n_views = self.vb.n
        if rec_capacity is None:
            # first guess: visible Gaussians ~ pixels, bounded to ~4 GB of records;
            # render() grows it to the device-reported count on overflow
            max_px = max(v.width * v.height for v in self.vb.views)
            rec_capacity = min(max(self.scene.n, 1), max(4096, max_px // 2),
                               max(4096, (4 << 30) // (G.RECORD_BYTES * n_views)))
        if pair_capacity is None:
            # ~4 pairs per record, bounded to ~8 GB of pair buffers (28 B / pair)
            pair_capacity = min(max(1 << 16, 4 * rec_capacity * n_views), (8 << 30) // 28)
        pair_capacity = min(pair_capacity, (1 << 32) - 1)
        rec_capacity = min(rec_capacity, ((1 << 32) - 1) // n_views)
        if self.proj is None or self.proj.rec_capacity != rec_capacity:
            self.proj = None
            self.proj = G.Projected(n_views, rec_capacity, device=self.device, contrib=self.with_contrib)
        if self.bins is None or self.bins.pair_capacity != pair_capacity:
            self.bins = None
            self.ws_bin = None
            self.bins = G.Bins(self.vb.total_tiles, pair_capacity, device=self.device, debug_keys=self.debug_keys,
                               binning=self.binning)
            self.ws_bin = torch.empty(G.bin_sort_workspace_bytes(pair_capacity, self.vb.total_tiles),
                                      dtype=torch.uint8, device=self.device)

    # ------------------------------------------------------------- hot path
    def run(self, stream=None, views=None, zero_status: bool = True):
        """Enqueue the whole hot path for the batch (asynchronous).  `views` may
        replace the batch's device descriptors (same sizes), e.g. poses written
        on the device by gs_pnp."""
        vb = self.vb if views is None else views
        if zero_status:
            self.proj.status.zero_()
        G.gs_project(self.scene, vb, self.params, self.proj, self.ws_proj, stream, scene_struct=self.scene_struct)
        G.gs_bin_sort(self.proj, vb, self.bins, self.ws_bin, stream)
        if self.images is None:
            return
        if self.do_backproject:
            # O13 fused into the compositing epilogue (same values as gs_backproject)
            G.gs_rasterize_backproject(self.scene, self.proj, self.bins, vb, self.params, self.images, self.a_min,
                                       self.xyz, self.valid, stream)
        else:
            G.gs_rasterize(self.scene, self.proj, self.bins, vb, self.params, self.images, stream)

    def status(self) -> int:
        return int(self.proj.status.item())

    def view_pair_counts(self):
        """Per-view pair counts of the last run (from the tile ranges), e.g. the
        costs of dist.shard_views' LPT assignment."""
        from .dist import view_costs_from_ranges
        offs = [self.vb.tile_offset(i) for i in range(self.vb.n)]
        nts = [((v.width + 15) // 16) * ((v.height + 15) // 16) for v in self.vb.views]
        return view_costs_from_ranges(self.bins.ranges, offs, nts)

    def render(self, max_retries: int = 4):
        """Run, and on capacity overflow grow the buffers to the reported sizes and re-run."""
        for _ in range(max_retries):
            self.run()
            st = self.status()
            if st == 0:
                return self
            rec_cap = self.proj.rec_capacity
            pair_cap = self.bins.pair_capacity
            if st & G.GS_STATUS_RECORD_OVERFLOW:
                rec_cap = int(self.proj.n_rec.max().item() * 1.1) + 64
            else:
                pair_cap = int(self.bins.n_pairs.item() * 1.1) + 1024
            self._alloc(rec_cap, pair_cap)
        raise G.GSError(f"capacity overflow persisted after {max_retries} retries")

    def fit_capacities(self, slack: float = 1.05):
        """Shrink/grow the buffers to the counts of the last successful run."""
        rec = int(self.proj.n_rec.max().item() * slack) + 64
        pairs = int(self.bins.n_pairs.item() * slack) + 1024
        self._alloc(rec, pairs)
        return self

    # ------------------------------------------------------------- outputs
    def view_images(self, i: int):
        out = self.images.view_planes(self.vb, i)
        if self.do_backproject:
            v = self.vb.views[i]
            o = self.vb.pix_offset(i)
            hw = v.width * v.height
            out["xyz"] = self.xyz[3 * o:3 * o + 3 * hw].view(3, v.height, v.width)
            out["valid"] = self.valid[o:o + hw].view(v.height, v.width)
        return out

    def view_records(self, i: int) -> torch.Tensor:
        n = min(int(self.proj.n_rec[i].item()), self.proj.rec_capacity)
        base = i * self.proj.rec_capacity
        return self.proj.records()[base:base + n]

    def n_pairs(self) -> int:
        return int(self.bins.n_pairs.item())

    def bytes_allocated(self) -> int:
        ts = [self.proj.rec, self.bins.sorted_rec, self.ws_bin, self.images.rgb, self.images.depth,
              self.images.alpha, self.images.feat, self.xyz, self.valid]
        return sum(t.numel() * t.element_size() for t in ts if t is not None)


class SignificanceScorer:
    """N1: Alg. 1 visibility + Eq. 4-6 significance over batches of views.

    ``add(renderer, fmaps)`` runs gs_visibility_score on a rendered batch (the
    renderer must be built with ``contrib=True``); ``scores()`` returns
    S(g) = S(G)/M (Eq. 6) with -inf where M = 0."""

    def __init__(self, scene: G.DeviceScene, eps: float = 1e-6, stride: int = 1):
        self.scene = scene
        self.eps = eps
        self.stride = stride
        dev = scene.pos.device
        self.score_sum = torch.zeros(scene.n, dtype=torch.int64, device=dev)
        self.count = torch.zeros(scene.n, dtype=torch.int32, device=dev)

    def add(self, r: "Renderer", fmaps: Optional[torch.Tensor] = None, stream=None):
        n_views = r.vb.n
        dev = self.count.device
        if getattr(r, "visible", None) is None or r.visible.numel() != n_views * r.proj.rec_capacity:
            r.visible = torch.empty(n_views * r.proj.rec_capacity, dtype=torch.uint8, device=dev)
            r.n_visible = torch.zeros(n_views, dtype=torch.int32, device=dev)
        ws = None
        if fmaps is not None:
            nb = G.visibility_workspace_bytes(r.vb, self.scene.feat_dim, self.stride)
            if getattr(r, "vis_ws", None) is None or r.vis_ws.numel() < nb:
                r.vis_ws = torch.empty(max(nb, 16), dtype=torch.uint8, device=dev)
            ws = r.vis_ws
        G.gs_visibility_score(r.proj, r.vb, self.eps, self.scene, r.visible, r.n_visible, self.score_sum, self.count,
                              fmaps, self.stride, ws, stream)
        return r.visible, r.n_visible

    def scores(self) -> torch.Tensor:
        s = self.score_sum.double() / G.FIXED_ONE
        m = self.count > 0
        out = torch.full_like(s, float("-inf"))
        out[m] = s[m] / self.count[m].double()
        return out


class Refiner:
    """N2 dense refinement: n rounds of render -> gs_match ->
    gs_pnp at the current poses of a batch of queries, then Algorithm 2
    (gs_verify_consistency).  Every round stays on the device: gs_pnp writes
    the refined pose into the gs_view slot the next round's gs_project reads,
    so the loop is one stream of launches with no host synchronisation and can
    be captured as a CUDA graph (``capture()``).

    query_feat: [B][D][H][W] f32 query feature maps (the query images'
    features at the rendering resolution); init_views: the B initial poses
    (equal sizes, H and W multiples of 8)."""

    def __init__(self, scene: G.DeviceScene, init_views: Sequence, query_feat: torch.Tensor, n_iters: int = 3,
                 tau_px: float = 3.0, n_hyp: int = 128, seed: int = 0, cap: int = 16384, match_tau: float = 0.1,
                 p_min: float = 0.05, a_min: float = 0.5, slack: float = 1.6, consistency_deg: float = 20.0):
        self.B = len(init_views)
        v0 = init_views[0]
        self.H, self.W, self.D = v0.height, v0.width, scene.feat_dim
        assert all(v.width == self.W and v.height == self.H for v in init_views)
        self.n_iters, self.tau_px, self.n_hyp, self.seed, self.cap = n_iters, tau_px, n_hyp, seed, cap
        self.match_tau, self.p_min, self.consistency_deg = match_tau, p_min, consistency_deg
        self.query = query_feat
        dev = query_feat.device
        self.r = Renderer(scene, init_views, a_min=a_min, backproject=True, device=dev)
        self.r.render()
        # capacities with slack: later rounds render at other poses
        self.r._alloc(int(self.r.proj.n_rec.max().item() * slack) + 256, int(self.r.bins.n_pairs.item() * slack) + 4096)
        nb = self.B * G.GS_VIEW_BYTES
        self.trace = torch.empty((n_iters + 1) * nb, dtype=torch.uint8, device=dev)
        self.trace[:nb].copy_(self.r.vb.dev)
        self.matches = G.Matches(self.B, self.H, self.W, with_points=True, device=dev)
        self.mws = torch.empty(G.match_workspace_bytes(self.B, self.D, self.H, self.W), dtype=torch.uint8, device=dev)
        self.pws = torch.empty(G.pnp_workspace_bytes(self.B, cap), dtype=torch.uint8, device=dev)
        self.stats = torch.zeros((n_iters, self.B, 4), dtype=torch.int32, device=dev)
        self.angle = torch.zeros(self.B * max(1, n_iters - 1), dtype=torch.float32, device=dev)
        self.dtrans = torch.zeros_like(self.angle)
        self.verdict = torch.zeros(self.B, dtype=torch.int32, device=dev)
        self.graph = None

    def slot(self, i: int) -> torch.Tensor:
        nb = self.B * G.GS_VIEW_BYTES
        return self.trace[i * nb:(i + 1) * nb]

    def run(self, stream=None):
        """Enqueue the n rounds + Algorithm 2 (asynchronous)."""
        self.r.proj.status.zero_()
        for i in range(self.n_iters):
            self.r.run(stream, views=G.ViewsAt(self.r.vb, self.slot(i)), zero_status=False)
            G.gs_match(self.query, self.r.images.feat, self.B, self.D, self.H, self.W, self.matches, self.mws,
                       tau=self.match_tau, p_min=self.p_min, rend_xyz=self.r.xyz, rend_valid=self.r.valid,
                       stream=stream)
            G.gs_pnp(self.matches.valid, self.matches.xyz, self.B, self.H, self.W, self.slot(i), self.slot(i + 1),
                     self.stats[i], self.pws, self.cap, tau_px=self.tau_px, n_hyp=self.n_hyp, seed=self.seed,
                     stream=stream)
        nb = self.B * G.GS_VIEW_BYTES
        G.gs_verify_consistency(self.trace[nb:], self.n_iters, self.B, self.angle, self.dtrans, self.verdict,
                                tau_deg=self.consistency_deg, stream=stream)

    def capture(self):
        """Record run() into a CUDA graph (after one eager run initialised every kernel)."""
        self.run()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                self.run(torch.cuda.current_stream())
        torch.cuda.current_stream().wait_stream(s)
        self.graph = g
        return g

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def status(self) -> int:
        return int(self.r.proj.status.item())

    def poses(self, i: int):
        """(R [B][3][3], t [B][3]) of trace slot i (0 = initial)."""
        return G.views_pose_array(self.slot(i), self.B)


class FeatureDistiller:
    """N4: Eq. 2 feature distillation with the geometry frozen -- per step: render
    the batch, L1 loss gradient against target feature maps (gs_feature_l1_grad),
    gs_feature_backward into dL/df, one gradient step on the scene's features
    (gs_feature_sgd, which also refreshes the fp16 copy the tcgen05 path reads)."""

    def __init__(self, scene: G.DeviceScene, views: Sequence, target: torch.Tensor, lr: float = 1.0):
        assert scene.feat is not None
        self.scene, self.lr = scene, lr
        self.r = Renderer(scene, views, backproject=False)
        self.r.render()
        self.target = target
        n_img = self.r.images.feat.numel()
        self.scale = 1.0 / n_img                      # mean absolute error over all channels and pixels
        self.gimg = torch.empty_like(self.r.images.feat)
        self.gfeat = torch.zeros_like(scene.feat)
        self.loss = torch.zeros(1, dtype=torch.float64, device=scene.feat.device)

    def step(self, stream=None) -> torch.Tensor:
        """One iteration; returns the device loss (of the features before the update)."""
        ensure_rendered(self.r, stream)
        self.loss.zero_()
        G.gs_feature_l1_grad(self.r.images.feat, self.target, self.scale, self.gimg, self.loss, stream)
        self.gfeat.zero_()
        G.gs_feature_backward(self.scene, self.r.proj, self.r.bins, self.r.vb, self.r.params, self.gimg,
                              self.gfeat, stream)
        G.gs_feature_sgd(self.scene.feat, self.gfeat, self.lr, self.scene.feat_h, stream)
        return self.loss


def ensure_rendered(r: Renderer, stream=None):
    """Run the hot path for a training step and check the device status (one sync):
    on a capacity overflow (Gaussians moved / grew since the buffers were sized) grow
    the buffers and re-render, so no loss or gradient is ever computed from a stale
    or partial render."""
    r.run(stream)
    if r.status() != 0:
        r.render()
        r.fit_capacities(slack=1.5)
        r.render()


def equal_size_runs(views, max_views: Optional[int] = None) -> list:
    """Runs of consecutive equal-size views as (first, count, height, width): the
    planes of a run are contiguous in gs_images, so one gs_dssim_grad call covers it.
    max_views splits longer runs, bounding gs_dssim_grad's workspace (12 B per pixel
    per plane of one call) -- SceneTrainer uses 64 views per call."""
    runs = []
    for i, v in enumerate(views):
        if runs and runs[-1][2:] == [v.height, v.width] and (max_views is None or runs[-1][1] < max_views):
            runs[-1][1] += 1
        else:
            runs.append([i, 1, v.height, v.width])
    return [tuple(r) for r in runs]


class SceneTrainer:
    """N4: a joint training step of Eq. 1, L = alpha L_f + beta L_rgb, with
    Eq. 2's L1 feature term and Eq. 3's L_rgb = (1 - lam) L1(I, I^a) + lam
    L_D-SSIM(I, I^r) (reading Q37: lam = 0.2 as in [3DGS]; reading Q38:
    I^a = a I^r + b per view and channel, trained jointly; appearance=False uses I^r).
    Per step: render the batch; gs_appearance_l1_grad (or gs_feature_l1_grad) on the
    RGB planes, gs_dssim_grad adding the D-SSIM gradient per run of equal-size views;
    for a feature scene gs_feature_l1_grad on the feature planes; gs_joint_backward to
    the records (the RGB terms and the feature term through the blend weights: the
    geometry receives L_f's gradient too); gs_mean_backward + gs_param_backward to
    every Gaussian parameter; gs_feature_backward to the features; then one
    gs_feature_sgd or gs_adam step per parameter plane (and the appearance
    parameters), gs_sanitize_scene, and the block bounds refreshed.  No
    densification / pruning."""

    PLANES = ("pos", "scale", "quat", "opacity", "sh")

    def __init__(self, scene: G.DeviceScene, views: Sequence, target_rgb: torch.Tensor,
                 target_feat: Optional[torch.Tensor] = None, lr: Optional[dict] = None, alpha: float = 1.0,
                 beta: float = 1.0, optimizer: str = "sgd", lam: float = 0.2, appearance: bool = True):
        self.scene = scene
        self.r = Renderer(scene, views, backproject=False)
        self.r.render().fit_capacities(slack=1.5)
        self.target_rgb, self.target_feat = target_rgb, target_feat
        # steps for losses that are means over all pixels (and channels)
        assert optimizer in ("sgd", "adam")
        self.optimizer, self.t = optimizer, 0
        if optimizer == "sgd":
            self.lr = {"pos": 1.0, "scale": 1e-2, "quat": 1e-1, "opacity": 1.0, "sh": 10.0, "feat": 1000.0,
                       "app": 0.01}
        else:   # Adam steps are scale-free: per-parameter step sizes in parameter units
            self.lr = {"pos": 1e-3, "scale": 1e-3, "quat": 1e-3, "opacity": 1e-2, "sh": 1e-2, "feat": 1e-2,
                       "app": 1e-3}
        self.lr.update(lr or {})
        dev = scene.pos.device
        self.rgb_scale = beta * (1.0 - lam) / self.r.images.rgb.numel()
        self.dssim_scale = beta * lam / self.r.images.rgb.numel()
        self.dssim_runs = equal_size_runs(self.r.vb.views, max_views=64)
        self.dssim_ws = None
        self.gout = G.Images(self.r.vb.total_pixels, 0, device=dev)
        self.gout.depth.zero_()
        self.gout.alpha.zero_()
        # Eq. 3's appearance-varied rendering I^a = a I^r + b (reading Q38): 3 planes per view
        self.appearance = appearance
        self.rgb_runs = equal_size_runs(self.r.vb.views)
        n_planes = 3 * self.r.vb.n
        self.app_a = torch.ones(n_planes, device=dev)
        self.app_b = torch.zeros(n_planes, device=dev)
        self.grad_app = (torch.zeros(n_planes, device=dev), torch.zeros(n_planes, device=dev))
        self.grec = torch.zeros(self.r.vb.n * self.r.proj.rec_capacity * 10, dtype=torch.float32, device=dev)
        self.grads = {k: torch.zeros_like(getattr(scene, k)) for k in self.PLANES}
        self.feat_scale = 0.0
        if target_feat is not None:
            assert scene.feat is not None
            self.feat_scale = alpha / self.r.images.feat.numel()
            self.gimg = torch.empty_like(self.r.images.feat)
            self.gfeat = torch.zeros_like(scene.feat)
        self.loss = torch.zeros(1, dtype=torch.float64, device=dev)
        self.opacity_min = float(self.r.params.alpha_min)
        self.scale_min = 1e-6
        self.sanitized = torch.zeros(1, dtype=torch.int64, device=dev)   # Gaussians clamped so far
        self.state = {}
        if optimizer == "adam":
            keys = list(self.PLANES) + (["feat"] if target_feat is not None else [])
            self.state = {k: (torch.zeros_like(getattr(scene, k)), torch.zeros_like(getattr(scene, k))) for k in keys}
            self.state["app_a"] = (torch.zeros_like(self.app_a), torch.zeros_like(self.app_a))
            self.state["app_b"] = (torch.zeros_like(self.app_b), torch.zeros_like(self.app_b))

    def _update(self, key, param, grad, param_h, stream, lr_key=None):
        lr = self.lr[lr_key or key]
        if self.optimizer == "sgd":
            G.gs_feature_sgd(param, grad, lr, param_h, stream)
        else:
            m, v = self.state[key]
            G.gs_adam(param, grad, m, v, lr, self.t, param_h=param_h, stream=stream)

    def step(self, stream=None) -> torch.Tensor:
        """One iteration; returns the device loss of the parameters before the update."""
        sc, r = self.scene, self.r
        self.t += 1
        ensure_rendered(r, stream)
        self.loss.zero_()
        if self.appearance:
            ga, gb = self.grad_app
            ga.zero_()
            gb.zero_()
            for i0, cnt, h, w in self.rgb_runs:
                o, n = 3 * r.vb.pix_offset(i0), 3 * cnt * h * w
                G.gs_appearance_l1_grad(r.images.rgb[o:o + n], self.target_rgb[o:o + n], 3 * cnt, h * w,
                                        self.app_a[3 * i0:3 * (i0 + cnt)], self.app_b[3 * i0:3 * (i0 + cnt)],
                                        self.rgb_scale, self.gout.rgb[o:o + n], ga[3 * i0:3 * (i0 + cnt)],
                                        gb[3 * i0:3 * (i0 + cnt)], self.loss, stream)
        else:
            G.gs_feature_l1_grad(r.images.rgb, self.target_rgb, self.rgb_scale, self.gout.rgb, self.loss, stream)
        if self.dssim_scale != 0.0:
            for i0, cnt, h, w in self.dssim_runs:
                o = 3 * r.vb.pix_offset(i0)
                n = 3 * cnt * h * w
                self.dssim_ws = G.gs_dssim_grad(r.images.rgb[o:o + n], self.target_rgb[o:o + n], 3 * cnt, h, w,
                                                self.dssim_scale, self.gout.rgb[o:o + n], self.loss, self.dssim_ws,
                                                stream)
        if self.target_feat is not None:
            # Eq. 2's gradient w.r.t. the rendered feature map (the geometry receives it
            # through gs_joint_backward, the features through gs_feature_backward)
            G.gs_feature_l1_grad(r.images.feat, self.target_feat, self.feat_scale, self.gimg, self.loss, stream)
        self.gout.set_feat(self.gimg if self.target_feat is not None else None,
                           sc.feat_dim if self.target_feat is not None else 0)
        self.grec.zero_()
        G.gs_joint_backward(sc, r.proj, r.bins, r.vb, r.params, r.images, self.gout, self.grec, stream)
        for g in self.grads.values():
            g.zero_()
        G.gs_mean_backward(sc, r.proj, r.vb, r.params, self.grec, self.grads["pos"], stream)
        G.gs_param_backward(sc, r.proj, r.vb, r.params, self.grec, self.grads["scale"], self.grads["quat"],
                            self.grads["opacity"], self.grads["sh"], stream)
        if self.target_feat is not None:
            self.gfeat.zero_()
            G.gs_feature_backward(sc, r.proj, r.bins, r.vb, r.params, self.gimg, self.gfeat, stream)
            self._update("feat", sc.feat, self.gfeat, sc.feat_h, stream)
        for k in self.PLANES:
            self._update(k, getattr(sc, k), self.grads[k], None, stream)
        if self.appearance:
            self._update("app_a", self.app_a, self.grad_app[0], None, stream, lr_key="app")
            self._update("app_b", self.app_b, self.grad_app[1], None, stream, lr_key="app")
        # keep every Gaussian renderable: opacity in [alpha_min, 1], scale > 0
        G.gs_sanitize_scene(sc, self.opacity_min, self.scale_min, self.sanitized, stream)
        if sc.block_bounds is not None:
            G.gs_scene_block_bounds(sc, stream)   # the means moved
        return self.loss
