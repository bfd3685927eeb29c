#!/usr/bin/env python
"""Benchmark of the B200 3DGS forward-rasterizer hot path (Hi^2-GSLoc).

One step = the whole hot path (gs_project -> gs_bin_sort -> gs_rasterize ->
gs_backproject) over one batch of views.  Default workload:
BASELINE.json configs[3] "C4" -- 5M-Gaussian aerial scene (SH 3, D = 32
features), 256 sampled 1024x768 poses, on one GPU.  Synthetic seeded data
(synth/), no trained weights.

  python bench.py [--gpus N --steps K --warmup W] [--config C4] [--scale 1.0]
  python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N
  python bench.py --impl reference      # the CPU oracle (the reference arm)

Rank 0 prints ONE JSON line.  See DESIGN.md §6 for the metric definitions.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "Mpixels/s and ms/view (RGB+depth)"
UNIT = "Mpixels/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--scale", type=float, default=1.0, help="Gaussian-count scale (1.0 = BASELINE size)")
    ap.add_argument("--views", type=int, default=0, help="limit views per rank (0 = config's batch)")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"],
                    help="N>1: strong = the config's pose batch sharded over the ranks (default, SURVEY §8(e)); "
                         "weak = every rank renders its own full batch")
    ap.add_argument("--no-gather", action="store_true",
                    help="N>1: skip the NCCL gather of RGB+depth+opacity (reported as render_only anyway)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="views per render/gather chunk of the sharded step (0 = a quarter of the largest shard)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the sharded chunked-gather step at N=1 too (exercises the N>1 code path)")
    ap.add_argument("--gather-transport", default="dense11", choices=["dense11", "f32"],
                    help="payload of the N > 1 gather: dense11 = GS_PACK_DENSE11 bytes (11 B/px, packed after "
                         "each chunk's render; reading Q39), f32 = the fp32 planes rendered straight into the "
                         "send buffer (20 B/px, lossless)")
    ap.add_argument("--force-gather", action="store_true",
                    help="sharded step with the per-chunk NCCL all_gather even at N = 1 (a one-rank NCCL group: "
                         "exercises the collective, comm stream and events of the N > 1 path on one GPU)")
    ap.add_argument("--feature-path", default="tcgen05", choices=["tcgen05", "mma_sync"],
                    help="feature contraction: tcgen05 (fp16 rows, TMEM) or mma.sync (fp32 rows)")
    ap.add_argument("--binning", default="tight", choices=["tight", "square"],
                    help="tile binning: tight alpha-ellipse tiles (N3, Q30) or the 3-sigma square (O8); same images")
    ap.add_argument("--separate-backproject", action="store_true",
                    help="time gs_rasterize + gs_backproject as two launches (default: the fused "
                         "gs_rasterize_backproject)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="also time the step replayed as one CUDA graph (default for batches of <= 8 views)")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="view chunks of the overlapped e2e measurement")
    ap.add_argument("--e2e-transport", default="dense11", choices=["dense11", "compact", "f32"],
                    help="D2H payload of the e2e leg: dense11 = fp16 RGB + unorm16 A + 24-bit depth (11 B/px), "
                         "compact = fp16 RGB + fp16 A + fp32 depth (12 B/px), f32 = the fp32 planes (20 B/px); "
                         "the line reports the other two as well")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0, help="(ncu) run only this many untimed steps")
    ap.add_argument("--n2", action="store_true",
                    help="also time N2 gs_match on (view i, view i+1) feature-map pairs of the rendered batch")
    ap.add_argument("--n2-pairs", type=int, default=64)
    ap.add_argument("--refine", type=int, default=0, metavar="B",
                    help="also time N2's n = 3 refinement loop (render -> gs_match -> gs_pnp, CUDA graph) for B "
                         "queries: query features rendered at B of the batch's poses, starts 1 deg / ~1.4 m off")
    ap.add_argument("--n4", action="store_true",
                    help="also time N4's feature backward (gs_feature_backward) over the batch")
    ap.add_argument("--n1", action="store_true",
                    help="also time N1 (per-Gaussian contributions + Alg. 1 visibility + Eq. 4-6 scoring "
                         "against stride-8 synthetic target maps) inside the step")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region: NVML polled every
    ~2 ms from a thread (short single-view regions last only milliseconds), falling
    back to `nvidia-smi -lms 100`."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown"}

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self.nvml = None
        self.samples = []
        self.max_mhz = None
        self.reasons = set()
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            dev = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            idx = int(dev.split(",")[self.gpu]) if dev and dev.split(",")[0].isdigit() else self.gpu
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.nvml = (pynvml, h)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _poll(self):
        pynvml, h = self.nvml
        while not self.stop.is_set():
            try:
                self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.nvml is not None and self.samples:
            return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi"}


# --------------------------------------------------------------------------- helpers
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def ncu_traffic(config_key: str):
    """The committed ncu record of one gs_rasterize launch in this configuration
    (profiles/ncu_traffic.json: DRAM bytes, issue activity, thread-instructions per
    pixel), or {}."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        d = json.load(f)
    return d.get(config_key) or {}


def workload(cfg: str, scale: float, rank: int, world: int, scaling: str, views_limit: int):
    import synth
    scene, views = synth.make_config(cfg, scale=scale)
    if cfg == "C4" and scaling == "weak" and world > 1 and rank > 0:
        # weak scaling: every rank renders its own full 256-pose batch (rank-seeded poses)
        ext = 1000.0 * math.sqrt(scale)
        views = synth.c4_views(extent=ext, seed=4 + 1000 * rank)
    return scene, views


def algorithmic_raster_bytes(n_pairs: int, n_visible: int, total_pixels: int, D: int, feat_bytes: int = 4,
                             fused_backproject: bool = False) -> int:
    """P*4 (sorted list) + V*(48 + D*feat_bytes) (records +
    feature rows, read once; 2-byte rows on the tcgen05 path) + H*W*(5 + D)*4
    (planar fp32 outputs) [+ H*W*13 (xyz + valid) when O13 is fused]."""
    return (4 * n_pairs + n_visible * (48 + feat_bytes * D) + total_pixels * (5 + D) * 4 +
            (13 * total_pixels if fused_backproject else 0))


# --------------------------------------------------------------------------- reference arm
_CPU_JOB = None


def _oracle_view(i):
    """Worker (forked): one view through the single-threaded oracle."""
    import oracle
    scene, views = _CPU_JOB
    t0 = time.perf_counter()
    oracle.render(scene, views[i], a_min=0.5)
    return views[i].width * views[i].height, time.perf_counter() - t0


def oracle_parallel(scene, views, picks):
    """Render views[picks] with independent single-threaded oracle processes, one
    view each, all at once (SURVEY.md §8(d) 'Oracle timing': min(C, views)
    processes on the host's C cores).  Returns (pixels, wall seconds, processes,
    per-view seconds)."""
    import multiprocessing as mp
    import oracle
    global _CPU_JOB
    oracle.build()
    _CPU_JOB = (scene, views)
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(len(picks)) as pool:
        res = pool.map(_oracle_view, picks, chunksize=1)
    wall = time.perf_counter() - t0
    _CPU_JOB = None
    return sum(p for p, _ in res), wall, len(picks), [t for _, t in res]


def cpu_processes(n_views: int) -> int:
    """min(host cores, views), bounded by host memory (~1 GB per oracle process)."""
    c = os.cpu_count() or 1
    try:
        import psutil
        c = min(c, max(1, int(psutil.virtual_memory().available / 1.0e9)))
    except ImportError:
        pass
    return max(1, min(c, n_views, 128))


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    import synth
    scene, views = synth.make_config(args.config, scale=args.scale)
    n = len(views)
    nproc = cpu_processes(n)
    times, pix = [], 0
    for s in range(args.warmup + args.steps):
        picks = [((s * nproc + k) * 37) % n for k in range(nproc)]
        px, wall, _, _ = oracle_parallel(scene, views, picks)
        if s >= args.warmup:
            times.append(wall)
            pix += px
    total = sum(times)
    value = pix / total / 1e6
    sample = (f"{nproc} of the {n} {args.config} views per step, one single-threaded C++ oracle process per view "
              f"on {nproc} host cores (project+bin+composite+backproject)")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "ms_per_view": 1e3 * total / (args.steps * nproc) * 1.0,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "f32 (decisions fp32 as the kernel, accumulations fp64)",
           "data": "synthetic", "config": {"workload": args.config, "scale": args.scale},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": nproc, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def cpu_baseline(scene, views):
    n = len(views)
    nproc = cpu_processes(n)
    picks = [(k * 97) % n for k in range(nproc)]
    px, wall, procs, per = oracle_parallel(scene, views, picks)
    return {"value": px / wall / 1e6, "unit": UNIT, "cores": procs, "kind": "oracle",
            "single_core_ms_per_view": 1e3 * float(np.median(per)), "host_cpu_count": os.cpu_count(),
            "sample": f"{procs} of {n} views, one single-threaded oracle process per view on {procs} host cores "
                      f"(project+bin+composite+backproject), {wall:.1f} s wall"}


# --------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    import paper_2507_15683_b200 as G
    from paper_2507_15683_b200 import dist as GD

    rank, world, local = GD.env_rank_world()
    use_pg = world > 1 or args.force_gather
    if use_pg:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", str(29500 + os.getpid() % 1000))
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())

    scene, views_all = workload(args.config, args.scale, rank, world, args.scaling, args.views)
    if args.views:
        views_all = views_all[:args.views]
    ds = G.DeviceScene(scene, device=dev, use_f16_features=args.feature_path == "tcgen05")
    stream = torch.cuda.current_stream()
    D = scene.feat_dim
    sharded = (world > 1 and args.scaling == "strong") or args.sharded or args.force_gather
    sharded_info = None
    if sharded:
        # cost-balanced shard of the pose batch (LPT over per-view pair
        # counts of one projection + binning pre-pass), per-chunk render into the gather
        # send buffer, one all_gather per chunk on a comm stream overlapped with the next
        # chunk's render
        pre = G.Renderer(ds, views_all, device=dev, binning=args.binning, alloc_images=False)
        pre.render()
        costs = pre.view_pair_counts()
        del pre
        torch.cuda.empty_cache()
        hw = views_all[0].width * views_all[0].height
        assert all(v.width * v.height == hw for v in views_all), "the gather needs equal-size views"
        chunk = args.chunk or max(1, -(-max(GD.shard_sizes(len(views_all), world, costs)) // 4))
        cg = GD.ChunkedGather(len(views_all), hw, world, rank, chunk, costs, device=dev,
                              always_gather=args.force_gather, payload=args.gather_transport)
        packed = args.gather_transport == "dense11"
        views = [views_all[i] for i in cg.mine]
        chunk_r = []
        for k in range(cg.n_chunks):
            cv = [views_all[i] for i in cg.chunk_views(k)]
            if not cv:
                chunk_r.append(None)
                continue
            rk = G.Renderer(ds, cv, device=dev, backproject=True, binning=args.binning,
                            out_planes=None if packed else cg.planes(k))
            rk.render()
            rk.fit_capacities()
            rk.render()
            chunk_r.append(rk)
        r = next(x for x in chunk_r if x is not None)
        chunks_rendered = sum(1 for x in chunk_r if x is not None)
        n_pairs = sum(x.n_pairs() for x in chunk_r if x is not None)
        n_visible = sum(int(x.proj.n_rec.sum().item()) for x in chunk_r if x is not None)
        total_px = sum(x.vb.total_pixels for x in chunk_r if x is not None)
        n_views = len(views)
    else:
        views = views_all
        r = G.Renderer(ds, views, device=dev, backproject=True, contrib=args.n1, binning=args.binning)
    scorer, fmaps = None, None
    if args.n1:
        if scene.feat_dim == 0 or sharded:
            raise SystemExit("--n1 needs a feature scene (C3 / C4) and the unsharded step")
        scorer = G.SignificanceScorer(ds, eps=1e-6, stride=8)
        g = torch.Generator(device=dev).manual_seed(1234 + rank)
        nmap = sum(scene.feat_dim * ((v.height + 7) // 8) * ((v.width + 7) // 8) for v in views)
        fmaps = torch.randn(nmap, generator=g, device=dev)
    if not sharded:
        r.render()
        r.fit_capacities()
        r.render()
        torch.cuda.synchronize()
        n_pairs = r.n_pairs()
        n_visible = int(r.proj.n_rec.sum().item())
        total_px = r.vb.total_pixels
        n_views = r.vb.n

    if args.profile_steps:
        for _ in range(args.profile_steps):
            if sharded:
                def prof_chunk(k):
                    if chunk_r[k] is not None:
                        chunk_r[k].run(stream)
                        if packed:
                            G.gs_pack_images(chunk_r[k].images, chunk_r[k].vb, cg.send[k], stream,
                                             fmt=G.GS_PACK_DENSE11)
                cg.step(prof_chunk, stream, gather=not args.no_gather)
            else:
                r.run()
        torch.cuda.synchronize()
        if world > 1:
            dist.destroy_process_group()
        return 0

    K = args.steps

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    def stage_pass(rr, e):
        """One hot-path pass of renderer rr with per-stage events e[0..5]."""
        rr.proj.status.zero_()
        e[0].record(stream)
        G.gs_project(rr.scene, rr.vb, rr.params, rr.proj, rr.ws_proj, stream, scene_struct=rr.scene_struct)
        e[1].record(stream)
        G.gs_bin_sort(rr.proj, rr.vb, rr.bins, rr.ws_bin, stream)
        e[2].record(stream)
        if args.separate_backproject:
            G.gs_rasterize(rr.scene, rr.proj, rr.bins, rr.vb, rr.params, rr.images, stream)
            e[3].record(stream)
            G.gs_backproject(rr.images, rr.vb, rr.a_min, rr.xyz, rr.valid, stream)
        else:
            G.gs_rasterize_backproject(rr.scene, rr.proj, rr.bins, rr.vb, rr.params, rr.images, rr.a_min, rr.xyz,
                                       rr.valid, stream)
            e[3].record(stream)
        e[4].record(stream)
        if scorer is not None:
            scorer.add(rr, fmaps, stream)
        e[5].record(stream)

    gather = sharded and (world > 1 or args.force_gather) and not args.no_gather
    with ClockSampler(torch.cuda.current_device() if world == 1 else local) as clk:
        if not sharded:
            # warm-up, then the timed region: CUDA events on the launching stream, per-stage
            # events for the roofline
            for _ in range(max(3, args.warmup)):
                r.run(stream)
                if scorer is not None:
                    scorer.add(r, fmaps, stream)
            torch.cuda.synchronize()
            ev = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(K)]
            start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            start.record(stream)
            for k in range(K):
                stage_pass(r, ev[k])
            end.record(stream)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            assert r.status() == 0, "capacity overflow inside the timed region"
            ms_total = start.elapsed_time(end)
            stage = np.array([[ev[k][j].elapsed_time(ev[k][j + 1]) for j in range(5)] for k in range(K)])
            step_ms = np.array([ev[k][0].elapsed_time(ev[k][5]) for k in range(K)])
        else:
            def render_chunk(k):
                if chunk_r[k] is not None:
                    chunk_r[k].run(stream)
                    if packed:   # the chunk's images -> its send buffer (GS_PACK_DENSE11)
                        G.gs_pack_images(chunk_r[k].images, chunk_r[k].vb, cg.send[k], stream,
                                         fmt=G.GS_PACK_DENSE11)

            def timed(gather_on):
                for _ in range(max(3, args.warmup)):
                    cg.step(render_chunk, stream, gather=gather_on)
                cg.wait(stream)
                torch.cuda.synchronize()
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
                if world > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                evs[0].record(stream)
                for k in range(K):
                    cg.step(render_chunk, stream, gather=gather_on)
                    cg.wait(stream)                      # the step ends when its gathers have landed
                    evs[k + 1].record(stream)
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                per = np.array([evs[k].elapsed_time(evs[k + 1]) for k in range(K)])
                return max_over_ranks(evs[0].elapsed_time(evs[K])), per

            ms_render, step_render = timed(False)
            if gather:
                ms_total, step_ms = timed(True)
            else:
                ms_total, step_ms = ms_render, step_render
            for x in chunk_r:
                assert x is None or x.status() == 0, "capacity overflow inside the timed region"
            # per-stage times of the rank's chunks (roofline of the dominant kernel)
            stage = np.zeros((K, 5))
            for k in range(K):
                evk = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in chunk_r]
                for q, x in enumerate(chunk_r):
                    if x is not None:
                        stage_pass(x, evk[q])
                torch.cuda.synchronize()
                for q, x in enumerate(chunk_r):
                    if x is not None:
                        stage[k] += [evk[q][j].elapsed_time(evk[q][j + 1]) for j in range(5)]
            all_px_r = sum_over_ranks(float(total_px))
            sharded_info = {
                "views_per_rank": [len(sh) for sh in cg.shards], "chunk": cg.chunk, "chunks": cg.n_chunks,
                "chunks_rendered": chunks_rendered,
                "assignment": "LPT over per-view pair counts of a gs_project + gs_bin_sort pre-pass",
                "render_only": {"value": all_px_r * K / (ms_render / 1e3) / 1e6, "ms_per_step": ms_render / K},
                "with_gather": None if not gather else {
                    "value": all_px_r * K / (ms_total / 1e3) / 1e6, "ms_per_step": ms_total / K,
                    "bytes_received_per_rank_per_step": cg.bytes_per_step,
                    "achieved_GBps": cg.bytes_per_step / (ms_total / K / 1e3) / 1e9,
                    "collective": "all_gather_into_tensor per chunk on a comm stream: " + (
                        "GS_PACK_DENSE11 bytes (fp16 RGB, unorm16 A, 24-bit depth; 11 B/px)" if packed
                        else "RGB + Dz + A fp32 planes (20 B/px)"),
                    "received_equals_sent": cg.check_own_slot()}}
    stage_ms = np.median(stage, axis=0)
    ms_total = max_over_ranks(ms_total)
    all_px = sum_over_ranks(float(total_px))
    all_views = sum_over_ranks(float(n_views))
    ms_step = ms_total / K
    value = all_px * K / (ms_total / 1e3) / 1e6
    step_stats = {"median": float(np.median(step_ms)), "p10": float(np.percentile(step_ms, 10)),
                  "p90": float(np.percentile(step_ms, 90)), "mean": float(np.mean(step_ms))}

    # e2e through the public API with host buffers: H2D of the pose batch from pinned
    # memory + the hot path + D2H of RGB + depth + opacity into pinned memory.
    # the same step replayed as one CUDA graph (single-view configs are also
    # timed as a graph -- their eager step is bound by launch gaps)
    graph_info = None
    if not sharded and scorer is None and (args.graph or n_views <= 8):
        gr = torch.cuda.CUDAGraph()
        gs_ = torch.cuda.Stream()
        gs_.wait_stream(stream)
        with torch.cuda.stream(gs_):
            r.run(gs_)
            with torch.cuda.graph(gr, stream=gs_):
                r.run(torch.cuda.current_stream())
        stream.wait_stream(gs_)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        g0.record(stream)
        for _ in range(K):
            gr.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        assert r.status() == 0
        ms_g = max_over_ranks(g0.elapsed_time(g1))
        graph_info = {"ms_per_step": ms_g / K, "value": all_px * K / (ms_g / 1e3) / 1e6,
                      "note": "the same step (project, bin_sort, rasterize + back-projection) captured once and "
                              "replayed as a CUDA graph"}
        del gr

    e2e = None
    if sharded:
        del chunk_r, r, cg
        torch.cuda.empty_cache()
        r = None
    if not args.no_e2e:
        # The batch in chunks, each with its own renderer buffers: chunk c's H2D (poses)
        # and render run on the compute stream while chunk c-1's RGB + depth + opacity
        # planes stream to pinned host memory on a copy stream -- the public API used
        # the way a caller overlaps PCIe with compute.
        n_chunks = max(1, min(args.e2e_chunks, n_views))
        bounds = [round(k * n_views / n_chunks) for k in range(n_chunks + 1)]
        chunk_views = [views[bounds[k]:bounds[k + 1]] for k in range(n_chunks)]
        r = None
        torch.cuda.empty_cache()
        rs = []
        for cv in chunk_views:
            rc = G.Renderer(ds, cv, device=dev, backproject=True, binning=args.binning)
            rc.render()
            rc.fit_capacities(1.02)
            rs.append(rc)
        px_off = np.cumsum([0] + [rc.vb.total_pixels for rc in rs])
        copy_stream = torch.cuda.Stream()
        copied = [torch.cuda.Event() for _ in rs]
        rendered = [torch.cuda.Event() for _ in rs]

        def measure_e2e(transport):
            compact = transport in ("compact", "dense11")
            fmt = G.GS_PACK_DENSE11 if transport == "dense11" else G.GS_PACK_COMPACT
            bpp = {"dense11": 11, "compact": 12, "f32": 20}[transport]
            host_out = torch.empty(bpp * total_px, dtype=torch.uint8, pin_memory=True)
            packed = [torch.empty(bpp * rc.vb.total_pixels + 16, dtype=torch.uint8, device=dev) for rc in rs] \
                if compact else None
            hf = host_out.view(torch.float32) if not compact else None

            def e2e_step(first):
                for k, rc in enumerate(rs):
                    if not first:
                        stream.wait_event(copied[k])          # chunk k's buffers were copied out
                    rc.vb.upload(stream)
                    rc.run(stream)
                    if compact:
                        G.gs_pack_images(rc.images, rc.vb, packed[k], stream, fmt=fmt)
                    rendered[k].record(stream)
                    copy_stream.wait_event(rendered[k])
                    with torch.cuda.stream(copy_stream):
                        o, m = int(px_off[k]), rc.vb.total_pixels
                        if compact:
                            host_out[bpp * o:bpp * (o + m)].copy_(packed[k][:bpp * m], non_blocking=True)
                        else:
                            hf[3 * o:3 * (o + m)].copy_(rc.images.rgb, non_blocking=True)
                            hf[3 * total_px + o:3 * total_px + o + m].copy_(rc.images.depth, non_blocking=True)
                            hf[4 * total_px + o:4 * total_px + o + m].copy_(rc.images.alpha, non_blocking=True)
                    copied[k].record(copy_stream)

            e2e_step(True)
            torch.cuda.synchronize()
            Ke = max(2, min(K, 5))
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            for _ in range(Ke):
                e2e_step(False)
            s1.record(copy_stream)
            torch.cuda.synchronize()
            ms_e = max_over_ranks(s0.elapsed_time(s1))
            del host_out, packed
            return {"value": all_px * Ke / (ms_e / 1e3) / 1e6, "unit": UNIT,
                    "h2d_bytes_per_step": int(sum(rc.vb.pinned.numel() for rc in rs)),
                    "d2h_bytes_per_step": int(bpp * total_px), "chunks": n_chunks,
                    "transport": {"dense11": "dense11: fp16 RGB + unorm16 A + 24-bit depth, 11 B/px "
                                             "(gs_pack_images GS_PACK_DENSE11, reading Q39)",
                                  "compact": "compact: fp16 RGB + fp16 A + fp32 depth, 12 B/px "
                                             "(gs_pack_images GS_PACK_COMPACT, reading Q39)",
                                  "f32": "fp32 RGB + depth + A planes, 20 B/px"}[transport],
                    "note": "pose upload + the whole step (incl. back-projection) + D2H of the step's RGB, depth, "
                            "opacity per chunk; D2H overlapped with the next chunk's render on a copy stream"}

        e2e = measure_e2e(args.e2e_transport)
        e2e["other_transports"] = []
        for t in ("dense11", "compact", "f32"):
            if t != args.e2e_transport:
                other = measure_e2e(t)
                e2e["other_transports"].append({"value": other["value"],
                                                "d2h_bytes_per_step": other["d2h_bytes_per_step"],
                                                "transport": other["transport"]})
        del rs
        torch.cuda.empty_cache()
    if r is None and (args.n2 or args.n4 or args.refine):
        r = G.Renderer(ds, views, device=dev, backproject=True, contrib=args.n1, binning=args.binning)
        r.render()

    # N2: coarse-to-fine matching of rendered feature maps, (view i -> query, view i+1 -> rendered)
    n2 = None
    if args.n2:
        D2 = scene.feat_dim
        H2, W2 = views[0].height, views[0].width
        if D2 not in (16, 32, 48, 64) or H2 % 8 or W2 % 8 or n_views < 2:
            raise SystemExit("--n2 needs D in {16,32,48,64}, sizes multiple of 8 and >= 2 views")
        Bp = max(1, min(args.n2_pairs, n_views - 1))
        hw = H2 * W2
        fq = r.images.feat[:Bp * D2 * hw]
        fr = r.images.feat[D2 * hw:(Bp + 1) * D2 * hw]
        mo = G.Matches(Bp, H2, W2, with_points=True, device=dev)
        mws = torch.empty(G.match_workspace_bytes(Bp, D2, H2, W2), dtype=torch.uint8, device=dev)
        xyz2, val2 = r.xyz[3 * hw:3 * hw * (Bp + 1)], r.valid[hw:hw * (Bp + 1)]

        def match():
            G.gs_match(fq, fr, Bp, D2, H2, W2, mo, mws, rend_xyz=xyz2, rend_valid=val2, stream=stream)

        for _ in range(3):
            match()
        torch.cuda.synchronize()
        m0, m1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        m0.record(stream)
        for _ in range(K):
            match()
        m1.record(stream)
        torch.cuda.synchronize()
        ms2 = m0.elapsed_time(m1) / K
        nc = (H2 // 8) * (W2 // 8)
        n2 = {"pairs": Bp, "ms": ms2, "ms_per_pair": ms2 / Bp, "fine_resolution": f"{W2}x{H2}", "feat_dim": D2,
              "coarse_cells": nc, "coarse_similarities_per_pair": nc * nc,
              "coarse_matches_per_pair": float((mo.coarse >= 0).sum().item()) / Bp,
              "fine_matches_per_pair": float((mo.peak >= 0).sum().item()) / Bp,
              "valid_2d3d_per_pair": float(mo.valid.sum().item()) / Bp,
              "coarse_gemm_tflops": 2.0 * 3 * 2 * 2 * nc * nc * D2 * Bp / (ms2 / 1e3) / 1e12,
              "gpu_launches": 5, "tau": 0.1, "p_min": 0.05}

    # N4: feature-field backward of Eq. 2 over the batch (random upstream gradient)
    n4 = None
    if args.n4:
        if scene.feat_dim == 0:
            raise SystemExit("--n4 needs a feature scene (C3 / C4)")
        g4 = torch.Generator(device=dev).manual_seed(99)
        gimg = torch.randn(r.images.feat.numel(), generator=g4, device=dev)
        gfeat = torch.zeros(scene.n * scene.feat_dim, dtype=torch.float32, device=dev)
        for _ in range(2):
            G.gs_feature_backward(ds, r.proj, r.bins, r.vb, r.params, gimg, gfeat, stream)
        torch.cuda.synchronize()
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Kb = max(2, min(K, 5))
        b0.record(stream)
        for _ in range(Kb):
            gfeat.zero_()
            G.gs_feature_backward(ds, r.proj, r.bins, r.vb, r.params, gimg, gfeat, stream)
        b1.record(stream)
        torch.cuda.synchronize()
        ms4 = b0.elapsed_time(b1) / Kb
        # radiance backward: random upstream gradients of RGB, depth, opacity
        gout = G.Images(total_px, 0, device=dev)
        for t in (gout.rgb, gout.depth, gout.alpha):
            t.normal_(generator=g4)
        grec = torch.zeros(n_views * r.proj.rec_capacity * 10, dtype=torch.float32, device=dev)
        G.gs_radiance_backward(r.proj, r.bins, r.vb, r.params, r.images, gout, grec, stream)
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(Kb):
            grec.zero_()
            G.gs_radiance_backward(r.proj, r.bins, r.vb, r.params, r.images, gout, grec, stream)
        b1.record(stream)
        torch.cuda.synchronize()
        msr = b0.elapsed_time(b1) / Kb
        # Eq. 1's joint record gradient: the radiance terms + the feature term through the
        # blend weights (gs_joint_backward, the upstream feature gradient = gimg)
        gout.set_feat(gimg, scene.feat_dim)
        G.gs_joint_backward(ds, r.proj, r.bins, r.vb, r.params, r.images, gout, grec, stream)
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(Kb):
            grec.zero_()
            G.gs_joint_backward(ds, r.proj, r.bins, r.vb, r.params, r.images, gout, grec, stream)
        b1.record(stream)
        torch.cuda.synchronize()
        msj = b0.elapsed_time(b1) / Kb
        gout.set_feat(None, 0)
        # projection backward: the record gradients to the 3D means and the other parameters
        nk = (scene.sh_degree + 1) ** 2
        gpos = torch.zeros(3 * scene.n, device=dev)
        gsc, gq = torch.zeros(3 * scene.n, device=dev), torch.zeros(4 * scene.n, device=dev)
        gop, gsh = torch.zeros(scene.n, device=dev), torch.zeros(nk * 3 * scene.n, device=dev)
        G.gs_mean_backward(ds, r.proj, r.vb, r.params, grec, gpos, stream)
        G.gs_param_backward(ds, r.proj, r.vb, r.params, grec, gsc, gq, gop, gsh, stream)
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(Kb):
            G.gs_mean_backward(ds, r.proj, r.vb, r.params, grec, gpos, stream)
            G.gs_param_backward(ds, r.proj, r.vb, r.params, grec, gsc, gq, gop, gsh, stream)
        b1.record(stream)
        torch.cuda.synchronize()
        msp = b0.elapsed_time(b1) / Kb
        del gpos, gsc, gq, gop, gsh
        # Eq. 3's D-SSIM loss + gradient (gs_dssim_grad) on the batch's RGB planes, one call per
        # run of equal-size views; target = the render with noise
        from paper_2507_15683_b200.pipeline import equal_size_runs
        runs = equal_size_runs(r.vb.views, max_views=64)
        tgt = (r.images.rgb + 0.05 * torch.randn(r.images.rgb.numel(), generator=g4, device=dev)).clamp_(0, 1)
        grgb = torch.zeros_like(r.images.rgb)
        lss = torch.zeros(1, dtype=torch.float64, device=dev)
        wsd = [None]     # one workspace reused by every call (<= 64 views each)

        def _dssim():
            for i0, cnt, h, w in runs:
                o, n = 3 * r.vb.pix_offset(i0), 3 * cnt * h * w
                wsd[0] = G.gs_dssim_grad(r.images.rgb[o:o + n], tgt[o:o + n], 3 * cnt, h, w,
                                         0.2 / r.images.rgb.numel(), grgb[o:o + n], lss, wsd[0], stream)
        _dssim()
        torch.cuda.synchronize()
        b0.record(stream)
        for _ in range(Kb):
            _dssim()
        b1.record(stream)
        torch.cuda.synchronize()
        msd = b0.elapsed_time(b1) / Kb
        dssim_bytes = 48 * r.images.rgb.numel()
        n4 = {"views": n_views, "feature_backward_ms": ms4, "feature_backward_ms_per_view": ms4 / n_views,
              "radiance_backward_ms": msr, "radiance_backward_ms_per_view": msr / n_views,
              "joint_backward_ms": msj, "joint_backward_ms_per_view": msj / n_views,
              "projection_backward_ms": msp, "dssim_grad_ms": msd, "dssim_grad_ms_per_view": msd / n_views,
              "dssim_grad_GBps": dssim_bytes / (msd * 1e-3) / 1e9, "feat_dim": scene.feat_dim,
              "gpu_launches": 7 + 2 * len(runs)}
        del tgt, grgb, wsd
        del gimg, gfeat, gout, grec

    # N2 refinement loop: B queries, n = 3 rounds, one CUDA graph
    refine = None
    if args.refine:
        import math as _m
        import synth
        Bq = max(1, min(args.refine, n_views))
        qv = views[:Bq]
        rq = G.Renderer(ds, qv, device=dev)
        rq.render()
        query = rq.images.feat.clone() if scene.feat_dim else None
        del rq
        if query is None:
            raise SystemExit("--refine needs a feature scene (C3 / C4)")
        rng = np.random.default_rng(7 + rank)
        init = []
        for v in qv:
            R = np.asarray(v.R, np.float64).reshape(3, 3)
            C = -R.T @ np.asarray(v.t, np.float64)
            ax = rng.standard_normal(3)
            ax /= np.linalg.norm(ax)
            th = _m.radians(1.0)
            Kx = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
            dR = np.eye(3) + _m.sin(th) * Kx + (1 - _m.cos(th)) * Kx @ Kx
            R0 = dR @ R
            C0 = C + np.array([1.0, -1.0, 0.3])
            init.append(synth.make_view(R0.astype(np.float32), (-R0 @ C0).astype(np.float32), v.fx, v.fy, v.cx, v.cy,
                                        v.width, v.height))
        ref = G.Refiner(ds, init, query, n_iters=3)
        ref.capture()
        for _ in range(2):
            ref.replay()
        torch.cuda.synchronize()
        r0e, r1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        Kr = max(2, min(K, 5))
        r0e.record()
        for _ in range(Kr):
            ref.replay()
        r1e.record()
        torch.cuda.synchronize()
        ms_r = r0e.elapsed_time(r1e) / Kr
        R0s, t0s = ref.poses(0)
        R3s, t3s = ref.poses(3)
        errs0, errs3 = [], []
        for b, v in enumerate(qv):
            Rg = np.asarray(v.R, np.float64).reshape(3, 3)
            Cg = -Rg.T @ np.asarray(v.t, np.float64)
            for (Rs, ts, out) in ((R0s, t0s, errs0), (R3s, t3s, errs3)):
                c = np.linalg.norm(Rs[b] - Rg) / (2 * _m.sqrt(2))
                out.append((_m.degrees(2 * _m.asin(min(1.0, c))), float(np.linalg.norm(-Rs[b].T @ ts[b] - Cg))))
        e0, e3 = np.median(np.array(errs0), 0), np.median(np.array(errs3), 0)
        refine = {"queries": Bq, "rounds": 3, "ms": ms_r, "ms_per_query": ms_r / Bq, "cuda_graph": True,
                  "median_rot_err_deg": {"initial": float(e0[0]), "refined": float(e3[0])},
                  "median_pos_err_m": {"initial": float(e0[1]), "refined": float(e3[1])},
                  "reliable_fraction": float((ref.verdict == -1).float().mean().item()),
                  "median_inliers_last_round": float(ref.stats[-1, :, 1].float().median().item()),
                  "resolution": f"{qv[0].width}x{qv[0].height}",
                  "launches_per_round": 12 + 5 + 1, "capacity_overflow": ref.status() != 0}
        del ref

    # roofline of the dominant kernel
    peak, peak_src = measured_peaks()
    dom = int(np.argmax(stage_ms[:4]))
    names = ["gs_project", "gs_bin_sort", "gs_rasterize", "gs_backproject", "n1_visibility_score"]
    D = scene.feat_dim
    tc_path = D in (16, 32, 48, 64) and args.feature_path == "tcgen05"
    fused = not args.separate_backproject
    raster_bytes = algorithmic_raster_bytes(n_pairs, n_visible, total_px, D, 2 if tc_path else 4, fused)
    achieved = raster_bytes / (stage_ms[2] / 1e3) / 1e9
    nrec = ncu_traffic(f"{args.config}@{args.scale}/{args.binning}/{'tcgen05' if tc_path else 'mma_sync'}")
    traffic = nrec.get("rasterize_dram_bytes_per_launch")
    roof = {"bound": "hbm", "kernel": "gs_rasterize", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": raster_bytes, "dominant_stage": names[dom],
            "ncu_issue_active": nrec.get("issue_active"),
            "ncu_thread_instructions_per_pixel": nrec.get("thread_instructions_per_pixel"),
            "note": "HBM roofline of the algorithmic bytes; the kernel is bound by instruction issue and "
                    "dependent latency, not bytes: ncu_issue_active / ncu_thread_instructions_per_pixel and "
                    "traffic come from one committed ncu launch of this configuration "
                    "(profiles/ncu_traffic.json, tools/gpu_traffic.sh; DESIGN.md §4.3b)"}
    # SURVEY §8(d) algorithmic bytes of the other stages: gs_project N*44 (geometry once per
    # batch) + V*12(L+1)^2 (SH of every visible record) + V*64 (records written); gs_bin_sort
    # V*16 (rectangle + depth read) + P*4 (sorted list) + T*8 (ranges)
    nk_sh = (scene.sh_degree + 1) ** 2
    T_tiles = sum(((v.width + 15) // 16) * ((v.height + 15) // 16) for v in views)
    proj_bytes = scene.n * 44 + n_visible * (12 * nk_sh + 64)
    bin_bytes = n_visible * 16 + n_pairs * 4 + T_tiles * 8
    stage_roofs = {
        "gs_project": {"bound": "hbm", "algorithmic_bytes": proj_bytes,
                       "achieved": proj_bytes / (stage_ms[0] / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                       "frac": proj_bytes / (stage_ms[0] / 1e3) / 1e9 / peak},
        "gs_bin_sort": {"bound": "hbm", "algorithmic_bytes": bin_bytes,
                        "achieved": bin_bytes / (stage_ms[1] / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": bin_bytes / (stage_ms[1] / 1e3) / 1e9 / peak}}
    launches_per_step = (3 if ds.n_blocks else 2) + 8 + 1 + (0 if fused else 1) + (1 if scorer is not None else 0)
    if sharded:
        launches_per_step = ((3 if ds.n_blocks else 2) + 8 + 1 + (1 if args.gather_transport == "dense11" else 0)) \
            * sharded_info["chunks_rendered"]

    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": args.warmup,
           "ms_per_step": ms_step, "ms_per_view": ms_step * world / all_views, "step_ms": step_stats,
           "higher_is_better": True, "scaling": args.scaling if world > 1 else "strong", "vs_baseline": None,
           "dtype": "f32 (RGB/depth/opacity fp32 FMA; features: fp16-rounded rows x hi+lo fp16 weights on tcgen05, "
                    "fp32 accumulate)" if D else "f32", "data": "synthetic",
           "config": {"workload": args.config, "scale": args.scale, "gaussians": scene.n, "views_per_rank": n_views,
                      "resolution": f"{views[0].width}x{views[0].height}", "sh_degree": scene.sh_degree,
                      "feat_dim": D, "l2": "inputs larger than L2 (scene %.2f GB, %.1f GB written per step)" % (
                          ds.nbytes() / 1e9, (total_px * (5 + D) * 4 + total_px * 13) / 1e9),
                      "gather": bool(gather), "n1": bool(args.n1), "binning": args.binning,
                      "backproject": "fused into gs_rasterize (gs_rasterize_backproject)" if fused else "separate",
                      "feature_path": (args.feature_path if scene.feat_dim in (16, 32, 48, 64) else "mma_sync")
                      if scene.feat_dim else None},
           "stages_ms": {n: float(m) for n, m in zip(names, stage_ms) if n != names[4] or scorer is not None},
           "counts": {"visible_records": n_visible, "pairs": n_pairs, "pixels": total_px},
           "roofline": roof, "stage_rooflines": stage_roofs, "gpu_launches": launches_per_step * K, "e2e": e2e,
           "clocks": clk.summary()}
    if sharded_info is not None:
        out["sharded"] = sharded_info
    if graph_info is not None:
        out["graph"] = graph_info
    if n2 is not None:
        out["n2"] = n2
    if refine is not None:
        out["refine"] = refine
    if n4 is not None:
        out["n4"] = n4
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(scene, views)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if use_pg:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
