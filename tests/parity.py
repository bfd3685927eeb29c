"""GPU-vs-oracle comparison helpers (BASELINE.json north_star tolerances,
SURVEY.md §8(c) 'Parity criteria').

* records: u, v, z, exponent coefficients, radius, tile rectangle bit-exact; rgb 1e-5
* keys (tile, depth_bits, gid) and tile ranges: bit-exact
* rgb, alpha: max abs 1e-3 on pixels not flagged by the oracle (Q20)
* depth Dz: |d| <= 1e-4 |Dz| where A >= 1e-3, else <= 1e-4 z_near
* features: max abs 1e-3 max(1, max|f|)
* flagged pixels (oracle O14, bands derived from the kernel's exp2 precision, DESIGN.md
  reading Q20): error <= 0.0105 max(1,|attr|) + 1e-3 (a flipped T-stop changes one
  blend of weight alpha T <= 1e-4/(1-0.99) = 0.01; a flipped 1/255 skip one of
  weight <= 1/255); their number over all pixels a test compares <= 1e-4 of them
  (SURVEY.md §8(c) parity criteria, FLAG_FRAC_MAX) -- assert_flag_budget
* back-projection: |dX| <= 1e-3 scene_scale (median valid zbar); valid masks
  equal except on flagged pixels
"""
import math

import numpy as np

RGB_TOL = 1e-3
DEPTH_REL = 1e-4
FEAT_TOL = 1e-3
FLAG_FRAC_MAX = 1e-4
FLAG_W = 0.0105


def decode_records(rec_i32: np.ndarray):
    """[n, 16] int32 words of gs_record -> dict of fields."""
    r = np.ascontiguousarray(rec_i32)
    f = r.view(np.float32)
    u32 = r.view(np.uint32)
    return dict(u=f[:, 0], v=f[:, 1], ecoef=f[:, 2:5], opacity=f[:, 5], e_cut=f[:, 6], rgb=f[:, 8:11],
                z=f[:, 11], gid=u32[:, 12], view=u32[:, 13] & 0xFFFF, radius=(u32[:, 13] >> 16).astype(np.float32),
                rect=np.stack([u32[:, 14] & 0xFFFF, u32[:, 14] >> 16, u32[:, 15] & 0xFFFF, u32[:, 15] >> 16], 1))


def check_records(gpu_rec: dict, orc_rec: dict, view_index: int):
    order = np.argsort(gpu_rec["gid"], kind="stable")
    g = {k: v[order] for k, v in gpu_rec.items()}
    np.testing.assert_array_equal(g["gid"], orc_rec["gid"].astype(np.uint32), err_msg="visible set differs")
    assert (g["view"] == view_index).all()
    for k in ("u", "v", "z"):
        np.testing.assert_array_equal(g[k].view(np.uint32), orc_rec[k].view(np.uint32), err_msg=f"{k} not bit-exact")
    # the record holds the exponent coefficients (k a, 2k b, k c), k = fp32(-log2(e)/2) (reading Q29)
    k = np.float32(-0.72134752044448170368)
    c = orc_rec["conic"].astype(np.float32)
    expect = np.stack([k * c[:, 0], (np.float32(2) * k) * c[:, 1], k * c[:, 2]], 1).astype(np.float32)
    np.testing.assert_array_equal(g["ecoef"].view(np.uint32), expect.view(np.uint32),
                                  err_msg="exponent coefficients not bit-exact")
    np.testing.assert_array_equal(g["e_cut"].view(np.uint32), orc_rec["e_cut"].view(np.uint32),
                                  err_msg="e_cut not bit-exact (reading Q30)")
    np.testing.assert_array_equal(g["radius"], np.minimum(orc_rec["radius"], 65535), err_msg="radius")
    np.testing.assert_array_equal(g["rect"].astype(np.int64), orc_rec["rect"].astype(np.int64), err_msg="rect")
    np.testing.assert_array_equal(g["opacity"], orc_rec["opacity"])
    np.testing.assert_allclose(g["rgb"], orc_rec["rgb"], rtol=1e-5, atol=1e-5, err_msg="SH rgb")


def check_keys(gk, orc_keys):
    tiles, depth, gid, ranges = gk
    assert len(tiles) == len(orc_keys["tile"]), f"pair count {len(tiles)} != oracle {len(orc_keys['tile'])}"
    np.testing.assert_array_equal(tiles, orc_keys["tile"], err_msg="tile keys")
    np.testing.assert_array_equal(depth, orc_keys["depth"], err_msg="depth keys")
    np.testing.assert_array_equal(gid, orc_keys["gid"], err_msg="gid keys")
    np.testing.assert_array_equal(ranges, orc_keys["ranges"], err_msg="ranges")


def check_images(gpu: dict, orc: dict, z_near: float = 0.2, report: dict = None):
    """Image parity; returns a stats dict."""
    flags = orc["flags"] != 0
    ok = ~flags
    stats = {}
    d_rgb = np.abs(gpu["rgb"] - orc["rgb"])
    d_a = np.abs(gpu["alpha"] - orc["alpha"])
    stats["rgb_max_err"] = float(d_rgb[:, ok].max(initial=0))
    stats["alpha_max_err"] = float(d_a[ok].max(initial=0))
    assert stats["rgb_max_err"] <= RGB_TOL, stats
    assert stats["alpha_max_err"] <= RGB_TOL, stats
    A = orc["alpha"]
    dz = np.abs(gpu["depth"].astype(np.float64) - orc["depth"])
    lim = np.where(A >= 1e-3, DEPTH_REL * np.abs(orc["depth"]), DEPTH_REL * z_near)
    stats["depth_max_rel_excess"] = float((dz / np.maximum(lim, 1e-30))[ok].max(initial=0))
    assert (dz[ok] <= lim[ok] * (1 + 1e-9)).all(), stats
    if orc.get("feat") is not None and orc["feat"].size:
        fmax = max(1.0, float(np.abs(orc["feat"]).max()))
        d_f = np.abs(gpu["feat"] - orc["feat"])
        stats["feat_max_err"] = float(d_f[:, ok].max(initial=0))
        assert stats["feat_max_err"] <= FEAT_TOL * fmax, stats
    nflag = int(flags.sum())
    stats["flagged"] = nflag
    stats["flagged_frac"] = nflag / flags.size
    if nflag:
        bound_rgb = FLAG_W * max(1.0, float(np.abs(orc["rgb"]).max())) + 1e-3
        assert d_rgb[:, flags].max() <= bound_rgb, stats
        assert d_a[flags].max() <= FLAG_W + 1e-3, stats
    stats["pixels"] = int(flags.size)
    stats["evals_per_pixel"] = orc.get("evals", 0) / max(1, flags.size)
    if report is not None:
        report.update(stats)
    log_stats("", stats)
    return stats


def check_backproject(gpu_xyz, gpu_valid, orc_xyz, orc_valid, flags, orc_depth, orc_alpha):
    ok = flags == 0
    np.testing.assert_array_equal(gpu_valid[ok], orc_valid[ok], err_msg="valid mask")
    both = (gpu_valid > 0) & (orc_valid > 0)
    if both.any():
        zbar = orc_depth[orc_valid > 0].astype(np.float64) / orc_alpha[orc_valid > 0]
        scale = float(np.median(zbar))
        err = np.linalg.norm(gpu_xyz[:, both].astype(np.float64) - orc_xyz[:, both], axis=0)
        assert err.max() <= 1e-3 * scale, (err.max(), scale)
    assert not gpu_xyz[:, gpu_valid == 0].any()


def _current_test() -> str:
    import os
    return os.environ.get("PYTEST_CURRENT_TEST", "").split(" ")[0]


def log_stats(test: str, stats: dict):
    """Append one parity record (flagged count / fraction, max errors) to the
    JSONL log ($GS_PARITY_LOG, default gpurun_out/parity_stats.jsonl)."""
    import json
    import os
    path = os.environ.get("GS_PARITY_LOG") or os.path.join(
        os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out", "parity_stats.jsonl")
    try:
        os.makedirs(os.path.dirname(path), exist_ok=True)
        with open(path, "a") as f:
            f.write(json.dumps({"test": test or _current_test(), **stats}) + "\n")
    except OSError:
        pass


def assert_flag_budget(stats_list, test: str = ""):
    """Flagged (O14) pixels over all the views a test compared: a fraction
    <= FLAG_FRAC_MAX of the n pixels compared ('fraction <=
    1e-4'), i.e. at most ceil(1e-4 n) pixels -- a test of fewer than 10^4 pixels
    may hold one flagged pixel (reading Q20)."""
    px = sum(s["pixels"] for s in stats_list)
    fl = sum(s["flagged"] for s in stats_list)
    log_stats((test or _current_test()) + "::total", {"pixels": px, "flagged": fl, "flagged_frac": fl / max(1, px), "views": len(stats_list)})
    assert fl <= math.ceil(FLAG_FRAC_MAX * px), (test, fl, px)
