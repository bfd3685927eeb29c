"""Time gs_dssim_grad (Eq. 3's D-SSIM + gradient, N4) on C4-sized RGB planes
(V views x 3 x 768 x 1024, inputs far larger than L2) with CUDA events on the
launching stream; print one JSON line with the HBM roofline of the algorithmic
bytes (48 B per pixel per plane: pass 1 reads x, y and writes 3 partials; pass 2
reads the partials, x, y and read-modify-writes the gradient)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_15683_b200 as G  # noqa: E402


def main(views=64, steps=10, warmup=3):
    H, W, C = 768, 1024, 3
    n = views * C * H * W
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand(n, device="cuda", generator=g)
    y = (x + 0.1 * torch.randn(n, device="cuda", generator=g)).clamp_(0, 1)
    grad = torch.zeros(n, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    ws = None
    s = torch.cuda.current_stream()
    for _ in range(warmup):
        ws = G.gs_dssim_grad(x, y, views * C, H, W, 1.0 / n, grad, loss, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(steps):
        ws = G.gs_dssim_grad(x, y, views * C, H, W, 1.0 / n, grad, loss, ws)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    peak = float(peaks["hbm_gbs"])   # measured copy bandwidth (burst: the kernel is timed alone)
    gbs = 48.0 * n / (ms * 1e-3) / 1e9
    print(json.dumps({"kernel": "gs_dssim_grad", "planes": views * C, "height": H, "width": W, "ms_per_call": ms,
                      "ms_per_view": ms / views, "algorithmic_bytes": 48 * n, "achieved_GBps": gbs,
                      "peak_GBps": peak, "frac": gbs / peak if peak else None}))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
