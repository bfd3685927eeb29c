"""Debug: SIMT efficiency of gs_rasterize's walk (build gs_rasterize.cu with
-DGS_RASTER_STATS into paper_2507_15683_b200/libgs_stats.so first, see
DESIGN.md §10).  Prints entry walks per warp-tile and the live-lane fraction."""
import ctypes, os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
os.environ["GS_LIB"] = os.path.join(os.environ["GRAFT_REPO_ROOT"], "paper_2507_15683_b200/libgs_stats.so")
import torch, numpy as np, synth
import paper_2507_15683_b200 as G
sc, vs = synth.make_config("C4", scale=1.0)
vs = vs[:32]
ds = G.DeviceScene(sc)
r = G.Renderer(ds, vs)
r.render(); r.fit_capacities(); r.render(); torch.cuda.synchronize()
L = G.lib()
out = (ctypes.c_ulonglong * 4)()
L.gs_debug_raster_stats(out)
r.run(); torch.cuda.synchronize()
L.gs_debug_raster_stats(out)
walks, live = out[0], out[1]
px = r.vb.total_pixels
print("entry-walks per warp-tile: %.1f" % (walks / (r.vb.total_tiles * 8)))
print("live lane fraction during walks: %.3f" % (live / (32.0 * walks)))
print("entry-walks per pixel-lane: %.1f, live per pixel: %.1f" % (walks * 32 / px, live / px))
print("walked entries with alpha >= alpha_min at some warp pixel: %.3f" % (out[2] / max(walks, 1)))
print("blends per pixel: %.1f" % (out[3] / px))
