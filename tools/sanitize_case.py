"""Small end-to-end invocation for compute-sanitizer runs:
C1 (+ D = 8 features, contributions, visibility) and a cropped aerial batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2507_15683_b200 as G  # noqa: E402
import synth  # noqa: E402

sc = synth.box_v1(1000, seed=11, feat_dim=8)
ds = G.DeviceScene(sc)
r = G.Renderer(ds, [synth.box_view()], contrib=True)
r.render()
scorer = G.SignificanceScorer(ds)
fm = torch.randn(8 * 64 * 64, device="cuda")
scorer.add(r, fm)
sc2, vs2 = synth.make_config("C4", scale=0.004)
vs2 = [synth.make_view(v.R, v.t, v.fx / 4, v.fy / 4, (v.cx + 0.5) / 4 - 0.5, (v.cy + 0.5) / 4 - 0.5, 256, 192)
       for v in vs2[:4]]
ds2 = G.DeviceScene(sc2)
r2 = G.Renderer(ds2, vs2)
r2.render()
sc3, vs3 = synth.make_config("C3", scale=0.01)
r3 = G.Renderer(G.DeviceScene(sc3), vs3[:2])
r3.render()
torch.cuda.synchronize()
print("sanitize case ok", int(r.n_pairs()), int(r2.n_pairs()), int(r3.n_pairs()))
