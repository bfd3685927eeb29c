"""Debug: SceneTrainer loss curves on the C1 box scene for a few learning-rate sets."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import dataclasses, numpy as np, torch, synth
import paper_2507_15683_b200 as G
base = synth.box_v1(1500, seed=21, sh_degree=1)
v = synth.box_view()
true = G.DeviceScene(base)
rt = G.Renderer(true, [v], backproject=False)
rt.render()
target = rt.images.rgb.clone()
rng = np.random.default_rng(5)
start = dataclasses.replace(base, pos=base.pos + rng.normal(0, 0.02, base.pos.shape).astype(np.float32),
                            sh=base.sh + rng.normal(0, 0.3, base.sh.shape).astype(np.float32))
for lr in ({}, {"pos": 1e-1, "sh": 1.0, "opacity": 1e-1}, {"pos": 1.0, "sh": 10.0, "opacity": 1.0, "scale": 1e-2}):
    ds = G.DeviceScene(start)
    t = G.SceneTrainer(ds, [v], target, lr=lr)
    losses = [float(t.step().item()) for _ in range(40)]
    print(lr, ["%.4f" % x for x in losses[::8]], t.r.status())
