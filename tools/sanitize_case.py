"""Small end-to-end invocation for compute-sanitizer runs:
C1 with D = 8 features (mma.sync path) + N1 contributions / visibility; a
cropped C4 batch with D = 32 (the tcgen05 / TMEM / mbarrier feature path), with
and without N1 contributions; the C3 pyramid's coarse levels (long-list sorts);
N2 matching on the rendered feature maps; the N4 backward kernels (feature,
joint, appearance, D-SSIM, projection) and one training step."""
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
# C4 crop: D = 32 on tcgen05 (256x192 views, multiples of 8 for N2)
sc2, vs2 = synth.make_config("C4", scale=0.004)
vs2 = [synth.make_view(v.R, v.t, v.fx / 4, v.fy / 4, (v.cx + 0.5) / 4 - 0.5, (v.cy + 0.5) / 4 - 0.5, 256, 192)
       for v in vs2[:4]]
ds2 = G.DeviceScene(sc2)
r2 = G.Renderer(ds2, vs2)
r2.render()
r2c = G.Renderer(ds2, vs2, contrib=True)      # tcgen05 path + N1 contributions
r2c.render()
sc3, vs3 = synth.make_config("C3", scale=0.01)
r3 = G.Renderer(G.DeviceScene(sc3), vs3[:2])
r3.render()
# N2: coarse-to-fine matching between rendered views 0 -> 1, 2 -> 3
H, W, D = 192, 256, 32
hw = H * W
mo = G.Matches(2, H, W, with_points=True)
mws = torch.empty(G.match_workspace_bytes(2, D, H, W), dtype=torch.uint8, device="cuda")
q = torch.cat([r2.images.feat[0:D * hw], r2.images.feat[2 * D * hw:3 * D * hw]])
rf = torch.cat([r2.images.feat[D * hw:2 * D * hw], r2.images.feat[3 * D * hw:4 * D * hw]])
xyz = torch.cat([r2.xyz[3 * hw:6 * hw], r2.xyz[9 * hw:12 * hw]])
val = torch.cat([r2.valid[hw:2 * hw], r2.valid[3 * hw:4 * hw]])
G.gs_match(q, rf, 2, D, H, W, mo, mws, rend_xyz=xyz, rend_valid=val)
# N4: backward kernels + a joint training step with appearance and D-SSIM
rng = np.random.default_rng(0)
gimg = torch.randn(r2.images.feat.numel(), device="cuda")
gfeat = torch.zeros(sc2.n * D, device="cuda")
G.gs_feature_backward(ds2, r2.proj, r2.bins, r2.vb, r2.params, gimg, gfeat)
gout = G.Images(r2.vb.total_pixels, 0)
for t in (gout.rgb, gout.depth, gout.alpha):
    t.normal_()
gout.set_feat(gimg, D)
grec = torch.zeros(r2.vb.n * r2.proj.rec_capacity * 10, device="cuda")
G.gs_joint_backward(ds2, r2.proj, r2.bins, r2.vb, r2.params, r2.images, gout, grec)
tgt = (r2.images.rgb + 0.05).contiguous()
t = G.SceneTrainer(G.DeviceScene(sc2), vs2[:2], tgt[:3 * 2 * hw].contiguous(),
                   target_feat=r2.images.feat[:2 * D * hw].contiguous(), optimizer="adam")
t.step()
torch.cuda.synchronize()
print("sanitize case ok", int(r.n_pairs()), int(r2.n_pairs()), int(r3.n_pairs()),
      int((mo.coarse >= 0).sum().item()))
