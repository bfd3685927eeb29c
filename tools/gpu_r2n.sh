cd $GRAFT_REPO_ROOT
O=gpurun_out/r2n; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/l5.log 2>&1
for k in big_sort_kernel scatter_kernel count_kernel; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 --launch-count 1 -o $O/${k}_C5x8 python bench.py --config C5 --views 8 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/n_$k.log 2>&1
done
python - <<'PY' > $O/list_lengths.txt
import sys, numpy as np, torch
sys.path.insert(0, '.')
import synth, paper_2507_15683_b200 as G
sc, vs = synth.make_config("C5")
r = G.Renderer(G.DeviceScene(sc), vs[:8]); r.render(); torch.cuda.synchronize()
rg = r.bins.ranges.view(-1, 2).cpu().numpy().view(np.uint32).astype(np.int64)
L = rg[:, 1] - rg[:, 0]
print("tiles", len(L), "pairs", L.sum(), "mean", L.mean(), "p50", np.median(L), "p90", np.percentile(L, 90), "p99", np.percentile(L, 99), "max", L.max())
for a, b in [(0, 32), (33, 256), (257, 512), (513, 2048), (2049, 8192), (8193, 10**9)]:
    m = (L >= a) & (L <= b); print(f"len {a}-{b}: tiles {m.sum()} pairs {L[m].sum()}")
PY
ls -la $O
