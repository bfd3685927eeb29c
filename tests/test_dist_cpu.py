"""Multi-process host logic of the pose-sharded path on CPU (gloo, world size 2):
view sharding (contiguous / LPT over pre-pass costs), the chunked gather of
dist.ChunkedGather (render straight into per-chunk send buffers, one collective
per chunk) and the assembly back to global view order.  Each rank "renders" its
shard with the CPU oracle (test infrastructure), so the gathered planes must
equal a single-process render bit for bit."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_15683_b200 import dist as GD  # noqa: E402


def test_shard_views_partition_properties():
    for n in (1, 7, 256):
        for world in (1, 2, 3, 8):
            shards = [GD.shard_views(n, world, r) for r in range(world)]
            flat = sorted(i for s in shards for i in s)
            assert flat == list(range(n))
            sizes = [len(s) for s in shards]
            assert max(sizes) - min(sizes) <= 1
            assert all(s == sorted(s) and (not s or s == list(range(s[0], s[-1] + 1))) for s in shards)


def test_cost_balanced_sharding():
    rng = np.random.default_rng(0)
    costs = rng.lognormal(0, 1, 256)
    for world in (2, 4, 8):
        shards = [GD.shard_views(256, world, r, costs) for r in range(world)]
        assert sorted(i for s in shards for i in s) == list(range(256))
        loads = [costs[s].sum() for s in shards]
        # LPT bound: max load <= mean + max single cost
        assert max(loads) <= np.mean(loads) + costs.max() + 1e-9
        assert shards == [GD.shard_views(256, world, r, costs) for r in range(world)]   # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _views(n_views):
    import synth
    return [synth.make_view(np.eye(3), [0.05 * i, -0.03 * i, 0.0], 48, 48, 23.5, 15.5, 48, 32) for i in range(n_views)]


def _oracle_render_chunk(cg, views, scene):
    """Fill chunk k's send buffer in the gs_images planar layout (what the GPU
    Renderer writes through out_planes): view j of the chunk at RGB 3 j hw,
    Dz / A at j hw."""
    import oracle

    def render(k):
        rgb, dep, alp = cg.planes(k)
        hw = cg.hw
        for j, i in enumerate(cg.chunk_views(k)):
            r = oracle.render(scene, views[i])
            rgb[3 * j * hw:3 * (j + 1) * hw] = torch.from_numpy(r["rgb"].reshape(-1))
            dep[j * hw:(j + 1) * hw] = torch.from_numpy(r["depth"].reshape(-1))
            alp[j * hw:(j + 1) * hw] = torch.from_numpy(r["alpha"].reshape(-1))
    return render


def _worker(rank, world, port, n_views, use_costs, chunk, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import synth
    scene = synth.box_v1(300, seed=9)
    views = _views(n_views)
    costs = [float(i % 3 + 1) for i in range(n_views)] if use_costs else None
    cg = GD.ChunkedGather(n_views, 48 * 32, world, rank, chunk, costs)
    assert cg.n_chunks == -(-max(len(s) for s in cg.shards) // chunk)
    render = _oracle_render_chunk(cg, views, scene)
    for _ in range(2):                       # two steps reuse the send / receive buffers
        cg.step(render)
    assert cg.check_own_slot()               # this rank's slot of every receive buffer = its send buffer
    full = cg.assemble()
    if rank == 0:
        torch.save(full, out_path)
    dist.barrier()
    dist.destroy_process_group()


def _single_process(n_views):
    import oracle
    import synth
    scene = synth.box_v1(300, seed=9)
    return [oracle.render(scene, v) for v in _views(n_views)]


@pytest.mark.parametrize("use_costs,chunk", [(False, 2), (True, 2), (True, 1), (False, 8)])
def test_gloo_chunked_gather_equals_single_process(tmp_path, use_costs, chunk):
    """dist.ChunkedGather (the bench's multi-GPU step: per-chunk render straight
    into the send buffer, one all_gather per chunk) at world size 2 assembles
    planes bit-identical to a single-process render."""
    import oracle
    oracle.build()
    n_views = 5
    out = str(tmp_path / "gathered.pt")
    mp.spawn(_worker, args=(2, _free_port(), n_views, use_costs, chunk, out), nprocs=2, join=True)
    full = torch.load(out)
    for i, r in enumerate(_single_process(n_views)):
        assert np.array_equal(full[i, 0:3].numpy(), r["rgb"].reshape(3, -1))
        assert np.array_equal(full[i, 3].numpy(), r["depth"].reshape(-1))
        assert np.array_equal(full[i, 4].numpy(), r["alpha"].reshape(-1))


def test_chunked_gather_world_one_is_the_render():
    import synth
    scene = synth.box_v1(300, seed=9)
    views = _views(3)
    cg = GD.ChunkedGather(3, 48 * 32, 1, 0, 2)
    cg.step(_oracle_render_chunk(cg, views, scene))
    full = cg.assemble()
    for i, r in enumerate(_single_process(3)):
        assert np.array_equal(full[i, 4].numpy(), r["alpha"].reshape(-1))


def test_view_costs_from_ranges():
    # two views of 3 and 2 tiles; lower-bound ranges (empty tiles start = end)
    ranges = torch.tensor([0, 4, 4, 4, 4, 9, 9, 10, 10, 10], dtype=torch.int32)
    assert GD.view_costs_from_ranges(ranges, [0, 3], [3, 2]) == [9.0, 1.0]


def test_bench_reference_arm_json():
    """bench.py --impl reference prints one JSON line with the contract keys."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "Mpixels/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0


def test_equal_size_runs_groups_consecutive_views():
    """SceneTrainer / bench --n4 call gs_dssim_grad once per run of consecutive
    equal-size views (their RGB planes are contiguous)."""
    from types import SimpleNamespace as V
    from paper_2507_15683_b200.pipeline import equal_size_runs
    vs = [V(height=768, width=1024)] * 3 + [V(height=480, width=640), V(height=768, width=1024)]
    assert equal_size_runs(vs) == [(0, 3, 768, 1024), (3, 1, 480, 640), (4, 1, 768, 1024)]
    assert equal_size_runs([]) == []
    assert len(equal_size_runs([V(height=8, width=8)] * 256)) == 1
    # bounded calls (gs_dssim_grad workspace): 256 views in groups of <= 64
    assert equal_size_runs([V(height=8, width=8)] * 130, max_views=64) == [(0, 64, 8, 8), (64, 64, 8, 8), (128, 2, 8, 8)]


def _worker_one(rank, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=0, world_size=1)
    import synth
    scene = synth.box_v1(300, seed=9)
    views = _views(3)
    cg = GD.ChunkedGather(3, 48 * 32, 1, 0, 2, always_gather=True)
    cg.step(_oracle_render_chunk(cg, views, scene))
    torch.save({"ok": cg.check_own_slot(), "recv": [t.clone() for t in cg.recv]}, out_path)
    dist.destroy_process_group()


def test_always_gather_one_rank_group(tmp_path):
    """--force-gather's host path: a one-rank group still issues the per-chunk collective
    (bench.py uses it to exercise the N > 1 step on one GPU); the receive buffers hold the
    rendered planes bit for bit."""
    import oracle
    oracle.build()
    out = str(tmp_path / "one.pt")
    mp.spawn(_worker_one, args=(_free_port(), out), nprocs=1, join=True)
    d = torch.load(out)
    assert d["ok"]
    r = _single_process(3)
    np.testing.assert_array_equal(d["recv"][0][4 * 2 * 48 * 32:4 * 2 * 48 * 32 + 48 * 32].numpy(),
                                  r[0]["alpha"].reshape(-1))


def _pack_dense11_np(rgb, depth, alpha):
    """Test-side writer of the GS_PACK_DENSE11 layout (include/gs.h) for the gloo test."""
    tp = depth.size
    out = np.zeros(11 * tp, np.uint8)
    out[:6 * tp] = rgb.reshape(3, tp).astype(np.float16).reshape(-1).view(np.uint8)
    a = np.rint(np.clip(alpha, 0, 1).astype(np.float32) * np.float32(65535)).astype(np.uint16)
    out[6 * tp:8 * tp] = a.view(np.uint8)
    d = (depth.astype(np.float32).view(np.uint32) + np.uint32(0x80)) >> np.uint32(8)
    b = np.stack([d & 0xFF, (d >> 8) & 0xFF, (d >> 16) & 0xFF], axis=1).astype(np.uint8)
    out[8 * tp:11 * tp] = b.reshape(-1)
    return out


def _worker_dense(rank, world, port, n_views, chunk, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    scene = synth.box_v1(300, seed=9)
    views = _views(n_views)
    hw = 48 * 32
    cg = GD.ChunkedGather(n_views, hw, world, rank, chunk, payload="dense11")

    def render(k):
        idx = cg.chunk_views(k)
        if not idx:
            return
        rs = [oracle.render(scene, views[i]) for i in idx]
        rgb = np.concatenate([r["rgb"].reshape(3, -1) for r in rs], axis=1)
        dep = np.concatenate([r["depth"].reshape(-1) for r in rs])
        alp = np.concatenate([r["alpha"].reshape(-1) for r in rs])
        b = _pack_dense11_np(rgb, dep, alp)
        cg.send[k][:b.size] = torch.from_numpy(b)

    cg.step(render)
    assert cg.check_own_slot()
    if rank == 0:
        torch.save({"recv": [t.clone() for t in cg.recv], "shards": cg.shards, "chunk": cg.chunk}, out_path)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_chunked_gather_dense11_payload(tmp_path):
    """The bench's default N > 1 payload: each rank packs its chunk's planes as GS_PACK_DENSE11
    bytes and gathers them; rank 0 decodes every rank's slot (unpack_dense11) to the oracle's
    planes within the format's rounding (fp16 RGB exact-rounded, A <= 0.5/65535, depth
    <= 2^-16 relative)."""
    import oracle
    oracle.build()
    n_views, chunk, hw = 5, 2, 48 * 32
    out = str(tmp_path / "dense.pt")
    mp.spawn(_worker_dense, args=(2, _free_port(), n_views, chunk, out), nprocs=2, join=True)
    d = torch.load(out)
    ref = _single_process(n_views)
    n = d["recv"][0].numel() // 2
    seen = 0
    for k, rv in enumerate(d["recv"]):
        for r in range(2):
            idx = d["shards"][r][k * d["chunk"]:(k + 1) * d["chunk"]]
            if not idx:
                continue
            rgb, dep, alp = GD_unpack(rv[r * n:(r + 1) * n].numpy(), len(idx) * hw)
            for j, g in enumerate(idx):
                sl = slice(j * hw, (j + 1) * hw)
                np.testing.assert_array_equal(rgb[:, sl], ref[g]["rgb"].reshape(3, -1).astype(np.float16).astype(np.float32))
                assert np.abs(alp[sl] - ref[g]["alpha"].reshape(-1)).max() <= 0.5 / 65535 + 1e-7
                z = ref[g]["depth"].reshape(-1).astype(np.float64)
                assert (np.abs(dep[sl].astype(np.float64) - z) <= z * 2.0 ** -16 + 1e-30).all()
                seen += 1
    assert seen == n_views


def GD_unpack(buf, tp):
    from paper_2507_15683_b200.gs import unpack_dense11
    return unpack_dense11(buf, tp)

