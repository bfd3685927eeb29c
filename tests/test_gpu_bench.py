"""bench.py's code paths on the GPU at small sizes (the driver runs the full-size
default): the JSON contract keys, the sharded (multi-GPU) step at N = 1 with
its chunk renderers writing into the gather send buffers, the CUDA-graph
timing of small batches and both e2e transports."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def _contract(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "step_ms"):
        assert k in d, k
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1
    assert d["clocks"]["samples"] > 0


def test_bench_sharded_step_and_e2e_transports():
    d = _bench("--config", "C4", "--scale", "0.02", "--views", "16", "--steps", "3", "--warmup", "3", "--sharded",
               "--chunk", "4", "--no-cpu-baseline")
    _contract(d)
    sh = d["sharded"]
    assert sh["chunks"] == 4 and sh["chunks_rendered"] == 4 and sum(sh["views_per_rank"]) == 16
    assert sh["render_only"]["value"] > 0
    e = d["e2e"]
    assert e["d2h_bytes_per_step"] == 11 * d["counts"]["pixels"]
    assert sorted(o["d2h_bytes_per_step"] for o in e["other_transports"]) == [12 * d["counts"]["pixels"],
                                                                           20 * d["counts"]["pixels"]]
    assert set(d["stage_rooflines"]) == {"gs_project", "gs_bin_sort"}


def test_bench_small_batch_graph_timing():
    d = _bench("--config", "C2", "--scale", "0.25", "--steps", "20", "--warmup", "3", "--no-cpu-baseline",
               "--e2e-transport", "f32")
    _contract(d)
    assert d["graph"]["ms_per_step"] > 0
    assert d["e2e"]["d2h_bytes_per_step"] == 20 * d["counts"]["pixels"]


def test_bench_force_gather_one_rank_nccl():
    """The N > 1 step on one GPU: sharded chunks, one NCCL all_gather_into_tensor per chunk
    on the comm stream (a one-rank group), the received planes equal to the rendered ones."""
    hw = 1024 * 768
    for transport, nbytes in (("dense11", 4 * ((11 * 4 * hw + 15) // 16 * 16)), ("f32", 4 * 5 * 4 * hw * 4)):
        d = _bench("--config", "C4", "--scale", "0.02", "--views", "16", "--steps", "3", "--warmup", "3",
                   "--force-gather", "--gather-transport", transport, "--chunk", "4", "--no-cpu-baseline", "--no-e2e")
        _contract(d)
        wg = d["sharded"]["with_gather"]
        assert wg is not None and wg["received_equals_sent"] is True
        assert wg["bytes_received_per_rank_per_step"] == nbytes

