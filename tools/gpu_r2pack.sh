cd $GRAFT_REPO_ROOT
# dense11 transport: parity tests, bench contract tests, C4 + C5 bench lines
O=gpurun_out/r2pack; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench.py -q -x -k "pack or bench" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
python - <<'PY'
import json
for c in ("C4", "C5"):
    d = json.loads(open(f"gpurun_out/r2pack/bench_{c}.json").read().strip().splitlines()[-1])
    e = d["e2e"]
    print(c, round(d["value"], 1), round(d["ms_per_step"], 3), "e2e", round(e["value"], 1), e["transport"][:8],
          [(round(o["value"], 1), o["transport"][:8]) for o in e["other_transports"]])
PY
