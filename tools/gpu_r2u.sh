cd $GRAFT_REPO_ROOT
O=gpurun_out/r2u; mkdir -p $O
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pose.py tests/test_gpu_n2.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
for f in bench_C4 bench_C5; do python -c "import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['stages_ms'])"; done
