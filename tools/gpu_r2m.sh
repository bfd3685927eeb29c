cd $GRAFT_REPO_ROOT
O=gpurun_out/r2m; mkdir -p $O
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/*.err $O/pytest.log
