cd $GRAFT_REPO_ROOT
O=gpurun_out/r2o; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/l4.log 2>&1
