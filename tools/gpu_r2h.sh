cd $GRAFT_REPO_ROOT
O=gpurun_out/r2h; mkdir -p $O
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 400 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_n1.py tests/test_gpu_n4.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
