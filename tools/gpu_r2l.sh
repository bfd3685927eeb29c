cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l; mkdir -p $O
timeout 600 python bench.py --config C2 --steps 300 --warmup 20 --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C3 --steps 100 --warmup 10 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C5.json 2> $O/bench_C5.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4.json 2> $O/bench_C4.err
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "c5 or C5" > $O/pytest_c5.log 2>&1; echo "rc=$?" >> $O/pytest_c5.log
tail -n 2 $O/*.err $O/pytest_c5.log
