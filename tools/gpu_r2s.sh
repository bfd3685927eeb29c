cd $GRAFT_REPO_ROOT
O=gpurun_out/r2s; mkdir -p $O
bash tools/var_bench.sh main se128n3 se64n6 > $O/var.txt 2>&1
cat $O/var.txt
timeout 600 python bench.py --config C5 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --config C2 --steps 300 --warmup 20 --no-e2e --no-cpu-baseline > $O/bench_C2.json 2> $O/bench_C2.err
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
