cd $GRAFT_REPO_ROOT
O=gpurun_out/r2p; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_n4.py tests/test_gpu_bench.py -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --n4 > $O/bench_C4_n4.json 2> $O/bench_C4_n4.err
