cd $GRAFT_REPO_ROOT
O=gpurun_out/r2j; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 600 python -m pytest tests/test_gpu_n1.py "tests/test_gpu_parity.py::test_square_and_tight_binning_keys_and_identical_images" -q > $O/pytest_n1.log 2>&1; echo "rc=$?" >> $O/pytest_n1.log
tail -n 3 $O/pytest_n1.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --n1 > $O/bench_C4_n1.json 2> $O/bench_C4_n1.err
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 300 python bench.py --config C3 --steps 20 --warmup 5 > $O/bench_C3.json 2> $O/bench_C3.err
tail -n 2 $O/*.err
