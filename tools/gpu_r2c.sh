cd $GRAFT_REPO_ROOT
O=gpurun_out/r2c; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 600 python -m pytest tests/test_gpu_alpha_band.py "tests/test_gpu_parity.py::test_c1_features_D8" -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --steps 5 --warmup 3 --sharded --no-e2e --no-cpu-baseline > $O/bench_C4_sharded.json 2> $O/bench_C4_sharded.err
tail -3 $O/*.err
