cd $GRAFT_REPO_ROOT
O=gpurun_out/r2e; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or tiny or contraction or empty or culled or c2_full or c4_batch" > $O/pytest_quick.log 2>&1; echo "rc=$?" >> $O/pytest_quick.log
tail -n 3 $O/pytest_quick.log
GS_DEBUG=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_new.json 2> $O/bench_new.err
GS_RASTER_LEGACY=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_legacy.json 2> $O/bench_legacy.err
GS_DEBUG=1 timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5_new.json 2> $O/bench_C5_new.err
GS_RASTER_LEGACY=1 timeout 300 python bench.py --config C5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_C5_legacy.json 2> $O/bench_C5_legacy.err
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_all.log 2>&1; echo "rc=$?" >> $O/pytest_all.log
tail -n 3 $O/pytest_all.log
