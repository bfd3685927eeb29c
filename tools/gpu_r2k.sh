cd $GRAFT_REPO_ROOT
O=gpurun_out/r2k; mkdir -p $O
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 600 python -m pytest tests/test_gpu_n1.py -q > $O/pytest_n1.log 2>&1; echo "rc=$?" >> $O/pytest_n1.log
tail -n 2 $O/pytest_n1.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --n1 > $O/bench_C4_n1.json 2> $O/bench_C4_n1.err
# the whole GPU suite and the sanitize case on the bounds-checked build (GS_CHECKS)
GS_LIB=$GRAFT_REPO_ROOT/paper_2507_15683_b200/_build/checks/libgs.so timeout 300 python tools/sanitize_case.py > $O/checks_case.log 2>&1; echo "rc=$?" >> $O/checks_case.log
GS_LIB=$GRAFT_REPO_ROOT/paper_2507_15683_b200/_build/checks/libgs.so timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_checks.log 2>&1; echo "rc=$?" >> $O/pytest_checks.log
tail -n 3 $O/checks_case.log $O/pytest_checks.log
