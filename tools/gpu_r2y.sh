cd $GRAFT_REPO_ROOT
O=gpurun_out/r2y; mkdir -p $O
for rep in 1 2; do for v in main old; do
  if [ "$v" == "main" ]; then L=paper_2507_15683_b200/libgs.so; else L=paper_2507_15683_b200/_build/var_$v/libgs.so; fi
  for c in C4 C5; do
  GS_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v $c', round(d['stages_ms']['gs_bin_sort'],3), round(d['ms_per_step'],3))"
  done
done; done > $O/var.txt
cat $O/var.txt
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "keys or tiny or c3 or c4 or c5 or c2" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 2 $O/pytest.log
