cd $GRAFT_REPO_ROOT
# A/B of the 4-entry walk (main) vs GS_WALK4=0 (now4) on C4 and C5, then the GPU suite
O=gpurun_out/r2z; mkdir -p $O
for rep in 1 2; do for v in main now4; do
  if [ "$v" == "main" ]; then L=paper_2507_15683_b200/libgs.so; else L=paper_2507_15683_b200/_build/var_$v/libgs.so; fi
  for c in C4 C5; do
  GS_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v $c', round(d['stages_ms']['gs_rasterize'],3), round(d['ms_per_step'],3))"
  done
done; done > $O/var.txt
cat $O/var.txt
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
