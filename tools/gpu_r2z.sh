cd $GRAFT_REPO_ROOT
# A/B of build variants (args; "main" = in-tree lib) on C4 and C5 (raster stage ms, step ms),
# then the GPU suite on the in-tree lib
O=gpurun_out/r2z; mkdir -p $O
VARS="${@:-main}"
for rep in 1 2; do for v in $VARS; do
  if [ "$v" == "main" ]; then L=paper_2507_15683_b200/libgs.so; else L=paper_2507_15683_b200/_build/var_$v/libgs.so; fi
  for c in C4 C5; do
  GS_DEBUG=1 GS_LIB=$L timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>$O/err_${v}_$c | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v $c', round(d['stages_ms']['gs_rasterize'],3), round(d['stages_ms']['gs_project'],3), round(d['stages_ms']['gs_bin_sort'],3), round(d['ms_per_step'],3))"
  grep -m1 "rasterize<" $O/err_${v}_$c
  done
done; done > $O/var.txt 2>&1
cat $O/var.txt
[ -n "$NOTEST" ] && exit 0
export GS_PARITY_LOG=$O/parity_stats.jsonl
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -n 3 $O/pytest.log
