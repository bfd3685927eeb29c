cd $GRAFT_REPO_ROOT
# usage: bash tools/var_bench.sh v1 v2 ... (variants under paper_2507_15683_b200/_build/var_*; "main" = in-tree lib)
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" == "main" ]; then L=paper_2507_15683_b200/libgs.so; else L=paper_2507_15683_b200/_build/var_$v/libgs.so; fi
  GS_DEBUG=1 GS_LIB=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/err_$v | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['stages_ms']['gs_rasterize'],3), round(d['ms_per_step'],3))"
  grep "rasterize<32" /tmp/err_$v | head -1
done; done
