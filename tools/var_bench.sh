cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in p64c64 p500c64 p500c200 p1000c500 p200c0; do
  GS_LIB=paper_2507_15683_b200/_build/var_$v/libgs.so python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read());print('$v', round(d['stages_ms']['gs_rasterize'],3))"
done; done
