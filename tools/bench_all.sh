#!/bin/bash
# every configuration of BASELINE.md §4 (run on the GPU box; results under gpurun_out/all/)
cd $GRAFT_REPO_ROOT
O=gpurun_out/all; mkdir -p $O
for c in C2 C3 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --n1 > $O/bench_C4_n1.json 2> $O/bench_C4_n1.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --n4 > $O/bench_C4_n4.json 2> $O/bench_C4_n4.err
ls -la $O
