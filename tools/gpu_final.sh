#!/bin/bash
# Round measurement set (run on the GPU box): bench lines for every config and
# extension, the ncu launch list of the default bench command, and a --set full
# capture of the dominant kernel.  Results under gpurun_out/$1.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-final}; mkdir -p $O
timeout 900 python bench.py > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python bench.py --impl reference > $O/bench_C4_reference.json 2> $O/bench_C4_reference.err
timeout 600 python bench.py --config C2 --steps 300 --warmup 20 > $O/bench_C2.json 2> $O/bench_C2.err
timeout 600 python bench.py --config C3 --steps 100 --warmup 10 > $O/bench_C3.json 2> $O/bench_C3.err
timeout 900 python bench.py --config C5 --steps 10 --warmup 3 > $O/bench_C5.json 2> $O/bench_C5.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --n1 > $O/bench_C4_n1.json 2> $O/bench_C4_n1.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --n4 > $O/bench_C4_n4.json 2> $O/bench_C4_n4.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --n2 --refine 32 > $O/bench_C4_n2.json 2> $O/bench_C4_n2.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --sharded > $O/bench_C4_sharded.json 2> $O/bench_C4_sharded.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --force-gather > $O/bench_C4_force_gather.json 2> $O/bench_C4_force_gather.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C5.csv python bench.py --config C5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch_C5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^rasterize -c 1 -o $O/full_raster_C4x16 python bench.py --views 16 --profile-steps 1 --no-e2e --no-cpu-baseline > $O/ncu_full.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
[ -n "$WITH_TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log; }
ls -la $O
