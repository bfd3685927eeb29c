cd $GRAFT_REPO_ROOT
# the N > 1 step on one GPU: one-rank NCCL group with the per-chunk gather
O=gpurun_out/r2fg; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bench.py -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -3 $O/pytest.log
timeout 600 python bench.py --force-gather --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_C4_force_gather.json 2> $O/fg.err
python -c "
import json; d=json.loads(open('$O/bench_C4_force_gather.json').read().strip().splitlines()[-1]); print(json.dumps(d['sharded'])[:800]); print(d['value'], d['ms_per_step'])"
tail -3 $O/fg.err
timeout 600 python bench.py --force-gather --gather-transport f32 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_C4_force_gather_f32.json 2> $O/fg32.err
python -c "
import json; d=json.loads(open('$O/bench_C4_force_gather_f32.json').read().strip().splitlines()[-1]); print(json.dumps(d['sharded']['with_gather'])[:500]); print(d['value'], d['ms_per_step'])"
