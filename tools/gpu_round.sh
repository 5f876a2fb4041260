#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list + full capture of the attention kernel.
# Usage (under gpurun):  bash tools/gpu_round.sh <tag>
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err
timeout 400 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
timeout 600 python bench.py --workload hy544p129f --steps 5 --no-cpu-baseline > $OUT/bench_hy544p.jsonl 2>> $OUT/bench.err
timeout 300 python tools/attn_perf.py --sdpa > $OUT/attn_perf.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd|copy_runs" --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o $OUT/prof_attn_osp python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_osp.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 \
    -o $OUT/prof_attn_hy720p8 python tools/attn_perf.py --shapes hy720p8 --reps 1 > $OUT/ncu_hy.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:copy_runs -s 4 -c 1 \
    -o $OUT/prof_copy python tools/sp_perf.py --workload osp480p93f --stages 1 --reps 1 > $OUT/ncu_copy.log 2>&1
timeout 400 python tools/sp_perf.py --stages 1,3,24 > $OUT/sp_perf.jsonl 2>&1
ls -la $OUT
