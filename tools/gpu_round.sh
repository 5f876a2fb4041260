#!/bin/bash
# One GPU session: tests, smoke, bench (both arms), ncu launch list + full capture of the attention kernel.
# Usage (under gpurun):  bash tools/gpu_round.sh <tag> [quick]
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/smi.csv 2>&1
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
SPA_PARITY_LOG=$OUT/parity_fullsize.jsonl timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
timeout 600 python bench.py > $OUT/bench.jsonl 2> $OUT/bench.err
timeout 600 python bench.py --spawn --steps 5 --no-cpu-baseline > $OUT/bench_spawn1.jsonl 2> $OUT/bench_spawn1.err
timeout 400 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.jsonl 2> $OUT/bench_reference.err
if [ "$2" != "quick" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_fwd|copy_runs|qkv|lse" --csv \
    --log-file $OUT/launches_bench.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 \
    -o $OUT/prof_attn_hy544p python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_hy544p.log 2>&1
fi
ls -la $OUT
