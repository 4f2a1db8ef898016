#!/bin/bash
# Warp-cooperative inverse square root on the latency paths: GPU parity of
# every path that uses it, then the per-epoch distill latency (C++ drop-in),
# the drop-in paver at config 1 (fresh Y / warm) and the default bench.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/wf
O=gpurun_out/wf
T="timeout -k 20"
$T 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
tail -2 $O/pytest_gpu.log
$T 600 oracle/_ref/distill_bench 1024 256 16 32 8 3 > $O/distill.txt 2>&1
cat $O/distill.txt
$T 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv oracle/_ref/distill_bench 32 256 4 32 2 1 > /dev/null 2>&1
python tools/ncu_table.py $O/launches.csv 2>&1 | tail -14
$T 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/bench_c2.json 2> $O/bench_c2.err
python -c "
import json; d=json.loads(open('$O/bench_c2.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['stages_ms']); print(json.dumps(d.get('e2e_dropin'))[:700])"
