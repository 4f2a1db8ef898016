#!/bin/bash
# A/B: per-epoch radix-2^16 checks against R-hat decoded during hashing
# (default) vs no square root per check (POSLO_CHECK16=sqrt: combs -> batched
# inversion -> encode(P) == R-hat by squares), config 3 at 2^30; launch list at 2^28.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/abs
out=gpurun_out/abs/ab.txt
: > $out
for rep in 1 2; do
  for v in "decode:POSLO_CHECK16=decode" "sqrt:POSLO_CHECK16=sqrt"; do
    n=${v%%:*}; e=${v#*:}
    env $e timeout 600 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > gpurun_out/abs/c3_$n.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/abs/c3_$n.log').read().strip().splitlines()[-1]); r=d['roofline']
print('epoch', '$n', d['ms_per_step'], r['stages_ms'], d['verdict'])" >> $out 2>&1
  done
done
for v in "decode:POSLO_CHECK16=decode" "sqrt:POSLO_CHECK16=sqrt"; do
  n=${v%%:*}; e=${v#*:}
  env $e POSLO_PIPE_PIECES=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_check|k_decode|k_batch_invert" --csv --log-file gpurun_out/abs/launch_$n.csv python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-dropin > /dev/null 2>&1
  python tools/ncu_table.py gpurun_out/abs/launch_$n.csv 2>&1 | tail -8 >> $out
done
cat $out
