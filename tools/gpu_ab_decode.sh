#!/bin/bash
# A/B: R-hat decode queued behind the seed kernel (beside the hashing, default)
# vs before the seeds (POSLO_DECODE_EARLY=1), configs 3 and 5 at 2^30.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/abd
out=gpurun_out/abd/ab.txt
: > $out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_distill.py tests/test_gpu_multi.py -x -q -p no:cacheprovider -k "large or resident or distill or determinism or byte_identical" 2>&1 | tail -1 >> $out
for rep in 1 2; do
  for v in "late:" "early:POSLO_DECODE_EARLY=1"; do
    n=${v%%:*}; e=${v#*:}
    for m in epoch tamper; do
      env $e timeout 600 python bench.py --mode $m --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > gpurun_out/abd/${m}_$n.log 2>&1
      python -c "
import json; d=json.loads(open('gpurun_out/abd/${m}_$n.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$m', '$n', d['ms_per_step'], r['stages_ms'], d['verdict'])" >> $out 2>&1
    done
  done
done
cat $out
