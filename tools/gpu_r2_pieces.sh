#!/bin/bash
# Epoch-piece pipelining A/B (POSLO_PIPE_PIECES=1 vs the default 8 pieces on
# two alternating hash streams) on config 4 (varlen) and config 3 (lean,
# 2^28), then the whole GPU suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/pieces.txt
: > $out
one() {  # tag pieces args...
  tag=$1; pc=$2; shift 2
  POSLO_PIPE_PIECES=$pc timeout 600 python bench.py "$@" --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/pieces_$tag.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/pieces_$tag.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$tag', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['value'], d['verdict'])" >> $out 2>&1
}
for rep in 1 2; do
  one c4_p8 8 --varlen --mode epoch --n2 1024 --log2n 24 --steps 5 --warmup 3
  one c4_p1 1 --varlen --mode epoch --n2 1024 --log2n 24 --steps 5 --warmup 3
  one c3_p8 8 --mode epoch --n2 1024 --log2n 28 --steps 5 --warmup 3
  one c3_p1 1 --mode epoch --n2 1024 --log2n 28 --steps 5 --warmup 3
  one c5_p8 8 --mode tamper --n2 1024 --log2n 26 --n-u 1024 --steps 3 --warmup 3
  one c5_p1 1 --mode tamper --n2 1024 --log2n 26 --n-u 1024 --steps 3 --warmup 3
done
cat $out
if [ -n "${SUITE:-}" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pieces_pytest_gpu.log 2>&1
  tail -3 gpurun_out/pieces_pytest_gpu.log
fi
