#!/bin/bash
# A/B of the check / decode kernels' occupancy (variant_<name>.so, tools/build_variant.sh)
# on config 5 (2^30, per-epoch checks + umbrella folds) and config 3: ms/step and stages.
#   VARS="base m5 base m5" bash tools/gpu_ab_checks.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/abc
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
out=gpurun_out/abc/ab_checks.txt
: > $out
for v in ${VARS:-base}; do
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  for m in tamper epoch; do
    timeout 600 python bench.py --mode $m --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > gpurun_out/abc/${m}_$v.log 2>&1
    python -c "
import json; d=json.loads(open('gpurun_out/abc/${m}_$v.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$m', '$v', d['ms_per_step'], r['stages_ms'], d['verdict'])" >> $out 2>&1
  done
done
cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so
cat $out
