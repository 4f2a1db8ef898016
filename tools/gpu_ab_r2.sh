#!/bin/bash
# A/B of kernel build variants (variant_<name>.so at the repo root, built by
# tools/build_variant.sh) on config 2 (lean kernel) and config 4 (variable-
# length kernel), alternating base/variant twice; then the integer pipe probe.
#   LEAN="base l5v base l5v" VAR="base v5v base v5v" bash tools/gpu_ab_r2.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/base.so
out=gpurun_out/ab_r2.txt
: > $out
run() {  # variant mode
  v=$1; m=$2
  if [ $v = base ]; then cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so; else cp variant_$v.so paper_2506_08781_b200/libposlo_gpu.so; fi
  if [ $m = lean ]; then
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/ab_${m}_$v.log 2>&1
  elif [ $m = varp1 ]; then
    POSLO_PIPE_PIECES=1 timeout 600 python bench.py --varlen --mode epoch --n2 1024 --log2n 24 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/ab_${m}_$v.log 2>&1
  else
    timeout 600 python bench.py --varlen --mode epoch --n2 1024 --log2n 24 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/ab_${m}_$v.log 2>&1
  fi
  python -c "
import json; d=json.loads(open('gpurun_out/ab_${m}_$v.log').read().strip().splitlines()[-1]); r=d['roofline']
print('$m', '$v', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['verdict'], d['clocks']['sm_mhz'])" >> $out 2>&1
}
for v in ${LEAN:-}; do run $v lean; done
for v in ${VAR:-}; do run $v var; done
for v in ${VARP1:-}; do run $v varp1; done
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_logfile.py tests/test_gpu_scale.py -q -p no:cacheprovider -x -k "length or ragged or varlen or log or large or chunked" > gpurun_out/ab_r2_tests.log 2>&1
  tail -3 gpurun_out/ab_r2_tests.log >> $out
fi
if [ -n "${NCU_VAR:-}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_var -c 1 -o /tmp/kv \
    python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > /dev/null 2>&1
  ncu -i /tmp/kv.ncu-rep --page raw --csv > gpurun_out/ab_ncu_var_raw.csv 2>&1
  ncu -i /tmp/kv.ncu-rep --page source --csv --print-source sass > gpurun_out/ab_ncu_var_sass.csv 2>&1
fi
cp /tmp/base.so paper_2506_08781_b200/libposlo_gpu.so
if [ -n "${PIPE:-}" ]; then timeout 300 python tools/pipe_probe.py > gpurun_out/ab_r2_pipe.log 2>&1; fi
if [ -n "${TESTVAR:-}" ]; then cp variant_$TESTVAR.so paper_2506_08781_b200/libposlo_gpu.so; fi > gpurun_out/ab_r2_pipe.log 2>&1
cat $out
