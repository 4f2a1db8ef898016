#!/bin/bash
# Round-2: comb-table build (one power chain per point, run-based radix-2^16
# fill with batch inversion) and the var-kernel warp rotation: parity tests,
# table kernel times from a launch list, var A/B (v3 = previous kernel), config 5.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/tab
O=gpurun_out/tab
T="timeout -k 20"
$T 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_multi.py tests/test_gpu_scale.py tests/test_gpu_fine.py -x -q -p no:cacheprovider > $O/tests.log 2>&1
tail -2 $O/tests.log
$T 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches_epoch.csv python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-dropin > /dev/null 2>&1
grep -i "table" $O/launches_epoch.csv | awk -F'","' '{print $5, $NF}' | head -12
cp paper_2506_08781_b200/libposlo_gpu.so /tmp/cur.so
for v in v3 cur v3 cur; do
  if [ $v = v3 ]; then cp variant_v3.so paper_2506_08781_b200/libposlo_gpu.so; else cp /tmp/cur.so paper_2506_08781_b200/libposlo_gpu.so; fi
  POSLO_PIPE_PIECES=1 $T 600 python bench.py --varlen --mode epoch --n2 1024 --log2n 24 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > $O/var_$v.json 2>&1
  python -c "
import json; d=json.loads(open('$O/var_$v.json').read().strip().splitlines()[-1]); r=d['roofline']
print('var', '$v', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['verdict'])"
done
cp /tmp/cur.so paper_2506_08781_b200/libposlo_gpu.so
$T 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 --no-dropin > $O/bench_c5.json 2>&1
python -c "
import json; d=json.loads(open('$O/bench_c5.json').read().strip().splitlines()[-1]); print('c5', d['value'], d['ms_per_step'], d['roofline']['stages_ms'])"
