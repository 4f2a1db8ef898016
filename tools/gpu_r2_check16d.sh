#!/bin/bash
# A/B of the radix-2^16 per-epoch checks (round 2, before the square-root-free default): thread per check against decoded
# R-hat (k_check_thread16d, default) vs encoding compare (POSLO_CHECK16=encode)
# for config 3, and distillation (config 5) with the decoded compare.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c16
O=gpurun_out/c16
T="timeout -k 20"
$T 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "batched_epoch_checks_large or resident or radix256" > $O/tests.log 2>&1
tail -2 $O/tests.log
for v in "dec:POSLO_CHECK16=decode" "enc:POSLO_CHECK16=encode"; do
  n=${v%%:*}; e=${v#*:}
  env $e $T 900 python bench.py --mode epoch --n2 1024 --log2n 30 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > $O/c3_$n.json 2> $O/c3_$n.err
done
$T 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > $O/c5_dec.json 2> $O/c5_dec.err
python - <<'PY'
import json
for f in ['c3_dec','c3_enc','c5_dec']:
    try:
        d=json.loads(open(f'gpurun_out/c16/{f}.json').read().strip().splitlines()[-1])
        print(f, d['value'], d['ms_per_step'], d['roofline']['stages_ms'])
    except Exception as e:
        print(f, 'ERR', e, open(f'gpurun_out/c16/{f}.err').read()[-800:])
PY
POSLO_CHECK16=decode ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_check_thread16 --csv --log-file $O/launch_c3.csv python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-dropin > /dev/null 2>&1
POSLO_CHECK16=encode ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_check_thread16 --csv --log-file $O/launch_c3_enc.csv python bench.py --mode epoch --n2 1024 --log2n 28 --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-dropin > /dev/null 2>&1
grep -h "k_check\|k_decode" $O/launch_c3.csv $O/launch_c3_enc.csv | awk -F'","' '{print $5, $NF}' | sort | uniq -c | head
echo done
