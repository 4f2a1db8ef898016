#!/bin/bash
# ncu --set full capture of the lean kernel (config 2) after moving every
# addition to the FMA pipe: raw metrics + per-SASS executed counts, and the
# default-bench launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/l5
O=gpurun_out/l5
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_l32r -c 1 -o /tmp/kl \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > $O/ncu_lean.log 2>&1
ncu -i /tmp/kl.ncu-rep --page raw --csv > $O/ncu_k_hash_s1_l32r_raw.csv 2>&1
ncu -i /tmp/kl.ncu-rep --page source --csv --print-source sass > $O/ncu_k_hash_s1_l32r_sass.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > /dev/null 2>&1
ls -la $O
