#!/bin/bash
# Round-2 ceiling evidence: ncu --set full captures of the two suite-1 hash
# kernels (config 2 lean kernel, config 4 variable-length kernel) exported as
# raw metrics and as per-SASS-instruction executed counts (source page), for
# the executed-ops-per-entry accounting in DESIGN.md; plus the integer pipe
# probe under the same clocks.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python tools/pipe_probe.py > gpurun_out/r2_pipe_probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_l32r -c 1 -o /tmp/kl \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/r2_ncu_lean.log 2>&1
ncu -i /tmp/kl.ncu-rep --page raw --csv > gpurun_out/r2_ncu_lean_raw.csv 2>&1
ncu -i /tmp/kl.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_ncu_lean_sass.csv 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_s1_var -c 1 -o /tmp/kv \
    python bench.py --varlen --mode epoch --n2 1024 --log2n 22 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/r2_ncu_var.log 2>&1
ncu -i /tmp/kv.ncu-rep --page raw --csv > gpurun_out/r2_ncu_var_raw.csv 2>&1
ncu -i /tmp/kv.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_ncu_var_sass.csv 2>&1
for f in gpurun_out/r2_ncu_*; do echo "$f $(wc -c < $f)"; done
