#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ds2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_distill_step -s 4 -c 1 -o /tmp/kds oracle/_ref/distill_bench 32 256 4 32 2 1 > gpurun_out/ds2/ncu.log 2>&1
ncu -i /tmp/kds.ncu-rep --page raw --csv > gpurun_out/ds2/raw.csv 2>&1
ncu -i /tmp/kds.ncu-rep --page source --csv --print-source sass > gpurun_out/ds2/sass.csv 2>&1
ncu -i /tmp/kds.ncu-rep --page source --csv --print-source cuda > gpurun_out/ds2/cuda.csv 2>&1
ls -la gpurun_out/ds2
