#!/bin/bash
# Distill step (fused check + folds): golden CCD parity through the step, the
# reference's distiller suite on the C++ drop-in, per-epoch latency.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ds
O=gpurun_out/ds
T="timeout -k 20"
$T 900 python -m pytest tests/test_gpu_distill.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider > $O/tests.log 2>&1
tail -2 $O/tests.log
$T 600 oracle/_ref/distill_bench 1024 256 16 32 8 3 > $O/distill.txt 2>&1
cat $O/distill.txt
$T 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv oracle/_ref/distill_bench 32 256 4 32 2 1 > /dev/null 2>&1
python tools/ncu_table.py $O/launches.csv 2>&1 | tail -12
