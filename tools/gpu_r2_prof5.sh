#!/bin/bash
# Host-side profile of the config-5 bench step (cProfile) and the fresh-Y cost.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/p5
O=gpurun_out/p5
T="timeout -k 20"
$T 900 python -m cProfile -o /tmp/c5.prof bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 --steps 3 --warmup 2 --e2e-steps 0 --no-dropin --no-cpu-baseline > $O/c5.json 2>&1
python -c "
import pstats; p=pstats.Stats('/tmp/c5.prof'); p.sort_stats('tottime').print_stats(25)" > $O/c5_prof.txt 2>&1
head -60 $O/c5_prof.txt
$T 300 oracle/_ref/dropin_bench 1 20 256 32 5 1 > $O/dropin20.txt 2>&1
$T 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "comb or group or config3 or config5 or table or check" > $O/tests.log 2>&1
tail -2 $O/tests.log
cat $O/dropin20.txt
