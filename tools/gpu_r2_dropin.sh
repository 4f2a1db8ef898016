#!/bin/bash
# Drop-in path measurements: dropin_bench (paver on the std::map input, host
# roofline probes) at 2^26 and 2^20, distill_bench (ColdCryptoData epoch by
# epoch + SeBVer) on the drop-in and on the unmodified reference, then the
# drop-in tests (the reference's own suites on the drop-ins).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/r2_dropin.txt
: > $out
for r in 1 2; do
  timeout 600 oracle/_ref/dropin_bench 1 26 256 32 3 1 >> $out 2>&1
  timeout 300 oracle/_ref/dropin_bench 1 20 256 32 5 1 >> $out 2>&1
done
timeout 600 oracle/_ref/distill_bench 1024 256 16 32 8 3 >> $out 2>&1
timeout 900 oracle/_ref/distill_bench_ref 1024 256 16 32 8 1 >> $out 2>&1
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_distill.py -q -p no:cacheprovider > gpurun_out/r2_dropin_tests.log 2>&1
tail -3 gpurun_out/r2_dropin_tests.log >> $out
cat $out
