#!/bin/bash
# compute-sanitizer over the smoke path and a slice of the GPU parity suite:
# memcheck (out-of-bounds / misaligned / leaks of device memory), racecheck
# (shared-memory hazards) and synccheck (illegal barriers) on the kernels the
# product path launches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/san
O=gpurun_out/san
S="compute-sanitizer --print-limit 20 --error-exitcode 9"
T="timeout -k 20"
$T 900 $S --tool memcheck python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/memcheck_smoke.log 2>&1; echo "memcheck smoke rc=$?"
$T 900 $S --tool racecheck python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/racecheck_smoke.log 2>&1; echo "racecheck smoke rc=$?"
$T 900 $S --tool synccheck python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/synccheck_smoke.log 2>&1; echo "synccheck smoke rc=$?"
$T 1500 $S --tool memcheck python -m pytest tests/test_gpu_parity.py tests/test_gpu_distill.py -x -q -p no:cacheprovider \
   -k "golden or stream or radix256 or commit_check or batched_epoch_checks_large or length or ragged or resident or distill or segfold or fold or paver" > $O/memcheck_parity.log 2>&1; echo "memcheck parity rc=$?"
tail -3 $O/memcheck_parity.log
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY" $O/*.log
$T 900 $S --tool racecheck python -m pytest tests/test_gpu_distill.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "distill or commit_check or segfold" > $O/racecheck_distill.log 2>&1; echo "racecheck distill rc=$?"
$T 900 $S --tool synccheck python -m pytest tests/test_gpu_distill.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "distill or commit_check or segfold" > $O/synccheck_distill.log 2>&1; echo "synccheck distill rc=$?"
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|passed\|failed" $O/racecheck_distill.log $O/synccheck_distill.log
# self-check: memcheck must flag a deliberate out-of-bounds write in a static-cudart .so loaded by Python
$T 300 $S --tool memcheck python -c "import ctypes; print('probe rc', ctypes.CDLL('tools/san_probe/liboob_probe.so').oob_probe())" > $O/memcheck_selfcheck.log 2>&1; echo "memcheck self-check rc=$? (9 = error found, as intended)"
grep -m3 "Invalid __global__ write\|ERROR SUMMARY" $O/memcheck_selfcheck.log
