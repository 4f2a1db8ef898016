#!/bin/bash
# Round-2 check on the B200: new tests first, then the whole GPU suite, then
# the drop-in bench at configs 1 and 2.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dropin.py tests/test_gpu_multirank.py -x -q \
    > gpurun_out/r2_new_tests.log 2>&1
echo "new tests rc=$?" >> gpurun_out/r2_new_tests.log
timeout 300 oracle/_ref/dropin_bench 1 20 256 32 5 1 > gpurun_out/r2_dropin_c1.json 2> gpurun_out/r2_dropin_c1.err
timeout 600 oracle/_ref/dropin_bench 1 26 256 32 3 1 > gpurun_out/r2_dropin_c2.json 2> gpurun_out/r2_dropin_c2.err
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2_pytest_gpu.log 2>&1
echo "gpu suite rc=$?" >> gpurun_out/r2_pytest_gpu.log
tail -3 gpurun_out/r2_new_tests.log gpurun_out/r2_pytest_gpu.log
cat gpurun_out/r2_dropin_c1.json gpurun_out/r2_dropin_c2.json
