#!/bin/bash
# Round-2 check on the B200: new tests first, then the whole GPU suite, then
# the default bench, the self-launched 2-rank bench (gloo on the one GPU) and
# the 2-rank per-epoch / tamper modes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_dropin.py tests/test_gpu_multirank.py -x -q \
    > gpurun_out/r2_new_tests.log 2>&1
echo "new tests rc=$?" >> gpurun_out/r2_new_tests.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2_pytest_gpu.log 2>&1
echo "gpu suite rc=$?" >> gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err
timeout 900 python bench.py --gpus 2 --no-dropin --steps 5 > gpurun_out/r2_bench_w2.json 2> gpurun_out/r2_bench_w2.err
timeout 900 python bench.py --gpus 2 --mode tamper --log2n 24 --n2 1024 --n-u 64 --steps 3 --e2e-steps 1 \
    > gpurun_out/r2_bench_w2_tamper.json 2> gpurun_out/r2_bench_w2_tamper.err
timeout 900 python bench.py --gpus 2 --mode epoch --log2n 24 --n2 1024 --steps 3 --e2e-steps 1 \
    > gpurun_out/r2_bench_w2_epoch.json 2> gpurun_out/r2_bench_w2_epoch.err
for f in gpurun_out/r2_new_tests.log gpurun_out/r2_pytest_gpu.log; do tail -n 4 $f; done
for f in gpurun_out/r2_bench_*.json; do echo "== $f"; head -c 1500 $f; echo; done
