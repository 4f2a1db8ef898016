#!/bin/bash
# Round-2 re-entry check on one B200: smoke, the whole GPU suite, default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/re
O=gpurun_out/re
T="timeout -k 20"
$T 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
tail -1 $O/smoke.log
$T 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
$T 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
tail -c 600 $O/bench_c2.json
echo done
