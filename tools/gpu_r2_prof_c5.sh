#!/bin/bash
# Config-5 step timeline: one distill step under torch.profiler (CUPTI kernel
# records incl. the C-ABI's own launches) after the timed region.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/c5
O=gpurun_out/c5
POSLO_PROFILE_STEP=$O/trace_c5.json timeout -k 20 900 python bench.py --mode tamper --n2 1024 --log2n 30 --tamper 1024 \
  --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --no-dropin > $O/bench_c5.json 2> $O/bench_c5.err
tail -c 300 $O/bench_c5.json; grep -A45 "profiled step" $O/bench_c5.err | head -60
gzip -f $O/trace_c5.json
echo done
