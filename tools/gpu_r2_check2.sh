#!/bin/bash
# Round-2 check after the multi-rank / pageable e2e changes
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_multi.py tests/test_gpu_dropin.py -x -q -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1
tail -3 gpurun_out/r2c_tests.log
timeout 900 python bench.py --no-dropin > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 900 python bench.py --gpus 2 --no-dropin --steps 5 > gpurun_out/r2c_bench_w2.json 2> gpurun_out/r2c_bench_w2.err
python - <<'PY'
import json
for f in ['gpurun_out/r2c_bench.json','gpurun_out/r2c_bench_w2.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['value'], d['ms_per_step'], json.dumps(d.get('e2e'))[:900])
    except Exception as e:
        print(f, 'ERR', e, open(f.replace('.json','.err')).read()[-1500:])
PY
