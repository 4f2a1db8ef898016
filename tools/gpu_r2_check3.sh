#!/bin/bash
# Round-2: pageable staging parity + bench lines (default, 2-rank)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout -k 20 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "chunked" > gpurun_out/r2d_tests.log 2>&1
tail -3 gpurun_out/r2d_tests.log
timeout -k 20 900 python bench.py --no-dropin > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
python - <<'PY'
import json
for f in ['gpurun_out/r2d_bench.json']:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d['value'], d['ms_per_step'], json.dumps(d.get('e2e'))[:1200])
    except Exception as e:
        print(f, 'ERR', e, open(f.replace('.json','.err')).read()[-1500:])
PY
