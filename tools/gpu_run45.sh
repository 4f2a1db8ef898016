cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_logfile.py -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_scan.log 2>&1
python - > gpurun_out/scan_speed.log 2>&1 <<'PY'
import time, numpy as np, sys
sys.path.insert(0, ".")
import bench
from paper_2506_08781_b200 import api
from paper_2506_08781_b200.logfile import RecordLog
n = 1 << 22
lens = bench.synth_varlen(5, 0, n).astype(np.int64)
pos = np.zeros(n + 1, dtype=np.int64); np.cumsum(lens + 4, out=pos[1:])
buf = np.full(int(pos[-1]), 0x41, dtype=np.uint8)
l32 = lens.astype(np.uint32).view(np.uint8).reshape(-1, 4)
for k in range(4): buf[pos[:-1] + k] = l32[:, k]
img = buf.tobytes()
v = api.Verifier(0)
RecordLog(img[:1 << 20 + 4], v) if False else None
for sc in ("device", "device", "host"):
    t = time.perf_counter(); log = RecordLog(img, v, scanner=sc); dt = time.perf_counter() - t
    print(sc, len(log), f"{dt*1e3:.1f} ms incl. H2D of {len(img)/1e9:.2f} GB")
PY
echo done
