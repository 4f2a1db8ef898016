"""Raw log image scan: device (image resident in HBM) vs host scanner, 2^22 syslog-style records."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2506_08781_b200 import synth as bench  # noqa: E402
from paper_2506_08781_b200 import _native as N  # noqa: E402
from paper_2506_08781_b200 import api  # noqa: E402

n = 1 << 22
lens = bench.synth_varlen(5, 0, n).astype(np.int64)
pos = np.zeros(n + 1, dtype=np.int64)
np.cumsum(lens + 4, out=pos[1:])
buf = np.full(int(pos[-1]), 0x41, dtype=np.uint8)
l32 = lens.astype(np.uint32).view(np.uint8).reshape(-1, 4)
for k in range(4):
    buf[pos[:-1] + k] = l32[:, k]
v = api.Verifier(0)
lib = v._lib
dev = torch.from_numpy(buf).cuda()
offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
cnt = ctypes.c_uint64()
err = N.PosloError()
for it in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    rc = lib.poslo_gpu_log_scan(v._ctx, ctypes.c_void_p(dev.data_ptr()), len(buf), 1, ctypes.c_void_p(offs.data_ptr()),
                                n + 1, ctypes.byref(cnt), ctypes.byref(err))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print("device-resident", rc, cnt.value, f"{dt * 1e3:.2f} ms", f"{len(buf) / dt / 1e9:.0f} GB/s")
ho = np.zeros(n + 2, dtype=np.uint64)
t = time.perf_counter()
rc = lib.poslo_log_scan(buf.ctypes.data, len(buf), ho.ctypes.data, n + 2, ctypes.byref(cnt), ctypes.byref(err))
dt = time.perf_counter() - t
print("host", rc, cnt.value, f"{dt * 1e3:.2f} ms", f"{len(buf) / dt / 1e9:.1f} GB/s")
assert np.array_equal(ho[:n + 1].astype(np.int64), offs.cpu().numpy())
print("offsets identical")
