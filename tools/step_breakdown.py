"""Per-stage device timings of one coarse PAVer step (config 2) via the
C-ABI's event timings: [seed, hash, finalize, sum, group, total] ms."""
import ctypes
import random
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2506_08781_b200 import _native as N
from paper_2506_08781_b200 import api

v = api.Verifier(0)
lib = v._lib
n2, n = 256, 1 << 26
n1 = n // n2
D = (n1 - 1).bit_length()
root = bytes(range(16))
ds = api.SeedStack(D, [api.SeedNode(D, 0, root)])
dsb = ds.serialize()
dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
log = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
err = N.PosloError()
assert lib.poslo_gpu_synth_log(v._ctx, 1, 0, n, 32, ctypes.c_void_p(log.data_ptr()), ctypes.byref(err)) == 0
epochs = np.arange(n1, dtype=np.uint32)
b = N.PosloBatch()
b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, log.data_ptr(), n * 32
b.offsets, b.entry_len, b.n_entries = None, 32, n
b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), D, 1
Y = v.exp_base((5).to_bytes(32, "little"))
S = (7).to_bytes(32, "little")
R = v.exp_base((9).to_bytes(32, "little"))
verdict = ctypes.c_uint8(0)
v.enable_timing(True)
for it in range(6):
    v._call(lib.poslo_gpu_paver, ctypes.byref(b), Y, S, R, None, ctypes.byref(verdict))
    t = v.last_timings()
    print(it, {k: round(x, 4) for k, x in t.items()})
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
ev0.record()
for it in range(10):
    v._call(lib.poslo_gpu_paver, ctypes.byref(b), Y, S, R, None, ctypes.byref(verdict))
ev1.record()
ev1.synchronize()
print("ms/step", ev0.elapsed_time(ev1) / 10)
