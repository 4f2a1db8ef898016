"""Log ingestion: the reference's flat log container (include/poslo/log_file.hpp:34-66,
records = LE32 length + bytes) read without splitting it into per-record objects.

`RecordLog` keeps the file image as one array plus the record header positions
from poslo_gpu_log_scan (speculative chunk walks on the device) or
poslo_log_scan (the host scanner); both raise FormatError exactly where
read_log throws. Batches built from it point the device at the file image
itself (poslo_batch.record_header = 4): the H2D copy is the file, no per-record
repacking. `epochs_of` is tools/poslo.cpp:32-40.
"""
import ctypes
import os
from typing import Optional

import numpy as np

from . import _native as N
from . import api
from .api import FormatError


class RecordLog:
    def __init__(self, raw: bytes, verifier: Optional[api.Verifier] = None, scanner: str = "device"):
        """scanner: "device" (poslo_gpu_log_scan, the default) or "host" (poslo_log_scan)."""
        self.raw = np.frombuffer(raw, dtype=np.uint8) if len(raw) else np.zeros(0, np.uint8)
        lib = N.load()
        n = ctypes.c_uint64(0)
        err = N.PosloError()
        buf = self.raw if len(self.raw) else np.zeros(1, np.uint8)
        cap = max(2, len(raw) // 4 + 1)  # every record takes >= 4 bytes
        offs = np.zeros(cap, dtype=np.uint64)
        if scanner == "host":
            rc = lib.poslo_log_scan(buf.ctypes.data, len(raw), offs.ctypes.data, cap, ctypes.byref(n),
                                    ctypes.byref(err))
        else:
            v = verifier or api.default_verifier()
            rc = lib.poslo_gpu_log_scan(v._ctx, buf.ctypes.data, len(raw), 0, offs.ctypes.data, cap, ctypes.byref(n),
                                        ctypes.byref(err))
        if rc:
            api._raise(rc, err)
        self.n = int(n.value)
        self.offsets = offs[:self.n + 1].copy()

    @staticmethod
    def read(path: str, verifier: Optional[api.Verifier] = None, scanner: str = "device") -> "RecordLog":
        """read_file + read_log (log_file.hpp:14-19, 34-51)."""
        if not os.path.exists(path):
            raise FormatError("cannot open " + path)
        with open(path, "rb") as f:
            return RecordLog(f.read(), verifier, scanner)

    def __len__(self):
        return self.n

    def record(self, t: int) -> bytes:
        return self.raw[int(self.offsets[t]) + 4:int(self.offsets[t + 1])].tobytes()

    def epochs_of(self, n2: int):
        """tools/poslo.cpp:32-40: the record count must be a nonzero multiple of n2."""
        if self.n == 0 or self.n % n2:
            raise FormatError("record count must be a nonzero multiple of n2")
        return self.n // n2

    def batch(self, suite: int, n2: int, ds: api.SeedStack, epochs: Optional[range] = None):
        """A poslo_batch over epochs of this log (all by default), zero-copy."""
        n1 = self.epochs_of(n2)
        epochs = range(n1) if epochs is None else epochs
        return RecordBatch(self, suite, n2, ds, list(epochs))


def write_log(path: str, records) -> None:
    """write_log (log_file.hpp:53-66) — test tooling."""
    out = bytearray()
    for r in records:
        out += len(r).to_bytes(4, "little") + bytes(r)
    tmp = path + ".tmp"
    with open(tmp, "wb") as f:
        f.write(out)
    os.replace(tmp, path)


class RecordBatch:
    """poslo_batch over consecutive epochs of a RecordLog (host-resident file image)."""

    def __init__(self, log: RecordLog, suite: int, n2: int, ds: api.SeedStack, epochs):
        self.log, self.suite, self.n2, self.ds = log, suite, n2, ds
        self.epochs = np.array(epochs, dtype=np.uint32)
        if len(self.epochs) and np.any(np.diff(self.epochs.astype(np.int64)) != 1):
            raise ValueError("record batches cover consecutive epochs")
        e0 = int(self.epochs[0]) if len(self.epochs) else 0
        t0, t1 = e0 * n2, (e0 + len(self.epochs)) * n2
        base = int(log.offsets[t0])
        self.offsets = (log.offsets[t0:t1 + 1] - np.uint64(base)).astype(np.uint64)
        self.payload = log.raw[base:int(log.offsets[t1])]
        self.n_entries = t1 - t0
        self.ds_bytes = ds.serialize()

    def cstruct(self) -> N.PosloBatch:
        b = N.PosloBatch()
        b.suite, b.n2 = self.suite, self.n2
        pay = self.payload if len(self.payload) else np.zeros(1, np.uint8)
        self._keep = pay
        b.payload, b.payload_bytes = pay.ctypes.data, len(self.payload)
        b.offsets, b.entry_len, b.n_entries = self.offsets.ctypes.data, 0, self.n_entries
        b.epochs = self.epochs.ctypes.data if len(self.epochs) else None
        b.epoch_starts, b.n_epochs = None, len(self.epochs)
        self._dsbuf = ctypes.create_string_buffer(self.ds_bytes, len(self.ds_bytes))
        b.ds, b.ds_len, b.ds_capacity = ctypes.addressof(self._dsbuf), len(self.ds_bytes), self.ds.capacity
        b.device_resident, b.ds_offsets, b.record_header = 0, None, 4
        return b


class ImageBatch:
    """poslo_batch over a WHOLE raw record image with no offsets
    (record_header = 4, offsets = NULL): the device finds the records itself
    and, for a host image, copies it in 64 MiB chunks with the record scan and
    the hashing of every completed epoch running behind the copy (read_log +
    epochs_of + verification in one call; the record count must be
    n_epochs x n2). `image`: bytes / uint8 array in host memory, or a device
    pointer with device_resident=True (then `nbytes` is required)."""

    def __init__(self, image, suite: int, n2: int, n_epochs: int, ds: api.SeedStack,
                 device_resident: bool = False, nbytes: Optional[int] = None):
        self.suite, self.n2, self.ds = suite, n2, ds
        self.device_resident = device_resident
        if device_resident:
            self._ptr, self._len = int(image), int(nbytes)
        else:
            arr = np.frombuffer(image, dtype=np.uint8) if isinstance(image, (bytes, bytearray)) else image
            self._keep = arr if len(arr) else np.zeros(1, np.uint8)
            self._ptr, self._len = self._keep.ctypes.data, len(arr)
        self.epochs = np.arange(n_epochs, dtype=np.uint32)
        self.ds_bytes = ds.serialize()

    def cstruct(self) -> N.PosloBatch:
        b = N.PosloBatch()
        b.suite, b.n2 = self.suite, self.n2
        b.payload, b.payload_bytes = self._ptr, self._len
        b.offsets, b.entry_len, b.n_entries = None, 0, len(self.epochs) * self.n2
        b.epochs = self.epochs.ctypes.data if len(self.epochs) else None
        b.epoch_starts, b.n_epochs = None, len(self.epochs)
        self._dsbuf = ctypes.create_string_buffer(self.ds_bytes, len(self.ds_bytes))
        b.ds, b.ds_len, b.ds_capacity = ctypes.addressof(self._dsbuf), len(self.ds_bytes), self.ds.capacity
        b.device_resident, b.ds_offsets, b.record_header = int(self.device_resident), None, 4
        return b
