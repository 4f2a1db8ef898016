"""Signed synthetic logs resident in HBM, for the bench and the scale /
multi-rank parity tests (SURVEY §8d "Synthetic inputs", "Fixtures at scale").

`SignedLog` is one shard of a global log: epochs [first_epoch, first_epoch +
n_epochs) of n2 entries each, entry bytes from the counter-based generator
(include/poslo_synth.h, by GLOBAL entry index, so any shard of any split
regenerates the same bytes), keys and per-epoch signatures by the reference's
own derivation on the device (PoslocSecretKey::kg / sig_epoch,
poslo_c.cpp:91-134: R-hat_i = alpha^(sum_j nonce_to_scalar(r, i, j)),
s-hat_i = r-hat_i - y e~_i), all from one 64-bit seed. Every shard of the same
(seed, D) shares y, the nonce seed and the seed-tree root, so shards of a G-way
split verify exactly as the whole log does.
"""
from __future__ import annotations

import ctypes
import random
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from . import api

L_ORDER = api.L


def synth_varlen(seed: int, first: int, n: int) -> np.ndarray:
    """numpy port of poslo_synth_varlen (include/poslo_synth.h)."""
    with np.errstate(over="ignore"):
        k = np.arange(first, first + n, dtype=np.uint64)
        z = np.uint64((seed ^ 0x6c656e677468) & (2**64 - 1)) + np.uint64(0x9E3779B97F4A7C15) * (
            (k << np.uint64(8)) + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (np.uint64(64) + z % np.uint64(961)).astype(np.uint64)


class SignedLog:
    def __init__(self, v: api.Verifier, first_epoch: int, n_epochs: int, n2: int, D: int, seed: int,
                 entry_len: int = 32, varlen: bool = False, suite: int = 1, sign: bool = True):
        import torch
        self.v, self.suite, self.n2, self.D, self.seed = v, suite, n2, D, seed
        self.first_epoch, self.n1 = first_epoch, n_epochs
        self.n = n_epochs * n2
        first = first_epoch * n2
        lib = v._lib
        rng = random.Random(seed)
        root = bytes(rng.getrandbits(8) for _ in range(16))
        self.ds = api.SeedStack(D, [api.SeedNode(D, 0, root)])  # the root discloses every epoch
        self.ds_bytes = self.ds.serialize()
        self._dsbuf = ctypes.create_string_buffer(self.ds_bytes, len(self.ds_bytes))
        y = rng.randrange(1, L_ORDER)
        self.y = y.to_bytes(32, "little")
        self.r_seed = bytes(rng.getrandbits(8) for _ in range(16))
        err = N.PosloError()
        self.offsets = None
        if varlen:
            lens = synth_varlen(seed, first, self.n)
            offs = np.zeros(self.n + 1, dtype=np.uint64)
            np.cumsum(lens, out=offs[1:])
            self.offsets_host = offs
            self.offsets = torch.from_numpy(offs.view(np.int64)).cuda()
            self.log = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
            rc = lib.poslo_gpu_synth_varlog(v._ctx, seed, first, self.n, ctypes.c_void_p(self.offsets.data_ptr()),
                                            ctypes.c_void_p(self.log.data_ptr()), ctypes.byref(err))
            self.entry_len = 0
        else:
            self.log = torch.empty(self.n * entry_len, dtype=torch.uint8, device="cuda")
            rc = lib.poslo_gpu_synth_log(v._ctx, seed, first, self.n, entry_len,
                                         ctypes.c_void_p(self.log.data_ptr()), ctypes.byref(err))
            self.entry_len = entry_len
        if rc:
            api._raise(rc, err)
        self.epochs = np.arange(first_epoch, first_epoch + n_epochs, dtype=np.uint32)
        self.payload_bytes = int(self.log.numel())
        self.tampered: Sequence[int] = []
        if sign:
            self._sign()

    # -- the C-ABI batch over the device log (or a host copy)
    def batch(self, device_resident: bool = True, payload_ptr: Optional[int] = None,
              offsets_ptr: Optional[int] = None) -> N.PosloBatch:
        b = N.PosloBatch()
        b.suite, b.n2 = self.suite, self.n2
        b.payload = payload_ptr if payload_ptr is not None else self.log.data_ptr()
        b.payload_bytes = self.payload_bytes
        if self.offsets is not None:  # device offsets for a device batch, else the host copy
            b.offsets = offsets_ptr if offsets_ptr is not None else (
                self.offsets.data_ptr() if device_resident else self.offsets_host.ctypes.data)
        else:
            b.offsets = None
        b.entry_len, b.n_entries = self.entry_len, self.n
        b.epochs, b.epoch_starts, b.n_epochs = self.epochs.ctypes.data, None, self.n1
        b.ds, b.ds_len, b.ds_capacity = ctypes.addressof(self._dsbuf), len(self.ds_bytes), self.D
        b.device_resident = 1 if device_resident else 0
        return b

    def _sign(self):
        import torch
        v, lib = self.v, self.v._lib
        r_hats = ctypes.create_string_buffer(max(self.n1, 1) * 32)
        v._call(lib.poslo_gpu_kg_commitments, self.suite, self.r_seed, ctypes.c_void_p(self.epochs.ctypes.data),
                self.n1, self.n2, r_hats, None)
        s_hats = ctypes.create_string_buffer(max(self.n1, 1) * 32)
        b = self.batch()
        v._call(lib.poslo_gpu_sig_epochs, ctypes.byref(b), self.r_seed, self.y, s_hats)
        self.r_hats = r_hats.raw[:32 * self.n1]
        self.s_hats = s_hats.raw[:32 * self.n1]
        self.Y = v.exp_base(self.y)
        # this shard's parts of the coarse aggregate (sum of s-hat, fold of R-hat)
        self.S_part = v.scalar_sum([self.s_hats[32 * k:32 * k + 32] for k in range(self.n1)])
        self.R_part = v.group_fold([self.r_hats[32 * k:32 * k + 32] for k in range(self.n1)])
        # signature arrays resident in HBM too (device-timed per-epoch steps)
        self.s_dev = torch.frombuffer(bytearray(self.s_hats or b"\0"), dtype=torch.uint8).cuda()
        self.r_dev = torch.frombuffer(bytearray(self.r_hats or b"\0"), dtype=torch.uint8).cuda()
        torch.cuda.synchronize()

    def tamper(self, k: int, seed: int) -> Sequence[int]:
        """Flips one bit of k seeded entries (after signing); returns their global
        entry indices, ascending."""
        import torch
        rng = random.Random(seed)
        local = sorted(rng.sample(range(self.n), min(k, self.n)))
        for t in local:
            off = int(self.offsets_host[t]) if self.offsets is not None else t * self.entry_len
            self.log[off] ^= 1
        torch.cuda.synchronize()
        first = self.first_epoch * self.n2
        self.tampered = [first + t for t in local]
        return self.tampered

    def bad_epochs(self):
        return sorted({t // self.n2 for t in self.tampered})
