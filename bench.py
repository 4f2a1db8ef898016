"""bench.py — verified log entries/sec of the B200 batch verifier.

Contract (see the task's bench contract and SURVEY.md §8d):
  python bench.py --gpus N --steps K --warmup W [--impl reference]
One process per GPU (torchrun for N > 1). A "step" is one full coarse-mode
PAVer pass (BASELINE.json config 2: 2^26 x 32-byte entries per GPU,
n2 = 256 -> 2^18 epochs, suite 1 / SHA-256) over a synthetic log already
resident in HBM: K0 seed derivation -> K1+K2 fused hash + segmented modular
sum -> e-hat fold -> K3 ristretto255 group check -> verdict to host. For
N > 1 each rank verifies its own contiguous epoch shard (weak scaling) and
the per-shard partial e-hat (32 B) is combined with an NCCL all-gather and a
rank-ordered device fold before the single group check on rank 0.

Extra keys: e2e (same metric through the C-ABI with the log in pinned HOST
memory, H2D inside the timed region), roofline (integer pipe, measured
peak), cpu_baseline (the reference's own paver, compiled from
/root/reference into oracle/_ref, on this host's cores), clocks, gpu_launches.
"""
import argparse
import ctypes
import json
import os
import random
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified log entries/sec (device-timed) at 1/2/4/8 B200 vs CPU ref"
L_ORDER = 2**252 + 27742317777372353535851937790883648493
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--log2n", type=int, default=26, help="entries per GPU = 2^log2n")
    ap.add_argument("--n2", type=int, default=256)
    ap.add_argument("--suite", type=int, default=1)
    ap.add_argument("--entry-len", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0x5EED)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-log2n", type=int, default=21)
    ap.add_argument("--varlen", action="store_true",
                    help="syslog-style entries of 64..1024 printable bytes (BASELINE config 4)")
    ap.add_argument("--mode", default="coarse", choices=["coarse", "epoch", "tamper"],
                    help="coarse: one aggregate (config 2); epoch: per-epoch verdicts (config 3); "
                         "tamper: k tampered entries localised by distillation (config 5)")
    ap.add_argument("--tamper", type=int, default=16, help="tampered entries per GPU (mode tamper)")
    ap.add_argument("--records", action="store_true",
                    help="with --varlen --mode epoch: also time file ingestion end to end (raw LE32-record image "
                         "in pinned host memory -> H2D -> device record scan -> in-place verification)")
    ap.add_argument("--n-u", type=int, default=1024, help="umbrellas over the whole job (mode tamper)")
    return ap.parse_args()


def synth_varlen(seed, first, n):
    """numpy port of poslo_synth_varlen (include/poslo_synth.h)."""
    import numpy as np
    with np.errstate(over="ignore"):
        k = np.arange(first, first + n, dtype=np.uint64)
        z = np.uint64((seed ^ 0x6c656e677468) & (2**64 - 1)) + np.uint64(0x9E3779B97F4A7C15) * ((k << np.uint64(8)) + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (np.uint64(64) + z % np.uint64(961)).astype(np.uint64)


def config_dict(a, n_gpus):
    if a.varlen:
        return {"workload": f"BASELINE config 4 (per GPU): 2^{a.log2n} syslog-style entries of 64..1024 printable "
                            f"bytes, {a.mode} verify (epoch = {a.n2} entries, suite {a.suite}), inputs resident in HBM",
                "entries_per_gpu": 1 << a.log2n, "entry_len": "U[64,1024] (mean 544)", "n2": a.n2,
                "suite": a.suite, "mode": a.mode,
                "parallelism": f"epoch-sharded x{n_gpus}" if n_gpus > 1 else "single GPU",
                "l2": "inputs larger than L2"}
    if a.mode == "tamper":
        return {"workload": f"BASELINE config 5 (per GPU): 2^{a.log2n} x {a.entry_len}-byte entries with {a.tamper} "
                            f"tampered entries, hierarchical localisation by coarse distillation (per-epoch verdicts, "
                            f"epoch = {a.n2} entries, + umbrella folds, n_u = {a.n_u} over the job; suite {a.suite}), "
                            f"inputs resident in HBM",
                "entries_per_gpu": 1 << a.log2n, "entry_len": a.entry_len, "n2": a.n2, "suite": a.suite,
                "mode": a.mode, "tampered_per_gpu": a.tamper, "n_u": a.n_u,
                "parallelism": f"epoch-sharded x{n_gpus}" if n_gpus > 1 else "single GPU",
                "l2": "inputs larger than L2 (2 GiB log per GPU vs 126 MB L2)"}
    return {
        "workload": (f"BASELINE config 2: 2^{a.log2n} x {a.entry_len}-byte entries per GPU, coarse single-aggregate "
                     f"PAVer (suite {a.suite}, n2={a.n2}), inputs resident in HBM") if a.mode == "coarse" else
                    (f"BASELINE config 3: 2^{a.log2n} x {a.entry_len}-byte entries per GPU, per-epoch verify "
                     f"(epoch = {a.n2} entries, {(1 << a.log2n) // a.n2} group checks; suite {a.suite}), inputs resident in HBM"),
        "entries_per_gpu": 1 << a.log2n,
        "entry_len": a.entry_len,
        "n2": a.n2,
        "suite": a.suite,
        "mode": a.mode,
        "parallelism": f"epoch-sharded x{n_gpus}" if n_gpus > 1 else "single GPU",
        "l2": "inputs larger than L2 (2 GiB log per GPU vs 126 MB L2)",
    }


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:  # NVML set up BEFORE the timed region, so even a short region gets samples
            import pynvml as nv
            nv.nvmlInit()
            self._h = nv.nvmlDeviceGetHandleByIndex(index)
            self._mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            self._nv = nv
        except Exception:
            self._nv = None

    def _sample_nvml(self):
        nv = self._nv
        bits = (0x8, 0x40, 0x20, 0x4)  # hw_slowdown, hw_thermal, sw_thermal, sw_power_cap
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append([str(sm), str(self._mx), ""] + ["Active" if r & bt else "Not Active" for bt in bits])

    def _sample_smi(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                  "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                 timeout=5).stdout.strip()
            if out:
                self.samples.append([x.strip() for x in out.split(",")])
        except Exception:
            pass

    def _run(self):
        # NVML samples every 5 ms (a 10-step timed region is ~130 ms); nvidia-smi if NVML is absent
        while not self._stop.is_set():
            if self._nv is not None:
                try:
                    self._sample_nvml()
                except Exception:
                    self._nv = None
                self._stop.wait(0.005)
            else:
                self._sample_smi()
                self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)
        if not self.samples:  # region shorter than one sampling period: one sample at its end
            if self._nv is not None:
                try:
                    self._sample_nvml()
                except Exception:
                    pass
            if not self.samples:
                self._sample_smi()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [int(s[0]) for s in self.samples if s[0].isdigit()]
        mx = [int(s[1]) for s in self.samples if s[1].isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------- CPU reference
def run_ref_tool(log2n, n2, entry_len, suite, seed, reps, mode="coarse"):
    if not os.path.exists(REF_TOOL):
        return None
    cmd = [REF_TOOL, "bench", str(suite), str(log2n), str(n2), str(entry_len), "0", str(seed), str(reps), mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    if out.returncode != 0:
        raise RuntimeError(f"ref_tool failed: {out.stderr.strip()}")
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(a):
    per_epoch = a.mode != "coarse"
    # varlen entries cost ~6.6x the compressions of a 32-byte one: a 16x smaller sample
    log2n = a.cpu_log2n - (4 if a.varlen else 0)
    r = run_ref_tool(log2n, a.n2, 0 if a.varlen else a.entry_len, a.suite, a.seed, 1,
                     "epoch" if per_epoch else "coarse")
    if r is None:
        return None
    what = ("the shipped per-epoch poslo::aver loop (proj/src/poslo_c.cpp:192-213, as acceptance.cpp:477-481), "
            "epochs sharded over all host threads" if per_epoch else
            "reference poslo::paver (proj/src/batch_verify.cpp:64-87)")
    shape = "syslog-style 64..1024-byte" if a.varlen else f"{a.entry_len}-byte"
    return {"value": round(r["eps_best"], 1), "unit": "entries/s", "cores": r["workers"],
            "kind": "reference",
            "sample": f"{what}, OpenSSL 3 + libsodium 1.0.20, on an epoch-aligned 2^{log2n}-entry prefix of the "
                      f"same synthetic {shape} log (n2={a.n2}, suite {a.suite}), workers={r['workers']} = all "
                      f"host threads, {cpu_model()}; {r['best_s']:.2f} s wall"}


def reference_arm(a, rank, world):
    if rank != 0:
        return 0
    log2n = min(a.cpu_log2n, 20)
    reps = a.warmup + a.steps
    r = run_ref_tool(log2n, a.n2, a.entry_len, a.suite, a.seed, reps)
    line = {"impl": "reference", "metric": METRIC, "unit": "entries/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic", "config": config_dict(a, world)}
    if r is None:
        line.update({"unavailable": "oracle/_ref/ref_tool not built (needs /root/reference at build time)"})
        print(json.dumps(line), flush=True)
        return 0
    times = r["times"][a.warmup:]
    t = sum(times) / len(times)
    value = (1 << log2n) / t
    line.update({
        "value": round(value, 1), "ms_per_step": round(t * 1e3, 3),
        "cpu_baseline": {"value": round(value, 1), "unit": "entries/s", "cores": r["workers"], "kind": "reference",
                         "sample": f"each step = reference paver over a 2^{log2n}-entry epoch-aligned sample of the "
                                   f"workload ({cpu_model()}, {r['workers']} threads)"},
        "e2e": {"value": round(value, 1), "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "verdict": bool(r["verdict"]),
    })
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- roofline helpers
def sass_ops_per_entry(lib_path, kernel_substr, entries_per_thread):  # static count (unrolled kernels only)
    """Integer-pipe instructions per entry of the hashing kernel, counted once
    from the shipped SASS (ALU + FMA pipe ops; memory/control excluded)."""
    try:
        out = subprocess.run(["cuobjdump", "-sass", lib_path], capture_output=True, text=True, timeout=300).stdout
    except Exception:
        return None
    blocks = out.split("Function : ")
    for blk in blocks:
        if kernel_substr in blk.split("\n", 1)[0]:
            n = 0
            for line in blk.splitlines():
                line = line.strip()
                if not line.startswith("/*") or "*/" not in line:
                    continue
                ins = line.split("*/", 1)[1].strip().split(" ")[0].strip("{").strip()
                if ins.startswith("@"):
                    ins = line.split("*/", 1)[1].strip().split(" ")[1]
                op = ins.split(".")[0]
                if op in ("LOP3", "SHF", "IADD3", "IMAD", "PRMT", "IADD", "LEA", "VIADD", "IABS", "SEL",
                          "ISETP", "SHL", "SHR", "IMNMX", "BMSK", "FLO", "POPC"):
                    n += 1
            return n / entries_per_thread
    return None


def int_peak(device):
    lib_path = os.path.join(ROOT, "paper_2506_08781_b200", "libposlo_microbench.so")
    if not os.path.exists(lib_path):
        return None
    lib = ctypes.CDLL(lib_path)
    lib.poslo_microbench_int_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_double)]
    res = {}
    for _ in range(3):  # best of three: the first pass can run before the clocks settle
        for mode, name in ((0, "alu"), (1, "fma"), (2, "dual"), (10, "lds")):
            v, ms = ctypes.c_double(), ctypes.c_double()
            if lib.poslo_microbench_int_peak(device, mode, ctypes.byref(v), ctypes.byref(ms)) == 0:
                res[name] = max(res.get(name, 0.0), v.value)
    return res


# ----------------------------------------------------------------- B200 arm
def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if a.impl == "reference":
        return reference_arm(a, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200 import _native as N

    # one process per GPU; POSLO_DIST_BACKEND=gloo lets the N > 1 path be
    # exercised with several ranks sharing one device (tests only)
    backend = os.environ.get("POSLO_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2506_08781_b200 import multi_gpu as MG
    v = api.Verifier(local)
    # one stream for torch's ops on the bench buffers AND the C-ABI's work, so
    # copies, kernels and the timing events are all ordered on it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    v.set_stream(stream.cuda_stream)
    lib = v._lib

    n = 1 << a.log2n
    L = a.entry_len
    n1_local = n // a.n2
    n1_total = n1_local * world
    D = max(1, (n1_total - 1).bit_length())
    rng = random.Random(a.seed)
    root = bytes(rng.getrandbits(8) for _ in range(16))
    ds = api.SeedStack(D, [api.SeedNode(D, 0, root)])  # fully disclosed tree: D PRFs per epoch

    # synthetic log of this rank's epochs, generated on the device
    import numpy as np
    err = N.PosloError()
    offsets_dev = None
    if a.varlen:
        lens = synth_varlen(a.seed, rank * n, n)
        offs = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(lens, out=offs[1:])
        payload_bytes = int(offs[-1])
        offsets_dev = torch.from_numpy(offs.view(np.int64)).cuda()
        log = torch.empty(payload_bytes, dtype=torch.uint8, device="cuda")
        rc = lib.poslo_gpu_synth_varlog(v._ctx, a.seed, rank * n, n, ctypes.c_void_p(offsets_dev.data_ptr()),
                                        ctypes.c_void_p(log.data_ptr()), ctypes.byref(err))
        L = 0
    else:
        payload_bytes = n * L
        log = torch.empty(n * L, dtype=torch.uint8, device="cuda")
        rc = lib.poslo_gpu_synth_log(v._ctx, a.seed, rank * n, n, L, ctypes.c_void_p(log.data_ptr()),
                                     ctypes.byref(err))
    assert rc == 0, err.message
    epochs = np.arange(rank * n1_local, (rank + 1) * n1_local, dtype=np.uint32)
    ds_bytes = ds.serialize()
    ds_buf = ctypes.create_string_buffer(ds_bytes, len(ds_bytes))

    host_offs = None

    def batch(payload_ptr, device_resident):
        b = N.PosloBatch()
        b.suite, b.n2, b.payload, b.payload_bytes = a.suite, a.n2, payload_ptr, payload_bytes
        if offsets_dev is not None:
            b.offsets = offsets_dev.data_ptr() if device_resident else host_offs.ctypes.data
        else:
            b.offsets = None
        b.entry_len, b.n_entries = L, n
        b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1_local
        b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(ds_buf), len(ds_bytes), D, device_resident
        return b

    bdev = batch(log.data_ptr(), 1)

    def call(fn, *args):
        e = N.PosloError()
        rc = fn(v._ctx, *args, ctypes.byref(e))
        if rc:
            raise RuntimeError(f"{fn.__name__}: {rc} {e.message.decode()}")

    # ---- fixture (untimed): keys and signatures by the reference's own
    # derivation (PoslocSecretKey::kg / sig_epoch, poslo_c.cpp:91-134) on the
    # device: secret y, nonce seed r, seed-tree root; R-hat_i = alpha^(sum_j
    # nonce_to_scalar(r, i, j)) and s-hat_i = r-hat_i - y e~_i for this rank's
    # epochs; the coarse aggregate folds them over every rank.
    y = rng.randrange(1, L_ORDER)
    y_le = y.to_bytes(32, "little")
    r_seed = bytes(rng.getrandbits(8) for _ in range(16))
    ep_arr = np.ascontiguousarray(epochs)
    r_hats_buf = ctypes.create_string_buffer(max(n1_local, 1) * 32)
    call(lib.poslo_gpu_kg_commitments, a.suite, r_seed, ctypes.c_void_p(ep_arr.ctypes.data), n1_local, a.n2,
         r_hats_buf, None)
    s_hats_buf = ctypes.create_string_buffer(max(n1_local, 1) * 32)
    call(lib.poslo_gpu_sig_epochs, ctypes.byref(bdev), r_seed, y_le, s_hats_buf)
    r_enc, s_bytes = r_hats_buf.raw[:32 * n1_local], s_hats_buf.raw[:32 * n1_local]
    R_part = v.group_fold([r_enc[32 * k:32 * k + 32] for k in range(n1_local)])
    S_part = v.scalar_sum([s_bytes[32 * k:32 * k + 32] for k in range(n1_local)])
    if world > 1:
        R_all, S_all = MG.all_gather_bytes(R_part), MG.all_gather_bytes(S_part)
    else:
        R_all, S_all = [R_part], [S_part]
    R = v.group_fold(R_all)
    s_le = v.scalar_sum(S_all)
    Y = v.exp_base(y_le)
    Yb, Sb, Rb = (ctypes.create_string_buffer(x, 32) for x in (Y, s_le, R))
    verdict = ctypes.c_uint8(0)
    e_part = ctypes.create_string_buffer(32)

    def step_single(b):
        call(lib.poslo_gpu_paver, ctypes.byref(b), Yb, Sb, Rb, None, ctypes.byref(verdict))
        return verdict.value

    def step_multi(b):
        # partial e-hat of this rank's epochs -> all-gather (NCCL/NVLink) ->
        # rank-ordered device fold mod l -> one group check on rank 0
        call(lib.poslo_gpu_agg_ekeys, ctypes.byref(b), None, e_part)
        gathered = b"".join(MG.all_gather_bytes(e_part.raw))
        ok = 1
        if rank == 0:
            eh = ctypes.create_string_buffer(32)
            call(lib.poslo_gpu_scalar_sum, world, gathered, eh)  # rank-ordered device fold mod l
            call(lib.poslo_gpu_group_check, 1, Yb, eh, Sb, Rb, ctypes.byref(verdict))
            ok = verdict.value
        return ok

    step = step_single if world == 1 else step_multi

    if a.mode == "epoch":
        # per-epoch signatures (kg/sig_epoch derivation above): one
        # verdict per epoch, no cross-rank exchange except the verdict count
        s_buf = ctypes.create_string_buffer(s_bytes, len(s_bytes))
        r_buf = ctypes.create_string_buffer(r_enc, len(r_enc))
        # signatures are inputs too: resident in HBM for the device-timed steps
        s_dev = torch.frombuffer(bytearray(s_bytes), dtype=torch.uint8).cuda()
        r_dev = torch.frombuffer(bytearray(r_enc), dtype=torch.uint8).cuda()
        verd = ctypes.create_string_buffer(n1_local)

        def sig_ptrs(b):
            if b.device_resident:
                return ctypes.c_void_p(s_dev.data_ptr()), ctypes.c_void_p(r_dev.data_ptr())
            return s_buf, r_buf

        def step_epoch(b):
            call(lib.poslo_gpu_epoch_verify, ctypes.byref(b), Yb, *sig_ptrs(b), verd, None)
            bad = n1_local - sum(verd.raw[:n1_local])
            if world > 1:
                bad = sum(int.from_bytes(x, "little") for x in MG.all_gather_bytes(bad.to_bytes(4, "little")))
            return 1 if bad == 0 else 0

        step = step_epoch

    if a.mode == "tamper":
        # per-epoch signatures as in epoch mode, then k seeded entries tampered (one bit
        # flipped after signing); a step distils every epoch: per-epoch verdicts (the
        # invalid-epoch list) + valid (s, R) folded per umbrella piece on the device
        s_buf = ctypes.create_string_buffer(s_bytes, len(s_bytes))
        r_buf = ctypes.create_string_buffer(r_enc, len(r_enc))
        s_dev = torch.frombuffer(bytearray(s_bytes), dtype=torch.uint8).cuda()
        r_dev = torch.frombuffer(bytearray(r_enc), dtype=torch.uint8).cuda()

        def sig_ptrs(b):
            if b.device_resident:
                return ctypes.c_void_p(s_dev.data_ptr()), ctypes.c_void_p(r_dev.data_ptr())
            return s_buf, r_buf

        trng = random.Random(a.seed * 7919 + rank)
        tampered = sorted(trng.sample(range(n), min(a.tamper, n)))
        for t in tampered:
            log[t * L] ^= 1
        torch.cuda.synchronize()
        expect_bad = sorted({t // a.n2 for t in tampered})
        w = max(1, n1_total // max(1, a.n_u))
        e0 = rank * n1_local
        cuts = [0] + [k for k in range(1, n1_local) if (e0 + k) % w == 0] + [n1_local]
        seg_arr = np.array(cuts, dtype=np.uint32)
        n_seg = len(cuts) - 1
        verd = ctypes.create_string_buffer(n1_local)
        seg_s = ctypes.create_string_buffer(32 * n_seg)
        seg_r = ctypes.create_string_buffer(32 * n_seg)

        def step_tamper(b):
            call(lib.poslo_gpu_distill_coarse, ctypes.byref(b), Yb, *sig_ptrs(b),
                 ctypes.c_void_p(seg_arr.ctypes.data), n_seg, verd, seg_s, seg_r)
            ok = 1
            if world > 1:
                ok = min(int(x[0]) for x in MG.all_gather_bytes(bytes([ok])))
            return ok

        step = step_tamper

    # ---- warm-up + correctness of the fixture
    for _ in range(a.warmup):
        ok = step(bdev)
    if a.mode == "tamper":
        raw = verd.raw
        found = [e0 + k for k in range(n1_local) if not raw[k]]
        assert found == [e0 + k for k in expect_bad], f"localisation mismatch: {found[:8]} vs {expect_bad[:8]}"
    if rank == 0:
        assert ok == 1, "verifier rejected a valid aggregate"
    # tamper check (untimed): one flipped bit must be rejected
    if world == 1 and a.mode != "tamper":
        saved = log[0].item()
        log[0] = saved ^ 1
        torch.cuda.synchronize()
        assert step(bdev) == 0, "tampered log accepted"
        log[0] = saved
        torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    v.enable_timing(True)
    hash_ms = []
    stage_ms = []
    launches = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            ok = step(bdev)
            st_ = v.last_timings()
            hash_ms.append(st_["hash"])
            stage_ms.append(st_)
            launches += v.last_launches()
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
    ms_per_step = ms / a.steps
    value = world * n / (ms_per_step * 1e-3)

    # ---- e2e: same metric through the C-ABI with the log in pinned HOST memory
    v.enable_timing(False)
    e2e = None
    if a.e2e_steps > 0:
        host = torch.empty(payload_bytes, dtype=torch.uint8, pin_memory=True)
        host.copy_(log)
        if offsets_dev is not None:
            # pinned like the log (a pageable source would make the driver stage it synchronously)
            host_offs_t = torch.empty(offsets_dev.numel(), dtype=torch.int64, pin_memory=True)
            host_offs_t.copy_(offsets_dev)
            host_offs = host_offs_t.numpy().view(np.uint64)
        bhost = batch(host.data_ptr(), 0)
        step(bhost)  # warm the staging buffers
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0.record(stream)
        for _ in range(a.e2e_steps):
            step(bhost)
        ev1.record(stream)
        ev1.synchronize()
        e2e_ms = max(ev0.elapsed_time(ev1), (time.perf_counter() - t0) * 1e3) / a.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_ms], device="cuda" if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = t.item()
        e2e_value = world * n / (e2e_ms * 1e-3)
        if os.environ.get("POSLO_BENCH_STAGES"):  # diagnostics: per-stage device times of one e2e step
            v.enable_timing(True)
            step(bhost)
            print("e2e stages (ms):", {k: round(x, 3) for k, x in v.last_timings().items()}, file=sys.stderr)
            v.enable_timing(False)
        # the e2e roof: plain pinned H2D of the same bytes (64 MiB chunks, one
        # stream) into the device log, which already holds exactly these bytes
        link_ms = []
        for _ in range(3):
            torch.cuda.synchronize()
            ev0.record(stream)
            for off in range(0, payload_bytes, 64 << 20):
                log[off:off + (64 << 20)].copy_(host[off:off + (64 << 20)], non_blocking=True)
            ev1.record(stream)
            ev1.synchronize()
            link_ms.append(ev0.elapsed_time(ev1))
        link_peak = payload_bytes / (min(link_ms) * 1e-3) / 1e9
        del host
        per_epoch_in = 64 * n1_local if a.mode in ("epoch", "tamper") else 32
        h2d = payload_bytes + (8 * (n + 1) if offsets_dev is not None else 0) + 4 * n1_local + len(ds_bytes) + 8 + per_epoch_in
        if a.mode == "tamper":
            h2d += 4 * (n_seg + 1)
        d2h = (n1_local if a.mode in ("epoch", "tamper") else 1) + 8 + (64 * n_seg if a.mode == "tamper" else 0)
        e2e = {"value": round(e2e_value, 1), "unit": "entries/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": round(e2e_ms, 3),
               "path": f"poslo_gpu_{dict(coarse='paver', epoch='epoch_verify', tamper='distill_coarse')[a.mode]}(device_resident=0) "
                       f"on a pinned host log, 64 MiB chunked H2D overlapped with hashing",
               "link": {"bound": "PCIe host->device", "achieved_gbs": round(h2d / (e2e_ms * 1e-3) / 1e9, 2),
                        "peak_gbs": round(link_peak, 2), "frac": round(h2d / (e2e_ms * 1e-3) / 1e9 / link_peak, 4),
                        "peak_source": "measured live: plain pinned H2D of the same log, 64 MiB chunks"}}

    # ---- e2e from a raw log image (log_file.hpp records): H2D, device record
    # scan (poslo_gpu_log_scan), per-epoch verification of the image in place
    records = None
    if a.records and a.varlen and a.mode == "epoch":
        lens_h = synth_varlen(a.seed, rank * n, n).astype(np.int64)
        hdr_pos = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens_h + 4, out=hdr_pos[1:])
        img_bytes = int(hdr_pos[-1])
        img = torch.empty(img_bytes, dtype=torch.uint8, pin_memory=True)
        img_np = img.numpy()
        payload_h = log.cpu().numpy()
        l32 = lens_h.astype(np.uint32).view(np.uint8).reshape(-1, 4)
        for k in range(4):
            img_np[hdr_pos[:-1] + k] = l32[:, k]
        offs_h = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(lens_h, out=offs_h[1:])
        for e in range(n1_local):  # payload bytes of epoch e behind their headers (per epoch: bounded memory)
            t0_, t1_ = e * a.n2, (e + 1) * a.n2
            seg = lens_h[t0_:t1_]
            dst = np.repeat(hdr_pos[t0_:t1_] + 4 - offs_h[t0_:t1_], seg) + np.arange(offs_h[t0_], offs_h[t1_])
            img_np[dst] = payload_h[offs_h[t0_]:offs_h[t1_]]
        cnt = ctypes.c_uint64()

        def step_records():
            # the raw image straight from pinned host memory: the C-ABI copies it in
            # 64 MiB chunks, scans each chunk's records on the device as it lands
            # and hashes every epoch whose records are complete, behind the copy
            rb = N.PosloBatch()
            rb.suite, rb.n2, rb.payload, rb.payload_bytes = a.suite, a.n2, img.data_ptr(), img_bytes
            rb.offsets, rb.entry_len, rb.n_entries = None, 0, n
            rb.epochs, rb.epoch_starts, rb.n_epochs = epochs.ctypes.data, None, n1_local
            rb.ds, rb.ds_len, rb.ds_capacity = ctypes.addressof(ds_buf), len(ds_bytes), D
            rb.device_resident, rb.record_header = 0, 4
            call(lib.poslo_gpu_epoch_verify, ctypes.byref(rb), Yb, s_buf, r_buf, verd, None)
            cnt.value = n
            return n1_local - sum(verd.raw[:n1_local])

        assert step_records() == 0 and cnt.value == n, "record-image verification failed"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = max(1, a.e2e_steps)
        for _ in range(reps):
            bad = step_records()
        torch.cuda.synchronize()
        rec_ms = (time.perf_counter() - t0) * 1e3 / reps
        assert bad == 0
        records = {"value": round(world * n / (rec_ms * 1e-3), 1), "unit": "entries/s", "ms_per_step": round(rec_ms, 3),
                   "h2d_bytes_per_step": img_bytes, "d2h_bytes_per_step": n1_local + 16,
                   "path": "raw LE32-record image (log_file.hpp) in pinned host memory -> poslo_gpu_epoch_verify("
                           "record_header=4, no offsets): 64 MiB chunked H2D, record scan and hashing per chunk behind "
                           "the copy"}
        del img

    if rank != 0:
        dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (integer ALU pipe)
    # Algorithmic work per SHA-256 compression (FIPS 180-4, 64 rounds + 48
    # schedule words), split by the pipe that can execute it on sm_100:
    #   ALU-only ops (rotations SHF.R.W, shifts, LOP3 logic): 64 x (6 + 4) + 48 x (4 + 2 + 2) = 1024
    #   additions (2-input, ALU IADD3 or FMA-pipe IMAD):      64 x 7 + 48 x 3 = 592
    # The ALU pipe is the binding roof (measured: 64 lanes/clk/SM for LOP3 and
    # SHF alike; IMAD.HI rotations on the FMA pipe run at a quarter of that),
    # so `achieved` counts the ALU-only ops: 3 compressions x 1024 per 32-byte
    # entry (onetime_seed, H(m||x), H(0x01||m||x)); hoisting is NOT subtracted.
    # `dual_pipe` is the secondary roof: all 1616 ops per compression against
    # the measured LOP3+IMAD dual-issue rate.
    ALU_OPS, ALL_OPS = 1024, 1616
    comps = 3.0 if a.suite == 1 and not a.varlen else None
    lean = a.suite == 1 and not a.varlen and a.entry_len == 32 and a.n2 <= 4096
    kname = "k_hash_s1_l32r" if lean else "k_hash_s1_l32c"
    if a.suite == 1 and a.varlen:  # ceil((L+25)/64) + ceil((L+26)/64) + 1 compressions per entry
        lens_np = synth_varlen(a.seed, rank * n, n).astype(np.int64)
        comps = float(((lens_np + 25 + 63) // 64 + (lens_np + 26 + 63) // 64 + 1).mean())
        kname = "k_hash_s1_var"
    peaks = int_peak(local) or {}
    hash_avg_ms = statistics.mean(hash_ms) if hash_ms else None
    peaks_file = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm_peak, hbm_src = 6534.5, "B200_PROFILING.md fallback"
    if os.path.exists(peaks_file):
        hbm_peak, hbm_src = json.load(open(peaks_file)).get("hbm_gbs", hbm_peak), "MEASURED_PEAKS.json hbm_gbs"
    roof = None
    if comps and hash_avg_ms and peaks.get("alu"):
        rate = n / (hash_avg_ms * 1e-3)  # entries/s through the hash kernel
        achieved = ALU_OPS * comps * rate / 1e12
        peak = peaks["alu"] / 1e12
        hbm_gbs = payload_bytes / (hash_avg_ms * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):  # dram bytes per launch from the committed `ncu --set full` capture
            tj = json.load(open(tf)).get(kname)
            if tj and tj.get("entries") == n:
                traffic = tj["dram_bytes"]
        roof = {"bound": "int32 ALU pipe", "kernel": kname, "achieved": round(achieved, 2), "peak": round(peak, 2),
                "unit": "Tops/s (int32 ALU-pipe lane-ops)", "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_unit": "bytes per launch (dram read + write, ncu --set full)",
                "algorithmic_bytes": payload_bytes,
                "ops_per_entry": ALU_OPS * comps,
                "ops_basis": f"{comps:.2f} SHA-256 compressions x 1024 ALU-only ops (64 rounds x 10 SHF/LOP3 + "
                             "48 schedule words x 8); additions excluded (FMA-pipe capable)",
                "ms_per_launch": round(hash_avg_ms, 4),
                "peak_source": "measured live: LOP3 chains, ALU pipe (paper_2506_08781_b200/csrc/microbench.cu)",
                "dual_pipe": {"achieved": round(ALL_OPS * comps * rate / 1e12, 2),
                              "peak": round(peaks.get("dual", 0) / 1e12, 2),
                              "frac": round(ALL_OPS * comps * rate / peaks["dual"], 4) if peaks.get("dual") else None,
                              "basis": "1616 ops per compression (1024 ALU-only + 592 two-input additions) vs the "
                                       "measured LOP3+IMAD dual-issue rate"},
                "hbm": {"achieved": round(hbm_gbs, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(hbm_gbs / hbm_peak, 4), "peak_source": hbm_src},
                "share_of_step": round(hash_avg_ms / ms_per_step, 4)}

    if a.suite == 2 and not a.varlen and a.entry_len == 32 and hash_avg_ms and peaks.get("lds"):
        # Suite 2 is bound by the AES T-table lookups (shared memory, one
        # 32-bit LDS per lookup): 17 AES-128 per entry (onetime_seed's second
        # MMO block - the first is hoisted per epoch - and 2 x 4 MDC-2 blocks of
        # 2 AES), each 160 state + 40 key-schedule lookups.
        LOOKUPS = 17 * 200
        rate = n / (hash_avg_ms * 1e-3)
        achieved = LOOKUPS * rate / 1e12
        peak = peaks["lds"] / 1e12
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf):
            tj = json.load(open(tf)).get("k_hash_s2")
            if tj and tj.get("entries") == n:
                traffic = tj["dram_bytes"]
        roof = {"bound": "shared-memory table lookups (LSU)", "kernel": "k_hash_s2_l32", "achieved": round(achieved, 3),
                "peak": round(peak, 3), "unit": "T lookups/s (32-bit LDS lanes)", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_unit": "bytes per launch (dram read + write, ncu --set full)",
                "algorithmic_bytes": payload_bytes, "ops_per_entry": LOOKUPS,
                "ops_basis": "17 AES-128 per 32-byte entry x (10 rounds x 16 T-table + 10 x 4 key-schedule lookups)",
                "ms_per_launch": round(hash_avg_ms, 4),
                "peak_source": "measured live: data-dependent LDS chains on a bank-replicated 256 x 32 table "
                               "(paper_2506_08781_b200/csrc/microbench.cu mode 10)",
                "alu_pipe": {"peak": round(peaks["alu"] / 1e12, 2), "unit": "Tops/s",
                             "note": "co-bound: PRMT byte picks, rotations and XORs of the rounds"},
                "share_of_step": round(hash_avg_ms / ms_per_step, 4)}

    if roof is not None and stage_ms:
        # device stage times of a step (C-ABI events on its stream): seed (K0), hash (K1+K2, with
        # the pipelined per-epoch checks when they overlap it), finalize, sum, group (K3), total
        roof["stages_ms"] = {k: round(statistics.mean(x[k] for x in stage_ms), 4) for k in stage_ms[0]}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "entries/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (counter-based log, include/poslo_synth.h); keys and signatures by the reference's kg/sig_epoch derivation, on the device",
        "config": config_dict(a, world),
        "e2e": e2e,
        **({"e2e_records": records} if records else {}),
        "roofline": roof,
        "gpu_launches": launches,
        "verdict": bool(ok),
        "clocks": clk.summary(),
        "log2_value": round(__import__("math").log2(value), 3),
    }
    if world == 1 and not a.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(a)
        except Exception as e:  # reported, never silently replaced
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
