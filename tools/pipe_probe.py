"""Integer pipe-rate probe (microbench.cu modes 0-7) on cuda:0: prints lane-ops/s
and lanes/clk/SM for each instruction form. Feeds the pipe-balancing design of
the SHA-256 hash kernel."""
import ctypes
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2506_08781_b200", "libposlo_microbench.so"))
lib.poslo_microbench_int_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                          ctypes.POINTER(ctypes.c_double)]
names = {0: "LOP3", 1: "IMAD reg", 2: "LOP3+IMAD reg", 3: "IMAD imm", 4: "LOP3+IMAD imm",
         5: "SHF.R.W", 6: "IMAD.HI imm", 7: "LOP3+IMAD.HI imm", 8: "IMAD.WIDE acc64", 9: "LOP3+IMAD.WIDE",
         10: "LDS table lookup", 11: "LOP3+IMAD R-R-R", 12: "LOP3+add reg", 13: "LOP3+add UR",
         14: "LOP3(3R)+IMAD R-R-R", 15: "LOP3(3R)+IMAD R-UR-R"}
out = {}
for rep in range(2):
    for m, n in names.items():
        v, ms = ctypes.c_double(), ctypes.c_double()
        assert lib.poslo_microbench_int_peak(0, m, ctypes.byref(v), ctypes.byref(ms)) == 0
        out[n] = max(out.get(n, 0.0), v.value)
clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                     capture_output=True, text=True).stdout.strip()
for n, v in out.items():
    print(f"{n:20s} {v / 1e12:7.2f} Tops/s  {v / (148 * 1.965e9):6.1f} lanes/clk/SM @1965")
print(json.dumps({"probe": out, "sm_mhz_after": clk}))
