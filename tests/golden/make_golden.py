"""Regenerates tests/golden/*.json from the UNMODIFIED reference compiled in
oracle/_ref (make -f oracle/Makefile.ref). Run here, where /root/reference
exists; the fixtures are committed so the GPU box never needs the reference.

  kat.json          primitives / scalar / group known answers (ref_tool kat)
  stream_*.json     signed coarse streams from the real signer (kg/sig_epoch,
                    deterministic randombytes) with every verifier output:
                    per-epoch e~, e^, paver/aver, per-epoch verdicts,
                    distillation invalid list, CCD bytes, SeBVer V/U/I bits.
  fine_*.json       signed POSLO-F streams (kg/sig_one) with aver_f_single per
                    entry, aver_f_batch, fine distillation CCD and SeBVer bits.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
TOOL = os.path.join(HERE, "..", "..", "oracle", "_ref", "ref_tool")

# name: (suite, n1, n2, n_u, entry_len (0 = random 1..64 / 1..31), seed, tampered entries)
STREAMS = {
    "stream_s1_mixed": (1, 8, 4, 2, 0, 1, []),
    "stream_s1_tamper": (1, 16, 8, 4, 32, 2, [5, 77]),
    "stream_s1_n256": (1, 8, 256, 4, 32, 3, [1000]),
    "stream_s2_mixed": (2, 8, 4, 4, 0, 4, [9]),
    "stream_s2_len32": (2, 4, 64, 2, 32, 5, []),
    "stream_s3_mixed": (3, 4, 4, 2, 0, 6, [3]),
    "stream_s1_clean_big": (1, 32, 16, 8, 48, 7, []),
}

# scheme F (POSLO-F): name: (suite, n1, n2, n_u, entry_len, seed, bpv_v, bpv_k, tampered entries)
FINE = {
    "fine_s1_tamper": (1, 8, 8, 4, 32, 11, 0, 0, [3, 7, 40]),
    "fine_s1_mixed_bpv": (1, 8, 4, 2, 0, 12, 16, 4, [9]),
    "fine_s2_mixed": (2, 4, 4, 2, 0, 13, 0, 0, [2]),
    "fine_s3_mixed": (3, 4, 4, 4, 0, 14, 8, 3, [15]),
}


def run(args, out):
    with open(os.path.join(HERE, out), "w") as f:
        subprocess.check_call([TOOL] + [str(a) for a in args], stdout=f)


def main():
    run(["kat"], "kat.json")
    for name, (s, n1, n2, nu, ln, seed, tam) in STREAMS.items():
        run(["golden", s, n1, n2, nu, ln, seed] + tam, name + ".json")
    for name, (s, n1, n2, nu, ln, seed, bv, bk, tam) in FINE.items():
        run(["golden_f", s, n1, n2, nu, ln, seed, bv, bk] + tam, name + ".json")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    sys.exit(main())
