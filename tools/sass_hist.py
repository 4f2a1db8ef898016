"""Executed-instruction accounting from an ncu source-page export
(`ncu -i X.ncu-rep --page source --csv --print-source sass`): per-opcode warp-
and thread-level executed counts, grouped by the pipe that retires them on
sm_100 (ALU: LOP3 SHF IADD3 PRMT ISETP SEL LEA ...; FMA: IMAD*, VIADD ...),
normalised per unit of work (--units N, e.g. SHA-256 compressions or entries).

usage: python tools/sass_hist.py export.csv --units N [--top 30] [--json out.json]
"""
import argparse
import collections
import csv
import json
import re

# pipe of each opcode family on sm_100 (B200). ALU = the integer/logic pipe
# (16 lanes/clk/SMSP); FMA = the IMAD-capable pipe (16 lanes/clk/SMSP);
# the rest issue to LSU / uniform / branch units.
ALU = {"LOP3", "SHF", "IADD3", "PRMT", "ISETP", "SEL", "LEA", "PLOP3", "FLO", "POPC", "VIMNMX",
       "IMNMX", "BMSK", "SGXT", "LOP", "SHL", "SHR", "ICMP", "P2R", "R2P", "BREV", "IABS", "CSETP",
       "FSETP", "FSEL", "VIADDMNMX", "LEA_HI"}
FMA = {"IMAD", "VIADD", "IDP", "IDP4A", "FFMA", "FADD", "FMUL", "HFMA2", "IMUL"}
MOVE = {"MOV", "CS2R", "S2R", "S2UR"}
LSU = {"LDS", "STS", "LDG", "STG", "LDC", "LDCU", "ATOMS", "ATOMG", "RED", "LDSM", "SHFL", "LD", "ST",
       "LDL", "STL", "ULDC"}


def opcode(src: str) -> str:
    s = re.sub(r"^@!?U?P[T\d]+\s+", "", src.strip())
    return s.split()[0] if s else ""


def pipe(op: str) -> str:
    fam = op.split(".")[0]
    if fam.startswith("U"):
        return "uniform"
    if fam in ALU:
        return "alu"
    if fam in FMA:
        return "fma"
    if fam in LSU:
        return "lsu"
    if fam in MOVE:
        return "move"
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--units", type=float, required=True, help="work units (compressions, entries) of the launch")
    ap.add_argument("--unit-name", default="unit")
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--json")
    a = ap.parse_args()
    lines = open(a.csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rd = csv.DictReader(lines[start:])
    warp = collections.Counter()
    thread = collections.Counter()
    for r in rd:
        op = opcode(r.get("Source", ""))
        if not op:
            continue
        try:
            w = float(r["Instructions Executed"] or 0)
            t = float(r.get("Predicated-On Thread Instructions Executed") or r["Thread Instructions Executed"] or 0)
        except (KeyError, ValueError):
            continue
        fam = op.split(".")[0]
        warp[fam] += w
        thread[fam] += t
    by_pipe_w = collections.Counter()
    by_pipe_t = collections.Counter()
    for fam in warp:
        by_pipe_w[pipe(fam)] += warp[fam]
        by_pipe_t[pipe(fam)] += thread[fam]
    u = a.units
    print(f"per {a.unit_name} (units = {u:.6g}); warp-level instructions x 32 / units, and thread-level (pred-on) / units")
    for p in sorted(by_pipe_w, key=lambda p: -by_pipe_w[p]):
        print(f"  {p:8s} {32 * by_pipe_w[p] / u:9.1f} lane-slots   {by_pipe_t[p] / u:9.1f} thread-ops")
    print(f"  {'total':8s} {32 * sum(by_pipe_w.values()) / u:9.1f} lane-slots   {sum(by_pipe_t.values()) / u:9.1f} thread-ops")
    print("top opcodes:")
    for fam, w in warp.most_common(a.top):
        print(f"  {fam:10s} {pipe(fam):8s} {32 * w / u:9.1f} {thread[fam] / u:9.1f}")
    if a.json:
        json.dump({"units": u, "unit_name": a.unit_name,
                   "per_unit_lane_slots": {p: 32 * v / u for p, v in by_pipe_w.items()},
                   "per_unit_thread_ops": {p: v / u for p, v in by_pipe_t.items()},
                   "per_unit_opcode_lane_slots": {f: 32 * v / u for f, v in warp.items()}},
                  open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
