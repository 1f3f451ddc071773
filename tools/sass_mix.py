#!/usr/bin/env python
"""Instruction mix and stall samples by SASS opcode class from an
`ncu --page source --csv` export (the SASS view).  usage: sass_mix.py file.csv"""
import collections
import csv
import sys

CLS = [("fp32", ("FFMA", "FADD", "FMUL", "FMNMX", "FSEL", "FSETP")), ("mufu", ("MUFU",)),
       ("lds/sts", ("LDS", "STS")), ("ldg/stg", ("LDG", "STG", "LDGSTS", "LDGDEPBAR", "DEPBAR")),
       ("bar/sync", ("BAR", "WARPSYNC", "NANOSLEEP")), ("shfl", ("SHFL",)),
       ("int/addr", ("IMAD", "IADD3", "LOP3", "SHF", "LEA", "ISETP", "IABS", "SEL", "PRMT", "IMNMX", "VIADD",
                     "VIMNMX", "I2F", "F2I", "LOP", "MOV", "S2R", "CS2R", "ULDC", "UMOV", "LDC", "UIADD3", "ULOP3",
                     "USHF", "ULEA", "UIMAD", "S2UR", "R2UR", "UISETP", "USEL", "UPRMT", "F2F", "I2FP", "F2IP",
                     "POPC", "FLO", "BREV", "PLOP3", "P2R", "R2P", "VOTE", "UMOV")),
       ("control", ("BRA", "EXIT", "BSYNC", "BSSY", "CALL", "RET", "BMOV", "YIELD", "NOP", "WARPSYNC"))]


def cls_of(op):
    for name, ops in CLS:
        if op in ops:
            return name
    return "other:" + op


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {c: i for i, c in enumerate(h)}
    ins = collections.Counter()
    smp = collections.Counter()
    tot_i = tot_s = 0
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        src = r[ix["Source"]].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        n = float(r[ix["Instructions Executed"]] or 0)
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        c = cls_of(op)
        ins[c] += n
        smp[c] += s
        tot_i += n
        tot_s += s
    print(f"{path}: {tot_i / 1e6:.1f}M warp-instructions")
    for c, n in ins.most_common():
        print(f"  {c:14s} inst {100 * n / tot_i:5.1f}%   stall-samples {100 * smp[c] / max(tot_s, 1):5.1f}%")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
