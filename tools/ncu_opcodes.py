"""Executed SASS instructions by opcode for one kernel of an ncu report.
Usage: python tools/ncu_opcodes.py report.ncu-rep kernel-regex"""
import collections
import csv
import io
import subprocess
import sys


def main(path, kre):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    agg = collections.Counter()
    tot = 0
    seen_kernel = 0
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            seen_kernel += 1
            if seen_kernel > 1:
                break
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            try:
                n = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            op = d["Source"].strip().split()
            if not op:
                continue
            o = op[0]
            if o.startswith("@"):
                o = op[1] if len(op) > 1 else o
            o = o.split(".")[0]
            agg[o] += n
            tot += n
    print(f"total {tot}")
    for o, n in agg.most_common(30):
        print(f"{o:12s} {n:12d} {100 * n / tot:5.1f}%")


if __name__ == "__main__":
    main(*sys.argv[1:])
