"""Top source lines of an ncu report by stall samples (needs -lineinfo).
Usage: python tools/ncu_lines.py report.ncu-rep [kernel-regex] [N]"""
import csv
import io
import subprocess
import sys


def main(path, kre=None, n=40):
    args = ["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kre:
        args += ["-k", f"regex:{kre}"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, hdr, recs = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            d["Source"] = r[1]
            try:
                s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
                ins = int(d.get("Instructions Executed", "0") or 0)
            except ValueError:
                continue
            if (s or ins) and d["Line No"].isdigit():
                stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and v.isdigit() and int(v)}
                top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
                recs.append((s, ins, fname, d["Line No"], d["Source"].strip()[:70], top))
    agg = {}
    for s_, ins, f, ln, src, top in recs:
        k = (f, ln)
        if k not in agg:
            agg[k] = [0, 0, src, {}]
        agg[k][0] += s_
        agg[k][1] += ins
        for name, v in top:
            agg[k][3][name] = agg[k][3].get(name, 0) + v
    recs = [(v[0], v[1], k[0], k[1], v[2], sorted(v[3].items(), key=lambda kv: -kv[1])[:3]) for k, v in agg.items()]
    tot = sum(r[0] for r in recs) or 1
    toti = sum(r[1] for r in recs) or 1
    print(f"total samples {tot}, warp-instructions {toti}")
    import os
    key = (lambda r: -r[1]) if os.environ.get("SORT") == "ins" else (lambda r: -r[0])
    for s, ins, f, ln, src, top in sorted(recs, key=key)[:int(n)]:
        print(f"{100*s/tot:5.1f}% {100*ins/toti:5.1f}%i {f}:{ln:5s} {src:70s} {top}")


if __name__ == "__main__":
    main(*sys.argv[1:])
