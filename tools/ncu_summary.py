"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
per-kernel table: launches, total ms, share.  Usage:
    python tools/ncu_summary.py gpurun_out/launches.csv [out.md]"""
import collections
import csv
import sys


def main(path, out=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        ms = {"ns": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "nsecond": v / 1e6, "ms": v, "msecond": v}.get(unit, v)
        name = d["Kernel Name"]
        name = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list: {path}", "", f"total device time {tot:.2f} ms over "
             f"{sum(v[0] for v in agg.values())} launches (serialised, cold-cache; compare shares)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k[:80]}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% |")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
