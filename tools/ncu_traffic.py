"""Per-tag DRAM traffic per launch from an ncu metrics CSV (--metrics
dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv),
written to profiles/ncu_traffic.json for bench.py's roofline `traffic` field.
A tag's launch is the group of kernels its ProfScope brackets (csrc), so the
per-launch traffic of a tag is the sum over its kernels divided by the tag's
launch count.  Usage: python tools/ncu_traffic.py launches.csv out.json"""
import collections
import csv
import json
import re
import sys

# kernel-name regex -> (tag, kernels per tag launch)
TAGS = [
    (r"k_normal_(rank|ws)", "sense_normal_y_cg"),
    (r"k_cg_update_r", "cg_update_rank"),
    (r"k_conv_tc_wgrad|k_wgrad_fold", "conv_tc_bwd_weight"),
    (r"k_conv_tc_t<\d+, 2>", "conv_tc_bwd_data"),
    (r"k_conv_tc_t<\d+, [01]>", "conv_tc_fwd"),
    (r"k_conv_tc(_pair)?<", "conv_tc_fwd_or_bwd_data"),
    (r"k_stats|k_stats_final|k_apply\b", "bnblock_fwd"),
    (r"k_bwd_reduce|k_bwd_final|k_bwd_apply", "bnblock_bwd"),
    (r"k_thin_wgrad|k_thin_wsum", "conv_thin_bwd_weight"),
    (r"k_thin_expand|k_thin_reduce", "conv_thin_fwd_or_bwd_data"),
    (r"k_fft_lines", "fft"),
]
# launches of each tag per ncu capture are counted from its anchor kernel
ANCHOR = {"sense_normal_y_cg": "k_normal_(rank|ws)", "cg_update_rank": "k_cg_update_r",
          "conv_tc_bwd_weight": "k_conv_tc_wgrad", "conv_tc_bwd_data": "k_conv_tc_t<\\d+, 2>",
          "conv_tc_fwd": "k_conv_tc_t<\\d+, [01]>", "conv_tc_fwd_or_bwd_data": "k_conv_tc(_pair)?<",
          "bnblock_fwd": "k_apply", "bnblock_bwd": "k_bwd_apply", "conv_thin_bwd_weight": "k_thin_wgrad",
          "conv_thin_fwd_or_bwd_data": "k_thin_(expand|reduce)", "fft": "k_fft_lines"}


def main(path, out):
    rows = list(csv.reader(open(path)))
    hdr = None
    per = collections.defaultdict(lambda: collections.defaultdict(float))  # launch id -> metric
    names = {}
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        lid = d["ID"]
        names[lid] = d["Kernel Name"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
        per[lid][d["Metric Name"]] = v * scale if "bytes" in d["Metric Name"] else v
    tot = collections.defaultdict(float)
    cnt = collections.defaultdict(int)
    for lid, m in per.items():
        n = names[lid]
        for rx, tag in TAGS:
            if re.search(rx, n):
                tot[tag] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                if re.search(ANCHOR[tag], n):
                    cnt[tag] += 1
                break
    res = {tag: tot[tag] / cnt[tag] for tag in tot if cnt[tag]}
    for a, b in (("conv_tc_fwd_or_bwd_data", ("conv_tc_fwd", "conv_tc_bwd_data")),
                 ("conv_thin_fwd_or_bwd_data", ("conv_thin_fwd", "conv_thin_bwd_data"))):
        if a in res:
            for t in b:
                res.setdefault(t, res[a])
    json.dump({k: round(v) for k, v in sorted(res.items())}, open(out, "w"), indent=1)
    print(json.dumps({k: f"{v / 1e6:.1f} MB" for k, v in sorted(res.items())}, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
