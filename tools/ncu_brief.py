"""Key metrics of an ncu --set full report: duration, throughput, occupancy,
stall breakdown, pipe utilisation, DRAM bytes.  Usage:
    python tools/ncu_brief.py report.ncu-rep [kernel-regex]"""
import csv
import io
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
        "launch__block_size", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_tmem_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]


def main(path, kre=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    for r in rows[2:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", "")
        if kre and not re.search(kre, name):
            continue
        print("==", name[:110])
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]}")
        st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v.replace(",", "") or 0))
              for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k
              and v]
        tot = sum(v for _, v in st) or 1
        print("   stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in sorted(st, key=lambda t: -t[1])[:7]))


if __name__ == "__main__":
    main(*sys.argv[1:])
