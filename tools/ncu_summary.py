"""Summarise an .ncu-rep (raw page) into the handful of numbers DESIGN.md / bench.py cite.
python tools/ncu_summary.py report.ncu-rep [more.ncu-rep ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64 pipe inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def main():
    for path in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")]
            print(f"== {path}: {name}")
            for key, label in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    print(f"   {label:24s} {r[i]} {units[i]}")
            stalls = []
            for i, k in enumerate(hdr):
                if "average_warps_issue_stalled" in k and "not_issued" not in k:
                    try:
                        v = float(r[i])
                    except ValueError:
                        continue
                    if v >= 0.1:
                        stalls.append((v, k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))


if __name__ == "__main__":
    main()
