"""Summarise raw-page CSVs written by tools/round_profile.sh: python tools/ncu_summary_csv.py a.raw.csv ..."""
import csv
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.sum", "fp64 pipe inst"),
    ("sm__inst_executed_pipe_tensor_op_dmma.sum", "dmma inst"),
    ("sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active", "dmma pipe active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "sm clock"),
]
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    if len(rows) < 3:
        print(f"== {path}: empty")
        continue
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print(f"== {path}: {r[hdr.index('Kernel Name')]}")
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                print(f"   {label:24s} {r[i]} {units[i]}")
        extra = [h for h in hdr if "dmma" in h.lower() and h not in dict(KEYS)]
        for h in extra[:6]:
            print(f"   {h:24s} {r[hdr.index(h)]}")
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
