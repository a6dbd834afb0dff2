"""Summarise an ncu --set full report (one block per kernel launch): duration, DRAM bytes and
throughput, SM / tensor-pipe utilisation, occupancy, registers, shared memory, top stall reasons.

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
want = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM by smem"),
    ("smsp__inst_executed.sum", "instructions (warp)"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]
# warp-stall breakdown: warps stalled on each reason per issue-active cycle (ncu's "Warp State")
SP, SS = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
stall = [i for i, x in enumerate(h) if x.startswith(SP) and x.endswith(SS)]
for r in rows[2:]:
    print("==", r[h.index("Kernel Name")][:110])
    for key, label in want:
        if key in h:
            i = h.index(key)
            print(f"  {label:28s} {r[i]:>14s} {units[i]}")
    def num(s):
        try:
            return float(str(s).replace(",", ""))
        except ValueError:
            return 0.0
    st = sorted(((num(r[i]), h[i][len(SP):-len(SS)]) for i in stall), reverse=True)[:6]
    print("  top stalls (warps/issue):   " + ", ".join(f"{n} {v:.2f}" for v, n in st))
