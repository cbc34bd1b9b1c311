"""One-line-per-kernel summary of an ncu --set full report (key roofline metrics).
Usage: python scripts/ncu_summary.py report.ncu-rep > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "hmma_active_cyc"),
    ("sm__cycles_active.avg", "sm_active_cyc"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "tma_ld_bytes"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn_smem"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
]
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
print(f"# ncu --set full summary of {rep.split('/')[-1]}")
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0]
    parts = [name]
    for k, short in KEYS:
        if k in h:
            i = h.index(k)
            parts.append(f"{short}={r[i]}{u[i] if u[i] else ''}")
    print("  ".join(parts))
