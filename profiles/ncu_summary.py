"""Compact summary of ncu --set full captures: one block per kernel launch.

  python profiles/ncu_summary.py gpurun_out/full_*.ncu-rep > profiles/rNN_ncu_full_summary.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__ops_path_tensor_src_tf32_dst_fp32.avg.pct_of_peak_sustained_elapsed", "tf32 ops % of peak"),
    ("sm__ops_path_tensor_src_bf16_dst_fp32.avg.pct_of_peak_sustained_elapsed", "bf16 ops % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(f"{path}: no data")
        return
    head, units = rows[0], rows[1]
    for row in rows[2:]:
        d = dict(zip(head, row))
        u = dict(zip(head, units))
        print(f"== {path}  launch {d.get('ID')}  {d.get('Kernel Name', '')[:90]}")
        for k, name in KEYS:
            if k in d:
                print(f"   {name:34s} {d[k]:>14s} {u.get(k, '')}")
        st = [(float(d[k]), k[len(STALLS):].replace("_per_issue_active.ratio", ""))
              for k in d if k.startswith(STALLS) and k.endswith("_per_issue_active.ratio") and d[k]]
        st.sort(reverse=True)
        print("   top stalls (warps per issue):   " + ", ".join(f"{n} {v:.2f}" for v, n in st[:5]))


for p in sys.argv[1:]:
    summarize(p)
