"""Summarise an ncu --set full report (raw page) into a small text file for profiles/.
  python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/out.txt
"""
import csv
import re
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
pat = (r"^(Kernel Name|gpu__time_duration.sum|dram__bytes_(read|write).sum|"
       r"dram__throughput.avg.pct_of_peak_sustained_elapsed|lts__t_sectors.avg.pct_of_peak_sustained_elapsed|"
       r"lts__throughput.avg.pct_of_peak_sustained_elapsed|lts__t_bytes.sum.per_second|"
       r"sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_(active|elapsed)|"
       r"sm__throughput.avg.pct_of_peak_sustained_elapsed|l1tex__throughput.avg.pct_of_peak_sustained_elapsed|"
       r"sm__cycles_elapsed.avg.per_second|launch__registers_per_thread|launch__grid_size|launch__block_size|"
       r"launch__shared_mem_per_block_dynamic|smsp__average_warps_issue_stalled_\w+_per_issue_active.ratio)$")
with open(out, "w") as f:
    f.write(f"# ncu --set full summary of {rep}\n")
    for vals in rows[2:]:
        for h, u, v in zip(hdr, units, vals):
            if re.search(pat, h):
                f.write(f"{h} [{u}] {v}\n")
print(open(out).read())
