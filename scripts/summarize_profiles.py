"""Copy the ncu evidence of a gpu_round.sh run from gpurun_out/ into profiles/:
the launch list, the selected raw metrics and the details pages of the
top-kernel captures. Usage: python scripts/summarize_profiles.py r01"""
import csv
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
           "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
           "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
           "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle"]

shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches_config5_step.csv"))
raw_rows, details = [], []
for rep in sorted(glob.glob(os.path.join(OUT, "prof_*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    d = dict(zip(h, v))
    u = dict(zip(h, units))

    def norm(m):
        # times in us, byte counts in MB (ncu scales units per row)
        x = d.get(m, "")
        try:
            val = float(x.replace(",", ""))
        except ValueError:
            return x
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6,
                 "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u.get(m, ""), 1.0)
        return f"{val * scale:.6g}"
    raw_rows.append([d.get("Kernel Name", "")] + [norm(m) for m in METRICS])
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    details.append(det)
with open(os.path.join(PROF, f"{tag}_top_kernels_raw.csv"), "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["Kernel Name"] + [m + (" [us]" if m.startswith("gpu__time") else " [MB]" if "bytes" in m else "")
                                  for m in METRICS])
    w.writerows(raw_rows)
with open(os.path.join(PROF, f"{tag}_top_kernels_details.csv"), "w") as f:
    f.write("\n".join(details))
print("wrote", len(raw_rows), "captures")
