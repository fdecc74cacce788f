"""Summarise one `ncu --set full` capture into profiles/<round>/:
<name>_summary.json (key metrics + stall shares), <name>_details.csv (the
details page) and <name>_source_lines.txt (per-source-line instructions, stall
samples and shared-memory wavefronts).

usage: python tools/ncu_summary.py <rep.ncu-rep> <round> <name>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, rnd, name = sys.argv[1:4]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
out = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out, exist_ok=True)


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
summ = {k: [v[h.index(k)], u[h.index(k)]] for k in KEYS if k in h}
stalls = {k.split("issue_stalled_")[1].split("_per_issue_active")[0]: float(v[i].replace(",", ""))
          for i, k in enumerate(h)
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") and v[i]}
tot = sum(stalls.values()) or 1.0
summ["stall_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(stalls.items(), key=lambda kv: -kv[1]) if x / tot > 0.01}
summ["kernel"] = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
json.dump(summ, open(os.path.join(out, name + "_summary.json"), "w"), indent=1)
open(os.path.join(out, name + "_details.csv"), "w").write(ncu("--page", "details", "--csv"))
src = ncu("--page", "source", "--print-source", "cuda,sass", "--csv")
tmp = os.path.join(out, ".src.csv")
open(tmp, "w").write(src)
lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), tmp, "60"],
                       capture_output=True, text=True).stdout
smem = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_smem.py"), tmp],
                      capture_output=True, text=True).stdout
os.remove(tmp)
open(os.path.join(out, name + "_source_lines.txt"), "w").write(
    "# per source line: % of warp instructions, % of stall samples\n" + lines +
    "\n# per source line: shared-memory wavefronts (excess = bank conflicts)\n" + smem)
print(json.dumps(summ, indent=1))
