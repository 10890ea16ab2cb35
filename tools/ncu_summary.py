"""Summarise ncu --set full captures as a markdown table (development):
python tools/ncu_summary.py a.ncu-rep b.ncu-rep ... > summary.md"""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("sm__cycles_elapsed.avg.per_second", "SM clock"),
        ("dram__bytes_read.sum", "DRAM read"), ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe %"),
        ("smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "DMMA cycles"),
        ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
print("| capture | kernel | " + " | ".join(k[1] for k in KEYS) + " |")
print("|" + "---|" * (len(KEYS) + 2))
for rep in sys.argv[1:]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")[-48:]
        cells = []
        for k, _ in KEYS:
            # section-prefixed names (e.g. TPC.TriageCompute.<metric>) match by suffix
            hk = k if k in d else next((h for h in hdr if h.endswith("." + k)), None)
            v = d.get(hk, "") if hk else ""
            cells.append(f"{v} {u.get(hk, '')}".strip() if v else "-")
        print(f"| {rep.split('/')[-1]} | `{name}` | " + " | ".join(cells) + " |")
