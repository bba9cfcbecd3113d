"""Print the key metrics and top stall reasons of an ncu report: python scripts/ncu_summary.py REP [REP2 ...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem LSU wavefronts %"),
]


def recs(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    units = dict(zip(rows[0], rows[1]))
    return [dict(zip(rows[0], r)) for r in rows[2:]], units


for rep in sys.argv[1:]:
    rs, units = recs(rep)
    for r in rs:
        print(f"== {rep}: {r.get('Kernel Name', '')[:60]}")
        for k, n in KEYS:
            print(f"  {n:28s} {r.get(k, '')} {units.get(k, '')}")
        items = []
        for k, v in r.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                try:
                    items.append((float(v.replace(",", "")), k[33:]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1.0
        print("  stalls: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(items, reverse=True)[:8]))
