"""Summarise an ncu launch list + a --set full capture into profiles/ (committed).

    python scripts/summarize_profile.py TAG [config] [traffic key]

Reads gpurun_out/launches_TAG.csv, gpurun_out/prof_TAG.ncu-rep, gpurun_out/bench_TAG.json
and writes profiles/TAG_launches.md, profiles/TAG_ncu_full.md, profiles/TAG_bench.json and
updates profiles/ncu_traffic.json (DRAM bytes per attention launch, read by bench.py) under
the traffic key bench.traffic_key gives the profiled command (default "<config>|streams|
fused|boost0|world1|layerseq0").
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def launches(tag):
    path = os.path.join(G, f"launches_{tag}.csv")
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows[hdr_i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        agg[name][0] += 1
        agg[name][1] += us
        total += us
    out = ["| kernel | launches | total µs (ncu, cold, serialised) | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / total:.1f}% |")
    return "\n".join(out), agg


def ncu_raw(tag):
    rep = os.path.join(G, f"prof_{tag}.ncu-rep")
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "registers/thread (launch)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def main():
    tag = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c5"
    tkey = sys.argv[3] if len(sys.argv) > 3 else f"{cfg}|streams|fused|boost0|world1|layerseq0"
    os.makedirs(P, exist_ok=True)
    table, agg = launches(tag)
    open(os.path.join(P, f"{tag}_launches.md"), "w").write(
        f"# ncu launch list ({tag}): `{os.environ.get('LCMD', 'python bench.py --steps 2 --warmup 3 --no-cpu-baseline --config ' + cfg)}`\n\n"
        "`ncu --metrics gpu__time_duration.sum --clock-control none`; every kernel of the run "
        "(fill, warm-up, timed steps, e2e).  Per-launch times are cold-cache and serialised: "
        "compare shares, not absolutes.\n\n" + table + "\n")
    recs = ncu_raw(tag)
    kname = os.environ.get("KNAME", "attn_fa_kernel")
    lines = [f"# ncu --set full of {kname} ({tag}, {cfg})\n"]

    def section(recs, title, labels):
        lines.append(f"## {title}\n")
        lines.append("| metric | " + " | ".join(labels[:len(recs)]) + " |")
        lines.append("|---|" + "---|" * len(recs))
        for k, name in KEYS:
            vals = [r.get(k, "") for r in recs]
            lines.append(f"| {name} (`{k}`) | " + " | ".join(vals) + " |")
        stalls = []
        for r in recs:
            items = []
            for k, v in r.items():
                if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
                    try:
                        items.append((float(v.replace(",", "")), k[33:]))
                    except ValueError:
                        pass
            tot = sum(v for v, _ in items) or 1.0
            stalls.append(", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(items, reverse=True)[:6]))
        lines.append("\nTop warp-stall reasons (pc sampling): " + " / ".join(stalls) + "\n")

    section(recs, os.environ.get("STITLE", "Fused step launch (the bench's dominant kernel): `-k regex:attn_fa -s 4 -c 1`, "
            f"one {cfg} step = build_instant + attend items in one persistent launch"), [os.environ.get("SLABEL", "fused step")])
    split_rep = os.path.join(G, f"prof_split_{tag}.ncu-rep")
    if os.path.exists(split_rep):
        txt = subprocess.run(["ncu", "-i", split_rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        srecs = [dict(zip(rows[0], r)) for r in rows[2:]]
        section(srecs, "Split API (`--api split`, `-s 8 -c 2`): launch 1 = build_instant, launch 2 = attend",
                ["build_instant", "attend"])
    open(os.path.join(P, f"{tag}_ncu_full.md"), "w").write("\n".join(lines) + "\n")
    # DRAM traffic per launch for bench.py's roofline.traffic (units from the raw page: MB or GB)
    units = {}
    txt = subprocess.run(["ncu", "-i", os.path.join(G, f"prof_{tag}.ncu-rep"), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    units = dict(zip(rows[0], rows[1]))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def b(r, k):
        return float(r[k].replace(",", "")) * scale.get(units.get(k, "byte"), 1)
    per = [b(r, "dram__bytes_read.sum") + b(r, "dram__bytes_write.sum") for r in recs]
    tp = os.path.join(P, "ncu_traffic.json")
    d = json.load(open(tp)) if os.path.exists(tp) else {}
    d[tkey] = {"dram_bytes_per_launch": sum(per) / len(per), "per_launch": per, "tag": tag}
    json.dump(d, open(tp, "w"), indent=1)
    bj = os.path.join(G, f"bench_{tag}.json")
    if os.path.exists(bj):
        open(os.path.join(P, f"{tag}_bench.json"), "w").write(open(bj).read())
    print(open(os.path.join(P, f"{tag}_ncu_full.md")).read())
    print(table)


if __name__ == "__main__":
    main()
