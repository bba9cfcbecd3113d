"""Top stalled SASS instructions of an ncu --set full capture (source page, sass view).

    ncu -i REP --page source --csv --print-source sass > x.csv; python scripts/ncu_sass_hot.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        ks.append(cur)
        continue
    if cur is not None:
        cur.append(r)
reasons = ["stall_long_sb", "stall_wait", "stall_short_sb", "stall_math", "stall_mio", "stall_barrier", "stall_branch_resolving",
           "stall_no_inst", "stall_selected", "stall_not_selected", "stall_lg", "stall_dispatch", "stall_sleep", "stall_misc"]
for ki, k in enumerate(ks):
    hdr = k[0]
    ix = {h: i for i, h in enumerate(hdr)}
    data = []
    for idx, r in enumerate(k[1:]):
        try:
            v = int(r[ix["Warp Stall Sampling (All Samples)"]])
        except (ValueError, IndexError):
            continue
        data.append((v, idx, r))
    tot = sum(v for v, _, _ in data)
    agg = {x: sum(int(r[ix[x]] or 0) for _, _, r in data) for x in reasons}
    print(f"== kernel {ki}: {tot} samples; " + ", ".join(f"{x[6:]} {100*v/tot:.1f}%" for x, v in sorted(agg.items(), key=lambda t: -t[1])[:8]))
    for v, idx, r in sorted(data, key=lambda t: -t[0])[:N]:
        br = sorted(((int(r[ix[x]] or 0), x[6:]) for x in reasons), reverse=True)[:3]
        print(f"{100*v/tot:5.2f}% #{idx:5d} {r[ix['Source']].strip()[:60]:60s} " + " ".join(f"{n}:{c}" for c, n in br if c))
