"""Per-source-line warp-stall samples of an ncu --set full capture of the tcgen05 kernel.

    python scripts/ncu_lines.py REP [LIB] [N]

Maps each SASS address of the capture's source page to its CUDA file:line with nvdisasm -g
on the kernel's cubin extracted from LIB (default paper_2605_01858_b200/libdscache.so; it
must be the library that was profiled) and prints the top N lines by samples with their
top stall reasons.
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2605_01858_b200/libdscache.so"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True).stdout.decode("latin-1")
rows = list(csv.reader(io.StringIO(txt)))
kname = rows[0][1]
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
# address -> line from the cubin
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
addr_line = {}
want = "attn_fa_kernel"
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    if want not in dis:
        continue
    cur_fn, cur_line = None, None
    for ln in dis.splitlines():
        m = re.match(r"\s*\.text\.(\S+):", ln)
        if m:
            cur_fn = m.group(1)
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            # inlined helper: report the kernel line it was called from
            mi = re.findall(r'inlined at "([^"]+)", line (\d+)', ln)
            if mi and os.environ.get("OUTER", "1") == "1":
                cur_line = f"{os.path.basename(mi[-1][0])}:{mi[-1][1]}"
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur_fn and want in cur_fn:
            addr_line[int(m.group(1), 16)] = cur_line
agg = defaultdict(lambda: defaultdict(float))
tot = 0.0
base = None
for r in rows[2:]:
    try:
        a = int(r[ix["Address"]], 16) if r[ix["Address"]].startswith("0x") else int(r[ix["Address"]])
        if base is None:
            base = a
        a -= base
        v = float(r[ix["Warp Stall Sampling (All Samples)"]])
    except (ValueError, IndexError, KeyError):
        continue
    line = addr_line.get(a, "?")
    agg[line]["_all"] += v
    tot += v
    for h in reasons:
        try:
            agg[line][h] += float(r[ix[h]])
        except ValueError:
            pass
print(f"{kname[:70]}: {tot:.0f} samples, {len(addr_line)} mapped addresses")
src_cache = {}
for line, d in sorted(agg.items(), key=lambda kv: -kv[1]["_all"])[:N]:
    top = sorted(((v, h[6:]) for h, v in d.items() if h != "_all"), reverse=True)[:3]
    code = ""
    if ":" in line:
        f, l = line.split(":")
        for path in glob.glob(f"paper_2605_01858_b200/csrc/{f}"):
            src_cache.setdefault(path, open(path).read().splitlines())
            code = src_cache[path][int(l) - 1].strip()[:70]
    print(f"{100 * d['_all'] / tot:5.1f}% {line:22s} {', '.join(f'{n} {100 * v / max(d[chr(95) + chr(97) + chr(108) + chr(108)], 1):.0f}%' for v, n in top):45s} {code}")
