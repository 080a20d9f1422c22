"""Attribute ncu warp-stall samples (SASS page) to CUDA source lines.

usage: python scripts/ncu_lines.py <report.ncu-rep> <kernel-mangled-name> <lib.so> [top] [demangled substring]
Needs -lineinfo builds; maps SASS offsets through nvdisasm --print-line-info.
"""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

rep, kname, lib = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# one section per profiled kernel: ["Kernel Name", name], header, rows...
# section filter: demangled-name substring (argv[5]); default the mangled name
kname_plain = sys.argv[5] if len(sys.argv) > 5 else kname
samples = []
take = False
hdr = ix = None
for r in rows:
    if r and r[0] == "Kernel Name":
        take = len(r) > 1 and kname_plain in r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        continue
    if not take or hdr is None or len(r) < len(hdr):
        continue
    samples.append((int(r[ix["Address"]], 16), int(r[ix["Warp Stall Sampling (All Samples)"]])))
base = min(a for a, _ in samples)
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
line_of = {}
for f in os.listdir(tmp):
    if not f.endswith(".cubin"):
        continue
    out = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, f)],
                         capture_output=True, text=True).stdout
    key = f".text.{kname}:"
    if key not in out:
        continue
    body = out.split(key, 1)[1].split(".text.", 1)[0]
    cur = None
    for ln in body.splitlines():
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            line_of[int(m.group(1), 16)] = cur
    break
agg = defaultdict(int)
for a, s in samples:
    agg[line_of.get(a - base, "?")] += s
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{100 * v / tot:6.2f}%  {k}")
