"""Aggregate an ncu SASS source page (CSV) by CUDA source line.

usage: python scripts/ncu_lines.py REPORT.ncu-rep CUBIN_NAME KERNEL_SUBSTR [N]
  CUBIN_NAME: the cubin inside libjsvd.so (e.g. batched.sm_100a.cubin); set
  JSVD_PROFILED_LIB to the exact .so that was profiled if the tree was rebuilt
Prints the top-N source lines by warp-stall samples with executed-instruction
counts (warp level) -- the map from profile to code used for the notes under
profiles/.  Needs ncu, cuobjdump and nvdisasm (no GPU)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, cub, ksub = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
LIB = os.environ.get("JSVD_PROFILED_LIB") or os.path.join(os.path.dirname(__file__), "..",
                                                          "paper_2202_08361_b200", "libjsvd.so")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ist, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Instructions Executed")
isrc = hdr.index("Source")
prof = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        prof.append((int(r[ia], 16), float(r[ist] or 0), float(r[iex] or 0), r[isrc]))
    except ValueError:
        pass
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", cub, os.path.abspath(LIB)], cwd=tmp, capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
line_of, cur, inside = {}, None, False
for l in dis.splitlines():
    if l.startswith("\t.text.") or l.startswith(".text."):
        pass
    m = re.match(r'\s*\.section\s+\.text\.(\S+),', l)
    if m:
        inside = ksub in m.group(1)
        continue
    if not inside:
        continue
    m = re.search(r'File "[^"]*/([^"/]+)", line (\d+)', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        line_of[int(m.group(1), 16)] = cur
base = min(a for a, _, _, _ in prof)  # ncu reports absolute addresses
prof = [(a - base, s, e, t) for a, s, e, t in prof]
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot_s = tot_e = 0.0
for a, s, e, _ in prof:
    k = line_of.get(a, "?")
    agg[k][0] += s
    agg[k][1] += e
    tot_s += s
    tot_e += e
print(f"total stall samples {tot_s:.0f}, executed warp instructions {tot_e:.3e}")
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{100*s/tot_s:6.2f}% stalls {100*e/tot_e:6.2f}% instr  {k}")
