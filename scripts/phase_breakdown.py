"""Per-phase breakdown of a kernel from an ncu capture -- the paper's Fig 5.4
(spade norms, club dots, heart test + Grammian, diamond EVD, star
rotations) for this repo's kernels.

usage: python scripts/phase_breakdown.py REPORT.ncu-rep CUBIN KERNEL_SUBSTR SOURCE.cu [LIB]

Each SASS instruction is attributed to its OUTERMOST source line in SOURCE.cu
(nvdisasm -gi follows the inlining chain), and each line to the phase whose
`// @phase NAME` marker precedes it in SOURCE.cu.  Prints, per phase, the share
of the warp-stall samples (where the warps spend their cycles) and of the
executed warp instructions.  Needs ncu, cuobjdump, nvdisasm (no GPU)."""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, cub, ksub, src = sys.argv[1:5]
lib = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(__file__), "..",
                                                         "paper_2202_08361_b200", "libjsvd.so")
srcname = os.path.basename(src)
phase_of_line, cur = {}, "prologue"
for i, l in enumerate(open(src), 1):
    m = re.search(r"//\s*@phase\s+(\S+)", l)
    if m:
        cur = m.group(1)
    phase_of_line[i] = cur

out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, ist, iex = (hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"),
                hdr.index("Instructions Executed"))
prof = []
for r in rows[2:]:
    try:
        prof.append((int(r[ia], 16), float(r[ist] or 0), float(r[iex] or 0)))
    except (ValueError, IndexError):
        pass
base = min(a for a, _, _ in prof)

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", cub, os.path.abspath(lib)], cwd=tmp, capture_output=True)
dis = subprocess.run(["nvdisasm", "-gi", os.path.join(tmp, cub)], capture_output=True,
                     text=True).stdout
line_at, inside, pending, last, saw_loc = {}, False, [], None, False
# (an instruction with no location in SOURCE keeps last = None: "outside")
for l in dis.splitlines():
    m = re.match(r"\s*\.section\s+\.text\.(\S+),", l)
    if m:
        inside = ksub in m.group(1)
        pending, last = [], None
        continue
    if not inside:
        continue
    if "//##" in l:
        saw_loc = True
        for f, n in re.findall(r'"([^"]+)", line (\d+)', l):
            if os.path.basename(f) == srcname:
                pending.append(int(n))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        line_at[int(m.group(1), 16)] = pending[-1] if pending else (last if not saw_loc else None)
        if pending:
            last = pending[-1]
        pending, saw_loc = [], False

agg = collections.defaultdict(lambda: [0.0, 0.0])
ts = te = 0.0
for a, s, e in prof:
    ln = line_at.get(a - base)
    ph = phase_of_line.get(ln, "prologue") if ln else f"outside {srcname}"
    agg[ph][0] += s
    agg[ph][1] += e
    ts += s
    te += e
order = list(dict.fromkeys(phase_of_line.values()))
print(f"{ksub}: {ts:.0f} stall samples, {te:.3e} warp instructions")
print(f"{'phase':28s} {'cycles (stall samples)':>24s} {'instructions':>14s}")
for ph in order + [p for p in agg if p not in order]:
    if ph in agg:
        s, e = agg[ph]
        print(f"{ph:28s} {100 * s / ts:23.1f}% {100 * e / te:13.1f}%")
