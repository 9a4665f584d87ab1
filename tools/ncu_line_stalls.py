"""Warp-stall samples of one kernel attributed to CUDA source lines.

    cuobjdump -xelf all paper_2003_05293_b200/_lib/libholospots_b200.so   # in a scratch dir
    nvdisasm -g hs_umma.sm_100a.cubin > umma.dis
    ncu -i report.ncu-rep --page source --csv > src.csv
    python tools/ncu_line_stalls.py umma.dis <mangled kernel name> src.csv [top]

ncu's source page (SASS view) carries per-instruction stall samples with
absolute addresses; `nvdisasm -g` gives each SASS offset's file:line.  The
report must come from the same build as the disassembled cubin.  Reads
files only (no GPU).
"""
import collections
import csv
import re
import sys

dis, func, csvf = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
lines = open(dis).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('.text.' + func + ':')][0]
cur, addr2line = None, {}
for l in lines[start + 1:]:
    if l.startswith('//---------------------') and '.text.' in l:
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]+)\*/\s+[@A-Z]', l)
    if m and cur:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvf)))
hdr = rows[1]
ai, si = hdr.index('Address'), hdr.index('Warp Stall Sampling (All Samples)')
ii = hdr.index('Instructions Executed')
base, tot = None, 0
agg, inst = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        a, s, n = int(r[ai], 16), int(r[si] or 0), int(r[ii] or 0)
    except (ValueError, IndexError):
        continue
    if base is None:
        base = a
    ln = addr2line.get(a - base, ('?', 0))
    agg[ln] += s
    inst[ln] += n
    tot += s
print(f"total samples {tot}, mapped SASS offsets {len(addr2line)}")
for ln, s in agg.most_common(top):
    print(f"{s / max(tot, 1) * 100:5.1f}%  {ln[0]}:{ln[1]}  inst={inst[ln]}")
