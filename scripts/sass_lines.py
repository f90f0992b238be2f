"""Attribute ncu SASS-level samples / executed instructions to CUDA source lines.

usage: python scripts/sass_lines.py <sass.csv from ncu --page source --print-source=sass>
       <nvdisasm --print-line-info dump> <kernel-mangled-substring> [topN]
"""
import collections, csv, re, sys

sass_csv, dis, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
lines = open(dis).read().splitlines()
start = next(k for k, l in enumerate(lines) if l.startswith("//----") and ".text." in l and kname in l)
end = next((k for k in range(start + 1, len(lines)) if lines[k].startswith("//----")), len(lines))
cur = None
off2line = {}
for l in lines[start:end]:
    m = re.search(r'line (\d+)', l)
    if l.strip().startswith("//## File") and m:
        cur = int(m.group(1))
    m2 = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m2 and cur is not None:
        off2line[int(m2.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
data = rows[2:]
iA, iS, iE = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][iA], 16)
samp = collections.Counter(); ex = collections.Counter()
for r in data:
    off = int(r[iA], 16) - base
    ln = off2line.get(off, -1)
    if r[iS].isdigit():
        samp[ln] += int(r[iS])
    if r[iE].isdigit():
        ex[ln] += int(r[iE])
tot = sum(samp.values())
for ln, c in samp.most_common(top):
    print(f"line {ln:5d}: {100 * c / tot:5.1f}% samples, {ex[ln]:>12d} instr")
