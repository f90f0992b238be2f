"""Attribute an ncu source-page capture (SASS) to source line ranges.

usage: sass_regions.py REP.ncu-rep OBJ.o KERNEL_SUBSTR SRC.cu [norm]
Regions are the top-level functions of SRC (detected from lines starting a
definition); prints executed instructions and stall samples per region and the
hottest lines.  norm divides instruction counts (e.g. warps * iterations).
"""
import collections, csv, os, re, subprocess, sys, tempfile

rep, obj, kname, srcf = sys.argv[1:5]
norm = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
               capture_output=True)
cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "--print-line-info", os.path.join(tmp, cubin)],
                     capture_output=True, text=True).stdout.splitlines()
start = next(k for k, l in enumerate(dis) if l.startswith("//----") and ".text." in l and kname in l)
end = next((k for k in range(start + 1, len(dis)) if dis[k].startswith("//----")), len(dis))
cur = None
off2line = {}
base_file = os.path.basename(srcf)
for l in dis[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m2 and cur is not None:
        off2line[int(m2.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = next(k for k, r in enumerate(rows) if "Address" in r)
hdr, data = rows[hi], rows[hi + 1:]
iA, iE = hdr.index("Address"), hdr.index("Instructions Executed")
iS = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][iA], 16)
src = {}
for f in {v[0] for v in off2line.values()}:
    for d in (os.path.dirname(srcf),):
        p = os.path.join(d, f)
        if os.path.exists(p):
            src[f] = open(p).read().splitlines()
# function regions: lines matching a function header in each file
regions = {}
for f, lines in src.items():
    heads = [(k + 1, re.sub(r"\s*\(.*", "", l).split()[-1])
             for k, l in enumerate(lines)
             if re.match(r"^(template|__device__|__global__|  __device__|struct)", l) is None and False]
    hs = []
    for k, l in enumerate(lines):
        m = re.match(r"^\s*(?:__device__|__global__).*?(\w+)\s*\(", l)
        if m and not l.strip().endswith(";"):
            hs.append((k + 1, m.group(1)))
    regions[f] = hs
def region(fl):
    f, ln = fl
    hs = regions.get(f, [])
    name = f
    for s, n in hs:
        if s <= ln:
            name = f"{f}:{n}"
    return name
ex, sa = collections.Counter(), collections.Counter()
exl, sal = collections.Counter(), collections.Counter()
for r in data:
    fl = off2line.get(int(r[iA], 16) - base, ("?", 0))
    e = int(r[iE]) if r[iE].isdigit() else 0
    s = int(r[iS]) if r[iS].isdigit() else 0
    ex[region(fl)] += e
    sa[region(fl)] += s
    exl[fl] += e
    sal[fl] += s
T, S = sum(ex.values()), max(1, sum(sa.values()))
print(f"total instr {T}  per-norm {T / norm:.0f}")
for n, c in ex.most_common():
    print(f"{n:40s} {100 * c / T:5.1f}% instr {c / norm:8.0f}/norm  {100 * sa[n] / S:5.1f}% stall")
print("--- hottest lines")
for fl, c in exl.most_common(25):
    f, ln = fl
    txt = src.get(f, [""] * (ln + 1))[ln - 1].strip()[:70] if ln > 0 and f in src else ""
    print(f"{f}:{ln:<5d} {100 * c / T:5.1f}% ex {100 * sal[fl] / S:5.1f}% st  {txt}")
