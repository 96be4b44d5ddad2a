"""Attribute ncu SASS-page samples/instructions to source functions and lines.
usage: python scripts/sass_lines.py OBJ.o KERNEL_SUBSTR SASS.csv SRC.cu [top]
(SASS.csv = ncu -i R.ncu-rep --page source --csv --print-source sass)"""
import collections, csv, os, re, subprocess, sys, tempfile

obj, ksub, sass_csv, src = sys.argv[1:5]
top = int(sys.argv[5]) if len(sys.argv) > 5 else 25
tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith('.cubin')][0]
dis = subprocess.run(['nvdisasm', '-gi', '-c', cub], capture_output=True, text=True).stdout.splitlines()
srcbase = os.path.basename(src)
# offset -> innermost line within src
in_k, pending, line_of = False, [], {}
for L in dis:
    if L.startswith('.text.'):
        in_k = ksub in L
        continue
    if not in_k:
        continue
    if L.strip().startswith('//## File'):
        pending.append(L)
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', L)
    if m:
        off = int(m.group(1), 16)
        best = None
        for c in pending:  # innermost first
            for f, ln in re.findall(r'File "([^"]+)", line (\d+)', c):
                if os.path.basename(f) == srcbase and best is None:
                    best = int(ln)
        if best is not None:
            line_of[off] = best
        elif off - 16 in line_of:
            line_of[off] = line_of[off - 16]
        pending = []
# function ranges in src
lines = open(src).read().splitlines()
funcs = []
for i, t in enumerate(lines, 1):
    m = re.match(r'^(?:static\s+)?(?:__global__|__device__)[^(]*?\b(\w+)\s*\(', t)
    if m and not t.rstrip().endswith(';'):
        funcs.append((i, m.group(1)))
def func_of(ln):
    name = '?'
    for s, f in funcs:
        if s <= ln:
            name = f
    return name
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ci, cs = hdr.index('Instructions Executed'), hdr.index('Warp Stall Sampling (All Samples)')
base = int(rows[2][0], 16)
byf, byl = collections.defaultdict(lambda: [0., 0.]), collections.defaultdict(lambda: [0., 0.])
T = [0., 0.]
for r in rows[2:]:
    if len(r) <= cs:
        continue
    off = int(r[0], 16) - base
    i, s = float(r[ci] or 0), float(r[cs] or 0)
    ln = line_of.get(off, -1)
    byf[func_of(ln)][0] += i; byf[func_of(ln)][1] += s
    byl[ln][0] += i; byl[ln][1] += s
    T[0] += i; T[1] += s
print(f"{'function':24s} {'instr%':>7s} {'stall%':>7s}")
for f, (i, s) in sorted(byf.items(), key=lambda kv: -kv[1][1]):
    print(f"{f:24s} {100*i/T[0]:7.1f} {100*s/T[1]:7.1f}")
print()
for ln, (i, s) in sorted(byl.items(), key=lambda kv: -kv[1][1])[:top]:
    txt = lines[ln - 1].strip()[:80] if 0 < ln <= len(lines) else ''
    print(f"{ln:5d} {100*i/T[0]:6.1f} {100*s/T[1]:6.1f}  {txt}")
