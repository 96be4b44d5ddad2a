"""Stall-reason breakdown per source function from an ncu SASS page CSV.
usage: python scripts/sass_stalls.py OBJ.o KERNEL_SUBSTR SASS.csv SRC.cu"""
import collections, csv, os, re, subprocess, sys, tempfile
obj, ksub, sass_csv, src = sys.argv[1:5]
tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith('.cubin')][0]
dis = subprocess.run(['nvdisasm', '-gi', '-c', cub], capture_output=True, text=True).stdout.splitlines()
srcbase = os.path.basename(src)
in_k, pending, line_of, op_of = False, [], {}, {}
for L in dis:
    if L.startswith('.text.'):
        in_k = ksub in L
        continue
    if not in_k:
        continue
    if L.strip().startswith('//## File'):
        pending.append(L); continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)', L)
    if m:
        off = int(m.group(1), 16)
        op_of[off] = m.group(3).split('.')[0]
        best = None
        for c in pending:
            for f, ln in re.findall(r'File "([^"]+)", line (\d+)', c):
                if os.path.basename(f) == srcbase and best is None:
                    best = int(ln)
        if best is not None: line_of[off] = best
        elif off - 16 in line_of: line_of[off] = line_of[off - 16]
        pending = []
lines = open(src).read().splitlines()
funcs = []
for i, t in enumerate(lines, 1):
    m = re.match(r'^(?:static\s+)?(?:__global__|__device__)[^(]*?\b(\w+)\s*\(', t)
    if m and not t.rstrip().endswith(';'): funcs.append((i, m.group(1)))
def func_of(ln):
    name = '?'
    for s, f in funcs:
        if s <= ln: name = f
    return name
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
reasons = [h for h in hdr if h.startswith('stall_') and '(' not in h]
ri = [hdr.index(h) for h in reasons]
ci = hdr.index('Instructions Executed')
base = int(rows[2][0], 16)
byf = collections.defaultdict(lambda: collections.Counter())
byop = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows[2:]:
    if len(r) <= max(ri): continue
    off = int(r[0], 16) - base
    f = func_of(line_of.get(off, -1))
    op = op_of.get(off, '?')
    ins = float(r[ci] or 0)
    byf[f]['inst'] += ins; byop[op]['inst'] += ins; tot['inst'] += ins
    for h, i in zip(reasons, ri):
        v = float(r[i] or 0)
        byf[f][h] += v; byop[op][h] += v; tot[h] += v
show = [h for h in reasons if tot[h] > 0.01 * sum(tot[x] for x in reasons)]
def table(d, title, top=18):
    print(f"{title:18s} {'inst%':>6s} " + " ".join(f"{h[6:]:>9s}" for h in show))
    for k, c in sorted(d.items(), key=lambda kv: -sum(kv[1][h] for h in reasons))[:top]:
        print(f"{k[:18]:18s} {100*c['inst']/tot['inst']:6.1f} " + " ".join(f"{100*c[h]/max(1,sum(tot[x] for x in reasons)):9.2f}" for h in show))
table(byf, 'function')
print()
table(byop, 'opcode')
