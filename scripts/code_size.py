"""Static SASS instruction count per source function (code-size audit):
python scripts/code_size.py OBJ.o SRC.cu"""
import collections, os, re, subprocess, sys, tempfile
obj, src = sys.argv[1:3]
tmp = tempfile.mkdtemp()
subprocess.run(['cuobjdump', '-xelf', 'all', os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith('.cubin')][0]
dis = subprocess.run(['nvdisasm', '-gi', '-c', cub], capture_output=True, text=True).stdout.splitlines()
lines = open(src).read().splitlines()
funcs = []
for i, t in enumerate(lines, 1):
    m = re.match(r'^(?:static\s+)?(?:__global__|__device__)[^(]*?\b(\w+)\s*\(', t)
    if m and not t.rstrip().endswith(';'):
        funcs.append((i, m.group(1)))
def func_of(ln):
    name = '?'
    for s0, f in funcs:
        if s0 <= ln:
            name = f
    return name
cnt = collections.Counter()
pending = []
base = os.path.basename(src)
for L in dis:
    if L.strip().startswith('//## File'):
        pending.append(L)
        continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/', L):
        best = None
        for c in pending:
            for f, ln in re.findall(r'File "([^"]+)", line (\d+)', c):
                if os.path.basename(f) == base and best is None:
                    best = int(ln)
        cnt[func_of(best) if best else '?'] += 1
        pending = []
for f, c in cnt.most_common(25):
    print(f"{c:7d} {f}")
