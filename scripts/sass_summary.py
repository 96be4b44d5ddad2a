"""Summarise an ncu SASS source page (csv): instruction mix and stall samples by opcode.
usage: ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv; python sass_summary.py s.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = hdr.index('Instructions Executed'); cs = hdr.index('Warp Stall Sampling (All Samples)')
agg = collections.defaultdict(lambda: [0.0, 0.0])
tot = [0.0, 0.0]
for r in rows[2:]:
    if len(r) <= cs: continue
    op = r[1].strip().split()
    if not op: continue
    o = op[0]
    if o.startswith('@'): o = op[1] if len(op) > 1 else o
    o = o.split('.')[0]
    i, s = float(r[ci] or 0), float(r[cs] or 0)
    agg[o][0] += i; agg[o][1] += s; tot[0] += i; tot[1] += s
print(f"total warp-instr {tot[0]:.3e}  stall samples {tot[1]:.0f}")
for o, (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{o:10s} instr {100*i/tot[0]:5.1f}%  samples {100*s/tot[1]:5.1f}%")
