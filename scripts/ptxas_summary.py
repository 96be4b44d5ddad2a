"""Per-kernel ptxas summary (registers, spills, stack) from build/build.log."""
import re
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "build/build.log").read().splitlines()
cur = None
rows = {}
for l in log:
    m = re.search(r"Compiling entry function '([^']+)' for 'sm_100a'", l)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", l)
    if m:
        rows[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", l)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    if "k_" in k:
        name = re.sub(r"^_ZN.*?(k_\w+?)(E|I|ENS|$).*", r"\1", k)
        print(f"{name[:40]:40s} {k[-30:]:30s} {v}")
