"""Instruction mix of the innermost loop holding >= N HMMA in a kernel's SASS."""
import collections
import re
import subprocess
import sys

obj, fun = sys.argv[1], sys.argv[2]
min_hmma = int(sys.argv[3]) if len(sys.argv) > 3 else 32
sass = subprocess.run(["cuobjdump", "-sass", "-fun", fun, obj], capture_output=True, text=True).stdout
ins = []
for l in sass.splitlines():
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
h = [a for a, t in ins if 'HMMA' in t]
best = None
for a, t in ins:
    mm = re.search(r'BRA.*0x([0-9a-f]+)', t)
    if mm:
        tgt = int(mm.group(1), 16)
        n = sum(1 for x in h if tgt <= x <= a)
        if tgt < a and n >= min_hmma and (best is None or a - tgt < best[1] - best[0]):
            best = (tgt, a)
tgt, a = best
body = [x for x in ins if tgt <= x[0] <= a]
op = lambda t: t.split()[1] if t.startswith('@') else t.split()[0]
c = collections.Counter(op(x[1]) for x in body)
print(hex(tgt), hex(a), len(body), "instructions")
print(dict(c.most_common(60)))
