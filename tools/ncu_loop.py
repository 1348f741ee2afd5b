"""Stall reasons + shared-memory wavefronts of a kernel's hot loop from an
ncu report (source page, SASS view)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
I = h.index("Instructions Executed")
S = h.index("Source")
W = h.index("Warp Stall Sampling (All Samples)")
stalls = [k for k in h if k.startswith("stall_") and "Not" not in k]
wf = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
wfi = h.index("L1 Wavefronts Shared Ideal") if "L1 Wavefronts Shared Ideal" in h else None


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


maxn = max(f(x[I]) for x in rows)
tot = collections.Counter()
st = collections.Counter()
ops = collections.Counter()
samples = 0
loop_samples = 0
wft = wfit = 0
for x in rows:
    n = f(x[I])
    samples += f(x[W])
    if n < 0.5 * maxn:
        continue
    loop_samples += f(x[W])
    op = x[S].split()[1] if x[S].startswith("@") else x[S].split()[0]
    ops[op] += n
    for k in stalls:
        st[k] += f(x[h.index(k)])
    if wf is not None:
        wft += f(x[wf])
        wfit += f(x[wfi])
print(f"samples total {samples:.0f}, hot loop {loop_samples:.0f} ({loop_samples / max(samples, 1):.0%})")
print("hot-loop stalls:", ", ".join(f"{k[6:]} {v:.0f}" for k, v in st.most_common(10)))
print(f"hot-loop shared wavefronts {wft:.0f} (ideal {wfit:.0f})")
print("hot-loop ops:", ", ".join(f"{k} {v:.0f}" for k, v in ops.most_common(25)))
