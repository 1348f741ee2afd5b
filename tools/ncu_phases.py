"""Stall samples per prologue phase of decode_fast_kernel (phases delimited
by the trace clock reads, SR_CLOCKLO) from an ncu --set full report."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h = r[1]
rows = r[2:]
S = h.index("Source")
W = h.index("Warp Stall Sampling (All Samples)")
stalls = [k for k in h if k.startswith("stall_") and "Not" not in k]


def f(x):
    try:
        return float(x or 0)
    except ValueError:
        return 0.0


marks = [i for i, x in enumerate(rows) if "SR_CLOCKLO" in x[S]]
for a, b in zip(marks, marks[1:]):
    st = collections.Counter()
    top = []
    tot = 0
    for x in rows[a:b]:
        w = f(x[W])
        tot += w
        for k in stalls:
            st[k[6:]] += f(x[h.index(k)])
        top.append((w, x[S][:60]))
    top.sort(reverse=True)
    print(f"[{a}-{b}] samples {tot:5.0f} {dict(st.most_common(4))}")
    for w, s in top[:3]:
        print("      ", w, s)
