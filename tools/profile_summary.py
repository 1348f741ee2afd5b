"""Summaries committed under profiles/: the ncu launch list of a bench run
(per-kernel count / time share) and the full-set capture of the decode kernel
(duration, DRAM bytes, throughput, occupancy, hot-loop stalls)."""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    K, V = h.index("Kernel Name"), h.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[1:]:
        name = r[K].split("(")[0]
        tot[name] += float(r[V])
        cnt[name] += 1
    allt = sum(tot.values())
    out = ["| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for name, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        out.append(f"| `{name}` | {cnt[name]} | {t / 1e3:.1f} | {t / cnt[name] / 1e3:.2f} | {t / allt:.1%} |")
    return "\n".join(out)


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, u, v = r[0], r[1], r[2]
    d = dict(zip(h, v))
    un = dict(zip(h, u))
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__bytes_read.sum.per_second", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
            "sm__cycles_active.avg"]
    out = {k: f"{d.get(k, 'n/a')} {un.get(k, '')}".strip() for k in keys}
    return out


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "launches":
        print(launches(path))
    else:
        print(json.dumps(full(path), indent=1))
