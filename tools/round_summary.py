"""Write profiles/<TAG>_summary.md and the JSON summaries from the outputs of
`TAG=<TAG> bash tools/gpu_round.sh` in gpurun_out/ (run here, after the
gpurun call has merged its files back).  Usage: python tools/round_summary.py r02"""
import csv
import gzip
import io
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT, PROF = ROOT / "gpurun_out", ROOT / "profiles"
sys.path.insert(0, str(ROOT / "tools"))
import profile_summary  # noqa: E402

RAW = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "sm__cycles_active.avg"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "--metrics", ",".join(RAW)],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    return [{k: f"{row[i]} {u[i]}".strip() for i, k in enumerate(h) if k in RAW or k == "Kernel Name"}
            for row in r[2:]]


def num(s):
    return float(s.split()[0].replace(",", ""))


def main(tag):
    bench = json.loads((OUT / f"bench_{tag}.json").read_text().strip().splitlines()[-1])
    ref = json.loads((OUT / f"bench_ref_{tag}.json").read_text().strip().splitlines()[-1])
    (PROF / f"{tag}_bench.json").write_text(json.dumps(bench) + "\n")
    (PROF / f"{tag}_bench_reference.json").write_text(json.dumps(ref) + "\n")
    with open(OUT / f"launches_{tag}.csv", "rb") as f, gzip.open(PROF / f"{tag}_launches.csv.gz", "wb") as g:
        g.write(f.read())
    shutil.copy(OUT / f"decode_fast_{tag}.ncu-rep", PROF / f"{tag}_decode_fast.ncu-rep")
    dec = profile_summary.full(str(OUT / f"decode_fast_{tag}.ncu-rep"))
    (PROF / f"{tag}_decode_fast_ncu_full.json").write_text(json.dumps(dec, indent=1) + "\n")
    fa = raw(OUT / f"prefill_tc_{tag}.ncu-rep")[0]
    an = raw(OUT / f"ans_tc_{tag}.ncu-rep")[0]
    src = f"tools/gpu_round.sh TAG={tag}: ncu --set full --clock-control none, 32K tokens " \
          "(tools/flash_tc_once.py / tools/ans_tc_once.py)"
    (PROF / f"{tag}_prefill_tc_ncu.json").write_text(
        json.dumps({"flash_tc_kernel": fa, "ans_tc_kernel": an, "source": src}, indent=1) + "\n")
    launches = profile_summary.launches(str(OUT / f"launches_{tag}.csv")).splitlines()[:16]
    rf = bench["roofline"]
    row = lambda d: (f"{num(d['gpu__time_duration.sum']):.2f} ms | "
                     f"{num(d['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']):.1f} % | "
                     f"{num(d['sm__cycles_elapsed.avg.per_second']):.2f} GHz | "
                     f"{num(d['dram__bytes_read.sum']):.1f} / {num(d['dram__bytes_write.sum']):.1f} MB | "
                     f"{num(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} % | "
                     f"{int(num(d['launch__registers_per_thread']))}")
    cfg1 = ref.get("config1_reference", {})
    md = f"""# Round {int(tag[1:])} profile summary

Commands (one B200 via gpurun, `TAG={tag} bash tools/gpu_round.sh`; this file and the JSON
summaries by `python tools/round_summary.py {tag}`):

* `python -m pytest tests -m gpu`; `__graft_entry__.smoke()` (logs: `gpurun_out/pytest_gpu_{tag}.log`)
* `python bench.py` -> `{tag}_bench.json` (no profiler)
* `python bench.py --impl reference --steps 2 --warmup 3` -> `{tag}_bench_reference.json`
* `ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline` -> launch list below (raw: `{tag}_launches.csv.gz`)
* `ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 64 -c 1 python bench.py ...` -> `{tag}_decode_fast_ncu_full.json` (report: `{tag}_decode_fast.ncu-rep`)
* `ncu --set full ... -k regex:flash_tc python tools/flash_tc_once.py 32768` and `-k regex:ans_tc_kernel python tools/ans_tc_once.py 32768` -> `{tag}_prefill_tc_ncu.json`
* encoder: `{tag}_encode_tc5.md`, `{tag}_encode_tc5_ncu.json`; parity maxima: `{tag}_parity_errors.md`

## Bench line (no profiler)

| key | value |
|---|---|
| value (batch x layers / s) | {bench['value']:.0f} tok/s ({bench['ms_per_step']:.4f} ms per 32-layer step) |
| e2e (pinned host q/k/v in, output back, public API) | {bench['e2e']['value']:.0f} tok/s |
| decode kernel per launch (graph of 32 attention launches) | {rf['launch_ms'] * 1e3:.1f} us |
| roofline (HBM) | {rf['achieved']:.0f} GB/s of {rf['peak']} GB/s measured = {rf['frac']:.3f} |
| algorithmic bytes per launch | {rf['algorithmic_bytes_per_launch'] / 1e6:.2f} MB |
| DRAM bytes per launch (ncu) | {dec['dram__bytes_read.sum']} read + {dec['dram__bytes_write.sum']} write |
| encode d8m256 (tcgen05) | {bench['encode']['value'] / 1e6:.1f} M tok/s ({bench['encode']['ms_per_layer']:.2f} ms per 128K-token layer) |
| encode d32m4096 (tcgen05 long-codebook) | {bench['encode_d32m4096']['value'] / 1e6:.1f} M tok/s |
| prefill, one layer at 128K (FA + AnS + selection + encode + layout) | {bench['prefill']['ms_per_layer']:.0f} ms ({bench['prefill']['tflops_attention']:.0f} TFLOP/s algorithmic) |
| CPU reference arm (reference package's own decode_step) | {ref['value']:.3f} layer-steps/s on {ref['cpu_baseline']['cores']} cores; config #1 on one core: {cfg1.get('prefill_ms_per_head', float('nan')):.0f} ms prefill + {cfg1.get('decode_step_ms_per_head', float('nan')):.1f} ms per decode step per head |
| clocks | {bench['clocks']} |

## Fused decode kernel (ncu --set full, one launch, cold caches, serialised)

| metric | value |
|---|---|
""" + "\n".join(f"| {k} | {v} |" for k, v in dec.items()) + f"""

The ncu duration ({dec['gpu__time_duration.sum']}) is a cold, serialised replay; in the graph the
same launch takes {rf['launch_ms'] * 1e3:.1f} us.

## Prefill kernels (ncu --set full, 32K tokens, 32 Q / 8 KV heads, causal)

| kernel | duration | tensor pipe (elapsed) | SM clock under load | DRAM read / write | issue active | registers |
|---|---|---|---|---|---|---|
| `flash_tc_kernel` | {row(fa)} |
| `ans_tc_kernel` | {row(an)} |

## Launch list of the bench command (cold, serialised per launch under ncu)

The ncu run covers the bench's setup (cache builds, the 128K prefill measurement, the encode
measurements) and the decode region; in the timed decode step the CUDA graph holds 32
`decode_fast_kernel` launches (plus one position update), so that kernel is the whole timed step.

""" + "\n".join(launches) + "\n"
    (PROF / f"{tag}_summary.md").write_text(md)
    print(md)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r02")
