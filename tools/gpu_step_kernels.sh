cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
CFG=${CFG:-cfg3_128k_d32m4096}
python tools/step_kernels.py $CFG 3 > gpurun_out/stepk_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/stepk_$CFG.csv python tools/step_kernels.py $CFG 3 > gpurun_out/stepk_ncu.log 2>&1; echo rc=$?
python - <<'PY'
import csv, collections, os
cfg=os.environ.get("CFG","cfg3_128k_d32m4096")
rows=[r for r in csv.reader(open(f"gpurun_out/stepk_{cfg}.csv")) if len(r)>10]
h=rows[0]; idx=h.index("Kernel Name"); vi=h.index("Metric Value")
ks=[(r[idx], float(r[vi])) for r in rows[1:] if r[h.index("Metric Name")]=="gpu__time_duration.sum"]
for name,t in ks[-20:]: print(f"{t/1000:9.1f} us  {name[:90]}")
PY
