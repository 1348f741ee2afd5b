cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fast or gqa or cache_case or pdl or one_split or sharded or peer or llama" > gpurun_out/pt_pdl.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt_pdl.log
python tools/trace_pdl.py
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --no-prefill --steps 50 > gpurun_out/bench_pdl.json 2> gpurun_out/bench_pdl.err; echo bench rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_pdl.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'frac',d['roofline']['frac'],'e2e',d['e2e']['value'])"
done
