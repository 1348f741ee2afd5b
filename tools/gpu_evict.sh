cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_ev.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt_ev.log
timeout 900 python bench.py --notation d32m4096 --no-prefill --steps 20 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo rc=$?
python -c "import json;d=json.loads(open('gpurun_out/bench_cfg3.json').read().strip().splitlines()[-1]);print('value',d['value'],'ms/step',d['ms_per_step'],'launch_ms',d['roofline']['launch_ms'],'e2e',d['e2e']['value'], 'launches', d['gpu_launches'])"
