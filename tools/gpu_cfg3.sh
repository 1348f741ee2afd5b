# config #3 shape at N=1 (128K, d32m4096 0.375-bit, staged kernel) through bench.py
cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
timeout 900 python bench.py --notation d32m4096 --no-prefill --steps 20 > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo rc=$?
tail -c 3000 gpurun_out/bench_cfg3.json; tail -3 gpurun_out/bench_cfg3.err
