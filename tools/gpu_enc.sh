cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
true
for N in d8m256 d32m4096 d16m4096 d16m256; do NOTATION=$N timeout 300 python tools/prefill_bench.py 32768; done 2>&1 | tee gpurun_out/prefill_enc.log
