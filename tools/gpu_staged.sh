cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "${PTK:-staged}" > gpurun_out/pt_staged.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pt_staged.log
timeout 600 python tools/staged_bench.py --kernels ${KERNELS:-2} ${SB_ARGS:-} > gpurun_out/staged_bench.log 2>&1; echo bench rc=$?; cat gpurun_out/staged_bench.log | tail -20
ANTKV_TC_BULK=0 timeout 600 python tools/staged_bench.py --kernels 2 --configs cfg3_128k_d32m4096,d16m4096_128k > gpurun_out/staged_bench0.log 2>&1; echo bench0 rc=$?; cat gpurun_out/staged_bench0.log | tail -20
