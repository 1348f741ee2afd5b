# ncu --set full of the staged decode kernel on one config (run under gpurun)
cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
CFG=${CFG:-cfg3_128k_d32m4096}
python tools/staged_bench.py --configs $CFG --kernels 2 --reps 4 > gpurun_out/ncu_plain_$CFG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_tc -s 2 -c 1 -o gpurun_out/staged_$CFG -f \
    python tools/staged_bench.py --configs $CFG --kernels 2 --reps 4 > gpurun_out/ncu_staged_$CFG.log 2>&1; echo ncu rc=$?
