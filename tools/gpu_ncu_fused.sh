# ncu --set full of the fused d8m256 decode kernel (attention-only launch, 128K)
cd ${GRAFT_REPO_ROOT:-/root/repo}
mkdir -p gpurun_out
TAG=${TAG:-f}
python tools/staged_bench.py --configs cfg1_128k_d8m256 --kernels 1 --reps 4 > gpurun_out/ncu_plain_fused.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 2 -c 1 -o gpurun_out/fused_$TAG -f \
    python tools/staged_bench.py --configs cfg1_128k_d8m256 --kernels 1 --reps 4 > gpurun_out/ncu_fused.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/fused_$TAG.ncu-rep --page raw --csv > gpurun_out/fused_${TAG}_raw.csv 2>/dev/null
