cd ${GRAFT_REPO_ROOT:-/root/repo}
for i in 1 2; do
python tools/ans_tc_check.py 32768 2>&1 | tail -1 | cut -c1-200
ANTKV_LIB=$PWD/gpurun_var/nopoly/libantkv_b200.so python tools/ans_tc_check.py 32768 2>&1 | tail -1 | cut -c1-200
done
