cd ${GRAFT_REPO_ROOT:-/root/repo}
timeout 900 python -m pytest tests -m gpu -x -q -k "tcgen05 or cache_case or gqa or anchor or ans" 2>&1 | tail -2
python tools/ans_tc_check.py 32768 2>&1 | tail -3
NOTATION=d8m256 python tools/prefill_bench.py 32768
