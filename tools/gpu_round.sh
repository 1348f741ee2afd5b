#!/bin/bash
# Full GPU pass used for the committed evidence (run under gpurun):
# parity tests, smoke, bench (both arms), ncu launch list + one full capture.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
if [ "${NCU:-1}" = 1 ]; then
  ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
      --log-file gpurun_out/launches_$TAG.csv \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:decode_fast -s 64 -c 1 \
      -o gpurun_out/decode_fast_$TAG -f \
      python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:'flash_tc|ans_tc' -c 2 \
      -o gpurun_out/prefill_tc_$TAG -f \
      python tools/flash_tc_once.py 32768 > gpurun_out/ncu_prefill_$TAG.log 2>&1; echo "ncu prefill rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:'ans_tc_kernel' -c 1 \
      -o gpurun_out/ans_tc_$TAG -f \
      python tools/ans_tc_once.py 32768 > gpurun_out/ncu_ans_$TAG.log 2>&1; echo "ncu ans rc=$?"
fi
tail -c 2500 gpurun_out/bench_$TAG.json; echo; cat gpurun_out/bench_ref_$TAG.json; tail -3 gpurun_out/pytest_gpu_$TAG.log
