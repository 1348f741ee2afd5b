#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-enc}
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-tc5} -s 2 -c 1 -o gpurun_out/ncu_$TAG -f python tools/enc_once.py ${NOTATION:-d8m256} > gpurun_out/ncu_$TAG.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_$TAG.log
