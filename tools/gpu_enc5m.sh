#!/bin/bash
for m in 0 1 2 3; do echo "mode $m"; ANTKV_TC5_MODE=$m timeout 120 python tools/enc_bench.py d8m256 2>&1 | tail -1 | cut -c1-80; done
