#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
rm -f gpurun_out/korf_dinit.jsonl
WORK_NUM=256 DINITS=14 bash tests/korf_dinit_sweep.sh > gpurun_out/korf_dinit.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench8.json 2> gpurun_out/r2_bench8.err
