#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
rm -f gpurun_out/mlp_ab.jsonl
for rep in 1 2; do
  BIDA_GPU_LIB=paper_2507_11916_b200/_lib/libbida_gpu_old.so timeout 300 python tests/mlp_ab.py --tag old --models "1610,1610;512,512" --n 2097152 --check 4096 >> gpurun_out/mlp_ab.jsonl 2>> gpurun_out/mlp_ab.err
  timeout 300 python tests/mlp_ab.py --tag fix3 --models "1610,1610;512,512" --n 2097152 --check 4096 >> gpurun_out/mlp_ab.jsonl 2>> gpurun_out/mlp_ab.err
done
timeout 900 python -m pytest tests/test_gpu_mlp.py -q -x -k "wide" > gpurun_out/wide_tests.log 2>&1
