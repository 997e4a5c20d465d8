#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
rm -f gpurun_out/mlp_ab.jsonl
for rep in 1 2; do
  BIDA_GPU_LIB=paper_2507_11916_b200/_lib/libbida_gpu_old.so timeout 300 python tests/mlp_ab.py --tag old --models "128,128;128,128,128;160,96;256;256,256" >> gpurun_out/mlp_ab.jsonl 2>> gpurun_out/mlp_ab.err
  timeout 300 python tests/mlp_ab.py --tag var3 --models "128,128;128,128,128;160,96;256;256,256" >> gpurun_out/mlp_ab.jsonl 2>> gpurun_out/mlp_ab.err
done
timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_mlp_pinned.py tests/test_gpu_pdb.py tests/test_gpu_graphs.py -q -x > gpurun_out/res_tests.log 2>&1
