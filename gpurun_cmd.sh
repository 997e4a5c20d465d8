#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
rm -f gpurun_out/mlp_ab.jsonl
for rep in 1 2; do
  for f in 0 1; do
    BIDA_MLP_BIAS_FOLD=$f timeout 300 python tests/mlp_ab.py --tag fold$f >> gpurun_out/mlp_ab.jsonl 2>> gpurun_out/mlp_ab.err
  done
done
timeout 900 python -m pytest tests/test_gpu_mlp.py tests/test_mlp_pinned.py tests/test_gpu_pdb.py tests/test_gpu_graphs.py -q -x > gpurun_out/fold_tests.log 2>&1
