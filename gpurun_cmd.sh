#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 300 python tests/trace_mlp.py --hidden 128,128 --tiles-per-cta 16 --warps 1,2,6 > gpurun_out/trace_base.txt 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full4.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke2.log 2>&1
