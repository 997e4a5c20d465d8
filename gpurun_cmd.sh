#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench11.json 2> gpurun_out/r2_bench11.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full7.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke5.log 2>&1
