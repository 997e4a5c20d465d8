#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench10.json 2> gpurun_out/r2_bench10.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full6.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke4.log 2>&1
