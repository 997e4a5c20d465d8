#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_final.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_final.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_bench_reference_final.json 2> gpurun_out/r2_bench_reference_final.err
