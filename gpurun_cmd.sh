#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench12.json 2> gpurun_out/r2_bench12.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full8.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke6.log 2>&1
python tests/profile_kernel.py --model mlp --hidden 128,128 --n 1048576 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:mlp_fused -s 1 -c 1 -o gpurun_out/r2_h128_v3 -f \
  python tests/profile_kernel.py --model mlp --hidden 128,128 --n 1048576 --launches 2 > gpurun_out/ncu_v3.log 2>&1
