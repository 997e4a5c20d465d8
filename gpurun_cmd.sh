#!/bin/bash
cd "$(dirname "$0")"
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench15.json 2> gpurun_out/r2_bench15.err
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full9.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke7.log 2>&1
python tests/profile_kernel.py --model mlp --hidden 128,128 --n 1048576 --launches 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:mlp_fused -s 1 -c 1 -o gpurun_out/r2_h128_v4 -f \
  python tests/profile_kernel.py --model mlp --hidden 128,128 --n 1048576 --launches 2 > gpurun_out/ncu_v4.log 2>&1
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-wide-leg --no-linear-leg --no-sweep --search-seconds 0"
$B > gpurun_out/launch_plain.json 2> gpurun_out/launch_plain.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default_r2d.csv $B > gpurun_out/ncu_launch.log 2>&1
