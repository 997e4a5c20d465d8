set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 3000 gpurun_out/bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --search-seconds 0 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_fused -c 1 -o gpurun_out/prof_v7_h128 -f python tests/profile_kernel.py --hidden 128,128 --n 1048576 --launches 2 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_wide -c 1 -o gpurun_out/prof_v7_h1610 -f python tests/profile_kernel.py --hidden 1610,1610 --n 262144 --launches 2 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mlp_wide -c 1 -o gpurun_out/prof_v7_h512 -f python tests/profile_kernel.py --hidden 512,512 --n 1048576 --launches 2 > gpurun_out/ncu3.log 2>&1
