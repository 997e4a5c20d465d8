cd "$(dirname "$0")"
rm -f gpurun_out/search_screen.jsonl
timeout 400 python bench.py > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
timeout 400 python tests/search_screen.py --lengths 16 --seeds 16 --seed0 2528 --gpu-limit 10 --cpu-limit 60 > gpurun_out/r2_screen3.log 2>&1
timeout 1500 python tests/search_screen.py --korf 8,4,1,5,7 --gpu-limit 300 --cpu-limit 300 > gpurun_out/r2_korf.log 2>&1
python tests/profile_kernel.py --model mlp --hidden 1610,1610 --n 262144 --launches 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mlp_wide -s 2 -c 1 -o gpurun_out/r2_h1610 python tests/profile_kernel.py --model mlp --hidden 1610,1610 --n 262144 --launches 3 > gpurun_out/ncu1.log 2>&1
BIDA_MLP_L2HINT=0 python tests/profile_kernel.py --model mlp --hidden 1610,1610 --n 262144 --launches 3 > gpurun_out/plain.log 2>&1 && \
BIDA_MLP_L2HINT=0 ncu --set full --clock-control none --import-source on -k regex:mlp_wide -s 2 -c 1 -o gpurun_out/r2_h1610_nohint python tests/profile_kernel.py --model mlp --hidden 1610,1610 --n 262144 --launches 3 > gpurun_out/ncu2.log 2>&1
python tests/profile_kernel.py --model linear --n 4194304 --launches 3 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:linear_thread -s 2 -c 1 -o gpurun_out/r2_linear python tests/profile_kernel.py --model linear --n 4194304 --launches 3 > gpurun_out/ncu3.log 2>&1
