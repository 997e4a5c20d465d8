cd "$(dirname "$0")"
rm -f gpurun_out/search_ab.jsonl
bash tests/search_ab.sh bida_search_fast_prev bida_search_fast 3 > gpurun_out/search_ab.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --search-seconds 0 --no-wide-leg --no-linear-leg --no-sweep > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_default.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --search-seconds 0 --no-wide-leg --no-linear-leg --no-sweep > gpurun_out/ncu_launch.log 2>&1
