cd "$(dirname "$0")"
rm -f gpurun_out/korf_sweep.jsonl
bash tests/korf_sweep.sh > gpurun_out/korf_sweep.log 2>&1
timeout 900 python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err
tests/cpp/bin/latency_breakdown none linear > gpurun_out/r2_latency_breakdown_linear2.jsonl 2>&1
