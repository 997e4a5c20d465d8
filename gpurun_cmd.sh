cd "$(dirname "$0")"
rm -f gpurun_out/search_configs.jsonl gpurun_out/parity_scale.jsonl gpurun_out/pdb_build.jsonl
timeout 900 python bench.py > gpurun_out/r2_bench6.json 2> gpurun_out/r2_bench6.err
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full3.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
