cd "$(dirname "$0")"
rm -f gpurun_out/search_configs.jsonl gpurun_out/parity_scale.jsonl gpurun_out/pdb_build.jsonl
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r2_gputests_full.log 2>&1
python tests/sanitizer_driver.py > gpurun_out/sanitizer_plain.log 2>&1 && \
timeout 1200 compute-sanitizer --tool memcheck --target-processes all --print-limit 50 python tests/sanitizer_driver.py > gpurun_out/r2_sanitizer_memcheck.txt 2>&1
