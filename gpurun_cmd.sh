cd "$(dirname "$0")"
rm -f gpurun_out/search_ab.jsonl
bash tests/search_ab.sh bida_search_fast_prev bida_search_fast 3 > gpurun_out/search_ab.log 2>&1
