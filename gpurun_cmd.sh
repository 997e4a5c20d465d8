cd "$(dirname "$0")"
rm -f gpurun_out/korf_dinit.jsonl
bash tests/korf_dinit_sweep.sh > gpurun_out/korf_dinit.log 2>&1
