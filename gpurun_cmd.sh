cd "$(dirname "$0")"
python - <<'PY'
from paper_2507_11916_b200.models import make_bmlp1
open("/tmp/h128.bmlp","wb").write(make_bmlp1("rc", hidden=[128,128], classes=21, ensemble=1, seed=2507))
PY
tests/cpp/bin/latency_breakdown /tmp/h128.bmlp mlp > gpurun_out/r2_latency_breakdown_mlp.jsonl 2>&1
tests/cpp/bin/latency_breakdown none linear > gpurun_out/r2_latency_breakdown_linear.jsonl 2>&1
timeout 300 python tests/int8_peak.py > gpurun_out/r2_int8_peak.log 2>&1
rm -f gpurun_out/search_screen.jsonl
timeout 1500 python tests/search_screen.py --lengths 14,15,16 --seeds 16 --seed0 2512 --gpu-limit 12 --cpu-limit 60 > gpurun_out/r2_screen2.log 2>&1
