"""Measured dense int8 peak on this B200: cuBLASLt int8
GEMM through torch._int_mm (the library figure, as MEASURED_PEAKS.json's
bf16_tflops is cuBLAS bf16) and the sustained tcgen05 kind::i8 floor on every
SM (tests/cpp/bin/mma_microbench sustained).  Prints JSON lines; the bench's
roofline denominator is taken from profiles/r2_int8_peak.json."""
import json
import os
import subprocess

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cublas_int8(n=16384, reps=20):
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return {"what": "cublas_int8_gemm", "m": n, "n": n, "k": n, "ms": ms, "tops": 2 * n ** 3 / (ms * 1e-3) / 1e12}


def bf16(n=16384, reps=20):
    a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        a @ b
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return {"what": "cublas_bf16_gemm", "m": n, "n": n, "k": n, "ms": ms, "tops": 2 * n ** 3 / (ms * 1e-3) / 1e12}


if __name__ == "__main__":
    rows = []
    for f in (bf16, cublas_int8):
        try:
            rows.append(f())
        except Exception as ex:  # noqa: BLE001
            rows.append({"what": f.__name__, "error": str(ex)[:200]})
        print(json.dumps(rows[-1]), flush=True)
    exe = os.path.join(ROOT, "tests", "cpp", "bin", "mma_microbench")
    out = subprocess.run([exe, "sustained"], capture_output=True, text=True, timeout=300)
    for line in out.stdout.splitlines():
        if line.startswith("{"):
            rows.append(json.loads(line))
            print(line, flush=True)
    sus = [r["tops"] for r in rows if r.get("what") == "int8_dense_sustained"]
    lib = [r["tops"] for r in rows if r.get("what") == "cublas_int8_gemm" and "tops" in r]
    summary = {"int8_tcgen05_sustained_tops": min(sus) if sus else None, "cublas_int8_tops": lib[0] if lib else None,
               "rows": rows}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(summary, open(os.path.join(ROOT, "gpurun_out", "int8_peak.json"), "w"), indent=1)
