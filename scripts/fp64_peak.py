"""Measure the FP64 roofline denominator on this B200 (cuBLAS DGEMM via torch).

Mirrors MEASURED_PEAKS.json's bf16 method: 8192^3 (2 N^3 flops) best of 10
(burst) and back-to-back for 4 s (sustained); CUDA events on the stream.
Writes profiles/fp64_peak.json.  Also a DMMA microbenchmark lives in
scripts/dmma_peak.cu (optional).
"""
import json, os, subprocess, time
import torch

N = 8192
a = torch.randn(N, N, dtype=torch.float64, device="cuda")
b = torch.randn(N, N, dtype=torch.float64, device="cuda")
c = torch.empty(N, N, dtype=torch.float64, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); torch.matmul(a, b, out=c); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
burst = 2 * N ** 3 / best / 1e12
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time(); n = 0
s.record()
while time.time() - t0 < 4.0:
    torch.matmul(a, b, out=c); n += 1
    if n % 8 == 0: torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
sust = 2 * N ** 3 * n / (s.elapsed_time(e) / 1e3) / 1e12
try:
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
except Exception:
    clk = ""
out = dict(fp64_dgemm_tflops_burst=burst, fp64_dgemm_tflops_sustained=sust, N=N, iters=n,
           gpu=torch.cuda.get_device_name(), clocks_after=clk,
           how="torch.matmul float64 8192^3 (cuBLAS DGEMM), best of 10 / 4 s back to back, CUDA events")
os.makedirs("profiles", exist_ok=True)
json.dump(out, open("profiles/fp64_peak.json", "w"), indent=1)
print(json.dumps(out))
