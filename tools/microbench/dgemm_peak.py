"""cuBLAS FP64 GEMM throughput on this B200 (a library reference beside the DMMA loop of
fp64_peaks.cu): torch.matmul float64, 8192^3, best of 10, CUDA events."""
import json

import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(2):
    torch.matmul(a, b)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"cublas_dgemm_8192_tflops": 2.0 * n ** 3 / (best * 1e-3) / 1e12, "ms": best,
                  "how": "torch.matmul float64 8192^3 (cuBLAS DGEMM), best of 10"}))
