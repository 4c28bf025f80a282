"""cuBLAS DGEMM (torch.matmul float64) burst and sustained throughput: the measured FP64 roofline."""
import json, time, torch
dev = "cuda:0"
out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev); b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    out[f"dgemm_{n}_burst_tflops"] = 2 * n**3 / (best * 1e-3) / 1e12
    t0 = time.time(); cnt = 0
    e0.record()
    while time.time() - t0 < 4.0:
        c = a @ b; cnt += 1
        if cnt % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    out[f"dgemm_{n}_sustained_tflops"] = 2 * n**3 * cnt / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps(out))
