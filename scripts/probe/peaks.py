"""Measure the FP64 / FP32 / TF32 / INT8 dense GEMM peaks the roofline needs (torch 8192^3, best of 10)."""
import json, torch
def bench(fn, flops, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); best = 1e9
    for _ in range(n):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e))
    return flops / best / 1e9
N = 8192; out = {}
a = torch.randn(N, N, device='cuda', dtype=torch.float64); b = torch.randn_like(a)
out['fp64_tflops'] = bench(lambda: a @ b, 2 * N**3)
a32 = a.float(); b32 = b.float()
torch.backends.cuda.matmul.allow_tf32 = False
out['fp32_tflops'] = bench(lambda: a32 @ b32, 2 * N**3)
torch.backends.cuda.matmul.allow_tf32 = True
out['tf32_tflops'] = bench(lambda: a32 @ b32, 2 * N**3)
ai = torch.randint(-127, 127, (N, N), device='cuda', dtype=torch.int8); bi = torch.randint(-127, 127, (N, N), device='cuda', dtype=torch.int8).t()
try:
    out['int8_tops'] = bench(lambda: torch._int_mm(ai, bi), 2 * N**3)
except Exception as ex:
    out['int8_tops'] = str(ex)
print(json.dumps(out))
