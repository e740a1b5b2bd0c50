"""Dev: measured dense TF32 / fp64 GEMM throughput and HBM copy bandwidth (context for rooflines)."""
import torch

def bench(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best

n = 8192
torch.backends.cuda.matmul.allow_tf32 = True
a = torch.randn(n, n, device="cuda"); b = torch.randn(n, n, device="cuda")
ms = bench(lambda: a @ b)
print(f"tf32 matmul {n}^3: {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
torch.backends.cuda.matmul.allow_tf32 = False
ms = bench(lambda: a @ b, 3)
print(f"fp32 (no tf32) matmul: {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
a64, b64 = a.double()[:4096, :4096], b.double()[:4096, :4096]
ms = bench(lambda: a64 @ b64, 3)
print(f"fp64 matmul 4096^3: {2*4096**3/ms/1e9:.1f} TFLOP/s", flush=True)
x = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda"); y = torch.empty_like(x)
ms = bench(lambda: y.copy_(x))
print(f"copy 2 GiB: {2*x.numel()*2/ms/1e6:.1f} GB/s", flush=True)
