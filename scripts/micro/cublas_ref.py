"""cuBLAS bf16 GEMM 8192^3 launches (the tensor-pipe reference for ncu)."""
import torch

a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    c = a @ b
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"cublas 8192^3 bf16: {ms:.3f} ms  {2 * 8192**3 / ms / 1e9:.1f} TFLOP/s")
