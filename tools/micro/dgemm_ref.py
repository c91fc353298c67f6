import torch, time
A = torch.randn(14384, 2000, dtype=torch.float64, device='cuda')
B = torch.randn(2000, 2000, dtype=torch.float64, device='cuda')
for _ in range(3): C = A @ B
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): C = A @ B
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("cuBLAS DGEMM 14384x2000x2000: %.3f ms, %.1f TFLOP/s" % (ms, 2 * 14384 * 2000 * 2000 / ms / 1e9))
