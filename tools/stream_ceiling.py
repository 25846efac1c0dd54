"""Practical HBM ceiling of K1's access pattern (read g and r, write r; 12 B per element) measured
with torch's own vectorized elementwise kernel (r.add_(g, alpha=a)) over the bench's buffers: 3
rotating 102 MB gradients + the 102 MB residual, CUDA events over 200 back-to-back launches.
Diagnostic only: the denominator K1 is compared with besides the copy peak."""
import torch

n = 25_557_032
gs = [torch.randn(n, device="cuda") for _ in range(3)]
r = torch.zeros(n, device="cuda")
for t in range(20):
    r.add_(gs[t % 3], alpha=0.1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(200):
    r.add_(gs[t % 3], alpha=0.1)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
print(f"r += a*g over {n} fp32: {ms * 1e3:.1f} us per launch, {12 * n / (ms * 1e-3) / 1e9:.0f} GB/s")
# the copy (8 B per element) for reference
dst = torch.empty(n, device="cuda")
e0.record()
for t in range(200):
    dst.copy_(gs[t % 3])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 200
print(f"copy: {ms * 1e3:.1f} us per launch, {8 * n / (ms * 1e-3) / 1e9:.0f} GB/s")
