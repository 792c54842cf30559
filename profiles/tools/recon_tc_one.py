"""One C3-shaped reconstruction block (1600 frames 256x256 R=16) on the tensor-core kernel, for ncu captures."""
import sys, torch
sys.path.insert(0, '.')
from paper_1609_04104_b200 import _ops as K
F, nx, ny, R = 1600, 256, 256, 16
g = torch.Generator(device="cuda").manual_seed(1)
a = torch.randn(F, nx, R, dtype=torch.complex64, device="cuda", generator=g)
b = torch.randn(F, ny, R, dtype=torch.complex64, device="cuda", generator=g)
gm = torch.randn(F, R, dtype=torch.complex64, device="cuda", generator=g)
out = torch.empty(F, nx, ny, dtype=torch.complex64, device="cuda")
for _ in range(4):
    K.reconstruct(a, b, gm, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    K.reconstruct(a, b, gm, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"tc F={F} {nx}x{ny} R={R}: {ms*1e3:.1f} us, writes {F*nx*ny*8/ms/1e6:.0f} GB/s")
