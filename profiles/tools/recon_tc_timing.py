import os, sys, torch
sys.path.insert(0, '.')
from paper_1609_04104_b200 import _ops as K
for (F, nx, ny, R) in [(1600, 256, 256, 16), (400, 256, 256, 32), (200, 512, 512, 8), (400, 256, 256, 5), (256, 1024, 1024, 32)]:
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn(F, nx, R, dtype=torch.complex64, device="cuda", generator=g)
    b = torch.randn(F, ny, R, dtype=torch.complex64, device="cuda", generator=g)
    gm = torch.randn(F, R, dtype=torch.complex64, device="cuda", generator=g)
    out = torch.empty(F, nx, ny, dtype=torch.complex64, device="cuda")
    res = {}
    for form in ("tc", "ffma"):
        os.environ["TT_RECON_FFMA"] = "1" if form == "ffma" else "0"
        for _ in range(3): K.reconstruct(a, b, gm, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(10): K.reconstruct(a, b, gm, out)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        res[form] = out.clone() if F * nx * ny < 2**28 else None
        print(f"{form:5s} F={F} {nx}x{ny} R={R}: {ms*1e3:8.1f} us, writes {F*nx*ny*8/ms/1e6:6.0f} GB/s", flush=True)
    if res["tc"] is not None:
        d = (res["tc"] - res["ffma"]).abs().max().item()
        print("   max|tc - ffma|", d, "max|x|", res["ffma"].abs().max().item())
    del out, res
