"""Column-FFT throughput (tt_fft_cols, in place): GB/s of read + write over the data, the two-level register
kernel (n = 64 ... 1024) against the shared-memory Stockham kernel (TT_FFT_STOCKHAM=1), errors against torch.fft."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1609_04104_b200 import _lib as L  # noqa: E402
from paper_1609_04104_b200 import _ops as K  # noqa: E402

L.load()
dev = L.device()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)


def run(shape, reps=10):
    torch.manual_seed(1)
    x = torch.randn(*shape, dtype=torch.complex64, device=dev)
    ref = torch.fft.fft(x, dim=-2, norm="ortho")
    for _ in range(3):
        K.fft_cols_(x.clone())
    ts = []
    for _ in range(reps):
        y = x.clone()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        K.fft_cols_(y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    err = float((y - ref).abs().max() / ref.abs().max())
    ms = sorted(ts)[len(ts) // 2]
    return ms, 2 * x.numel() * 8 / ms / 1e6, err, y


for shape in [(1600, 256, 256), (400, 512, 512), (100, 1024, 1024), (6400, 128, 128), (6400, 64, 64),
              (64, 256, 16), (64, 256, 20)]:
    os.environ.pop("TT_FFT_STOCKHAM", None)
    ms1, bw1, err1, y1 = run(shape)
    os.environ["TT_FFT_STOCKHAM"] = "1"
    ms0, bw0, err0, y0 = run(shape)
    os.environ.pop("TT_FFT_STOCKHAM", None)
    xi = torch.randn(3, shape[1], 37, dtype=torch.complex64, device=dev)
    ei = float((K.fft_cols(xi, inverse=True) - torch.fft.ifft(xi, dim=-2, norm="ortho")).abs().max())
    print(f"{shape}: register two-level {ms1:.3f} ms {bw1:.0f} GB/s (err {err1:.1e}) | Stockham radix-4 in smem "
          f"{ms0:.3f} ms {bw0:.0f} GB/s (err {err0:.1e}) | inverse, 37 columns: err {ei:.1e}")


def timed(fn, x, reps=10):
    for _ in range(3):
        fn(x.clone())
    ts = []
    for _ in range(reps):
        y = x.clone()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn(y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2], y


def fft2_transposed(y):  # the 2-D transform before the row kernel: column pass, transposed copy, column pass
    return K.fft_cols_(K.fft_cols_(y).transpose(1, 2).contiguous()).transpose(1, 2)


print("rows / 2-D (in place; GB/s = one read + one write of the data per pass)")
for shape in [(1600, 256, 256), (400, 512, 512), (100, 1024, 1024), (6400, 128, 128), (6400, 64, 64)]:
    torch.manual_seed(2)
    x = torch.randn(*shape, dtype=torch.complex64, device=dev)
    nb = 2 * x.numel() * 8
    ms_r, yr = timed(K.fft_rows_, x)
    er = float((yr - torch.fft.fft(x, dim=-1, norm="ortho")).abs().max())
    ms_2, y2 = timed(K.fft2_, x)
    e2 = float((y2 - torch.fft.fft2(x, norm="ortho")).abs().max())
    ms_t, _ = timed(fft2_transposed, x)
    print(f"{shape}: rows {ms_r:.3f} ms {nb / ms_r / 1e6:.0f} GB/s (err {er:.1e}) | 2-D cols+rows {ms_2:.3f} ms "
          f"{2 * nb / ms_2 / 1e6:.0f} GB/s (err {e2:.1e}) | 2-D by transposed copy {ms_t:.3f} ms")
