"""GPU parity of the value kernels: column FFT (ortho convention), 2-D DFT by
two column passes, reconstruction, rebalance."""

import numpy as np
import pytest

from conftest import load_golden, rel
from oracle import tt_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 5, 7, 64, 100, 128, 256, 1000, 1024, 4096])
@pytest.mark.parametrize("inverse", [False, True])
def test_fft_cols_matches_numpy(n, inverse):
    import torch

    from paper_1609_04104_b200 import _ops as K

    rng = np.random.default_rng(n)
    x = (rng.standard_normal((3, n, 11)) + 1j * rng.standard_normal((3, n, 11))).astype(np.complex64)
    got = K.fft_cols(torch.from_numpy(x).cuda(), inverse).cpu().numpy()
    want = np.stack([O.fft_cols(x[b], inverse) for b in range(3)])
    assert rel(got, want) < 2e-6


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("ncols", [1, 16, 20, 37])
def test_fft_register_kernel_matches_numpy_and_the_stockham_kernel(monkeypatch, n, ncols):
    """The two-level register kernel (n = 64 ... 1024) on whole and ragged column blocks, both directions,
    against numpy and against the shared-memory Stockham kernel it replaced (TT_FFT_STOCKHAM=1)."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    rng = np.random.default_rng(n + ncols)
    x = (rng.standard_normal((2, n, ncols)) + 1j * rng.standard_normal((2, n, ncols))).astype(np.complex64)
    xd = torch.from_numpy(x).cuda()
    for inverse in (False, True):
        monkeypatch.delenv("TT_FFT_STOCKHAM", raising=False)
        got = K.fft_cols(xd, inverse).cpu().numpy()
        monkeypatch.setenv("TT_FFT_STOCKHAM", "1")
        old = K.fft_cols(xd, inverse).cpu().numpy()
        want = np.stack([O.fft_cols(x[b], inverse) for b in range(2)])
        assert rel(got, want) < 2e-6
        assert rel(got, old) < 2e-6
    monkeypatch.delenv("TT_FFT_STOCKHAM", raising=False)
    back = K.fft_cols(K.fft_cols(xd, False), True).cpu().numpy()  # unitary round trip
    assert rel(back, x) < 2e-6


@pytest.mark.parametrize("n", [16, 32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("lead", [(1,), (5,), (3, 37), (2, 70)])
def test_fft_rows_matches_numpy(n, lead):
    """The row transform (last axis, in place) on whole and ragged row blocks, both directions."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    rng = np.random.default_rng(n + len(lead))
    x = (rng.standard_normal(lead + (n,)) + 1j * rng.standard_normal(lead + (n,))).astype(np.complex64)
    for inverse in (False, True):
        got = K.fft_rows_(torch.from_numpy(x).cuda(), inverse).cpu().numpy()
        f = np.fft.ifft if inverse else np.fft.fft
        assert rel(got, f(x.astype(np.complex128), axis=-1, norm="ortho")) < 2e-6
    with pytest.raises(Exception):
        K.fft_rows_(torch.zeros(4, 100, dtype=torch.complex64, device="cuda"))  # not a register-kernel length


@pytest.mark.parametrize("shape", [(2, 256, 256), (3, 64, 128), (2, 100, 256), (2, 256, 100), (1, 1024, 512),
                                   (5, 32, 32), (4, 16, 32)])
def test_fft2_matches_numpy(shape):
    """2-D ortho DFT as a column pass and a row pass (no transposes when the row length is one of the row
    kernel's; the transposed fallback otherwise), both directions and the round trip."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    rng = np.random.default_rng(sum(shape))
    x = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex64)
    xd = torch.from_numpy(x).cuda()
    for inverse in (False, True):
        f = np.fft.ifft2 if inverse else np.fft.fft2
        assert rel(K.fft2(xd, inverse).cpu().numpy(), f(x.astype(np.complex128), norm="ortho")) < 3e-6
    assert rel(K.fft2_(K.fft2(xd), inverse=True).cpu().numpy(), x) < 3e-6


def test_dft2_delta_roundtrip_and_golden():
    import paper_1609_04104_b200 as tt

    x = np.zeros((4, 6), complex)
    x[0, 0] = 1.0
    np.testing.assert_allclose(tt.unitary_dft2(x), np.full((4, 6), 1 / np.sqrt(24)), atol=1e-7)
    g = load_golden("value_cases")
    assert rel(tt.unitary_dft2(g["dft_in"]), g["dft_out"]) < 1e-6
    assert rel(tt.unitary_dft2(g["dft_in"], inverse=True), g["idft_out"]) < 1e-6
    F = tt.unitary_dft_matrix(6)
    np.testing.assert_allclose(F, F.T, atol=1e-7)


def test_synthesis_reconstruction_rebalance_golden():
    import paper_1609_04104_b200 as tt

    g = load_golden("value_cases")
    A, B, gm = g["A"], g["B"], g["gamma"]
    sub = tt.TensorSubspace((A, B))
    assert rel(tt.synthesize_slice(sub, gm), g["synth"]) < 1e-6
    est = tt.reconstruct_frame(sub, gm)
    assert rel(est.kspace, g["synth"]) < 1e-6
    assert rel(est.image, g["image"]) < 1e-5
    rb = tt.rebalance(sub)
    assert rel(rb.factors[0], g["rebal_A"]) < 1e-6 and rel(rb.factors[1], g["rebal_B"]) < 1e-6
    with pytest.raises(ValueError):
        tt.synthesize_slice(sub, np.zeros(3))


@pytest.mark.parametrize("shape", [(256, 256, 20, 7), (128, 96, 10, 3), (1024, 1024, 32, 2), (50, 70, 64, 2)])
def test_batched_reconstruct_matches_outer_product(shape):
    import torch

    from paper_1609_04104_b200 import _ops as K

    nx, ny, R, F = shape
    rng = np.random.default_rng(nx + R)
    A = (rng.standard_normal((F, nx, R)) + 1j * rng.standard_normal((F, nx, R))).astype(np.complex64)
    B = (rng.standard_normal((F, ny, R)) + 1j * rng.standard_normal((F, ny, R))).astype(np.complex64)
    gm = (rng.standard_normal((F, R)) + 1j * rng.standard_normal((F, R))).astype(np.complex64)
    X = K.reconstruct(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.from_numpy(gm).cuda()).cpu().numpy()
    for f in range(F):
        assert rel(X[f], O.synth(A[f], B[f], gm[f])) < 1e-5


@pytest.mark.parametrize("shape", [(256, 256, 16, 5), (128, 128, 8, 3), (130, 77, 5, 2), (33, 300, 32, 2),
                                   (512, 384, 24, 2), (256, 256, 20, 3), (1, 1, 1, 1), (200, 129, 9, 2)])
def test_reconstruct_tensor_core_form(shape, monkeypatch):
    """R <= 32 runs on tcgen05 (3xTF32, tt_recon_tc.cu): against the complex128 outer product element by
    element, scaled by sum_r |a'_ir| |b_jr| (the bound both fp32 forms share), and against the CUDA-core
    form (TT_RECON_FFMA=1); ragged tiles, odd ny, R not a multiple of 4, several frames per launch."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    nx, ny, R, F = shape
    rng = np.random.default_rng(nx * 7 + R)
    A = (rng.standard_normal((F, nx, R)) + 1j * rng.standard_normal((F, nx, R))).astype(np.complex64)
    B = (rng.standard_normal((F, ny, R)) + 1j * rng.standard_normal((F, ny, R))).astype(np.complex64)
    gm = (rng.standard_normal((F, R)) + 1j * rng.standard_normal((F, R))).astype(np.complex64)
    a, b, g = (torch.from_numpy(v).cuda() for v in (A, B, gm))
    Xt = K.reconstruct(a, b, g).cpu().numpy()
    monkeypatch.setenv("TT_RECON_FFMA", "1")
    Xf = K.reconstruct(a, b, g).cpu().numpy()
    for f in range(F):
        a2 = A[f].astype(np.complex128) * gm[f].astype(np.complex128)
        ex = a2 @ B[f].astype(np.complex128).T
        bound = np.abs(a2) @ np.abs(B[f].astype(np.complex128)).T
        assert np.max(np.abs(Xt[f] - ex) / bound) < 4e-6
        assert np.max(np.abs(Xf[f] - ex) / bound) < 4e-6
        assert rel(Xt[f], ex) < 2e-6


@pytest.mark.parametrize("shape,offset", [((200, 136, 12, 3), 0), ((200, 136, 12, 3), 1), ((130, 258, 16, 2), 2),
                                          ((128, 128, 4, 2), 3)])
def test_reconstruct_writes_only_its_frames(shape, offset):
    """The tensor-core reconstruction's bulk tensor stores are clipped to the frames (ragged tiles in
    both dimensions); an output at an 8-byte-only aligned address and factors at one take the plain-store
    and scalar-load paths. Guard elements around the output stay untouched; repeated launches (the
    per-launch tile counters) agree bit for bit."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    nx, ny, R, F = shape
    rng = np.random.default_rng(nx + ny + offset)
    A = (rng.standard_normal((F, nx, R)) + 1j * rng.standard_normal((F, nx, R))).astype(np.complex64)
    B = (rng.standard_normal((F, ny, R)) + 1j * rng.standard_normal((F, ny, R))).astype(np.complex64)
    gm = (rng.standard_normal((F, R)) + 1j * rng.standard_normal((F, R))).astype(np.complex64)

    def shifted(x):  # a contiguous copy whose address is offset complex64 elements past an aligned base
        buf = torch.empty(x.size + offset, dtype=torch.complex64, device="cuda")
        v = buf[offset:].view(x.shape)
        v.copy_(torch.from_numpy(x))
        return v

    a, b, g = shifted(A), shifted(B), shifted(gm)
    guard = 4096
    sentinel = complex(-7.5, 3.25)
    buf = torch.full((guard + offset + F * nx * ny + guard,), sentinel, dtype=torch.complex64, device="cuda")
    out = buf[guard + offset:guard + offset + F * nx * ny].view(F, nx, ny)
    K.reconstruct(a, b, g, out)
    first = out.clone()
    for _ in range(3):
        K.reconstruct(a, b, g, out)
    torch.cuda.synchronize()
    assert torch.equal(first, out)
    host = buf.cpu().numpy()
    assert np.all(host[:guard + offset] == np.complex64(sentinel))
    assert np.all(host[guard + offset + F * nx * ny:] == np.complex64(sentinel))
    X = out.cpu().numpy()
    for f in range(F):
        assert rel(X[f], O.synth(A[f], B[f], gm[f])) < 1e-5


@pytest.mark.parametrize("n,ncols", [(256, 1), (256, 20), (256, 33), (1024, 64), (2048, 5), (8, 70)])
def test_fft_cols_column_blocking(n, ncols):
    """Column counts that split over several CTAs (up to 32 whole columns per CTA, fewer at large n)
    with a partial last block, odd log2 n (one radix-2 pass) and even log2 n."""
    import torch

    from paper_1609_04104_b200 import _ops as K

    rng = np.random.default_rng(n + ncols)
    x = (rng.standard_normal((2, n, ncols)) + 1j * rng.standard_normal((2, n, ncols))).astype(np.complex64)
    for inverse in (False, True):
        got = K.fft_cols(torch.from_numpy(x).cuda(), inverse).cpu().numpy()
        want = np.stack([O.fft_cols(x[b], inverse) for b in range(2)])
        assert rel(got, want) < 2e-6


def test_nmse_matches_reference_semantics():
    """metrics.nmse (metrics.py:53-62): value against the oracle, per-frame batch form, ValueError for
    a shape mismatch and for an all-zero reference."""
    import paper_1609_04104_b200 as tt

    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 40, 24)) + 1j * rng.standard_normal((3, 40, 24))
    y = x + 0.1 * (rng.standard_normal(x.shape) + 1j * rng.standard_normal(x.shape))
    assert abs(tt.nmse(x, y) - O.nmse(x, y)) <= 1e-5 * O.nmse(x, y)
    per = tt.nmse_frames(x, y).cpu().numpy()
    want = np.array([O.nmse(x[f], y[f]) for f in range(3)])
    assert np.max(np.abs(per - want) / want) < 1e-5
    assert tt.nmse(x.real, y.real) == pytest.approx(O.nmse(x.real, y.real), rel=1e-5)
    a, b = tt.nmse_frames(x, y), tt.nmse_frames(x, y)
    assert bool((a == b).all())  # fixed summation order
    with pytest.raises(ValueError):
        tt.nmse(x, y[:, :, :5])
    with pytest.raises(ValueError):
        tt.nmse(np.zeros((4, 4)), np.ones((4, 4)))
