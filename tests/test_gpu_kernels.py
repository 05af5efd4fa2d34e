"""GPU parity of the kernels behind the C ABI against the reference's own
outputs (tests/golden, from the unmodified reference library) and fp64
restatements.  Mirrors proj/tests/test_tensor.cpp.

Tolerances: K1 (pure data movement) bit-exact; contractions 1e-5 relative
Frobenius on represented values (test_tensor.cpp:120-155)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, tc_gemm

pytestmark = pytest.mark.gpu


def rel_frob(a, b):
    return np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300)


def test_transpose_golden_bit_exact(gpu):
    tr = np.load(os.path.join(GOLDEN, "transpose.npz"))
    for i in range(int(tr["n"])):
        got = gpu.transpose(tr[f"in{i}"], list(tr[f"perm{i}"]))
        want = tr[f"out{i}"]
        assert got.shape == want.shape
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), i


def test_transpose_identity_involution_and_large_bit_permutations(gpu):
    rng = np.random.default_rng(1)
    t = (rng.random((2, 3, 4)) + 1j * rng.random((2, 3, 4))).astype(np.complex64)
    assert np.array_equal(gpu.transpose(t, [0, 1, 2]), t)
    u = gpu.transpose(gpu.transpose(t, [2, 0, 1]), [1, 2, 0])
    assert np.array_equal(u, t)
    for rank in (7, 11, 17, 20, 23):
        x = (rng.random(2**rank) - 0.5 + 1j * (rng.random(2**rank) - 0.5)).astype(np.complex64).reshape([2] * rank)
        perm = list(rng.permutation(rank))
        assert np.array_equal(gpu.transpose(x, perm), np.transpose(x, perm))
    # innermost axis kept (contiguous runs) and fully reversed
    x = (rng.random(2**16) + 0j).astype(np.complex64).reshape([2] * 16)
    for perm in ([1, 0] + list(range(2, 16)), list(range(15, -1, -1))):
        assert np.array_equal(gpu.transpose(x, perm), np.transpose(x, perm))


def test_transpose_rejects_non_permutations(gpu):
    t = np.zeros((2, 2), np.complex64)
    with pytest.raises(gpu.InvalidArgument):
        gpu.transpose(t, [0, 0])
    with pytest.raises(gpu.InvalidArgument):
        gpu.transpose(t, [0, 5])


def test_contract_golden_matches_reference(gpu):
    ct = np.load(os.path.join(GOLDEN, "contract.npz"))
    for i in range(int(ct["n"])):
        l, r, o = list(ct[f"l{i}"]), list(ct[f"r{i}"]), list(ct[f"o{i}"])
        a = ct[f"a{i}"].reshape([2] * len(l)) if l else ct[f"a{i}"].reshape(())
        b = ct[f"b{i}"].reshape([2] * len(r)) if r else ct[f"b{i}"].reshape(())
        got, scale, fl = gpu.contract(l, a, 0.0, r, b, 0.0, o, normalize=True)
        want = ct[f"c{i}"]
        wscale = float(ct[f"scale{i}"][0])
        assert fl == int(ct[f"flops{i}"][0])
        got_v = got.astype(np.complex128) * 2.0**scale
        want_v = want.reshape(got.shape).astype(np.complex128) * 2.0**wscale
        assert rel_frob(got_v, want_v) < 1e-5, i
        if np.abs(got).max() > 0:
            assert 0.5 < np.abs(got).max() <= 1.0  # normalized like normalize_inplace


def test_contract_general_extents_vs_fp64(gpu):
    # test_tensor.cpp:120-129: rank-4 x rank-4, two shared labels, mixed extents
    rng = np.random.default_rng(7)
    for _ in range(8):
        a = (rng.random((2, 3, 4, 2)) - 0.5 + 1j * (rng.random((2, 3, 4, 2)) - 0.5)).astype(np.complex64)
        b = (rng.random((4, 2, 3, 2)) - 0.5 + 1j * (rng.random((4, 2, 3, 2)) - 0.5)).astype(np.complex64)
        got, scale, fl = gpu.contract([1, 2, 3, 4], a, 0.0, [3, 4, 5, 6], b, 0.0)
        want = np.einsum("ijkl,klmn->ijmn", a.astype(np.complex128), b.astype(np.complex128))
        assert rel_frob(got.astype(np.complex128), want) < 1e-5
        assert fl == gpu.flop_count(a.size, b.size, want.size)


def test_contract_identity_scalar_and_errors(gpu):
    eye = np.eye(2, dtype=np.complex64)
    c, s, fl = gpu.contract([0, 1], eye, 0.0, [1, 2], eye, 0.0)
    assert fl == 64 and np.array_equal(c, eye)  # test_tensor.cpp:100-110
    t = (np.arange(6) + 1j).astype(np.complex64).reshape(3, 2)
    c, s, _ = gpu.contract([], np.ones((), np.complex64), 0.0, [0, 1], t, 0.0)
    assert np.array_equal(c, t)  # test_tensor.cpp:112-118
    with pytest.raises(gpu.InvalidArgument, match="extent mismatch"):
        gpu.contract([0, 1], np.zeros((2, 3), np.complex64), 0.0, [1, 2], np.zeros((4, 2), np.complex64), 0.0)


def test_normalize_inplace(gpu):
    # test_tensor.cpp:193-240
    t = np.ones(4, np.complex64)
    nz, ls = gpu.normalize_inplace(t)
    assert nz and ls == 0.0 and np.array_equal(t, np.ones(4, np.complex64))
    t = np.full(2, 2.0**-20, np.complex64)
    nz, ls = gpu.normalize_inplace(t)
    assert nz and ls == -20.0 and np.array_equal(t, np.ones(2, np.complex64))
    rng = np.random.default_rng(3)
    for _ in range(10):
        t = (rng.random(32) - 0.5 + 1j * (rng.random(32) - 0.5)).astype(np.complex64)
        before = t.astype(np.complex128).copy()
        nz, ls = gpu.normalize_inplace(t)
        assert nz
        assert np.allclose(t.astype(np.complex128) * 2.0**ls, before, rtol=1e-6, atol=0)
        assert 0.5 < np.abs(t).max() <= 1.0
        again = t.copy()
        nz2, ls2 = gpu.normalize_inplace(again, ls)
        assert np.array_equal(again, t) and ls2 == ls
    z = np.zeros(3, np.complex64)
    nz, ls = gpu.normalize_inplace(z)
    assert not nz and ls == 0.0


@pytest.mark.parametrize("m,n,k,ta,tb", [(1000, 300, 700, 0, 0), (512, 256, 256, 1, 0), (333, 129, 65, 0, 1),
                                         (64, 128, 1, 1, 1), (8, 8, 1 << 16, 0, 0), (1, 1, 1 << 20, 0, 0),
                                         (1 << 14, 256, 256, 0, 0),
                                         # narrow-N kernel (n <= 16, m >= 1024): T / N layouts, ragged k and n
                                         (1 << 20, 16, 16, 1, 0), (5000, 16, 16, 0, 0), (4099, 7, 40, 0, 1),
                                         (3000, 16, 33, 1, 1), (2048, 1, 256, 0, 0), (1024, 16, 1, 1, 0),
                                         (1 << 17, 32, 16, 1, 1), (5000, 29, 70, 0, 0), (1100, 17, 8, 1, 0)])
def test_cgemm_device_shapes_vs_fp64(gpu, m, n, k, ta, tb):
    import torch
    g = torch.Generator().manual_seed(m * 7 + n * 3 + k)
    A = torch.complex(torch.rand(m, k, generator=g) - 0.5, torch.rand(m, k, generator=g) - 0.5)
    B = torch.complex(torch.rand(k, n, generator=g) - 0.5, torch.rand(k, n, generator=g) - 0.5)
    want = (A.to(torch.complex128) @ B.to(torch.complex128))
    dA = (A.t().contiguous() if ta else A).cuda()
    dB = (B.t().contiguous() if tb else B).cuda()
    dC = torch.zeros(m, n, dtype=torch.complex64, device="cuda")
    rc = gpu.lib().qsg_cgemm_dev(dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), m, n, k, ta, tb, None)
    gpu._check(rc)
    torch.cuda.synchronize()
    got = dC.cpu().to(torch.complex128)
    err = (got - want).abs().norm() / want.abs().norm()
    assert err < 1e-5 * max(1.0, (k / 4096) ** 0.5), float(err)


@pytest.mark.parametrize("m,n,k,tb", [(128, 64, 16, 0), (256, 128, 64, 0), (1024, 256, 256, 0), (512, 192, 80, 1),
                                      (4096, 128, 1024, 0), (1 << 15, 256, 256, 0),
                                      # narrow-N CTA-pair variants (BN = 32 / 64 / 128 real columns)
                                      (1 << 14, 16, 256, 0), (2048, 32, 64, 1), (1024, 64, 512, 0), (768, 48, 32, 0),
                                      # fp16 kernel with a half k-block tail (2k % 64 == 32)
                                      (512, 128, 16, 0), (1024, 64, 48, 1), (256, 32, 80, 0)])
@pytest.mark.parametrize("prec", ["f16", "f16split", "tf32"])
def test_cgemm_tensor_core_vs_fp64(gpu, m, n, k, tb, prec, monkeypatch):
    """tcgen05 path (3xFP16 with operand scaling on CTA-pair shapes, 3xTF32
    otherwise or with QSG_TC_PREC=tf32): FP32-level accuracy (1e-5 relative
    Frobenius, the reference's TTGT tolerance, test_tensor.cpp:120-155)."""
    import torch
    monkeypatch.setenv("QSG_TC_PREC", "tf32" if prec == "tf32" else "f16")
    monkeypatch.setenv("QSG_TC_SPLITA", "1" if prec.startswith("f16split") else "0")
    g = torch.Generator().manual_seed(m + 3 * n + 7 * k)
    A = torch.complex(torch.rand(m, k, generator=g) - 0.5, torch.rand(m, k, generator=g) - 0.5)
    B = torch.complex(torch.rand(k, n, generator=g) - 0.5, torch.rand(k, n, generator=g) - 0.5)
    want = A.to(torch.complex128) @ B.to(torch.complex128)
    dA = A.cuda()
    dB = (B.t().contiguous() if tb else B).cuda()
    dC = torch.zeros(m, n, dtype=torch.complex64, device="cuda")
    tc_gemm(gpu, dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), m, n, k, tb)
    torch.cuda.synchronize()
    got = dC.cpu().to(torch.complex128)
    err = float((got - want).abs().norm() / want.abs().norm())
    assert err < 1e-5, err
    # and agrees with the FP32 SIMT kernel to the same level
    dC2 = torch.zeros_like(dC)
    gpu._check(gpu.lib().qsg_cgemm_dev(dA.data_ptr(), dB.data_ptr(), dC2.data_ptr(), m, n, k, 0, tb, None))
    torch.cuda.synchronize()
    assert float((dC2.cpu().to(torch.complex128) - got).abs().norm() / want.abs().norm()) < 1e-5


@pytest.mark.parametrize("prec", ["f16", "tf32"])
def test_cgemm_tensor_core_dynamic_range(gpu, prec, monkeypatch):
    """Rows of A spanning 2^0 .. 2^-30 and a B with tiny entries: the fp16
    split's per-operand power-of-two scaling keeps every row whose scale is
    within 2^-14 of the operand max at FP32-level relative accuracy, and
    the rest within an absolute error far below FP32's normwise error."""
    import torch
    monkeypatch.setenv("QSG_TC_PREC", prec)
    m, n, k = 1024, 128, 256
    g = torch.Generator().manual_seed(11)
    A = torch.complex(torch.rand(m, k, generator=g) - 0.5, torch.rand(m, k, generator=g) - 0.5)
    B = torch.complex(torch.rand(k, n, generator=g) - 0.5, torch.rand(k, n, generator=g) - 0.5) * 2.0 ** -40
    rs = torch.tensor([2.0 ** -(i % 31) for i in range(m)])
    A = A * rs[:, None]
    want = A.to(torch.complex128) @ B.to(torch.complex128)
    dC = torch.zeros(m, n, dtype=torch.complex64, device="cuda")
    dA, dB = A.cuda(), B.cuda()
    tc_gemm(gpu, dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), m, n, k, 0)
    torch.cuda.synchronize()
    got = dC.cpu().to(torch.complex128)
    row_err = (got - want).abs().norm(dim=1) / want.abs().norm(dim=1)
    near = torch.tensor([(i % 31) <= 14 for i in range(m)])
    assert float(row_err[near].max()) < 1e-5
    abs_err = float((got - want).abs().max() / want.abs().max())
    assert abs_err < 5e-6


def test_accumulate_kernel_matches_fp64(gpu):
    """K3 (batch_amplitudes accumulation, src/sampler.cpp:28-34) through the C
    ABI: acc += double(fin) * 2^log_scale, per-slice contribution kept."""
    import torch
    g = torch.Generator().manual_seed(5)
    fin = torch.complex(torch.rand(1024, generator=g), torch.rand(1024, generator=g)).cuda()
    acc = torch.ones(1024, dtype=torch.complex128, device="cuda")
    per = torch.zeros(1024, dtype=torch.complex128, device="cuda")
    gpu._check(gpu.lib().qsg_accumulate_dev(fin.data_ptr(), -3.0, 1024, acc.data_ptr(), per.data_ptr(), None))
    torch.cuda.synchronize()
    want = fin.cpu().to(torch.complex128) * 2.0 ** -3
    assert torch.equal(per.cpu(), want)
    assert torch.equal(acc.cpu(), want + 1)


@pytest.mark.parametrize("m,n,k,tb", [(512, 4096, 4096, 0), (256, 4096, 8192, 1), (1024, 8192, 4096, 0)])
def test_cgemm_tensor_core_3m_matches_fp64_and_embedding(gpu, monkeypatch, m, n, k, tb):
    """3M (Gauss) complex products on the tensor-core path (n, k >= 4096):
    P1 = Ar Br, P2 = Ai Bi, P3 = (Ar + Ai)(Br + Bi) as three 3xFP16 real
    GEMMs + a combine pass.  FP32-level accuracy vs fp64 (1e-5 relative
    Frobenius, the reference's TTGT tolerance) and agreement with the 2x2
    embedding path (QSG_TC_3M=0)."""
    import torch
    g = torch.Generator().manual_seed(m + n + k)
    A = torch.complex(torch.rand(m, k, generator=g) - 0.5, torch.rand(m, k, generator=g) - 0.5)
    B = torch.complex(torch.rand(k, n, generator=g) - 0.5, torch.rand(k, n, generator=g) - 0.5)
    want = A.to(torch.complex128) @ B.to(torch.complex128)
    dA = A.cuda()
    dB = (B.t().contiguous() if tb else B).cuda()
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("QSG_TC_3M", mode)
        dC = torch.zeros(m, n, dtype=torch.complex64, device="cuda")
        tc_gemm(gpu, dA.data_ptr(), dB.data_ptr(), dC.data_ptr(), m, n, k, tb)
        out[mode] = dC.cpu().to(torch.complex128)
    for mode, got in out.items():
        err = float((got - want).abs().norm() / want.abs().norm())
        assert err < 1e-5, (mode, err)
    assert float((out["1"] - out["0"]).abs().norm() / want.abs().norm()) < 1e-5
