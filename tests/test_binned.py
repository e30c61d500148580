"""Per-pixel binned polynomial LUT (north_star stage with no reference
counterpart, SURVEY.md row a14 -- parity against gelsim unpinned).  Pinned
instead: the one-bin table IS gelsim's PolyLut, both in the CPU restatement
(against the reference restatement) and on the GPU (bit-identical to K1)."""
import numpy as np
import pytest

from oracle import gelsim_oracle as O
from oracle.binned_oracle import bin_index, depth_to_rgb_binned as oracle_binned
from paper_2408_06506_b200 import synthetic
from paper_2408_06506_b200.binned import BinnedPolyLut, vignetted_lut


def _setup(size=(80, 60), n=3, cid=91):
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    return synthetic.depth_batch(cam, bg, n, config_id=cid), lut


def test_bin_index_floor_rule():
    assert list(bin_index(10, 3)) == [0, 0, 0, 0, 1, 1, 1, 2, 2, 2]
    assert list(bin_index(5, 5)) == [0, 1, 2, 3, 4]
    assert list(bin_index(7, 1)) == [0] * 7


def test_one_bin_restatement_is_the_global_lut():
    d, lut = _setup()
    b = BinnedPolyLut.from_poly_lut(lut)
    np.testing.assert_allclose(oracle_binned(d, b.coeffs, b.degree), O.depth_to_rgb(d, lut.coeffs, lut.degree),
                               rtol=0, atol=1e-15)


def test_restatement_uses_each_bins_table():
    d, lut = _setup()
    v = vignetted_lut(lut, bins=(3, 4))
    got = oracle_binned(d, v.coeffs, v.degree)
    H, W = d.shape[-2:]
    for (y, x) in ((0, 0), (H - 1, W - 1), (H // 2, W // 3), (25, 61)):
        by, bx = y * 3 // H, x * 4 // W
        ref = O.depth_to_rgb(d, v.coeffs[by, bx], v.degree)[..., y, x, :]
        np.testing.assert_allclose(got[..., y, x, :], ref, rtol=0, atol=1e-15)


def test_binned_lut_validation():
    _, lut = _setup()
    with pytest.raises(ValueError):
        BinnedPolyLut(degree=2, coeffs=np.zeros((2, 2, 3, 5)), image_size=(80, 60))
    with pytest.raises(ValueError):
        BinnedPolyLut(degree=2, coeffs=np.zeros((61, 1, 3, 6)), image_size=(80, 60))
    with pytest.raises(ValueError):
        BinnedPolyLut(degree=5, coeffs=np.zeros((1, 1, 3, 21)), image_size=(80, 60))


@pytest.mark.gpu
@pytest.mark.parametrize("size", [(320, 240), (80, 60), (37, 29)])
@pytest.mark.parametrize("deg", [2, 3, 4])
def test_gpu_one_bin_equals_k1_bit_exact(size, deg):
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned_device
    from paper_2408_06506_b200.render import depth_to_rgb_device
    _, cam, bg, _, _ = synthetic.sensor_setup(size)
    lut = synthetic.synthetic_lut(size, degree=deg, gradient_scale=synthetic.lut_scale(size))
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 4, config_id=92)).cuda()
    ref_u8 = torch.empty(d.shape + (3,), dtype=torch.uint8, device="cuda")
    ref_f = torch.empty(d.shape + (3,), dtype=torch.float32, device="cuda")
    depth_to_rgb_device(d, lut, out_u8=ref_u8, out_f32=ref_f)
    for bins in ((1, 1), (3, 5), (size[1], 1)):
        b = BinnedPolyLut.from_poly_lut(lut, bins)
        u8 = torch.empty_like(ref_u8)
        f = torch.empty_like(ref_f)
        depth_to_rgb_binned_device(d, b, out_u8=u8, out_f32=f)
        torch.cuda.synchronize()
        assert torch.equal(u8, ref_u8), bins
        assert torch.equal(f, ref_f), bins


@pytest.mark.gpu
@pytest.mark.parametrize("size,bins", [((320, 240), (6, 8)), ((640, 480), (12, 16)), ((37, 29), (29, 37)),
                                       ((80, 60), (7, 3))])
def test_gpu_binned_vs_restatement(size, bins):
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned
    d, lut = _setup(size, n=2, cid=93)
    lut = synthetic.synthetic_lut(size, degree=2, gradient_scale=synthetic.lut_scale(size))
    v = vignetted_lut(lut, bins=bins, falloff=0.4)
    ref = O.to_uint8(oracle_binned(d, v.coeffs, v.degree))
    got = depth_to_rgb_binned(torch.from_numpy(d).cuda(), v, out_dtype=np.uint8).cpu().numpy()
    diff = np.abs(got.astype(int) - ref.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
    f64 = depth_to_rgb_binned(d, v)  # numpy in -> float64 numpy out
    assert f64.dtype == np.float64 and f64.shape == d.shape + (3,)
    np.testing.assert_allclose(f64, oracle_binned(d, v.coeffs, v.degree), rtol=0, atol=2e-6)


@pytest.mark.gpu
def test_gpu_binned_errors():
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned
    from paper_2408_06506_b200.errors import LutResolutionMismatch
    d, lut = _setup()
    v = vignetted_lut(lut, bins=(2, 2))
    with pytest.raises(LutResolutionMismatch):
        depth_to_rgb_binned(torch.from_numpy(d[..., :-1]).cuda().contiguous(), v)
    big = BinnedPolyLut(degree=4, coeffs=np.zeros((60, 80, 3, 15)), image_size=(80, 60))
    with pytest.raises(ValueError):  # table larger than shared memory, odd x-bin edges: no kernel takes it
        depth_to_rgb_binned(torch.from_numpy(d).cuda(), big)


@pytest.mark.gpu
@pytest.mark.parametrize("deg,bins", [(4, (24, 32)), (3, (48, 40)), (4, (60, 40))])
def test_gpu_large_tables_on_the_band_pipeline(deg, bins):
    """Tables too large for the per-quad kernel's shared memory run on the
    band pipeline, which reads the coefficients through L1 at degrees 3-4:
    same results as the CPU restatement (uint8 within one step)."""
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned
    size = (320, 240)
    d, _ = _setup(size, n=2, cid=97)
    lut = synthetic.synthetic_lut(size, degree=deg, gradient_scale=synthetic.lut_scale(size))
    v = vignetted_lut(lut, bins=bins, falloff=0.4)
    ref = O.to_uint8(oracle_binned(d, v.coeffs, v.degree))
    got = depth_to_rgb_binned(torch.from_numpy(d).cuda(), v, out_dtype=np.uint8).cpu().numpy()
    diff = np.abs(got.astype(int) - ref.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
    np.testing.assert_allclose(depth_to_rgb_binned(d, v), oracle_binned(d, v.coeffs, v.degree), rtol=0, atol=2e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("deg,bins,n", [(3, (24, 32), 6), (3, (12, 40), 6), (3, (3, 80), 6), (2, (24, 32), 300),
                                        (2, (6, 8), 300), (2, (7, 40), 300), (2, (240, 2), 40), (2, (13, 16), 1)])
def test_gpu_band_pipeline_binned_equals_simple_kernel(monkeypatch, deg, bins, n):
    """K1's band pipeline (rgb_bulk_kernel<..., BIN>, forced for every bin
    width here) and the per-quad kernel evaluate the same FMA sequence per
    pixel, so they agree bit for bit.  At degree 2 the band pipeline keeps
    each thread's coefficient sets in registers across rows and work units:
    hundreds of images make every CTA revisit its band, and bin heights that
    do not divide the 8-row thread blocks (7, 13 bins over 240 rows) make the
    sets change inside a thread's rows."""
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned_device
    size = (320, 240)
    d, lut = _setup(size, n=6, cid=95)
    d = np.ascontiguousarray(d[np.arange(n) % len(d)] + (np.arange(n) % 7)[:, None, None].astype(np.float32) * 1e-4)
    lut = synthetic.synthetic_lut(size, degree=deg, gradient_scale=synthetic.lut_scale(size))
    v = vignetted_lut(lut, bins=bins, falloff=0.3)
    dd = torch.from_numpy(d).cuda()
    a = torch.empty(dd.shape + (3,), dtype=torch.uint8, device="cuda")
    fa = torch.empty(dd.shape + (3,), dtype=torch.float32, device="cuda")
    monkeypatch.setenv("TACSL_BINNED_BAND", "1")
    depth_to_rgb_binned_device(dd, v, out_u8=a, out_f32=fa)
    monkeypatch.delenv("TACSL_BINNED_BAND")
    monkeypatch.setenv("TACSL_BINNED_SIMPLE", "1")
    b = torch.empty_like(a)
    fb = torch.empty_like(fa)
    depth_to_rgb_binned_device(dd, v, out_u8=b, out_f32=fb)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(fa, fb)


@pytest.mark.gpu
@pytest.mark.parametrize("deg", [3, 4])
def test_gpu_band_pipeline_table_in_smem_equals_l1(monkeypatch, deg):
    """At degrees 3-4 the band pipeline reads its band's y bins from shared
    memory; with TACSL_BINNED_L1 it reads the whole table through L1.  Same
    FMA sequence, same bits (hundreds of images: CTAs keep their band)."""
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned_device
    size = (320, 240)
    d, _ = _setup(size, n=6, cid=98)
    d = np.ascontiguousarray(d[np.arange(300) % len(d)])
    lut = synthetic.synthetic_lut(size, degree=deg, gradient_scale=synthetic.lut_scale(size))
    v = vignetted_lut(lut, bins=(24, 32), falloff=0.3)
    dd = torch.from_numpy(d).cuda()
    a = torch.empty(dd.shape + (3,), dtype=torch.uint8, device="cuda")
    fa = torch.empty(dd.shape + (3,), dtype=torch.float32, device="cuda")
    depth_to_rgb_binned_device(dd, v, out_u8=a, out_f32=fa)
    monkeypatch.setenv("TACSL_BINNED_L1", "1")
    b = torch.empty_like(a)
    fb = torch.empty_like(fa)
    depth_to_rgb_binned_device(dd, v, out_u8=b, out_f32=fb)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(fa, fb)


@pytest.mark.gpu
@pytest.mark.parametrize("size,scalar", [((1283, 12), False), ((1600, 10), True), ((2050, 6), True)])
def test_gpu_binned_wide_rows(monkeypatch, size, scalar):
    """Rows wider than 4 x the per-quad kernel's threads: every
    column is written (the generic kernel strides its quads)."""
    import torch
    from paper_2408_06506_b200.binned import depth_to_rgb_binned
    if scalar:
        monkeypatch.setenv("TACSL_BINNED_SCALAR", "1")
    W, H = size
    rng = np.random.default_rng(W)
    d = rng.uniform(0.02, 0.0202, size=(2, H, W)).astype(np.float32)
    lut = synthetic.synthetic_lut(size, degree=2, gradient_scale=synthetic.lut_scale(size) * 0.1)
    v = vignetted_lut(lut, bins=(3, 5), falloff=0.4)
    ref = O.to_uint8(oracle_binned(d, v.coeffs, v.degree))
    got = depth_to_rgb_binned(torch.from_numpy(d).cuda(), v, out_dtype=np.uint8).cpu().numpy()
    diff = np.abs(got.astype(int) - ref.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
