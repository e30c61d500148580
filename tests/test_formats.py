"""On-disk formats against files written by the
reference's own writers (tests/golden/ref.lut, ref.tff)."""
import numpy as np
import pytest

from paper_2408_06506_b200 import formats
from paper_2408_06506_b200.render import synthetic_lut
from paper_2408_06506_b200.tactile import ForceField

GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def test_read_reference_lut_file():
    lut = formats.read_lut(GOLDEN / "ref.lut")
    ref = synthetic_lut((320, 240), degree=3, seed=4)
    assert lut.degree == 3 and lut.image_size == (320, 240)
    assert lut.sensor_id == "gelpad-A" and lut.calibrated_on == "2026-01-15"
    assert lut.residual_rms == pytest.approx(0.00123)
    np.testing.assert_array_equal(lut.coeffs, ref.coeffs)  # %.17g round-trips float64 exactly


def test_write_lut_is_byte_identical_to_reference(tmp_path):
    lut = synthetic_lut((320, 240), degree=3, seed=4)
    lut.sensor_id, lut.calibrated_on, lut.residual_rms = "gelpad-A", "2026-01-15", 0.00123
    p = tmp_path / "pad.lut"
    formats.write_lut(lut, p)
    assert p.read_bytes() == (GOLDEN / "ref.lut").read_bytes()


def test_lut_reader_rejects_bad_files(tmp_path):
    p = tmp_path / "x.lut"
    p.write_text("NOT-A-LUT\n")
    with pytest.raises(ValueError):
        formats.read_lut(p)


def test_tff_reference_file_roundtrip(tmp_path, golden):
    z = golden("ff")
    frames = formats.read_force_field_frames(GOLDEN / "ref.tff")
    assert len(frames) == 2
    for e in (0, 1):
        np.testing.assert_array_equal(frames[e].f_n, z["f_n"][e].astype(np.float32).astype(np.float64))
        np.testing.assert_array_equal(frames[e].f_t, z["f_t"][e].astype(np.float32).astype(np.float64))
    p = tmp_path / "ours.tff"
    formats.write_force_field_frames(p, [ForceField(f_n=z["f_n"][e], f_t=z["f_t"][e]) for e in (0, 1)])
    assert p.read_bytes() == (GOLDEN / "ref.tff").read_bytes()
    raw = p.read_bytes()
    assert raw[:4] == b"TFF1" and int.from_bytes(raw[4:8], "little") == 20


def test_tff_rejects_batched_field(tmp_path):
    with pytest.raises(ValueError):
        formats.write_force_field_frames(tmp_path / "x.tff", [ForceField(np.zeros((2, 3, 4, 3)),
                                                                         np.zeros((2, 3, 4, 3)))])


def test_shear_map_image_shape():
    img = formats.shear_map_image(ForceField(f_n=np.zeros((4, 6, 3)), f_t=np.zeros((4, 6, 3))), upscale=8)
    assert img.shape == (32, 48, 3) and img.dtype == np.uint8


@pytest.mark.gpu
def test_export_from_device_matches_reference_file(tmp_path, golden):
    import torch
    z = golden("ff")
    f_n = torch.from_numpy(z["f_n"][:2]).cuda()
    f_t = torch.from_numpy(z["f_t"][:2]).cuda()
    p = tmp_path / "dev.tff"
    assert formats.export_force_field_frames(p, f_n, f_t) == 2
    assert p.read_bytes() == (GOLDEN / "ref.tff").read_bytes()
