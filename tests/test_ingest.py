"""Raw slice ingest: the reference's loader contract (tests/test_volume.py:220-290
of the reference) for the host loader and for load_raw_slices_device, which
must return the same Volume and leave it resident on the device."""

import numpy as np
import pytest

import paper_1609_01317_b200 as vc
from paper_1609_01317_b200 import Volume, load_raw_slices, save_raw_slices


def _loaders():
    return [pytest.param(load_raw_slices, id="host"),
            pytest.param(vc.load_raw_slices_device, id="device", marks=pytest.mark.gpu)]


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.mark.parametrize("load", _loaders())
def test_raw_slice_roundtrip_little_and_big(tmp_path, rng, load):
    arr = rng.integers(0, 4096, size=(5, 6, 7), dtype=np.uint16)
    arr[0, 0, 0], arr[4, 5, 6] = 65535, 40000  # above int16 range: unsigned min/max on device
    vol = Volume.from_array(arr, spacing=(1, 1, 2))
    for endian in ("little", "big"):
        pattern = str(tmp_path / f"ct_{endian}.{{index:03d}}.raw")
        assert len(save_raw_slices(vol, pattern, endian)) == 5
        back = load(pattern, 7, 6, 5, endian, spacing=(1, 1, 2))
        assert np.array_equal(back.as_array(), arr)
        assert back.spacing == (1.0, 1.0, 2.0)
        assert (back.value_min, back.value_max) == (int(arr.min()), 65535)
        assert back.data.dtype == np.uint16 and not back.data.flags.writeable


@pytest.mark.parametrize("load", _loaders())
def test_raw_slice_first_index_offset(tmp_path, rng, load):
    arr = rng.integers(0, 100, size=(3, 4, 4), dtype=np.uint16)
    pattern = str(tmp_path / "s{index}.raw")
    save_raw_slices(Volume.from_array(arr), pattern, first_index=10)
    assert np.array_equal(load(pattern, 4, 4, 3, first_index=10).as_array(), arr)


@pytest.mark.parametrize("load", _loaders())
def test_load_missing_slice_names_path(tmp_path, load):
    with pytest.raises(OSError) as exc:
        load(str(tmp_path / "gone{index}.raw"), 4, 4, 2)
    assert "gone0.raw" in str(exc.value)


@pytest.mark.parametrize("load", _loaders())
def test_load_short_slice_fails_with_size_message(tmp_path, load):
    (tmp_path / "short0.raw").write_bytes(b"\x00" * 10)
    with pytest.raises(OSError) as exc:
        load(str(tmp_path / "short{index}.raw"), 4, 4, 1)
    assert "32 bytes" in str(exc.value) and "short0.raw" in str(exc.value)


@pytest.mark.parametrize("load", _loaders())
def test_load_long_slice_fails(tmp_path, load):
    (tmp_path / "long0.raw").write_bytes(b"\x00" * 34)
    with pytest.raises(OSError):
        load(str(tmp_path / "long{index}.raw"), 4, 4, 1)


@pytest.mark.parametrize("load", _loaders())
def test_load_rejects_pattern_without_placeholder(tmp_path, load):
    (tmp_path / "flat.raw").write_bytes(b"\x00" * 32)
    with pytest.raises(ValueError):
        load(str(tmp_path / "flat.raw"), 4, 4, 2)
    assert load(str(tmp_path / "flat.raw"), 4, 4, 1).dims == (4, 4, 1)


@pytest.mark.parametrize("load", _loaders())
def test_strict_12bit_rejects_wide_values(tmp_path, load):
    np.full((1, 2, 2), 4096, np.uint16).astype("<u2").tofile(tmp_path / "wide0.raw")
    pattern = str(tmp_path / "wide{index}.raw")
    with pytest.raises(ValueError):
        load(pattern, 2, 2, 1, strict_12bit=True)
    assert load(pattern, 2, 2, 1).value_max == 4096


@pytest.mark.parametrize("load", _loaders())
def test_load_validates_geometry_and_endianness(tmp_path, load):
    with pytest.raises(ValueError):
        load(str(tmp_path / "x{index}"), 0, 4, 1)
    with pytest.raises(ValueError):
        load(str(tmp_path / "x{index}"), 4, 4, 1, endianness="middle")
    (tmp_path / "x0").write_bytes(b"\x00" * 32)
    with pytest.raises(ValueError):
        load(str(tmp_path / "x{index}"), 4, 4, 1, spacing=(1, 0, 1))


def test_raw_slice_layout_is_row_major_x_fastest(tmp_path):
    arr = np.arange(2 * 3 * 4, dtype=np.uint16).reshape(2, 3, 4)
    save_raw_slices(Volume.from_array(arr), str(tmp_path / "lay.{index}.raw"), "little")
    raw = np.fromfile(tmp_path / "lay.0.raw", dtype="<u2")
    assert raw[0] == arr[0, 0, 0] and raw[1] == arr[0, 0, 1] and raw[4] == arr[0, 1, 0]


# ------------------------------------------------------------------ device residency


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [1, 3, 7, 64])
def test_device_ingest_is_resident_and_renders_like_host_load(tmp_path, chunk):
    """Chunked ingest (chunk sizes that do / do not divide the slice count)
    leaves the exact voxels in HBM: the frame from the adopted device copy is
    identical to the frame of the host-loaded volume uploaded the usual way."""
    from paper_1609_01317_b200.volume import device_volume

    src = vc.make_phantom("shell", (40, 36, 30), r_inner=8, r_outer=13, value=1500)
    pattern = str(tmp_path / "ph.{index:02d}.raw")
    save_raw_slices(src, pattern, "big")
    vol = vc.load_raw_slices_device(pattern, 40, 36, 30, "big", chunk_slices=chunk,
                                    prepass_ops=("zucker-hummel",))
    dv = device_volume(vol)
    assert dv.dims == (40, 36, 30)
    assert device_volume(vol) is dv  # cached: no second upload
    assert dv.gradient_prepass(vc.OperatorKind.ZUCKER_HUMMEL.code) != 0
    import ctypes

    from paper_1609_01317_b200 import _native

    back = np.empty(src.data.size, np.uint16)  # the library's own copy, read back
    _native.check(_native.load().vc_memcpy_to_host(back.ctypes.data, ctypes.c_void_p(dv.data_ptr()),
                                                   back.nbytes, None))
    assert np.array_equal(back, src.data)

    host_vol = vc.load_raw_slices(pattern, 40, 36, 30, "big")
    scene = vc.default_scene(vol)
    for grad in ("taps", "volume"):
        st = vc.RenderSettings(width=96, height=72, operator=vc.OperatorKind.ZUCKER_HUMMEL,
                               gradient_source=grad)
        a = vc.render_frame(vol, scene, st)
        b = vc.render_frame(host_vol, vc.default_scene(host_vol), st)
        assert np.array_equal(a.pixels, b.pixels)
