"""CPU: HCF1 raw channel images and binary PPM (io.cpp:450-536) through the C++ drop-in and
the Python loaders, against files the compiled reference writes and its own error cases."""
import ctypes
import subprocess

import numpy as np
import pytest

import oracle
from conftest import ROOT

SRC = ROOT / "tests" / "cpp" / "test_image_io.cpp"


@pytest.fixture(scope="module")
def ref():
    r = oracle.reference(81)
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    return r


@pytest.fixture(scope="module")
def prog(tmp_path_factory):
    from paper_2602_18741_b200 import build

    lib = build.build()
    out = tmp_path_factory.mktemp("img") / "test_image_io"
    cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT / 'include'}", str(SRC), f"-L{lib.parent}", "-lhadacodec_b200",
           f"-Wl,-rpath,{lib.parent}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


@pytest.mark.parametrize("shape", [(3, 2, 5), (64, 48, 6), (1, 1, 1), (17, 9, 81)])
def test_raw_image_round_trip_byte_identical(ref, prog, tmp_path, shape):
    from paper_2602_18741_b200 import api

    w, h, c = shape
    data = (np.arange(w * h * c, dtype=np.float32) * 0.125 - 1.0)
    data[::7] = np.float32(np.nan) if c > 1 else data[::7]
    a, b = tmp_path / "a.hcf", tmp_path / "b.hcf"
    assert ref.ref_write_raw_image(str(a).encode(), w, h, c, data) == 0
    r = subprocess.run([str(prog), "raw", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert b.read_bytes() == a.read_bytes()
    img = api.read_raw_image(a, device="cpu")
    assert tuple(img.shape) == (h, w, c) and img.numpy().tobytes() == data.tobytes()
    api.write_raw_image(tmp_path / "c.hcf", img)
    assert (tmp_path / "c.hcf").read_bytes() == a.read_bytes()


RAW_BAD = [b"JUNKJUNKJUNK", b"HCF1\x02\x00", b"HCF1" + np.array([0, 2, 3], np.uint32).tobytes(),
           b"HCF1" + np.array([70000, 2, 3], np.uint32).tobytes(),
           b"HCF1" + np.array([2, 2, 2], np.uint32).tobytes() + b"\x00" * 12]


@pytest.mark.parametrize("case", range(len(RAW_BAD)))
def test_raw_image_errors_like_reference(ref, prog, tmp_path, case):
    from paper_2602_18741_b200 import api

    a = tmp_path / "bad.hcf"
    a.write_bytes(RAW_BAD[case])
    w, h, c = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    err = ctypes.create_string_buffer(256)
    assert ref.ref_read_raw_image(str(a).encode(), ctypes.byref(w), ctypes.byref(h), ctypes.byref(c),
                                  np.zeros(64, np.float32), 64, err, 256) == 1
    r = subprocess.run([str(prog), "raw", str(a), str(tmp_path / "o.hcf")], capture_output=True, text=True)
    assert r.returncode == 3
    assert err.value.decode().split(": ", 1)[1] in r.stderr  # same cause
    with pytest.raises(ValueError):
        api.read_raw_image(a, device="cpu")


def test_ppm_round_trip_byte_identical(ref, prog, tmp_path):
    rgb = (np.arange(5 * 3 * 3) * 17 % 256).astype(np.uint8)
    a, b = tmp_path / "a.ppm", tmp_path / "b.ppm"
    assert ref.ref_write_ppm(str(a).encode(), 5, 3, rgb.tobytes(), rgb.size) == 0
    r = subprocess.run([str(prog), "ppm", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert b.read_bytes() == a.read_bytes()


PPM_CASES = [b"P6\n# comment\n2 1\n# another one\n255\n" + bytes(range(6)),   # comments
             b"P6 2 1 255 " + bytes(range(6)) + b"extra",                      # trailing bytes ignored
             b"P3\n2 1\n255\n" + bytes(6), b"P6\n2 1\n65535\n" + bytes(12), b"P6\n2 x\n255\n" + bytes(6),
             b"P6\n2 1\n255\n" + bytes(5), b"P6\n2", b"", b"P6\n2 1 255", b"P6\n-2 1\n255\n" + bytes(6)]


@pytest.mark.parametrize("case", range(len(PPM_CASES)))
def test_ppm_reader_matches_reference(ref, prog, tmp_path, case):
    a = tmp_path / "a.ppm"
    a.write_bytes(PPM_CASES[case])
    w, h = ctypes.c_int(), ctypes.c_int()
    buf = ctypes.create_string_buffer(64)
    err = ctypes.create_string_buffer(256)
    rc = ref.ref_read_ppm(str(a).encode(), ctypes.byref(w), ctypes.byref(h), buf, 64, err, 256)
    r = subprocess.run([str(prog), "ppm", str(a), str(tmp_path / "o.ppm")], capture_output=True, text=True)
    if rc == 0:
        assert r.returncode == 0, r.stderr
        assert r.stdout.split() == [str(w.value), str(h.value)]
        assert (tmp_path / "o.ppm").read_bytes().endswith(buf.raw[: w.value * h.value * 3])
    else:
        assert r.returncode == 3
        assert err.value.decode().split(": ", 1)[1] in r.stderr
