"""CPU: codec weight files (io.cpp:370-403) — the C++ drop-in's load / save against files the
compiled reference writes (byte-identical re-save), and the Python loader's doubles."""
import ctypes
import subprocess

import numpy as np
import pytest

import oracle
from conftest import ROOT

SRC = ROOT / "tests" / "cpp" / "test_weights_io.cpp"


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
    out = tmp_path_factory.mktemp("w") / "test_weights_io"
    cmd = ["g++", "-std=c++17", "-O1", f"-I{ROOT / 'include'}", str(SRC), f"-L{lib.parent}", "-lhadacodec_b200",
           f"-Wl,-rpath,{lib.parent}", "-o", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return out


def _weights(k, seed):
    rng = np.random.default_rng(seed)
    re_ = rng.normal(0, 0.3, (k, 81)) * 10.0 ** rng.integers(-12, 3, (k, 81))
    rd = rng.normal(0, 0.3, (81, k))
    re_[0, :4] = [0.1, 1.0 / 3.0, -0.0, 1e-300]
    return np.ascontiguousarray(re_), np.ascontiguousarray(rd)


@pytest.mark.parametrize("k", [3, 6, 9])
def test_weight_file_resave_is_byte_identical(ref, prog, tmp_path, k):
    re_, rd = _weights(k, k)
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    lw = np.array([1.0, 0.5, 0.25, 0.125, 3e-7])
    assert ref.ref_save_codec_weights(str(a).encode(), k, 10.0, re_.reshape(-1), rd.reshape(-1), 2602, lw, 41) == 0
    r = subprocess.run([str(prog), str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert b.read_bytes() == a.read_bytes()
    # and the reference loads ours to the same doubles
    kk, beta = ctypes.c_int(), ctypes.c_double()
    e2, d2 = np.zeros(k * 81), np.zeros(81 * k)
    err = ctypes.create_string_buffer(256)
    assert ref.ref_load_codec_weights(str(b).encode(), ctypes.byref(kk), ctypes.byref(beta), e2, d2, k * 81, err,
                                      256) == 0
    assert e2.tobytes() == re_.reshape(-1).tobytes() and d2.tobytes() == rd.reshape(-1).tobytes()


def test_python_loader_reads_reference_doubles(ref, tmp_path):
    from paper_2602_18741_b200 import api

    re_, rd = _weights(6, 1)
    a = tmp_path / "a.json"
    assert ref.ref_save_codec_weights(str(a).encode(), 6, 7.5, re_.reshape(-1), rd.reshape(-1), 1, np.zeros(5), 0) == 0
    w = api.load_codec_weights(a)
    assert w["k"] == 6 and w["n"] == 81 and w["beta"] == 7.5
    assert w["raw_enc"].tobytes() == re_.tobytes() and w["raw_dec"].tobytes() == rd.tobytes()


BAD = [
    '{"format": "upsampler-weights", "k": 6}',
    '{"format": "codec-weights", "k": 5, "n": 81, "beta": 10.0, "raw_enc": [], "raw_dec": []}',
    '{"format": "codec-weights", "k": 6, "n": 81, "beta": 10.0, "raw_enc": [1.0], "raw_dec": [1.0]}',
    '{"format": "codec-weights", "k": 6',
    '[1, 2, 3]',
]


@pytest.mark.parametrize("case", range(len(BAD)))
def test_malformed_weight_files_rejected_like_reference(ref, prog, tmp_path, case):
    from paper_2602_18741_b200 import api

    a = tmp_path / "bad.json"
    a.write_text(BAD[case])
    kk, beta = ctypes.c_int(), ctypes.c_double()
    e2 = np.zeros(1024)
    err = ctypes.create_string_buffer(256)
    assert ref.ref_load_codec_weights(str(a).encode(), ctypes.byref(kk), ctypes.byref(beta), e2, e2, 1024, err,
                                      256) == 1
    r = subprocess.run([str(prog), str(a), str(tmp_path / "out.json")], capture_output=True, text=True)
    assert r.returncode == 3, (r.returncode, r.stderr)
    with pytest.raises(ValueError):
        api.load_codec_weights(a)


def _up_weights(k, hidden, seed):
    rng = np.random.default_rng(seed)
    return [rng.normal(0, 0.3, hidden * 3), rng.normal(0, 0.1, hidden), rng.normal(0, 0.1, hidden * hidden),
            rng.normal(0, 0.1, hidden), rng.normal(0, 0.2, k * hidden), rng.normal(0, 0.1, k)]


@pytest.mark.parametrize("k,hidden", [(6, 32), (9, 128)])
def test_upsampler_weight_file_resave_is_byte_identical(ref, prog, tmp_path, k, hidden):
    """test_io.cpp:196-212 (upsampler weight JSON round trip), against the reference's writer."""
    ws = _up_weights(k, hidden, hidden)
    a, b = tmp_path / "up.json", tmp_path / "up2.json"
    assert ref.ref_save_upsampler_weights(str(a).encode(), k, hidden, *ws, 123) == 0
    r = subprocess.run([str(prog), "upsampler", str(a), str(b)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert f"k={k} hidden={hidden} epochs=123" in r.stdout
    assert b.read_bytes() == a.read_bytes()


def test_weight_loaders_reject_each_others_files(ref, prog, tmp_path):
    """test_io.cpp:175-194: the upsampler loader rejects codec files and vice versa."""
    re_, rd = _weights(6, 2)
    codec, up = tmp_path / "c.json", tmp_path / "u.json"
    assert ref.ref_save_codec_weights(str(codec).encode(), 6, 10.0, re_.reshape(-1), rd.reshape(-1), 1, np.zeros(5),
                                      0) == 0
    assert ref.ref_save_upsampler_weights(str(up).encode(), 6, 16, *_up_weights(6, 16, 1), 0) == 0
    r = subprocess.run([str(prog), "upsampler", str(codec), str(tmp_path / "x.json")], capture_output=True, text=True)
    assert r.returncode == 3 and "not an upsampler weights file" in r.stderr
    r = subprocess.run([str(prog), str(up), str(tmp_path / "y.json")], capture_output=True, text=True)
    assert r.returncode == 3 and "not a codec weights file" in r.stderr
