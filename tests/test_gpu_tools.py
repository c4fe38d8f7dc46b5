"""GPU: the reference's encode / decode tools (tools/main.cpp:285-328) as device pipelines —
spectra CSV (%.9g, io.cpp:119-186), resample (spectrum.cpp:60-98), the fp64 codec
(codec.cpp:36-71) and the codes CSV — byte-identical to the compiled reference (oracle/_ref)
running the same tool steps."""
import ctypes

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N = 81


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


@pytest.fixture(scope="module")
def ref():
    r = oracle.reference(N)
    if r is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    return r


def _raw(k, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-0.5, 0.5, (k, N)) / np.sqrt(N), rng.uniform(-0.5, 0.5, (N, k)) / np.sqrt(N))


def _spectra_text(seed, rows, grid, ids):
    """A spectra CSV as a measurement tool would write it: any grid, %.9g-ish values."""
    rng = np.random.default_rng(seed)
    head = (["id"] if ids else []) + ["%.9g" % w for w in grid]
    lines = [",".join(head)]
    for r in range(rows):
        v = np.clip(rng.normal(0.5, 0.3, len(grid)), 0, None) * rng.uniform(0.1, 3.0)
        cells = (["s%05d_%s" % (r, "abc"[r % 3])] if ids else []) + ["%.*g" % (int(rng.integers(3, 17)), x) for x in v]
        lines.append(", ".join(cells) if r % 7 == 0 else ",".join(cells))
        if r % 11 == 0:
            lines.append("  ")
    return ("\n".join(lines) + "\n").encode()


GRIDS = {"1nm_360_830": np.arange(360.0, 830.5, 1.0), "5nm_400_700": np.arange(400.0, 700.5, 5.0),
         "irregular": np.cumsum(np.r_[372.5, np.random.default_rng(3).uniform(0.5, 9.0, 70)]),
         "narrow_450_650": np.linspace(450.0, 650.0, 17), "single": np.array([555.0]),
         "half_nm_941": np.arange(360.0, 830.25, 0.5)}  # > 512 cells per row: the one-lane fallback


@pytest.mark.parametrize("grid_name", list(GRIDS))
@pytest.mark.parametrize("ids", [True, False])
def test_encode_tool_matches_reference(api, ctx, ref, tmp_path, grid_name, ids):
    k = 6
    re_, rd = _raw(k, 7)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    data = _spectra_text(len(grid_name), 700, GRIDS[grid_name], ids)
    src, out = tmp_path / "s.csv", tmp_path / "codes.csv"
    src.write_bytes(data)
    err = ctypes.create_string_buffer(512)
    assert ref.ref_run_encode(str(src).encode(), k, 10.0, np.ascontiguousarray(re_.reshape(-1)),
                              np.ascontiguousarray(rd.reshape(-1)), str(out).encode(), err, 512) == 0, err.value
    got = api.encode_tool(codec, data)
    assert got == out.read_bytes()


@pytest.mark.parametrize("k", [3, 6, 9])
def test_decode_tool_matches_reference(api, ctx, ref, tmp_path, k):
    re_, rd = _raw(k, k)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    rng = np.random.default_rng(k)
    Z = rng.lognormal(-1, 2, (900, k)) * (rng.random((900, k)) > 0.1)
    data = api.codes_csv(ctx, torch.from_numpy(Z).cuda(), ids=["c%d" % i for i in range(900)])
    src, out = tmp_path / "codes.csv", tmp_path / "s.csv"
    src.write_bytes(data)
    err = ctypes.create_string_buffer(512)
    assert ref.ref_run_decode(str(src).encode(), k, 10.0, np.ascontiguousarray(re_.reshape(-1)),
                              np.ascontiguousarray(rd.reshape(-1)), str(out).encode(), err, 512) == 0, err.value
    got = api.decode_tool(codec, data)
    assert got == out.read_bytes()
    # encode(decode(z)) through both tools' files, once more through the reference
    data2 = _spectra_text(1, 5, GRIDS["5nm_400_700"], True)
    assert api.encode_tool(codec, api.decode_tool(codec, data)).startswith(b"id,c0")
    assert data2


def test_decode_rejects_negative_codes_like_reference(api, ctx, ref, tmp_path):
    k = 6
    re_, rd = _raw(k, 1)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    Z = np.abs(np.random.default_rng(0).normal(size=(50, k)))
    Z[37, 2] = -1e-300
    data = api.codes_csv(ctx, torch.from_numpy(Z).cuda(), ids=[str(i) for i in range(50)])
    src, out = tmp_path / "codes.csv", tmp_path / "s.csv"
    src.write_bytes(data)
    err = ctypes.create_string_buffer(512)
    assert ref.ref_run_decode(str(src).encode(), k, 10.0, np.ascontiguousarray(re_.reshape(-1)),
                              np.ascontiguousarray(rd.reshape(-1)), str(out).encode(), err, 512) == 1
    assert b"non-negative" in err.value
    with pytest.raises(ArithmeticError, match="row 37"):
        api.decode_tool(codec, data)


def test_resample_rejects_bad_grids(api, ctx):
    k = 6
    re_, rd = _raw(k, 2)
    codec = api.Codec.from_raw(ctx, re_, rd, beta=10.0)
    v = torch.ones(3, 4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="strictly increasing"):
        api.encode_resampled(codec, np.array([400.0, 500.0, 500.0, 600.0]), v)
    with pytest.raises(ValueError, match="strictly increasing"):
        api.encode_resampled(codec, np.array([400.0, 390.0, 500.0, 600.0]), v)


@pytest.mark.parametrize("with_ids", [True, False])
def test_spectra_csv_writer_matches_reference(api, ctx, ref, tmp_path, with_ids):
    from paper_2602_18741_b200.colorimetry import wavelengths

    rng = np.random.default_rng(5)
    rows = 3000
    V = rng.lognormal(0, 25, (rows, N)) * rng.choice([-1.0, 1.0], (rows, N))
    V[rng.random((rows, N)) < 0.03] = 0.0
    V[0, :6] = [0.1, 1.0 / 3.0, 2.5e-310, -0.0, 123456789.5, 0.5e-4]
    ids = ["row%d" % r for r in range(rows)] if with_ids else None
    got = api.spectra_csv(ctx, torch.from_numpy(V).cuda(), wavelengths(N), ids=ids)
    path = tmp_path / "s.csv"
    if with_ids:
        blob = "".join(ids).encode()
        lens = np.array([len(i) for i in ids], np.int64)
        spans = np.stack([np.r_[0, np.cumsum(lens)[:-1]], lens], 1).astype(np.int64).copy()
        assert ref.ref_write_spectra_csv(str(path).encode(), np.ascontiguousarray(V.reshape(-1)), rows, blob,
                                         spans.ctypes.data) == 0
    else:
        assert ref.ref_write_spectra_csv(str(path).encode(), np.ascontiguousarray(V.reshape(-1)), rows, b"",
                                         None) == 0
    assert got == path.read_bytes()
    # every cell is glibc's %.9g
    cells = got.decode().splitlines()[1].split(",")[1 if with_ids else 0:]
    assert cells == ["%.9g" % x for x in V[0]]


def test_g9_matches_glibc_on_hard_values(api, ctx):
    """%.9g on values whose 10th digit makes an exact tie (dyadic rationals), widened floats
    and every exponent range."""
    rng = np.random.default_rng(9)
    n = 81 * 2000
    v = np.concatenate([rng.integers(1, 2**40, n // 4) / 2.0 ** rng.integers(0, 60, n // 4),
                        rng.normal(0, 1, n // 4).astype(np.float32).astype(np.float64) * 2.0 ** rng.integers(-60, 60, n // 4),
                        rng.integers(0, 2**63 - 1, n // 4, dtype=np.int64).view(np.float64),
                        rng.integers(1, 2**52, n // 4, dtype=np.int64).view(np.float64)])
    v = v[np.isfinite(v)]
    v = v[: (v.size // N) * N].reshape(-1, N)
    from paper_2602_18741_b200.colorimetry import wavelengths

    got = api.spectra_csv(ctx, torch.from_numpy(v).cuda(), wavelengths(N)).decode().splitlines()[1:]
    want = [",".join("%.9g" % x for x in row) for row in v]
    bad = [(g, w) for g, w in zip(got, want) if g != w]
    assert not bad, bad[:2]


@pytest.mark.parametrize("ids", [True, False])
def test_spectra_csv_reader_matches_reference(api, ctx, ref, tmp_path, ids):
    data = _spectra_text(11, 2500, GRIDS["irregular"], ids)
    path = tmp_path / "s.csv"
    path.write_bytes(data)
    has_id, m, rows = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    wl = np.zeros(512)
    vals = np.zeros(2500 * 80)
    idbuf = ctypes.create_string_buffer(2500 * 16)
    assert ref.ref_read_spectra_csv(str(path).encode(), ctypes.byref(has_id), wl, 512, ctypes.byref(m),
                                    ctypes.byref(rows), vals, vals.size, idbuf, len(idbuf)) == 0
    gwl, gids, gvals, _ = api.read_spectra_csv(ctx, data)
    assert gwl.tobytes() == wl[: m.value].tobytes()
    assert gvals.cpu().numpy().tobytes() == vals[: rows.value * m.value].tobytes()
    if ids:
        assert gids == idbuf.value.decode().split("\n")[: rows.value]
    else:
        assert gids is None and has_id.value == 0


SPECTRA_BAD = [
    b"",                                   # missing header
    b"id\nx\n",                            # empty wavelength header
    b"400,500,x\n1,2,3\n",                 # bad wavelength
    b"400,500\n1,2,3\n",                   # wrong cell count
    b"id,400,500\na,1\n",                  # wrong cell count with ids
    b"400,500\n1,2e999\n",                 # out of range
    b"400,500\n1,2z\n",                    # trailing junk
]


@pytest.mark.parametrize("case", range(len(SPECTRA_BAD)))
def test_spectra_csv_reader_errors_match_reference(api, ctx, ref, tmp_path, case):
    data = SPECTRA_BAD[case]
    path = tmp_path / "s.csv"
    path.write_bytes(data)
    has_id, m, rows = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    wl, vals = np.zeros(16), np.zeros(64)
    idbuf = ctypes.create_string_buffer(512)
    assert ref.ref_read_spectra_csv(str(path).encode(), ctypes.byref(has_id), wl, 16, ctypes.byref(m),
                                    ctypes.byref(rows), vals, vals.size, idbuf, len(idbuf)) == 1
    with pytest.raises(ValueError):
        api.read_spectra_csv(ctx, data)


@pytest.mark.parametrize("k", [3, 6, 9])
def test_fp64_encode_decode_bit_identical_to_reference(api, ctx, ref, k):
    """hc_encode_f64 / hc_decode_f64 (the drop-in's by-value encode / decode) against the
    reference's encode / decode on the same (float-valued) weights and inputs."""
    rng = np.random.default_rng(40 + k)
    E = rng.uniform(0, 1, (k, N)).astype(np.float32)
    D = rng.uniform(0, 1, (N, k)).astype(np.float32)
    codec = api.Codec(ctx, E, D)
    rows = 4096
    S = rng.uniform(0, 2, (rows, N)).astype(np.float32)
    Z = api.encode_f64(codec, torch.from_numpy(S.astype(np.float64)).cuda()).cpu().numpy()
    Zr = np.zeros((rows, k))
    ref.ref_encode_rows_d(E.reshape(-1), k, S.reshape(-1), rows, Zr.reshape(-1), 1)
    assert Z.tobytes() == Zr.tobytes()
    Sd = api.decode_f64(codec, torch.from_numpy(Z).cuda()).cpu().numpy()
    Sr = np.zeros((rows, N))
    assert ref.ref_decode_rows_d(np.ascontiguousarray(D.reshape(-1)), k, np.ascontiguousarray(Z.reshape(-1)), rows,
                                 Sr.reshape(-1)) == 0
    assert Sd.tobytes() == Sr.tobytes()


@pytest.mark.parametrize("kind", ["junk", "short", "range", "ok"])
def test_long_line_errors_report_the_reference_line(api, ctx, ref, tmp_path, kind):
    """Errors inside long (cooperatively parsed) spectra rows: same first bad line."""
    lines = _spectra_text(3, 1500, GRIDS["1nm_360_830"], True).decode().split("\n")
    if kind == "junk":
        cells = lines[901].split(",")
        cells[200] = cells[200] + "x"
        lines[901] = ",".join(cells)
        cells = lines[1200].split(",")
        cells[3] = "abc"
        lines[1200] = ",".join(cells)
    elif kind == "short":
        lines[640] = ",".join(lines[640].split(",")[:-1])
    elif kind == "range":
        cells = lines[77].split(",")
        cells[-1] = "1e-400"
        lines[77] = ",".join(cells)
    data = "\n".join(lines).encode()
    path = tmp_path / "s.csv"
    path.write_bytes(data)
    has_id, m, rows = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    wl, vals = np.zeros(1024), np.zeros(1500 * 480)
    idbuf = ctypes.create_string_buffer(1500 * 16 + 1024)
    rc = ref.ref_read_spectra_csv(str(path).encode(), ctypes.byref(has_id), wl, 1024, ctypes.byref(m),
                                  ctypes.byref(rows), vals, vals.size, idbuf, len(idbuf))
    if kind == "ok":
        assert rc == 0
        _, _, gv, _ = api.read_spectra_csv(ctx, data)
        assert gv.cpu().numpy().tobytes() == vals[: rows.value * m.value].tobytes()
        return
    assert rc == 1
    line = idbuf.value.decode().split(":")[1]
    with pytest.raises(ValueError, match=rf"\(line {line}\)"):
        api.read_spectra_csv(ctx, data)
