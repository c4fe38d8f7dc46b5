"""GPU formats: print_g17 ("%.17g", io.cpp:108-112) and the codes CSV
(write_codes_csv, io.cpp:312-330) produced on the device, byte-identical to glibc's printf
(which Python's "%.17g" reproduces exactly) and to the reference's own writer (oracle/_ref)."""
import struct

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    from paper_2602_18741_b200 import api as a

    return a


@pytest.fixture(scope="module")
def ctx(api):
    return api.Context(0)


def _values(seed: int, n: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2**63 - 1, n, dtype=np.int64).view(np.float64)          # every exponent
    bits = bits[np.isfinite(bits)]
    uni = rng.random(n)                                                              # [0, 1)
    ints = rng.integers(-10**17, 10**17, n).astype(np.float64)                      # integers, 1e17 edge
    f32 = rng.normal(0, 1, n).astype(np.float32).astype(np.float64) * 10.0 ** rng.integers(-12, 12, n)
    f32w = rng.normal(0, 1, n).astype(np.float32).astype(np.float64) * 2.0 ** rng.integers(-60, 60, n)  # widened floats
    dyad = rng.integers(1, 2**40, n) / 2.0 ** rng.integers(0, 70, n)                # exact 17th-digit ties
    sub = rng.integers(1, 2**52, n // 10, dtype=np.int64).view(np.float64)          # subnormals
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1.7976931348623157e308, 2.2250738585072014e-308,
                        1e-5, 1e-4, 0.0001234, 1e16, 1e17, 9.9999999999999995e16, 99999999999999999.0,
                        1234567890123456.75, 1234567890123456.25, 0.1, 0.5, 1.0, 123.0, 2.0**63, 2.0**-1074,
                        0.30000000000000004, 9.5367431640625e-07, 1e22, 1e23, 4.35e-6])
    return np.concatenate([bits, uni, -uni, ints, f32, f32w, -dyad, dyad, sub, special])


def test_format_g17_matches_glibc(api, ctx):
    v = _values(7, 200_000)
    got = api.format_g17(ctx, torch.from_numpy(v).cuda())
    want = ["%.17g" % x for x in v]
    bad = [(x, g, w) for x, g, w in zip(v, got, want) if g != w]
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:5]}"


@pytest.mark.parametrize("rows,k", [(1, 6), (1000, 9), (70_001, 6), (0, 3)])
def test_codes_csv_matches_reference_writer(api, ctx, tmp_path, rows, k):
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    rng = np.random.default_rng(rows + k)
    Z = (rng.lognormal(-1, 2, (rows, k)) * (rng.random((rows, k)) > 0.05)).astype(np.float32)
    got = api.codes_csv(ctx, torch.from_numpy(Z).cuda().reshape(rows, k), first_id=1000)
    path = tmp_path / "codes.csv"
    assert ref.ref_write_codes_csv(str(path).encode(), np.ascontiguousarray(Z.reshape(-1)), rows, k, 1000) == 0
    want = path.read_bytes()
    assert got == want  # rows == 0: "id\n" (the reference's k is 0 for no codes)


def _ids_blob(ids):
    enc = [i.encode() for i in ids]
    off = np.zeros(len(enc) + 1, np.int64)
    np.cumsum([len(e) for e in enc], out=off[1:])
    return b"".join(enc) or b"\0", off


@pytest.mark.parametrize("rows,k", [(2, 6), (5000, 9), (0, 6)])
def test_codes_csv_double_codes_string_ids_match_reference_writer(api, ctx, tmp_path, rows, k):
    """The reference's own signature: LatentCode (double) values and arbitrary string ids."""
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    rng = np.random.default_rng(rows)
    if rows == 2:  # test_io.cpp "codes CSV round trip and validation"
        Z = np.array([[0.1, 0.25, 1.0 / 3.0, 0.0, 5e-17, 2.0], [1, 2, 3, 4, 5, 6]], np.float64)
        ids = ["x", "y"]
    else:
        Z = rng.lognormal(0, 30, (rows, k)) * rng.choice([-1.0, 1.0], (rows, k))
        Z[rng.random((rows, k)) < 0.05] = 0.0
        ids = [("row%d" % r) if r % 3 else ("sample_%x-%d" % (r * 7919, r)) for r in range(rows)]
    got = api.codes_csv(ctx, torch.from_numpy(Z).cuda().reshape(rows, k), ids=ids)
    blob, off = _ids_blob(ids)
    path = tmp_path / "codes.csv"
    assert ref.ref_write_codes_csv_ids(str(path).encode(), np.ascontiguousarray(Z.reshape(-1)), rows, k, blob, off) == 0
    assert got == path.read_bytes()
    if rows:
        back_ids, back = api.read_codes_csv(ctx, got)
        assert back_ids == ids
        assert back.cpu().numpy().tobytes() == Z.tobytes()  # %.17g round-trips doubles bit-exactly


def _glibc_strtod(cells):
    """(value, status) as the reference's parse_double sees them: std::stod = strtod + ERANGE
    -> throw, and the whole cell must be consumed (io.cpp:78-88)."""
    import ctypes

    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.strtod.restype = ctypes.c_double
    libc.strtod.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_char_p)]
    vals, sts = [], []
    for c in cells:
        ctypes.set_errno(0)
        end = ctypes.c_char_p()
        v = libc.strtod(c, ctypes.byref(end))
        rest = end.value if end.value is not None else b""
        consumed = len(c) - len(rest)
        err = ctypes.get_errno()
        if consumed == 0 or consumed != len(c):
            st = 1
        elif err:
            st = 2
        else:
            st = 0
        vals.append(v)
        sts.append(st)
    return np.array(vals), np.array(sts)


def test_parse_doubles_matches_glibc_strtod(api, ctx):
    rng = np.random.default_rng(3)
    cells = [b"0", b"-0", b"1", b"+1.5", b".5", b"5.", b"1e5", b"1E-5", b"1e+", b"1e5x", b"abc", b"", b"-", b".",
             b"inf", b"-Infinity", b"NaN", b"nan(123)", b"infx", b"0x1p3", b"0x1.8p-1", b"0X.8", b"0x", b"0x1p-1074",
             b"0x1p-1075", b"0x1.0000000000001p0", b"4.9406564584124654e-324", b"2.2250738585072014e-308",
             b"2.2250738585072009e-308", b"1e-320", b"1e309", b"1.7976931348623157e308", b"1.7976931348623159e308",
             b"1e-400", b"0.000000000000000000000000000001", b"123456789012345678901234567890",
             b"9007199254740993", b"9007199254740992.5", b"1.00000000000000011102230246251565404236316680908203125",
             b"1.00000000000000011102230246251565404236316680908203124", b"2.4703282292062327e-324",
             b"2.4703282292062328e-324", b"00012.50", b"1_0", b"1,5", b" 1"]
    # %.17g strings of every exponent, short decimals, long digit strings
    bits = rng.integers(0, 2**63 - 1, 30000, dtype=np.int64).view(np.float64)
    cells += [("%.17g" % v).encode() for v in bits if np.isfinite(v)]
    cells += [("%.*g" % (int(p), v)).encode() for p, v in zip(rng.integers(1, 17, 20000), rng.lognormal(0, 30, 20000))]
    cells += [("%de%d" % (int(a), int(b))).encode() for a, b in zip(rng.integers(1, 10**15, 5000), rng.integers(-340, 320, 5000))]
    long_digits = ["".join(rng.choice(list("0123456789"), int(n))) for n in rng.integers(20, 60, 2000)]
    cells += [(d[:3] + "." + d[3:] + "e" + str(int(e))).encode() for d, e in zip(long_digits, rng.integers(-320, 300, 2000))]
    got, gst = api.parse_doubles(ctx, cells)
    want, wst = _glibc_strtod(cells)
    bad = []
    for c, g, s, w, t in zip(cells, got, gst, want, wst):
        same = (s == t) and (t != 0 or (np.isnan(g) and np.isnan(w)) or g.tobytes() == w.tobytes())
        if not same:
            bad.append((c, g, s, w, t))
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:6]}"


def _ref_read(ref, path, cap_rows=200_000, k=9):
    import ctypes

    rows, kk = ctypes.c_int64(), ctypes.c_int()
    codes = np.zeros(cap_rows * k, np.float64)
    ids = ctypes.create_string_buffer(cap_rows * 24 + 4096)
    rc = ref.ref_read_codes_csv(str(path).encode(), ctypes.byref(rows), ctypes.byref(kk), codes, codes.size, ids,
                                len(ids))
    if rc:
        return None, ids.value.decode()
    n = rows.value * kk.value
    return (ids.value.decode().split("\n")[:rows.value], codes[:n].reshape(rows.value, kk.value)), None


@pytest.mark.parametrize("rows,k", [(1, 3), (5000, 6), (123_457, 9)])
def test_codes_csv_round_trip_matches_reference_reader(api, ctx, tmp_path, rows, k):
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    rng = np.random.default_rng(rows)
    Z = (rng.lognormal(-1, 3, (rows, k)) * (rng.random((rows, k)) > 0.05)).astype(np.float32)
    data = api.codes_csv(ctx, torch.from_numpy(Z).cuda(), first_id=7)
    path = tmp_path / "c.csv"
    path.write_bytes(data)
    ids, codes = api.read_codes_csv(ctx, data)
    (rids, rcodes), err = _ref_read(ref, path, rows, k)
    assert err is None
    assert ids == rids == [str(7 + r) for r in range(rows)]
    got = codes.cpu().numpy()
    assert got.tobytes() == rcodes.tobytes()
    assert np.array_equal(got, Z.astype(np.float64))  # %.17g round-trips the widened floats exactly


CASES = [
    b"id,c0,c1\na,1,2\nb,3.5,-4e-3\n",
    b"\n  \nid , c0 ,c1\r\n  x , 1e5 , .5 \r\n\n y,inf,-0x1p-3\n",   # blank lines, CRLF, spaces, inf, hex
    b"id,c0\nr0,1\nr1,2",                                          # no trailing newline
    b"id,c0,c1\na,1\n",                                            # wrong cell count
    b"id,c0,c1\na,1,2x\n",                                         # trailing junk
    b"id,c0,c1\na,1,1e400\n",                                      # out of range
    b"ix,c0\na,1\n",                                               # bad header
    b"id,c0,c2\na,1,2\n",                                          # bad header column
    b"   \n\n",                                                    # missing header
    b"id,c0,c1\n,1,2\nb,,3\n",                                     # empty id, empty cell
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_codes_csv_reader_edge_cases_match_reference(api, ctx, tmp_path, case):
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    data = CASES[case]
    path = tmp_path / "c.csv"
    path.write_bytes(data)
    want, err = _ref_read(ref, path, 16, 4)
    if err is not None:
        with pytest.raises(ValueError):
            api.read_codes_csv(ctx, data)
        return
    ids, codes = api.read_codes_csv(ctx, data)
    assert ids == want[0]
    assert codes.cpu().numpy().tobytes() == want[1].tobytes()


def _messy_csv(seed: int, rows: int, k: int) -> bytes:
    """Valid codes CSV with the whitespace, blank lines, long lines and number spellings
    read_codes_csv accepts: isspace bytes (\\t \\v \\f \\r, space) around cells and next to
    newlines, >19-digit decimals (exact path), leading zeros, exponents, hex, inf."""
    rng = np.random.default_rng(seed)
    ws = [b"", b" ", b"\t", b"\x0b", b"\x0c", b"\r", b"  \x0b"]
    out = [b"id," + b",".join(b"c%d" % j for j in range(k)) + b"\n"]
    for r in range(rows):
        if rng.random() < 0.05:
            out.append(rng.choice(ws) + b"\n")  # blank (whitespace-only) line
        cells = [b"r%d" % r]
        for _ in range(k):
            kind = rng.integers(0, 6)
            if kind == 0:
                cells.append(b"%.17g" % rng.lognormal(0, 20))
            elif kind == 1:
                cells.append(b"0.000" + bytes(rng.integers(48, 58, rng.integers(20, 60)).astype(np.uint8)))
            elif kind == 2:
                cells.append(b"-%de%d" % (rng.integers(1, 10**9), rng.integers(-300, 290)))
            elif kind == 3:
                cells.append(b"00%d.%d" % (rng.integers(0, 1000), rng.integers(0, 10**6)))
            elif kind == 4:
                cells.append(b"0x1.%xp%d" % (rng.integers(0, 2**40), rng.integers(-1000, 1000)))
            else:
                cells.append(b"%.9g" % rng.standard_normal())
        pad = b" " * int(rng.integers(300, 900)) if rng.random() < 0.02 else b""  # long lines
        line = b",".join(bytes(rng.choice(ws)) + c + bytes(rng.choice(ws)) for c in cells)
        out.append(bytes(rng.choice(ws)) + line + pad + bytes(rng.choice(ws)) + b"\n")
    return b"".join(out)


@pytest.mark.parametrize("shift", [0, 1, 3, 7, 13])
def test_codes_csv_reader_messy_text_unaligned_matches_reference(api, ctx, tmp_path, shift):
    ref = oracle.reference(81)
    if ref is None:
        pytest.skip("compiled reference (oracle/_ref) not built")
    rows, k = 3000, 5
    data = _messy_csv(shift, rows, k)
    assert len(data) > 4 * 16384  # several newline chunks
    path = tmp_path / "c.csv"
    path.write_bytes(data)
    (rids, rcodes), err = _ref_read(ref, path, rows, k)
    assert err is None, err
    buf = torch.zeros(len(data) + 32, dtype=torch.uint8, device="cuda")
    buf[shift:shift + len(data)] = torch.frombuffer(bytearray(data), dtype=torch.uint8).cuda()
    ids, codes = api.read_codes_csv(ctx, data, text=buf[shift:shift + len(data)])
    assert ids == rids
    assert codes.cpu().numpy().tobytes() == rcodes.tobytes()
