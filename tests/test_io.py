"""Instance bundles and the CSV result contract (csrc/io.hpp via the C ABI).

Ports the reference's tests/test_io.cpp cases (cited per test) and pins the
implementation against the reference's OWN io.cpp, compiled unmodified by
oracle/Makefile.ref into oracle/_ref/libref_io.so (skipped when that build
is absent): bundles written here load bit-exactly there and vice versa,
format_double / fnv1a64 / CsvWriter produce the same bytes.  CPU only.
"""
import ctypes as C
import math
import os
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "libref_io.so")


@pytest.fixture(scope="module")
def io():
    from paper_2405_00366_b200 import io as IO
    return IO


@pytest.fixture(scope="module")
def ref():
    if not os.path.exists(REF_IO):
        pytest.skip("reference io build oracle/_ref/libref_io.so not available")
    L = C.CDLL(REF_IO)
    vp = C.c_void_p
    L.ref_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
    L.ref_fnv1a64.restype = C.c_uint64
    L.ref_fnv1a64.argtypes = [C.c_char_p, C.c_uint64]
    L.ref_save_generated.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                     C.c_int, C.c_char_p]
    L.ref_load_instance.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, vp, vp, vp, vp]
    L.ref_csv.argtypes = [C.c_char_p, vp, C.c_int, vp, C.c_int, vp, vp, C.c_int]
    return L


def ref_fmt(ref, v):
    b = C.create_string_buffer(40)
    assert ref.ref_format_double(v, b, 40) == 0
    return b.value.decode()


def ref_load(ref, d):
    N, M, ht, sd = C.c_int(), C.c_int(), C.c_int(), C.c_uint64()
    meta = (C.c_double * 3)()
    assert ref.ref_load_instance(d.encode(), C.byref(N), C.byref(M), C.byref(ht), meta,
                                 C.byref(sd), None, None, None, None) == 0
    A = np.zeros((M.value, N.value), order="F")
    y = np.zeros(M.value)
    x = np.zeros(N.value)
    xi = np.zeros(N.value, np.int32)
    assert ref.ref_load_instance(d.encode(), C.byref(N), C.byref(M), C.byref(ht), meta,
                                 C.byref(sd), A.ctypes.data, y.ctypes.data, x.ctypes.data,
                                 xi.ctypes.data) == 0
    return dict(A=A, y=y, x=x if ht.value else None, xi=xi if ht.value else None,
                a=meta[0], alpha=meta[1], nu=meta[2], seed=sd.value)


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


# ---------------------------------------------------------------- ports of test_io.cpp

def test_format_double_round_trips_bitwise(io):
    """test_io.cpp:40-49."""
    for v in (0.0, -0.0, 1.0 / 3.0, 1e-300, -2.5e300, 0.125, 0.39215686, 6.02e23, -1.0 / 7.0):
        s = io.format_double(v)
        assert struct.pack("<d", float(s)) == struct.pack("<d", v), (v, s)


def test_hash_published_vectors(io):
    """test_io.cpp:51-56 (FNV-1a 64 test vectors)."""
    assert io.fnv1a64("") == 0xcbf29ce484222325
    assert io.fnv1a64("a") == 0xaf63dc4c8601ec8c
    assert io.hex64(0xcbf29ce484222325) == "cbf29ce484222325"
    assert io.hex64(0) == "0000000000000000"


def test_csv_writer_comments_header_rows(io, tmp_path):
    """test_io.cpp:58-77."""
    p = str(tmp_path / "basic.csv")
    with io.CsvWriter(p, ["alg test", "note two"], ["x", "y", "label"]) as w:
        w.row([io.cell(0.5), io.cell(3), "abc"])
        w.row([io.cell(-1.25), io.cell(1 << 40), "def"])
    lines = open(p).read().split("\n")
    assert lines[:5] == ["# alg test", "# note two", "x,y,label",
                         io.format_double(0.5) + ",3,abc",
                         io.format_double(-1.25) + ",1099511627776,def"]
    assert lines[5:] == [""]


def test_csv_writer_rejects_wrong_arity(io, tmp_path):
    """test_io.cpp:79-84."""
    from paper_2405_00366_b200 import InputError
    w = io.CsvWriter(str(tmp_path / "arity.csv"), [], ["a", "b"])
    with pytest.raises(InputError):
        w.row(["1"])
    with pytest.raises(InputError):
        w.row(["1", "2", "3"])
    w.close()


def test_bundle_round_trip_with_truth(io, tmp_path):
    """test_io.cpp:127-142: gen_instance(17, 0.7, 0.3, 0.2, 12345) survives exactly."""
    import paper_2405_00366_b200 as P
    inst = P.gen_instance(17, 0.7, 0.3, 0.2, 12345)
    d = str(tmp_path / "bundle_truth")
    io.save_instance(inst, d)
    back = io.load_instance(d)
    assert np.array_equal(bits(back.A), bits(inst.A))
    assert np.array_equal(bits(back.y), bits(inst.y))
    assert back.has_truth()
    assert np.array_equal(bits(back.x_true), bits(inst.x_true))
    assert np.array_equal(back.xi_true, inst.xi_true)
    assert (back.nu, back.seed, back.a, back.alpha) == (inst.nu, inst.seed, inst.a, inst.alpha)


def test_bundle_round_trip_without_truth(io, tmp_path):
    """test_io.cpp:144-155."""
    import paper_2405_00366_b200 as P
    inst = P.gen_instance(9, 0.6, 0.2, 0.0, 3)
    inst.x_true = inst.xi_true = None
    d = str(tmp_path / "bundle_blind")
    io.save_instance(inst, d)
    assert not os.path.exists(os.path.join(d, "truth.csv"))
    back = io.load_instance(d)
    assert np.array_equal(bits(back.A), bits(inst.A))
    assert np.array_equal(bits(back.y), bits(inst.y))
    assert not back.has_truth()


def test_bundle_count_mismatch_is_input_error(io, tmp_path):
    """io.cpp:139-152: row / column counts must match meta.json."""
    import paper_2405_00366_b200 as P
    inst = P.gen_instance(11, 0.6, 0.2, 0.01, 5)
    d = str(tmp_path / "bad")
    io.save_instance(inst, d)
    txt = open(os.path.join(d, "A.csv")).read().split("\n")
    open(os.path.join(d, "A.csv"), "w").write("\n".join(txt[1:]))  # one row short
    with pytest.raises(P.InputError, match="row count"):
        io.load_instance(d)
    io.save_instance(inst, d)
    rows = open(os.path.join(d, "A.csv")).read().split("\n")
    rows[0] = rows[0].rsplit(",", 1)[0]  # one column short
    open(os.path.join(d, "A.csv"), "w").write("\n".join(rows))
    with pytest.raises(P.InputError, match="column count"):
        io.load_instance(d)
    with pytest.raises(P.InputError):
        io.load_instance(str(tmp_path / "missing"))


def test_load_bundles_sorted_by_seed(io, tmp_path):
    """cmd_run --load (tools/main.cpp:390-400)."""
    import paper_2405_00366_b200 as P
    for s in (7, 2, 5):
        io.save_instance(P.gen_instance(8, 0.5, 0.25, 0.01, s), str(tmp_path / f"i{s}"))
    (tmp_path / "not_a_bundle").mkdir()
    assert [i.seed for i in io.load_bundles(str(tmp_path))] == [2, 5, 7]


def test_history_and_summary_tables(io, tmp_path):
    """Column contracts: history (orchestrator.cpp:253-264, test_orchestrator.cpp:
    388-392), summary (main.cpp:449-462, NaN for failed trials), failures
    (main.cpp:476-489, commas in reasons replaced by ';')."""
    import paper_2405_00366_b200 as P
    assert io.history_csv_columns() == ["trial", "i", "eta", "hamiltonian", "rmse", "hamming",
                                        "seconds"]
    insts = [P.gen_instance(8, 0.5, 0.25, 0.01, s) for s in (1, 2)]
    hist = [dict(i=0, eta=0.8, hamiltonian=-1.5, rmse=0.25, hamming=0.125, seconds=math.nan),
            dict(i=1, eta=0.18, hamiltonian=-2.0, rmse=0.125, hamming=0.0, seconds=math.nan)]
    ok = dict(failed=False, final_rmse=0.125, final_hamming=0.0, min_hamiltonian=-2.0,
              history=hist, fail_alternation=-1, fail_reason="")
    bad = dict(failed=True, final_rmse=0.5, final_hamming=0.5, min_hamiltonian=-1.0,
               history=hist[:1], fail_alternation=0, fail_reason="mfz_step: x, y")
    n = io.write_run_tables(str(tmp_path), insts, [ok, bad], "mfz-bn", "00ff00ff00ff00ff")
    assert n == 1
    s = open(tmp_path / "summary.csv").read().split("\n")
    assert s[:3] == ["# config 00ff00ff00ff00ff", "# rng mt19937_64-boxmuller-v1", "# seeds 1 2"]
    assert s[3] == ",".join(io.SUMMARY_COLUMNS)
    assert s[4] == "mfz-bn,0.25,0.5,0.01,1,0.125,0,-2"
    assert s[5] == "mfz-bn,0.25,0.5,0.01,2,nan,nan,nan"
    h = open(tmp_path / "history_mfz-bn.csv").read().split("\n")
    assert h[3] == "trial,i,eta,hamiltonian,rmse,hamming,seconds"
    assert h[4] == "0,0,0.8,-1.5,0.25,0.125,nan" and h[6] == "1,0,0.8,-1.5,0.25,0.125,nan"
    f = open(tmp_path / "failures.csv").read().split("\n")
    assert f[4] == "mfz-bn,0.25,0.5,0.01,2,0,mfz_step: x; y"


# ------------------------------------------------- pins against the reference's io.cpp

def test_format_double_matches_reference(io, ref):
    rng = np.random.default_rng(0)
    vals = list(rng.normal(size=300)) + list(rng.normal(size=100) * 10.0 ** rng.integers(
        -300, 300, size=100)) + [0.0, -0.0, 5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                                 0.1, 0.2, 0.3, 1.0, 100.0, 1e21, 1e-7, float("inf"), float("nan")]
    for v in vals:
        assert io.format_double(v) == ref_fmt(ref, float(v))


def test_format_double_matches_reference_random_bits(io, ref):
    """20000 doubles drawn as random 64-bit patterns (every exponent, denormals, NaN
    payloads, infinities): byte-identical to the reference's format_double (io.cpp:18-25).
    (A 100000-value run of the same loop is also clean.)"""
    vals = np.random.default_rng(1).integers(0, 2 ** 64, size=20000, dtype=np.uint64).view(np.float64)
    for v in vals:
        assert io.format_double(float(v)) == ref_fmt(ref, float(v))


def test_fnv1a64_matches_reference(io, ref):
    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 64, 1000):
        b = bytes(rng.integers(0, 256, size=n, dtype=np.uint8))
        assert io.fnv1a64(b) == ref.ref_fnv1a64(b, n)


@pytest.mark.parametrize("truth", [1, 0])
def test_reference_bundle_loads_bit_exactly_here(io, ref, tmp_path, truth):
    import paper_2405_00366_b200 as P
    d = str(tmp_path / f"ref{truth}")
    assert ref.ref_save_generated(23, 0.6, 0.2, 0.05, 99, truth, d.encode()) == 0
    back = io.load_instance(d)
    inst = P.gen_instance(23, 0.6, 0.2, 0.05, 99)  # the same generator stream (test_pins.py)
    assert np.array_equal(bits(back.A), bits(inst.A))
    assert np.array_equal(bits(back.y), bits(inst.y))
    assert back.has_truth() == bool(truth)
    if truth:
        assert np.array_equal(bits(back.x_true), bits(inst.x_true))
        assert np.array_equal(back.xi_true, inst.xi_true)
    assert (back.a, back.alpha, back.nu, back.seed) == (0.2, 0.6, 0.05, 99)


def test_bundle_written_here_loads_bit_exactly_in_reference(io, ref, tmp_path):
    import paper_2405_00366_b200 as P
    inst = P.gen_instance(31, 0.7, 0.3, 0.01, 2024)
    d = str(tmp_path / "ours")
    io.save_instance(inst, d)
    r = ref_load(ref, d)
    assert np.array_equal(bits(r["A"]), bits(inst.A))
    assert np.array_equal(bits(r["y"]), bits(inst.y))
    assert np.array_equal(bits(r["x"]), bits(inst.x_true))
    assert np.array_equal(r["xi"], inst.xi_true)
    assert (r["a"], r["alpha"], r["nu"], r["seed"]) == (0.3, 0.7, 0.01, 2024)
    # same bytes as the reference's own writer, meta.json included
    d2 = str(tmp_path / "theirs")
    assert ref.ref_save_generated(31, 0.7, 0.3, 0.01, 2024, 1, d2.encode()) == 0
    for f in ("A.csv", "y.csv", "truth.csv", "meta.json"):
        assert open(os.path.join(d, f), "rb").read() == open(os.path.join(d2, f), "rb").read(), f


def test_csv_bytes_match_reference(io, ref, tmp_path):
    comments, cols = ["config abc", "seeds 1 2 3"], ["backend", "a", "n"]
    rows = [["mfz-bn", io.cell(0.1), io.cell(3)], ["mfz-cn", io.cell(-2.5e-300), io.cell(1 << 40)],
            ["x"]]
    ours = str(tmp_path / "ours.csv")
    w = io.CsvWriter(ours, comments, cols)
    rejected = 0
    for r in rows:
        try:
            w.row(r)
        except Exception:
            rejected += 1
    w.close()
    theirs = str(tmp_path / "theirs.csv")
    enc = lambda xs: (C.c_char_p * len(xs))(*[x.encode() for x in xs])  # noqa: E731
    flat = [c for r in rows for c in r]
    widths = (C.c_int * len(rows))(*[len(r) for r in rows])
    n = ref.ref_csv(theirs.encode(), enc(comments), len(comments), enc(cols), len(cols),
                    enc(flat), widths, len(rows))
    assert n == rejected == 1
    assert open(ours, "rb").read() == open(theirs, "rb").read()
