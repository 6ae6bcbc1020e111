"""Cross-pins of the random streams and the instance generator.

Three independent implementations must agree bit for bit:
  * the reference's own rng.hpp + datagen.cpp, compiled from /root/reference
    by oracle/Makefile.ref into oracle/_ref/libref.so (skipped if not built);
  * the C oracle's restatement (oracle/oracle.c);
  * the product's host generator in libcimcs_gpu.so (std::mt19937_64).
CPU only (the product calls here are host functions).
"""
import ctypes as C
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libref.so")


def _ref():
    if not os.path.exists(REF_SO):
        mk = os.path.join(ROOT, "oracle", "Makefile.ref")
        if os.path.isdir("/root/reference/proj"):
            import subprocess
            subprocess.check_call(["make", "-s", "-C", os.path.dirname(mk), "-f", "Makefile.ref"])
        else:
            pytest.skip("reference build oracle/_ref not available")
    L = C.CDLL(REF_SO)
    L.ref_gen_instance.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_gauss.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
    L.ref_raw.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
    L.ref_uniform_below.restype = C.c_uint64
    L.ref_uniform_below.argtypes = [C.c_uint64, C.c_uint64]
    return L


@pytest.mark.parametrize("seed", [0, 1, 7, 5489, 2**63 + 12345])
def test_oracle_rng_matches_reference_rng(O, seed):
    L = _ref()
    n = 2000
    raw = np.zeros(n, np.uint64)
    L.ref_raw(seed, n, raw.ctypes.data)
    r = O.Rng(seed)
    assert [r.raw() for _ in range(n)] == [int(v) for v in raw]
    g = np.zeros(n)
    L.ref_gauss(seed, n, g.ctypes.data)
    r = O.Rng(seed)
    assert np.array_equal(np.array([r.gauss() for _ in range(n)]), g)
    for bound in (1, 3, 1000, 2**40 + 7):
        r = O.Rng(seed)
        assert r.uniform_below(bound) == L.ref_uniform_below(seed, bound)


@pytest.mark.parametrize("args", [(500, 0.6, 0.2, 0.01, 0), (40, 0.5, 0.2, 0.1, 3),
                                  (2000, 0.5, 0.1, 0.01, 1), (12, 8 / 12, 0.25, 0.0, 11)])
def test_oracle_datagen_matches_reference(O, args):
    L = _ref()
    N = args[0]
    inst = O.gen_instance(*args)
    A = np.zeros((inst.M, N), order="F")
    y, x = np.zeros(inst.M), np.zeros(N)
    xi = np.zeros(N, np.int32)
    M = C.c_int()
    assert L.ref_gen_instance(*args, A.ctypes.data, y.ctypes.data, x.ctypes.data,
                              xi.ctypes.data, C.byref(M)) == 0
    assert M.value == inst.M
    assert np.array_equal(A, inst.A)
    assert np.array_equal(x, inst.x_true)
    assert np.array_equal(xi, inst.xi_true)
    # y = A w + noise: the shim's GEMV is sequential like the oracle's
    assert np.array_equal(y, inst.y)


@pytest.mark.parametrize("args", [(500, 0.6, 0.2, 0.01, 0), (2000, 0.5, 0.1, 0.01, 5),
                                  (64, 0.3, 0.05, 0.01, 9)])
def test_product_generator_matches_oracle(O, args):
    from paper_2405_00366_b200 import cimcs as P
    a = P.gen_instance(*args)
    b = O.gen_instance(*args)
    assert np.array_equal(a.A, b.A)
    assert np.array_equal(a.y, b.y)
    assert np.array_equal(a.x_true, b.x_true)
    assert np.array_equal(a.xi_true, b.xi_true)


def test_product_batch_generator(O):
    from paper_2405_00366_b200 import cimcs as P
    params = [(0.5, 0.1, 0.01, s) for s in range(1, 6)]
    many = P.gen_instances(200, params, threads=3)
    for p, inst in zip(params, many):
        ref = O.gen_instance(200, *p)
        assert np.array_equal(inst.A, ref.A) and np.array_equal(inst.y, ref.y)


def test_mix_seed_matches(O):
    from paper_2405_00366_b200 import cimcs as P
    for base, salt in ((0, 1), (1, 0), (123456789, 7), (2**64 - 1, 3)):
        assert P.mix_seed(base, salt) == O.mix_seed(base, salt)


@pytest.mark.parametrize("threads", [2, 5])
def test_parallel_matrix_generator_matches_oracle(O, threads):
    """Large A (config 4 path): one thread draws the raw words in stream order,
    the Box-Muller transform and the column-major scatter run on `threads`
    workers; the result is the sequential stream bit for bit (ragged last chunk)."""
    from paper_2405_00366_b200 import cimcs as P
    args = (3001, 0.7, 0.1, 0.01, 11)  # M = 2101 rows: 32 chunks of 64 + a ragged one
    inst = P.gen_instances(args[0], [args[1:]], threads=threads)[0]
    ref = O.gen_instance(*args)
    assert np.array_equal(inst.A, ref.A) and np.array_equal(inst.y, ref.y)
    assert np.array_equal(inst.x_true, ref.x_true) and np.array_equal(inst.xi_true, ref.xi_true)


def test_generator_random_parameters_three_way(O):
    """80 random (N, alpha, a, nu, seed) including the edges (N = 1, alpha = 1 / N or 1,
    a = 0 or 1, nu = 0): the product's host generator, the oracle and the reference's own
    datagen.cpp agree bit for bit on A, y, x, xi and M, and reject the same inputs."""
    from paper_2405_00366_b200 import cimcs as P
    L = _ref()
    rng = np.random.default_rng(0)
    compared = 0
    for _ in range(80):
        N = int(rng.choice([1, 2, 3, 7, 12, 33, 100, 257]))
        alpha = float(rng.choice([rng.uniform(0.01, 1.0), 1.0, 1.0 / N, 0.5]))
        a = float(rng.choice([rng.uniform(0.0, 1.0), 0.0, 1.0, 1.0 / N]))
        nu = float(rng.choice([0.0, 0.01, 1.0]))
        seed = int(rng.integers(0, 2 ** 63))
        try:
            pi = P.gen_instance(N, alpha, a, nu, seed)
        except Exception:  # noqa: BLE001
            pi = None
        try:
            oi = O.gen_instance(N, alpha, a, nu, seed)
        except Exception:  # noqa: BLE001
            oi = None
        assert (pi is None) == (oi is None), (N, alpha, a, nu, seed)
        if pi is None:
            continue
        A = np.zeros((oi.M, N), order="F")
        y, x = np.zeros(oi.M), np.zeros(N)
        xi = np.zeros(N, np.int32)
        M = C.c_int()
        assert L.ref_gen_instance(N, alpha, a, nu, seed, A.ctypes.data, y.ctypes.data,
                                  x.ctypes.data, xi.ctypes.data, C.byref(M)) == 0
        assert M.value == pi.M == oi.M
        for inst in (pi, oi):
            assert np.array_equal(inst.A, A) and np.array_equal(inst.y, y)
            assert np.array_equal(inst.x_true, x) and np.array_equal(inst.xi_true, xi)
        compared += 1
    assert compared >= 60
