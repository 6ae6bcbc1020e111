"""Counter-based instances generated on the GPU (a documented
deviation: Philox4x32-10 streams instead of the reference's sequential
mt19937_64 stream).  The instances are not the reference's; the tests pin the
recipe (shapes, exact support size, A ~ N(0, 1/M), y = A(xi.x) + nu N(0,1) in
gen_instance's summation order), determinism, and that the solver on a
generated instance equals the oracle on the same (downloaded) numbers."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gen(P, N, params, dtype="f64"):
    ctx = P.Context(0, dtype)
    ctx.set_generated_problems(N, params)
    return ctx


def test_recipe_shapes_and_statistics(gpu):
    N, al, a = 2000, 0.5, 0.1
    with _gen(gpu, N, [(al, a, 0.0, 7)]) as ctx:
        inst = ctx.get_instance(0)
    M, K = gpu.gen_dims(N, al, a)
    assert inst.A.shape == (M, N) and int(inst.xi_true.sum()) == K
    A = inst.A
    n = A.size
    assert abs(A.mean()) < 5.0 / math.sqrt(M) / math.sqrt(n)
    assert abs(A.var() * M - 1.0) < 0.01
    assert abs(inst.x_true.mean()) < 5.0 / math.sqrt(N) and abs(inst.x_true.var() - 1.0) < 0.1
    # nu = 0: y = A (xi . x), summed over the support in ascending order
    y = np.zeros(M)
    for r in np.flatnonzero(inst.xi_true):
        y = y + A[:, r] * inst.x_true[r]
    assert np.array_equal(inst.y, y)


def test_noise_and_determinism(gpu):
    N = 1000
    with _gen(gpu, N, [(0.6, 0.2, 0.05, 3), (0.4, 0.1, 0.0, 4)]) as c1, \
            _gen(gpu, N, [(0.6, 0.2, 0.05, 3), (0.4, 0.1, 0.0, 4)]) as c2:
        for b in range(2):
            i1, i2 = c1.get_instance(b), c2.get_instance(b)
            for f in ("A", "y", "x_true", "xi_true"):
                assert np.array_equal(getattr(i1, f), getattr(i2, f))
        i0 = c1.get_instance(0)
    res = i0.y - i0.A @ (i0.xi_true * i0.x_true)
    assert abs(res.std() / 0.05 - 1.0) < 0.1
    with _gen(gpu, N, [(0.6, 0.2, 0.05, 5)]) as c3:
        assert not np.array_equal(c3.get_instance(0).A, i0.A)


def test_solve_on_generated_instance_matches_oracle(gpu, O):
    """fp64 solve on the resident generated instance == the oracle on the same
    numbers (canonical order, bitwise)."""
    with _gen(gpu, 300, [(0.6, 0.2, 0.01, 11)]) as ctx:
        inst = ctx.get_instance(0)
        ctx.build_coupling()
        seed = O.mix_seed(11, 1)
        res = ctx.solve(1, "mfz-bn", gpu.baseline_params(velo=3, n_steps=300), [seed])
    oi = O.Instance(inst.A, inst.y, inst.x_true, inst.xi_true)
    ref = O.Problem(oi, O.CANON).alternating_minimize(O.MFZ_BN, O.baseline_params(velo=3, n_steps=300),
                                                      O.Rng(seed))
    assert np.array_equal(res["R"][0, 0], ref["R"])
    assert np.array_equal(res["sigma"][0, 0], ref["sigma"])
