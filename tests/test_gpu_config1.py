"""Parity at the benchmark scale: BASELINE config 1 in full (64 instances x 16
replicas, N=2000, M=1000, 20 alternations x 1000 Euler steps, linear pump,
Jacobi refit) -- the workload bench.py credits.

* fp64: the GPU solve (DMMA symmetric path) is bitwise the oracle in the GPU's
  canonical order; checked on 4 trajectories re-solved on the host cores (the
  whole batch is ~20 CPU-hours).  The oracle's canonical and LITERAL orders agree
  on the supports of all 64 instances (profiles/r02_literal_study.json), and
  LITERAL is bitwise the reference's own code (tests/test_ref_solver.py).
* fp32 (declared tolerance, fixed before the round-2
  measurements): against the fp64 run on the same seeds, over all 1024
  trajectories -- mean final RMSE, mean Hamming loss and the mean best-replica RMSE
  each within 1 % relative; the paired mean RMSE difference within 4 standard
  errors; where the supports agree, RMSE within 1e-5 relative; no trajectory
  fails that the fp64 run does not.  Support identity is NOT an fp32 criterion:
  per-step fp32 state rounding alone moves 25 % of the fp64 supports
  (profiles/r02_precision_study.json).
"""
import concurrent.futures as cf
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def config1(gpu):
    from paper_2405_00366_b200 import workloads as W
    insts, R, hp, _ = W.config1(0, 64)
    seeds = gpu.replica_seeds(insts, R, "mfz-bn")
    return insts, R, hp, seeds


def _solve(gpu, config1, dtype):
    insts, R, hp, seeds = config1
    with gpu.Context(0, dtype) as ctx:
        ctx.set_problems(insts)
        ctx.build_coupling()
        res = ctx.solve(R, "mfz-bn", hp, seeds)
        res["order"] = ctx.canon_order()
    return res


@pytest.fixture(scope="module")
def f64(gpu, config1):
    return _solve(gpu, config1, "f64")


def test_fp64_config1_bitwise_subset(gpu, O, config1, f64):
    insts, R, _, seeds = config1
    hp = O.baseline_params()
    picks = [(0, 0), (17, 5), (42, 11), (63, 15)]

    def one(br):
        b, r = br
        inst = insts[b]
        p = O.Problem(O.Instance(inst.A, inst.y, inst.x_true, inst.xi_true), O.CANON,
                      *f64["order"])
        return p.alternating_minimize(O.MFZ_BN, hp, O.Rng(int(seeds[b, r])))

    with cf.ThreadPoolExecutor(len(picks)) as ex:
        refs = list(ex.map(one, picks))
    assert (f64["fail_alt"] < 0).all()
    for (b, r), ref in zip(picks, refs):
        assert np.array_equal(f64["R"][b, r], ref["R"]), (b, r)
        assert np.array_equal(f64["sigma"][b, r], ref["sigma"]), (b, r)


def test_fp32_config1_declared_tolerance(gpu, config1, f64):
    import bench
    res = _solve(gpu, config1, "f32")
    par = bench.parity_vs_f64(f64, res, "f32")
    assert par["pass"], par
