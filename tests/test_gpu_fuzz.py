"""Randomised shapes (tools/shape_fuzz.py): N from 33 to 3000 around the cluster, tile and
segment edges, batches of 1..33, replica counts that pad, MFZ-BN / MFZ-CN / Positive-P,
Jacobi and CG refits, track_best, world-1 sharded contexts and option toggles, 2-5
alternations -- fp64 bitwise against the oracle in the context's canonical order, fp32
finite on the same problems.  (Longer runs, 270 cases, and the two bugs they found are
recorded in profiles/r02_shape_fuzz.log.)"""
import importlib.util
import os

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [11])
def test_random_shapes(gpu, O, seed):
    spec = importlib.util.spec_from_file_location("shape_fuzz",
                                                  os.path.join(ROOT, "tools", "shape_fuzz.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.run(6, seed, quiet=True) == 0


def test_context_reuse_sequences(gpu, O):
    """tools/reuse_fuzz.py: one fp64 and one fp32 context driven through random sequences
    of set_problems / solve calls whose shapes, per-instance M, replica counts, schedules
    and backends change from call to call (cached graphs, schedules, state and pump
    buffers must follow): every fp64 solve bitwise equal to the oracle, fp32 finite."""
    spec = importlib.util.spec_from_file_location("reuse_fuzz",
                                                  os.path.join(ROOT, "tools", "reuse_fuzz.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.run(3, 5, quiet=True) == 0


def test_low_level_abi_random_shapes(gpu, O):
    """tools/abi_fuzz.py: cimcs_mfz_step, cimcs_run_cim, cimcs_cdp_minimize (Jacobi and CG)
    and cimcs_score on random shapes of an fp64 context, bitwise against the oracle (scorer
    scalars 1e-12 relative)."""
    spec = importlib.util.spec_from_file_location("abi_fuzz", os.path.join(ROOT, "tools", "abi_fuzz.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert mod.run(4, 9, quiet=True) == 0
