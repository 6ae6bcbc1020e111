"""Bundles -> GPU batch -> CSV tables, end to end (paper_2405_00366_b200.run):
the bundle loader feeds the B200 solver bit-exact inputs, and the summary /
history rows carry the oracle's results (fp64: sigma/R bitwise, scalars within
1e-12 relative; tables round-trip the doubles exactly)."""
import csv
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_bundles_to_tables_match_oracle(gpu, O, tmp_path):
    from paper_2405_00366_b200 import io as IO
    from paper_2405_00366_b200 import run as RUN
    src = tmp_path / "bundles"
    for s in (11, 4):
        IO.save_instance(gpu.gen_instance(120, 0.5, 0.15, 0.01, s), str(src / f"inst{s}"))
    hp = gpu.baseline_params(velo=3, n_steps=200)
    out = tmp_path / "out"
    assert RUN.run(str(src), str(out), "mfz-bn", 1, "f64", hp) == 0
    rows = [r for r in csv.reader(open(out / "summary.csv")) if r and not r[0].startswith("#")]
    assert rows[0] == list(IO.SUMMARY_COLUMNS)
    assert [int(r[4]) for r in rows[1:]] == [4, 11]  # bundles sorted by seed
    ohp = O.baseline_params(velo=3, n_steps=200)
    hist = [r for r in csv.reader(open(out / "history_mfz-bn.csv")) if r and r[0] != "trial"
            and not r[0].startswith("#")]
    for k, s in enumerate((4, 11)):
        inst = O.gen_instance(120, 0.5, 0.15, 0.01, s)
        p = O.Problem(O.Instance(inst.A, inst.y, inst.x_true, inst.xi_true), O.CANON)
        ref = p.alternating_minimize(O.MFZ_BN, ohp, O.Rng(int(O.mix_seed(s, 1))))
        assert not ref["failed"]
        last = ref["history"][-1]
        r = rows[1 + k]
        assert math.isclose(float(r[5]), last["rmse"], rel_tol=1e-12)
        assert float(r[6]) == last["hamming"]
        assert math.isclose(float(r[7]), min(h["hamiltonian"] for h in ref["history"]),
                            rel_tol=1e-12)
        mine = [h for h in hist if int(h[0]) == k]
        assert len(mine) == len(ref["history"]) == 4
        for h, g in zip(mine, ref["history"]):
            assert int(h[1]) == g["i"] and float(h[2]) == g["eta"]
