"""Regenerate the committed golden fixtures (run in the build container).

* ref_rng.npz / ref_instances.npz: outputs of the REFERENCE's own rng.hpp and
  datagen.cpp, compiled unmodified from /root/reference by oracle/Makefile.ref
  (oracle/_ref/libref.so).  They pin the oracle's and the product's
  generators on machines without /root/reference.
* oracle_config0.npz: the C oracle's fp64 solve of BASELINE config 0
  (gen_instance(500, 0.6, 0.2, 0.01, 0), MFZ-BN, dt 0.01, linear pump 0->1.2,
  20 alternations x 1000 steps, seed mix_seed(0, 1)) in the canonical order
  (bitwise target of the GPU fp64 path) and in the reference-literal
  matrix-free order (A^T(A w)).
"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402

SEEDS = [0, 1, 7, 5489, 2**63 + 12345]
INSTANCES = [(40, 0.5, 0.2, 0.1, 3), (12, 8 / 12, 0.25, 0.0, 11), (500, 0.6, 0.2, 0.01, 0),
             (64, 0.3, 0.05, 0.01, 9)]


def ref_lib():
    so = os.path.join(ROOT, "oracle", "_ref", "libref.so")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "-f", "Makefile.ref"])
    L = C.CDLL(so)
    L.ref_gen_instance.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                   C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    L.ref_gauss.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
    L.ref_raw.argtypes = [C.c_uint64, C.c_int, C.c_void_p]
    return L


def main():
    L = ref_lib()
    rng = {}
    for s in SEEDS:
        raw = np.zeros(1000, np.uint64)
        g = np.zeros(1000)
        L.ref_raw(s, 1000, raw.ctypes.data)
        L.ref_gauss(s, 1000, g.ctypes.data)
        rng[f"raw_{s}"] = raw
        rng[f"gauss_{s}"] = g
    np.savez_compressed(os.path.join(HERE, "ref_rng.npz"), seeds=np.array(SEEDS, np.uint64), **rng)
    inst = {}
    for k, (N, al, a, nu, s) in enumerate(INSTANCES):
        M = O.round_half_away(al * N)  # datagen.cpp:22
        A = np.zeros((M, N), order="F")
        y, x = np.zeros(M), np.zeros(N)
        xi = np.zeros(N, np.int32)
        Mo = C.c_int()
        assert L.ref_gen_instance(N, al, a, nu, s, A.ctypes.data, y.ctypes.data, x.ctypes.data,
                                  xi.ctypes.data, C.byref(Mo)) == 0
        inst[f"args_{k}"] = np.array([N, al, a, nu, s], np.float64)
        inst[f"A_{k}"], inst[f"y_{k}"], inst[f"x_{k}"], inst[f"xi_{k}"] = A, y, x, xi
    np.savez_compressed(os.path.join(HERE, "ref_instances.npz"), n=len(INSTANCES), **inst)

    g0 = O.gen_instance(500, 0.6, 0.2, 0.01, 0)
    hp = O.baseline_params()
    seed = O.mix_seed(0, 1)
    out = {"seed": np.array([seed], np.uint64)}
    for name, mode in (("canon", O.CANON), ("literal", O.LITERAL)):
        res = O.Problem(g0, mode).alternating_minimize(O.MFZ_BN, hp, O.Rng(seed))
        out[f"{name}_R"] = res["R"]
        out[f"{name}_sigma"] = res["sigma"]
        for f in ("hamiltonian", "rmse", "hamming", "min_e", "median_e", "eta"):
            out[f"{name}_{f}"] = np.array([h[f] for h in res["history"]])
        out[f"{name}_support"] = np.array([h["support"] for h in res["history"]], np.int32)
    np.savez_compressed(os.path.join(HERE, "oracle_config0.npz"), **out)
    print("golden fixtures written")


if __name__ == "__main__":
    main()
