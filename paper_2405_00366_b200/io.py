"""Instance bundles and the CSV result contract (the data formats either side
of the hot path), over the C ABI (csrc/io.hpp).

Mirrors the reference's io module (include/cimcs/io.hpp): ``format_double``,
``fnv1a64``/``hex64``, ``save_instance``/``load_instance`` (io.cpp:86-167),
``CsvWriter`` (io.cpp:169-196), and the run tables of ``cimcs run``:
summary.csv (tools/main.cpp:449-462), history_<backend>.csv
(orchestrator.cpp:253-264) and failures.csv (main.cpp:476-489).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from typing import Iterable, Sequence

import numpy as np

from ._lib import load
from .cimcs import Instance, InputError, _check

RNG_ALGORITHM = "mt19937_64-boxmuller-v1"  # rng.hpp:12
SUMMARY_COLUMNS = ("backend", "a", "alpha", "nu", "seed", "final_rmse", "final_hamming",
                   "min_hamiltonian")                                  # main.cpp:450-451
FAILURE_COLUMNS = ("backend", "a", "alpha", "nu", "seed", "alternation", "reason")  # :477


def history_csv_columns() -> list[str]:
    """orchestrator.cpp:253-255."""
    return ["trial", "i", "eta", "hamiltonian", "rmse", "hamming", "seconds"]


def format_double(v: float) -> str:
    """io.cpp:18-25: the shortest %.15g/%.16g/%.17g text that round-trips."""
    buf = C.create_string_buffer(40)
    _check(load().cimcs_format_double(float(v), buf, 40))
    return buf.value.decode()


def fnv1a64(data: bytes | str) -> int:
    """io.cpp:27-34."""
    b = data.encode() if isinstance(data, str) else bytes(data)
    return int(load().cimcs_fnv1a64(b, len(b)))


def hex64(v: int) -> str:
    """io.cpp:36-40."""
    return "%016x" % (v & 0xFFFFFFFFFFFFFFFF)


def cell(v) -> str:
    """CsvWriter::cell (io.hpp:41-43): doubles round-trip, integers in decimal."""
    if isinstance(v, (bool, np.bool_)):
        return str(int(v))
    if isinstance(v, (int, np.integer)):
        return str(int(v))
    if isinstance(v, (float, np.floating)):
        return format_double(float(v))
    return str(v)


def save_instance(inst: Instance, dir: str) -> None:
    """save_instance, io.cpp:86-125 (A.csv row-major, y.csv, truth.csv, meta.json)."""
    A = np.asfortranarray(inst.A, dtype=np.float64)
    y = np.ascontiguousarray(inst.y, dtype=np.float64)
    M, N = A.shape
    if y.shape != (M,):
        raise InputError("save_instance: y must have M entries")
    xp = xip = None
    if inst.has_truth():
        x = np.ascontiguousarray(inst.x_true, dtype=np.float64)
        xi = np.ascontiguousarray(inst.xi_true, dtype=np.int32)
        if x.shape != (N,) or xi.shape != (N,):
            raise InputError("save_instance: truth must have N entries")
        xp, xip = x.ctypes.data, xi.ctypes.data
    _check(load().cimcs_save_instance(os.fsencode(dir), N, M, A.ctypes.data, y.ctypes.data,
                                      xp, xip, float(inst.a), float(inst.alpha), float(inst.nu),
                                      int(inst.seed)))


def load_instance(dir: str) -> Instance:
    """load_instance, io.cpp:127-167 (row/column count checks are input errors)."""
    L = load()
    N, M, ht = C.c_int32(), C.c_int32(), C.c_int32()
    a, al, nu, sd = C.c_double(), C.c_double(), C.c_double(), C.c_uint64()
    d = os.fsencode(dir)
    _check(L.cimcs_load_instance(d, C.byref(N), C.byref(M), C.byref(ht), C.byref(a),
                                 C.byref(al), C.byref(nu), C.byref(sd), None, None, None, None))
    A = np.zeros((M.value, N.value), order="F")
    y = np.zeros(M.value)
    x = np.zeros(N.value) if ht.value else None
    xi = np.zeros(N.value, np.int32) if ht.value else None
    _check(L.cimcs_load_instance(d, C.byref(N), C.byref(M), C.byref(ht), None, None, None, None,
                                 A.ctypes.data, y.ctypes.data,
                                 None if x is None else x.ctypes.data,
                                 None if xi is None else xi.ctypes.data))
    return Instance(A, y, x, xi, a.value, al.value, nu.value, int(sd.value))


def load_bundles(root: str) -> list[Instance]:
    """cmd_run --load (tools/main.cpp:390-400): every sub-directory holding a
    meta.json, sorted by seed."""
    out = [load_instance(os.path.join(root, e)) for e in sorted(os.listdir(root))
           if os.path.isfile(os.path.join(root, e, "meta.json"))]
    if not out:
        from .cimcs import ConfigError
        raise ConfigError(f"no instance bundles found under {root}")
    return sorted(out, key=lambda i: i.seed)


def _strs(xs: Sequence[str]):
    enc = [x.encode() for x in xs]
    arr = (C.c_char_p * max(1, len(enc)))(*enc)
    return arr, enc


class CsvWriter:
    """CsvWriter, io.hpp:31-48: comments ("# " prefixed), header, rows; the file
    is written by close() (the reference writes in its destructor)."""

    def __init__(self, path: str, comments: Sequence[str], columns: Sequence[str]):
        self._h = C.c_void_p()
        ca, self._keep_c = _strs(list(comments))
        cb, self._keep_h = _strs(list(columns))
        _check(load().cimcs_csv_open(os.fsencode(path), ca, len(comments), cb, len(columns),
                                     C.byref(self._h)))

    def row(self, cells: Sequence) -> None:
        arr, keep = _strs([c if isinstance(c, str) else cell(c) for c in cells])
        _check(load().cimcs_csv_row(self._h, arr, len(keep)))

    def close(self) -> None:
        if self._h:
            h, self._h = self._h, C.c_void_p()
            _check(load().cimcs_csv_close(h))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def csv_comments(config_hash: str, seeds: Iterable[int]) -> list[str]:
    """tools/main.cpp:251-259: config hash, rng name, instance seed list."""
    return ["config " + config_hash, "rng " + RNG_ALGORITHM,
            "seeds " + " ".join(str(int(s)) for s in seeds)]


def append_history_rows(w: CsvWriter, trial: int, history: Sequence[dict]) -> None:
    """orchestrator.cpp:257-264."""
    for h in history:
        w.row([int(trial), int(h["i"]), float(h["eta"]), float(h["hamiltonian"]),
               float(h["rmse"]), float(h["hamming"]), float(h.get("seconds", math.nan))])


def write_run_tables(out_dir: str, instances: Sequence[Instance], trials: Sequence[dict],
                     backend: str, config_hash: str = "0" * 16) -> int:
    """The tables of cmd_run (tools/main.cpp:445-490) for one backend: trials[k]
    is the trial dict (cimcs.solve / Context.trial) of instances[k].  Returns the
    number of failed trials."""
    os.makedirs(out_dir, exist_ok=True)
    comments = csv_comments(config_hash, [i.seed for i in instances])
    failures = 0
    with CsvWriter(os.path.join(out_dir, "summary.csv"), comments, SUMMARY_COLUMNS) as w:
        for inst, t in zip(instances, trials):
            bad = bool(t["failed"])
            failures += bad
            w.row([backend, float(inst.a), float(inst.alpha), float(inst.nu), int(inst.seed),
                   math.nan if bad else float(t["final_rmse"]),
                   math.nan if bad else float(t["final_hamming"]),
                   math.nan if bad else float(t["min_hamiltonian"])])
    with CsvWriter(os.path.join(out_dir, f"history_{backend}.csv"), comments,
                   history_csv_columns()) as w:
        for k, t in enumerate(trials):
            append_history_rows(w, k, t["history"])
    if failures:
        with CsvWriter(os.path.join(out_dir, "failures.csv"), comments, FAILURE_COLUMNS) as w:
            for inst, t in zip(instances, trials):
                if t["failed"]:
                    w.row([backend, float(inst.a), float(inst.alpha), float(inst.nu),
                           int(inst.seed), int(t["fail_alternation"]),
                           str(t["fail_reason"]).replace(",", ";")])
    return failures
