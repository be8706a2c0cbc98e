"""oracle — TEST INFRASTRUCTURE ONLY (never on the product path).

A plain CPU evaluation of an LMFAO aggregate batch by materialising the natural
join tuple by tuple (oracle.cpp; PAPER.md P:336-347 problem statement, P:716-724
join tree).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` leg may import this package.  It shares no code with
paper_1906_08687_b200/ (the CUDA path); this file has its own marshalling of the
synth objects into the oracle's text spec.

Every function of oracle.cpp is pinned by tests/test_oracle_pins.py (hand DBs
with literal values, brute force via an independent pandas materialisation,
closed forms, the paper's worked examples); see DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.cpp with g++ (no FP contraction, so products round exactly
    as written; OpenMP for the THREADS fact-row chunks)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fopenmp", "-std=c++17", "-shared", "-fPIC",
                               "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_eval.restype = ctypes.c_void_p
        lib.oracle_eval.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_char_p, ctypes.c_int]
        lib.oracle_nqueries.argtypes = [ctypes.c_void_p]
        lib.oracle_shape.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        lib.oracle_fetch.argtypes = [ctypes.c_void_p, ctypes.c_int] + [ctypes.c_void_p] * 4
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


@dataclass
class OracleResult:
    keys: np.ndarray      # [n_groups, n_groupby] int64, ascending lexicographic
    vals: np.ndarray      # [n_groups, n_udafs] float64 (long-double sums rounded once)
    counts: np.ndarray    # [n_groups] uint64 join multiplicity of the group
    absmass: np.ndarray   # [n_groups, n_udafs] Σ|term| (tolerance fallback, R14)


def host_cores() -> int:
    """Threads the oracle may use on this host (its CPU affinity)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _spec(db, batch, root_range=None, threads=1, acc="longdouble"):
    lines, ptrs, keep = [], [], []
    for r in db.relations:
        lines.append(f"REL {r.name} {r.nrows} {len(r.cols)}")
        for c, v in r.cols.items():
            if v.dtype == np.int32:
                a = np.ascontiguousarray(v, dtype=np.int32)
                lines.append(f"COL {c} I")
            else:
                a = np.ascontiguousarray(v, dtype=np.float64)
                lines.append(f"COL {c} D")
            keep.append(a)
            ptrs.append(a.ctypes.data if a.size else 0)
    lines.append(f"ROOT {db.root}")
    if root_range is not None:
        lines.append(f"RANGE {int(root_range[0])} {int(root_range[1])}")
    lines.append(f"THREADS {int(threads)}")
    lines.append("ACC " + {"longdouble": "LONGDOUBLE", "neumaier": "NEUMAIER"}[acc])
    for p, c in db.edges:
        lines.append(f"EDGE {p} {c}")
    for q in batch:
        head = f"QUERY {len(q.groupby)} " + " ".join(q.groupby) + f" {len(q.udafs)}"
        lines.append(head)
        for u in q.udafs:
            lines.append(f"UDAF {len(u)}")
            for p in u:
                parts = [f"PROD {float(p.coeff).hex()} {len(p.factors)}"]
                for f in p.factors:
                    parts.append(f"{int(f.kind)} {f.attr if f.attr is not None else '-'} {float(f.param).hex()}")
                lines.append(" ".join(parts))
    return "\n".join(lines) + "\n", ptrs, keep


def evaluate(db, batch, root_range=None, threads=1, acc="longdouble") -> list:
    """Evaluate every query of `batch` over the natural join of `db`.
    root_range=(lo, hi) restricts the root relation to rows [lo, hi).
    threads: contiguous root-row chunks enumerated in parallel with private group
    tables merged in chunk order (0 = every host core).  acc: "longdouble" (default)
    or "neumaier" (compensated double)."""
    lib = _load()
    if threads == 0:
        threads = host_cores()
    spec, ptrs, keep = _spec(db, batch, root_range, threads, acc)
    arr = (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)
    err = ctypes.create_string_buffer(512)
    h = lib.oracle_eval(spec.encode(), arr, err, 512)
    if not h:
        raise ValueError("oracle: " + err.value.decode())
    try:
        out = []
        for q in range(lib.oracle_nqueries(h)):
            ng, ngb, nu = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int()
            lib.oracle_shape(h, q, ctypes.byref(ng), ctypes.byref(ngb), ctypes.byref(nu))
            keys = np.zeros((ng.value, ngb.value), dtype=np.int64)
            vals = np.zeros((ng.value, nu.value), dtype=np.float64)
            counts = np.zeros(ng.value, dtype=np.uint64)
            absm = np.zeros((ng.value, nu.value), dtype=np.float64)
            lib.oracle_fetch(h, q, keys.ctypes.data, vals.ctypes.data, counts.ctypes.data, absm.ctypes.data)
            out.append(OracleResult(keys, vals, counts, absm))
        return out
    finally:
        lib.oracle_free(h)
        del keep
