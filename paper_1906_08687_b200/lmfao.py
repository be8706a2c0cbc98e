"""Thin ctypes binding of liblmfao_gpu (include/lmfao_gpu.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no CPU fallback — if the shared library is missing the
import fails loudly.  Function names follow the C ABI (lmfao_create,
lmfao_add_relation, ...); `Engine` is a convenience wrapper over them.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LMFAO_LIB") or os.path.join(_HERE, "liblmfao_gpu.so")  # LMFAO_LIB: A/B builds

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1906_08687_b200.build` "
                      "(or __graft_entry__.build()); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

# status codes (lmfao_status)
STATUS = {0: "LMFAO_OK", 1: "LMFAO_ERR_INVALID_ARG", 2: "LMFAO_ERR_STATE", 3: "LMFAO_ERR_UNKNOWN_ATTR",
          4: "LMFAO_ERR_TYPE", 5: "LMFAO_ERR_CYCLIC_TREE", 6: "LMFAO_ERR_DISCONNECTED_TREE",
          7: "LMFAO_ERR_RUNNING_INTERSECTION", 8: "LMFAO_ERR_UNSUPPORTED", 9: "LMFAO_ERR_OOM",
          10: "LMFAO_ERR_CUDA", 11: "LMFAO_ERR_NCCL"}
INT32, FP64 = 0, 1
F_CONST, F_IDENT, F_LT, F_LE, F_GT, F_GE, F_EQ, F_NE, F_IN = range(9)
UNIQUE_ID_BYTES = 128
COLS_HOST, COLS_DEVICE, COLS_HOST_DEFERRED = 0, 1, 2


class lmfao_factor(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("attr", ctypes.c_int32), ("param", ctypes.c_double)]


class lmfao_product(ctypes.Structure):
    _fields_ = [("coeff", ctypes.c_double), ("n_factors", ctypes.c_int32),
                ("factors", ctypes.POINTER(lmfao_factor))]


class lmfao_udaf(ctypes.Structure):
    _fields_ = [("n_products", ctypes.c_int32), ("products", ctypes.POINTER(lmfao_product))]


_P = ctypes.c_void_p
_i32p = ctypes.POINTER(ctypes.c_int32)
_SIGS = {
    "lmfao_unique_id": [_P],
    "lmfao_create": [ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(_P)],
    "lmfao_destroy": [_P],
    "lmfao_add_relation": [_P, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.c_char_p),
                           _i32p, ctypes.POINTER(_P), ctypes.c_int, _i32p],
    "lmfao_attr_id": [_P, ctypes.c_char_p, _i32p],
    "lmfao_set_join_tree": [_P, ctypes.c_int32, ctypes.c_int32, _i32p, _i32p],
    "lmfao_set_root_shard": [_P, ctypes.c_int32, ctypes.c_int32],
    "lmfao_prepare": [_P],
    "lmfao_add_query": [_P, ctypes.c_int32, _i32p, ctypes.c_int32, ctypes.POINTER(lmfao_udaf), _i32p],
    "lmfao_plan": [_P],
    "lmfao_reset_batch": [_P],
    "lmfao_run": [_P, _P],
    "lmfao_result_shape": [_P, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), _i32p, _i32p],
    "lmfao_fetch": [_P, ctypes.c_int32, _P, _P, _P],
    "lmfao_result_device": [_P, ctypes.c_int32, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_P)],
    "lmfao_plan_info": [_P, ctypes.c_char_p, ctypes.c_int64],
    "lmfao_profile": [_P, ctypes.c_int],
    "lmfao_profile_read": [_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)],
    "lmfao_create_loopback": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(_P)],
    "lmfao_gather_result": [_P, ctypes.c_int32, ctypes.c_int32],
    "lmfao_set_condition": [_P, ctypes.c_int32, ctypes.POINTER(lmfao_factor)],
    "lmfao_shard_range": [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.c_int64)],
    "lmfao_owner_range": [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.c_int64)],
}
for _name, _args in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = ctypes.c_int
_lib.lmfao_last_error.argtypes = [_P]
_lib.lmfao_last_error.restype = ctypes.c_char_p

EXPORTED = list(_SIGS) + ["lmfao_last_error"]


class LmfaoError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


def lmfao_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(UNIQUE_ID_BYTES)
    s = _lib.lmfao_unique_id(buf)
    if s:
        raise LmfaoError(s, "lmfao_unique_id failed")
    return buf.raw


def _struct_dtype(cls):
    """numpy dtype with the same field offsets as a ctypes Structure (pointers as uint64)."""
    names, formats, offsets = [], [], []
    for name, ct in cls._fields_:
        names.append(name)
        formats.append({ctypes.c_int32: np.int32, ctypes.c_double: np.float64}.get(ct, np.uint64))
        offsets.append(getattr(cls, name).offset)
    return np.dtype({"names": names, "formats": formats, "offsets": offsets, "itemsize": ctypes.sizeof(cls)})


_FACTOR_DT, _PRODUCT_DT, _UDAF_DT = (_struct_dtype(c) for c in (lmfao_factor, lmfao_product, lmfao_udaf))


def _udaf_structs(udafs, attr_id):
    """udafs: list of products; product = (coeff, [(kind, attr_name|None, param), ...]) or an
    object with .coeff/.factors whose factors have .kind/.attr/.param.  Returns the lmfao_udaf
    array (three flat numpy buffers laid out as the C structs) and the buffers to keep alive."""
    ids = {}
    fk, fa, fp, pc, pn, ps, un, us = [], [], [], [], [], [], [], []
    for u in udafs:
        us.append(len(pc))
        un.append(len(u))
        for p in u:
            coeff, factors = (p.coeff, p.factors) if hasattr(p, "coeff") else p
            ps.append(len(fk))
            pn.append(len(factors))
            pc.append(float(coeff))
            for f in factors:
                kind, attr, param = (f.kind, f.attr, f.param) if hasattr(f, "kind") else f
                fk.append(int(kind))
                if attr is None:
                    fa.append(-1)
                else:
                    a = ids.get(attr)
                    if a is None:
                        a = ids[attr] = attr_id(attr)
                    fa.append(a)
                fp.append(float(param))
    F = np.zeros(max(1, len(fk)), _FACTOR_DT)
    F["kind"][:len(fk)], F["attr"][:len(fk)], F["param"][:len(fk)] = fk, fa, fp
    P = np.zeros(max(1, len(pc)), _PRODUCT_DT)
    P["coeff"][:len(pc)], P["n_factors"][:len(pc)] = pc, pn
    P["factors"][:len(pc)] = F.ctypes.data + np.asarray(ps, np.uint64) * np.uint64(F.itemsize)
    U = np.zeros(max(1, len(un)), _UDAF_DT)
    U["n_products"][:len(un)] = un
    U["products"][:len(un)] = P.ctypes.data + np.asarray(us, np.uint64) * np.uint64(P.itemsize)
    return ctypes.cast(U.ctypes.data, ctypes.POINTER(lmfao_udaf)), (F, P, U)


def shard_range(nrows: int, part: int, nparts: int):
    """lmfao_shard_range (host only): the rows [lo, hi) of the sorted root kept by `part`."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    s = _lib.lmfao_shard_range(nrows, part, nparts, ctypes.byref(lo), ctypes.byref(hi))
    if s:
        raise LmfaoError(s, "lmfao_shard_range")
    return lo.value, hi.value


def owner_range(ncells: int, rank: int, world: int):
    """lmfao_owner_range (host only): the cells [lo, hi) of a distributed output owned by `rank`."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    s = _lib.lmfao_owner_range(ncells, rank, world, ctypes.byref(lo), ctypes.byref(hi))
    if s:
        raise LmfaoError(s, "lmfao_owner_range")
    return lo.value, hi.value


class Engine:
    """One lmfao_ctx (one process, one GPU).  loopback=group name: a rank of an in-process
    group of contexts on one device (lmfao_create_loopback; tests of the multi-GPU path)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, unique_id: bytes | None = None,
                 loopback: str | None = None):
        h = _P()
        if loopback is not None:
            s = _lib.lmfao_create_loopback(device, rank, world, loopback.encode(), ctypes.byref(h))
        else:
            uid = ctypes.create_string_buffer(unique_id, UNIQUE_ID_BYTES) if unique_id is not None else None
            s = _lib.lmfao_create(device, rank, world, uid, ctypes.byref(h))
        if s:
            raise LmfaoError(s, "lmfao_create failed (no CUDA device?)")
        self.h = h
        self.rel_ids = {}
        self.query_ids = []
        self._deferred = []  # host buffers of LMFAO_COLS_HOST_DEFERRED relations, until plan

    def _check(self, s):
        if s:
            raise LmfaoError(s, _lib.lmfao_last_error(self.h).decode())

    def close(self):
        if self.h:
            _lib.lmfao_destroy(self.h)
            self.h = None
        self._deferred = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add_relation(self, name: str, cols: dict, deferred: bool | None = None) -> int:
        """cols: name -> numpy array or torch tensor (all host or all on this device).
        deferred (default: True for pinned host tensors): LMFAO_COLS_HOST_DEFERRED — the
        copies happen inside prepare(), overlapped with it; the Engine keeps the buffers
        alive until then."""
        names = list(cols)
        arrs, dtypes, ptrs, on_dev = [], [], [], None
        for c in names:
            v = cols[c]
            if hasattr(v, "data_ptr"):  # torch tensor
                dev = v.is_cuda
                if on_dev is None:
                    on_dev = dev
                elif on_dev != dev:
                    raise ValueError("all columns must be on the same side (host or device)")
                v = v.contiguous()
                dtypes.append(INT32 if str(v.dtype) == "torch.int32" else FP64)
                ptrs.append(v.data_ptr())
                arrs.append(v)
            else:
                a = np.ascontiguousarray(v)
                if a.dtype == np.int32:
                    dtypes.append(INT32)
                elif a.dtype == np.float64:
                    dtypes.append(FP64)
                else:
                    raise TypeError(f"column {c}: dtype {a.dtype} (int32 or float64 expected)")
                on_dev = on_dev or False
                arrs.append(a)
                ptrs.append(a.ctypes.data)
        n = len(arrs[0]) if arrs else 0
        if deferred is None:
            deferred = not on_dev and all(hasattr(a, "is_pinned") and a.is_pinned() for a in arrs)
        mode = COLS_DEVICE if on_dev else (COLS_HOST_DEFERRED if deferred else COLS_HOST)
        cn = (ctypes.c_char_p * len(names))(*[x.encode() for x in names])
        dt = (ctypes.c_int32 * len(names))(*dtypes)
        cp = (_P * len(names))(*ptrs)
        rid = ctypes.c_int32()
        self._check(_lib.lmfao_add_relation(self.h, name.encode(), n, len(names), cn, dt, cp, mode,
                                            ctypes.byref(rid)))
        if mode == COLS_HOST_DEFERRED:
            self._deferred.append(arrs)
        self.rel_ids[name] = rid.value
        return rid.value

    def attr_id(self, name: str) -> int:
        a = ctypes.c_int32()
        self._check(_lib.lmfao_attr_id(self.h, name.encode(), ctypes.byref(a)))
        return a.value

    def set_join_tree(self, root: str, edges):
        p = (ctypes.c_int32 * max(1, len(edges)))(*[self.rel_ids[e[0]] for e in edges])
        c = (ctypes.c_int32 * max(1, len(edges)))(*[self.rel_ids[e[1]] for e in edges])
        self._check(_lib.lmfao_set_join_tree(self.h, self.rel_ids[root], len(edges), p, c))

    def set_root_shard(self, part: int, nparts: int):
        self._check(_lib.lmfao_set_root_shard(self.h, part, nparts))

    def prepare(self):
        self._check(_lib.lmfao_prepare(self.h))

    def add_query(self, groupby, udafs) -> int:
        gb = (ctypes.c_int32 * max(1, len(groupby)))(*[self.attr_id(g) for g in groupby])
        arr, keep = _udaf_structs(udafs, self.attr_id)
        q = ctypes.c_int32()
        self._check(_lib.lmfao_add_query(self.h, len(groupby), gb, len(udafs), arr, ctypes.byref(q)))
        del keep
        self.query_ids.append(q.value)
        return q.value

    def plan(self):
        try:
            self._check(_lib.lmfao_plan(self.h))
        finally:
            self._deferred = []  # plan has waited for the deferred host columns (else close() drops them)

    def reset_batch(self):
        """Drop the batch and plan, keep the prepared relations (lmfao_reset_batch)."""
        self._check(_lib.lmfao_reset_batch(self.h))
        self.query_ids = []

    def run(self, stream: int | None = None):
        self._check(_lib.lmfao_run(self.h, _P(stream) if stream else None))

    def result_shape(self, q: int):
        ng, ngb, nu = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        self._check(_lib.lmfao_result_shape(self.h, q, ctypes.byref(ng), ctypes.byref(ngb), ctypes.byref(nu)))
        return ng.value, ngb.value, nu.value

    def fetch(self, q: int):
        ng, ngb, nu = self.result_shape(q)
        keys = np.zeros((ng, ngb), dtype=np.int32)
        vals = np.zeros((ng, nu), dtype=np.float64)
        counts = np.zeros(ng, dtype=np.uint64)
        self._check(_lib.lmfao_fetch(self.h, q, keys.ctypes.data if keys.size else None,
                                     vals.ctypes.data if vals.size else None, counts.ctypes.data if ng else None))
        return keys, vals, counts

    def set_condition(self, factors):
        """Dynamic path condition (lmfao_set_condition): factors = [(kind, attr name, param)] or
        synth.Factor objects, all predicates; replaces the planned batch's condition."""
        fs = []
        for f in factors:
            kind, attr, param = (f.kind, f.attr, f.param) if hasattr(f, "kind") else f
            fs.append(lmfao_factor(int(kind), self.attr_id(attr), float(param)))
        arr = (lmfao_factor * max(1, len(fs)))(*fs)
        self._check(_lib.lmfao_set_condition(self.h, len(fs), arr))

    def gather_result(self, q: int, root: int = 0):
        """Collective: assemble a distributed result on rank `root` (lmfao_gather_result)."""
        self._check(_lib.lmfao_gather_result(self.h, q, root))

    def result_device(self, q: int):
        k, v, c = _P(), _P(), _P()
        self._check(_lib.lmfao_result_device(self.h, q, ctypes.byref(k), ctypes.byref(v), ctypes.byref(c)))
        return k.value, v.value, c.value

    def profile(self, enable: bool = True):
        self._check(_lib.lmfao_profile(self.h, int(enable)))

    def profile_read(self):
        t, n = ctypes.c_double(), ctypes.c_int64()
        self._check(_lib.lmfao_profile_read(self.h, ctypes.byref(t), ctypes.byref(n)))
        return t.value, n.value

    def plan_info(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        self._check(_lib.lmfao_plan_info(self.h, buf, 1 << 16))
        return json.loads(buf.value.decode())


def load(engine: Engine, db, batch, columns=None):
    """Registers a database (relations with .name/.cols, .root, .edges) and a
    batch (queries with .groupby/.udafs) on `engine`, through prepare; returns
    the query ids.  `columns` optionally maps relation name -> dict of columns
    (e.g. torch tensors already on the device) replacing rel.cols."""
    for r in db.relations:
        engine.add_relation(r.name, columns[r.name] if columns else r.cols)
    engine.set_join_tree(db.root, list(db.edges))
    engine.prepare()
    return [engine.add_query(list(q.groupby), list(q.udafs)) for q in batch]
