"""CPU-side checks of the boundary: the C-ABI library loads and exports every
symbol include/lmfao_gpu.h declares (no compute calls without a GPU); the
product path has no CPU fallback."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    h = open(os.path.join(ROOT, "include", "lmfao_gpu.h")).read()
    return sorted(set(re.findall(r"LMFAO_API\s+[\w\s\*]+?\b(lmfao_\w+)\s*\(", h)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ["lmfao_create", "lmfao_add_relation", "lmfao_set_join_tree", "lmfao_prepare", "lmfao_add_query",
              "lmfao_plan", "lmfao_run", "lmfao_fetch", "lmfao_result_shape", "lmfao_result_device"]:
        assert n in names


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_1906_08687_b200 import lmfao
    lib = ctypes.CDLL(lmfao.LIB_PATH)
    for n in _declared():
        assert hasattr(lib, n), n
    assert sorted(lmfao.EXPORTED) == _declared()


def test_no_cpu_fallback_without_gpu():
    import torch

    from paper_1906_08687_b200 import lmfao
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lmfao.LmfaoError) as ei:
        lmfao.Engine()
    assert ei.value.name == "LMFAO_ERR_CUDA"


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1906_08687_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                src = open(os.path.join(dp, f), errors="ignore").read()
                assert "import oracle" not in src and "from oracle" not in src and "oracle.cpp" not in src, f


def test_udaf_marshalling_matches_c_layout():
    """The binding lays the UDAF batch out as the lmfao_udaf / lmfao_product / lmfao_factor
    structs of include/lmfao_gpu.h; read it back through the ctypes struct view."""
    import synth
    from paper_1906_08687_b200 import lmfao
    udafs = [[synth.Product(1.0, ())],
             [synth.Product(2.5, (synth.ident("a"), synth.Factor(synth.F_LE, "b", 0.25)))],
             [synth.Product(-1.0, (synth.ident("b"),)), synth.Product(3.0, (synth.Factor(lmfao.F_CONST, None, 4.0),))],
             [(0.5, [(lmfao.F_EQ, "a", 7.0)])]]
    ids = {"a": 3, "b": 9}
    arr, keep = lmfao._udaf_structs(udafs, ids.__getitem__)
    for j, u in enumerate(udafs):
        assert arr[j].n_products == len(u)
        for i, p in enumerate(u):
            coeff, factors = (p.coeff, p.factors) if hasattr(p, "coeff") else p
            pr = arr[j].products[i]
            assert pr.coeff == coeff and pr.n_factors == len(factors)
            for k, f in enumerate(factors):
                kind, attr, param = (f.kind, f.attr, f.param) if hasattr(f, "kind") else f
                got = pr.factors[k]
                assert (got.kind, got.attr, got.param) == (int(kind), -1 if attr is None else ids[attr], float(param))
