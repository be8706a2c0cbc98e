"""Test helpers: a tiny UDAF mini-language for fixtures, and the parity comparator.

Mini-language (fixtures only): terms separated by '+', factors by '*';
a number is a constant factor (SUM(1) is "1"), a name is the identity
function, "[x<=2]" is the Kronecker delta 1_{x<=2}.
"""
import re

import numpy as np

import synth

_OPS = {"<=": synth.F_LE, ">=": synth.F_GE, "!=": synth.F_NE, "<": synth.F_LT, ">": synth.F_GT, "==": synth.F_EQ}


def parse_factor(tok):
    tok = tok.strip()
    if tok.startswith("["):
        m = re.match(r"\[\s*(\w+)\s*(<=|>=|!=|==|<|>)\s*([-+0-9.eE]+)\s*\]", tok)
        return synth.Factor(_OPS[m.group(2)], m.group(1), float(m.group(3)))
    try:
        return synth.Factor(synth.F_CONST, None, float(tok))
    except ValueError:
        return synth.Factor(synth.F_IDENT, tok)


def parse_udaf(s):
    prods = []
    for term in s.split("+"):
        fs = [parse_factor(t) for t in term.split("*")]
        prods.append(synth.Product(1.0, tuple(fs)))
    return prods


def query(groupby, udafs):
    return synth.Query(list(groupby), [parse_udaf(u) for u in udafs])


def float_close(g, o, absmass, rel=1e-9, fallback_frac=1e-3, fallback_abs=1e-12):
    """Acceptance criterion (reading R14): |g-o| <= rel*|o|, or, when
    |o| < fallback_frac*A (A = oracle's Σ|term|), |g-o| <= fallback_abs*A."""
    g = np.asarray(g, dtype=np.float64)
    o = np.asarray(o, dtype=np.float64)
    A = np.asarray(absmass, dtype=np.float64)
    err = np.abs(g - o)
    ok = err <= rel * np.abs(o)
    fb = np.abs(o) < fallback_frac * A
    ok |= fb & (err <= fallback_abs * A)
    ok |= (A == 0) & (g == 0)
    return ok
