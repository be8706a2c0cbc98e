"""Downstream consumers of the batch results (host-side, cheap).

* Ridge linear regression over the covar matrix (§3 "Ridge linear regression",
  P:364-402; the optimiser of §6: batch gradient descent with Armijo
  backtracking line search and Barzilai-Borwein step sizes).  The covar matrix
  C[j][k] = Σ_{x ∈ D} X_j X_k (with X_0 ≡ 1 for the intercept) is the result of the covariance
  batch; every gradient step is C-sized work, the data is never touched again.
* Mutual information and the Chow-Liu tree: MI(X_i, X_j) from the count queries
  Q_∅, Q_{i}, Q_{j}, Q_{i,j} of the Chow-Liu batch with the 4-ary function
  f(α, β, γ, δ) = δ/α · log(αδ / (βγ)) summed over the groups (a, b) of Q_{i,j}; the tree is a
  maximum-weight spanning tree over the MI weights (reading R19 in DESIGN.md).
* A CART regression tree grown with node batches over the prepared relations (NEXT-1).

These run on the host over results that `lmfao_fetch` returned; they import nothing from
the oracle.
"""
from __future__ import annotations

import math

import numpy as np


# ------------------------------------------------------------------ covar matrix
def covar_matrix(features, values):
    """The (n+1)x(n+1) covar matrix [1, x_1..x_n] from the values of a covariance batch laid out
    as synth.covar_batch: COUNT, SUM(x_i), SUM(x_i x_j) for i <= j."""
    n = len(features)
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size != (n + 1) * (n + 2) // 2:
        raise ValueError(f"{v.size} values for {n} features")
    C = np.empty((n + 1, n + 1))
    C[0, 0] = v[0]
    C[0, 1:] = C[1:, 0] = v[1:n + 1]
    k = n + 1
    for i in range(n):
        for j in range(i, n):
            C[i + 1, j + 1] = C[j + 1, i + 1] = v[k]
            k += 1
    return C


# ------------------------------------------------------------------ ridge regression by BGD
def ridge_objective(C, label, theta, lam):
    """J(θ) = 1/(2|D|) Σ_x (Σ_j θ_j X_j − X_label)^2 + λ/2 ||θ||^2, from C alone:
    with θ' = θ and θ'_label = −1, Σ_x (θ'·X)^2 = θ'ᵀ C θ'.  θ ranges over the columns other
    than `label` (the intercept column 0 included)."""
    tp = _extend(theta, label, C.shape[0])
    return 0.5 * tp @ C @ tp / C[0, 0] + 0.5 * lam * theta @ theta


def ridge_gradient(C, label, theta, lam):
    """∇_k J = (1/|D|) Σ_j θ'_j C[j][k] + λ θ_k for k ≠ label."""
    tp = _extend(theta, label, C.shape[0])
    g = C @ tp / C[0, 0]
    return np.delete(g, label) + lam * theta


def _extend(theta, label, m):
    tp = np.empty(m)
    tp[:label] = theta[:label]
    tp[label] = -1.0
    tp[label + 1:] = theta[label:]
    return tp


def ridge_bgd(C, label, lam=1e-3, tol=1e-10, max_iter=100_000, armijo_c=1e-4, shrink=0.5):
    """Batch gradient descent with Armijo backtracking and Barzilai-Borwein step sizes over the
    covar matrix.  Returns (θ, iterations, converged)."""
    m = C.shape[0]
    theta = np.zeros(m - 1)
    g = ridge_gradient(C, label, theta, lam)
    J = ridge_objective(C, label, theta, lam)
    s = 1.0
    prev = None
    stall = 0
    for it in range(1, max_iter + 1):
        gg = g @ g
        if math.sqrt(gg) <= tol * max(1.0, abs(J)) or stall >= 50:
            # converged, or at the floating-point floor: 50 steps without a decrease of J
            # beyond its rounding (BB steps then only wander inside the noise of ∇J)
            return theta, it - 1, True
        if prev is not None:  # Barzilai-Borwein: s = Δθ·Δθ / Δθ·Δg
            dt, dg = theta - prev[0], g - prev[1]
            den = dt @ dg
            s = (dt @ dt) / den if den > 0 else 1.0
        while True:  # Armijo: sufficient decrease along −g
            cand = theta - s * g
            Jc = ridge_objective(C, label, cand, lam)
            if Jc <= J - armijo_c * s * gg or s < 1e-300:
                break
            s *= shrink
        prev = (theta, g)
        stall = stall + 1 if J - Jc <= 1e-15 * max(1.0, abs(J)) else 0
        theta, J = cand, Jc
        g = ridge_gradient(C, label, theta, lam)
    return theta, max_iter, False


def ridge_closed_form(C, label, lam):
    """The minimiser of J: (C_ff/|D| + λI) θ = C_{f,label}/|D| (normal equations)."""
    keep = [j for j in range(C.shape[0]) if j != label]
    A = C[np.ix_(keep, keep)] / C[0, 0] + lam * np.eye(len(keep))
    b = C[keep, label] / C[0, 0]
    return np.linalg.solve(A, b)


# ------------------------------------------------------------------ MI and Chow-Liu
def mutual_information(total, marg_i, marg_j, pair):
    """MI(X_i, X_j) = Σ_{(a,b)} f(α, β_a, γ_b, δ_ab), f = δ/α · log(αδ/(βγ)).
    total = α = |D|; marg_i / marg_j: value -> count (Q_{i}, Q_{j}); pair: (a, b) -> count."""
    a = float(total)
    mi = 0.0
    for (u, v), d in pair.items():
        if d > 0:
            mi += d / a * math.log(a * d / (marg_i[u] * marg_j[v]))
    return mi


def mi_matrix(attrs, results):
    """MI for every pair from the results of synth.mi_batch(attrs): the pair queries in
    itertools.combinations order, then the single-attribute queries, then COUNT; each result
    is (keys, values, counts) as lmfao_fetch returns it."""
    n = len(attrs)
    npair = n * (n - 1) // 2
    marg = []
    for q in range(npair, npair + n):
        keys, _, counts = results[q]
        marg.append({int(k[0]): int(c) for k, c in zip(keys, counts)})
    total = int(results[npair + n][2][0])
    M = np.zeros((n, n))
    q = 0
    for i in range(n):
        for j in range(i + 1, n):
            keys, _, counts = results[q]
            pair = {(int(k[0]), int(k[1])): int(c) for k, c in zip(keys, counts)}
            M[i, j] = M[j, i] = mutual_information(total, marg[i], marg[j], pair)
            q += 1
    return M


def chow_liu_tree(M):
    """Maximum-weight spanning tree over the MI matrix (Kruskal: heaviest edges first, skipping
    those that close a cycle); returns the n-1 edges (i, j), i < j, in the order they were added."""
    n = M.shape[0]
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    edges = sorted(((M[i, j], i, j) for i in range(n) for j in range(i + 1, n)), key=lambda e: (-e[0], e[1], e[2]))
    tree = []
    for w, i, j in edges:
        ri, rj = find(i), find(j)
        if ri != rj:
            parent[ri] = rj
            tree.append((i, j))
            if len(tree) == n - 1:
                break
    return tree


# ------------------------------------------------------------------ CART regression tree
F_LE, F_GT, F_GE, F_IDENT, F_IN = 3, 4, 5, 1, 8  # lmfao_fkind


def _mask(values):
    return float(sum(1 << int(v) for v in values))


def regression_tree(engine, features, target, thresholds, max_depth=4, min_split=1000, categoricals=(),
                    dynamic=True):
    """A CART regression tree (§3 "Decision trees" P:480-555; §6: depth 4, min split
    1000, 20 buckets) grown over the prepared relations of `engine`.

    Every node computes one batch: with α the node's path condition, RT(α, y·α, y²·α) for the
    node and for every candidate condition A ≤ t (the rt.cu path takes α as a row filter), and
    Q(X; α·y^p) for every categorical X.  dynamic=True ("dynamic
    functions"): the batch is planned once, with a placeholder condition y ≥ -inf, and each
    node only rebinds α (lmfao_set_condition) before its run; dynamic=False re-plans the batch
    per node (lmfao_reset_batch + add_query + plan).  The split with the largest variance
    reduction SSE(node) − SSE(left) − SSE(right), SSE = Σy² − (Σy)²/n, is taken; the right
    side's sums are the node's minus the left's.  A categorical X splits by set inclusion (P:484,
    LMFAO_F_IN; values in [0, 52]): its categories in increasing order of mean y (then value),
    cut after each prefix.  A node with fewer than `min_split` rows, at `max_depth`, or without a
    split that reduces SSE is a leaf.  Returns nested dicts."""
    y = [(F_IDENT, target, 0.0)]
    placeholder = [(F_GE, target, float("-inf"))]

    def batch(path):
        udafs = [[(1.0, path + y * p)] for p in range(3)]
        for a in features:
            for t in thresholds:
                cond = path + [(F_LE, a, float(t))]
                udafs += [[(1.0, cond + y * p)] for p in range(3)]
        q = engine.add_query([], udafs)
        qc = [engine.add_query([x], [[(1.0, path + y * p)] for p in range(3)]) for x in categoricals]
        return q, qc

    if dynamic:
        engine.reset_batch()
        q_dyn, qc_dyn = batch(placeholder)
        engine.plan()

    def node(path, depth):
        if dynamic:
            engine.set_condition(path if path else placeholder)
            q, qc = q_dyn, qc_dyn
        else:
            engine.reset_batch()
            q, qc = batch(path)
            engine.plan()
        engine.run()
        v = engine.fetch(q)[1][0]
        n, s, s2 = v[0], v[1], v[2]
        out = {"n": int(round(n)), "mean": s / n if n > 0 else 0.0, "path": [tuple(c) for c in path]}
        if depth == max_depth or n < min_split:
            return out
        sse = s2 - s * s / n
        best = None

        def consider(nl, sl, s2l, split):
            nonlocal best
            nr, sr, s2r = n - nl, s - sl, s2 - s2l
            if nl < 0.5 or nr < 0.5:
                return
            gain = sse - (s2l - sl * sl / nl) - (s2r - sr * sr / nr)
            if best is None or gain > best[0]:
                best = (gain, split)

        k = 3
        for a in features:
            for t in thresholds:
                consider(v[k], v[k + 1], v[k + 2], ("num", a, float(t)))
                k += 3
        for x, qx in zip(categoricals, qc):
            keys, vals, _ = engine.fetch(qx)
            cats = [(vals[i, 1] / vals[i, 0], int(keys[i, 0]), vals[i]) for i in range(len(keys)) if vals[i, 0] > 0]
            if not cats or any(c < 0 or c > 52 for _, c, _ in cats):
                continue
            cats.sort(key=lambda e: (e[0], e[1]))
            acc = np.zeros(3)
            for i in range(len(cats) - 1):
                acc = acc + cats[i][2]
                left = [c for _, c, _ in cats[:i + 1]]
                right = [c for _, c, _ in cats[i + 1:]]
                consider(acc[0], acc[1], acc[2], ("cat", x, _mask(left), _mask(right)))
        if best is None or best[0] <= 0.0:
            return out
        split = best[1]
        if split[0] == "num":
            _, a, t = split
            out.update(feature=a, threshold=t,
                       left=node(path + [(F_LE, a, t)], depth + 1), right=node(path + [(F_GT, a, t)], depth + 1))
        else:
            _, x, ml, mr = split
            out.update(feature=x, categories=ml,
                       left=node(path + [(F_IN, x, ml)], depth + 1), right=node(path + [(F_IN, x, mr)], depth + 1))
        return out

    return node([], 0)


# ------------------------------------------------------------------ root assignment
def assign_roots(schemas, sizes, batch):
    """LMFAO's root choice per query (§4): every query gives each relation the
    fraction of its group-by attributes that the relation holds (a query without group-by
    attributes gives every relation 1/m); relations are then taken in decreasing total weight
    (ties: the larger relation) and each becomes the root of every still-unassigned query
    that gave it a positive weight.  schemas: relation -> set of attribute names; sizes:
    relation -> row count; batch: queries with .groupby.  Returns one relation per query."""
    names = list(schemas)
    m = len(names)
    w = []
    for q in batch:
        gb = list(q.groupby)
        if gb:
            w.append({r: sum(a in schemas[r] for a in gb) / len(gb) for r in names})
        else:
            w.append({r: 1.0 / m for r in names})
    total = {r: sum(x[r] for x in w) for r in names}
    order = sorted(names, key=lambda r: (-total[r], -sizes[r], names.index(r)))
    root = [None] * len(batch)
    for r in order:
        for i in range(len(batch)):
            if root[i] is None and w[i][r] > 0:
                root[i] = r
    return root


def reroot(edges, root):
    """The edges (parent, child) of the same undirected join tree re-oriented away from root."""
    adj = {}
    for p, c in edges:
        adj.setdefault(p, []).append(c)
        adj.setdefault(c, []).append(p)
    out, seen, stack = [], {root}, [root]
    while stack:
        u = stack.pop()
        for v in adj.get(u, []):
            if v not in seen:
                seen.add(v)
                out.append((u, v))
                stack.append(v)
    return out
