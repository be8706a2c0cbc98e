"""World-size-2 tests of the multi-GPU host logic on CPU (gloo), through the library's own
partition functions (lmfao_shard_range / lmfao_owner_range: host-only C ABI calls, no GPU):
each rank evaluates its contiguous shard of the root (the oracle stands in for the per-rank
GPU scan, which needs a device), then the ranks combine partial aggregates the three ways
lmfao_run does —
  * all-reduce of a small output (complete on every rank),
  * reduce-scatter of a dense table by owner cell range,
  * exchange of sparse groups to the owner of their cell, merged there,
— and lmfao_gather_result's rule (the ranks' groups concatenated in rank order) rebuilds the
whole-root oracle's table in canonical order on rank 0.  Also the unique-id broadcast and
max-over-ranks timing helpers."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cell_layout(db, q):
    doms = []
    for a in q.groupby:
        rel = next(r for r in db.relations if a in r.cols)
        doms.append(np.unique(rel.cols[a]))
    return doms


def _cells(keys, doms):
    cell = np.zeros(len(keys), dtype=np.int64)
    for i, d in enumerate(doms):
        cell = cell * len(d) + np.searchsorted(d, keys[:, i])
    return cell


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1906_08687_b200 import lmfao
        from paper_1906_08687_b200.parallel import broadcast_bytes, max_over_ranks
        uid = broadcast_bytes(dist, bytes(range(128)) if rank == 0 else None, 128, rank)
        assert uid == bytes(range(128))
        assert max_over_ranks(dist, [float(rank + 1), 10.0 - rank]) == [float(world), 10.0]
        w = synth.config5(fact_rows=9_001, dim_rows=(20, 60, 200, 400), cube_doms=(5, 11, 17))
        batch = w.batch[:-1] + [synth.Query([], w.batch[-1].udafs[:30])]
        N = w.db.rel("F").nrows
        lo, hi = lmfao.shard_range(N, rank, world)
        part = oracle.evaluate(w.db, batch, root_range=(lo, hi))
        full = oracle.evaluate(w.db, batch) if rank == 0 else None
        for qi, (qq, r) in enumerate(zip(batch, part)):
            doms = _cell_layout(w.db, qq)
            ncell = int(np.prod([len(d) for d in doms])) if doms else 1
            nu = r.vals.shape[1]
            cells = _cells(r.keys, doms)
            replicated = qi % 3 == 0 or not qq.groupby
            if replicated:  # (1) all-reduce: complete on every rank
                vals = torch.zeros((ncell, nu), dtype=torch.float64)
                cnts = torch.zeros(ncell, dtype=torch.int64)
                vals[cells] = torch.from_numpy(r.vals)
                cnts[cells] = torch.from_numpy(r.counts.astype(np.int64))
                dist.all_reduce(vals)
                dist.all_reduce(cnts)
                pres = torch.nonzero(cnts).flatten().numpy()
                mine = (pres, vals[pres].numpy(), cnts[pres].numpy())
                olo, ohi = 0, ncell
            elif qi % 3 == 1:  # (2) reduce-scatter by owner range (dense, padded to world chunks)
                chunk = (ncell + world - 1) // world
                vals = torch.zeros((chunk * world, nu), dtype=torch.float64)
                cnts = torch.zeros(chunk * world, dtype=torch.int64)
                vals[cells] = torch.from_numpy(r.vals)
                cnts[cells] = torch.from_numpy(r.counts.astype(np.int64))
                ov = torch.zeros((chunk, nu), dtype=torch.float64)
                oc = torch.zeros(chunk, dtype=torch.int64)
                dist.reduce_scatter(ov, list(vals.split(chunk)))
                dist.reduce_scatter(oc, list(cnts.split(chunk)))
                olo, ohi = lmfao.owner_range(ncell, rank, world)
                assert olo == min(ncell, chunk * rank)
                n = ohi - olo
                pres = torch.nonzero(oc[:n]).flatten().numpy()
                mine = (olo + pres, ov[pres].numpy(), oc[pres].numpy())
            else:  # (3) sparse exchange: every local group to the owner of its cell, merged there
                owner = np.array([next(p for p in range(world)
                                       if lmfao.owner_range(ncell, p, world)[0] <= c < lmfao.owner_range(ncell, p, world)[1])
                                  for c in cells], dtype=np.int64)
                sends = [[(int(c), r.vals[i].tolist(), int(r.counts[i])) for i, c in enumerate(cells) if owner[i] == p]
                         for p in range(world)]
                recv = [None] * world
                dist.all_gather_object(recv, sends)
                got = {}
                for src in range(world):  # merge in source-rank order
                    for c, v, n in recv[src][rank]:
                        a = got.setdefault(c, [np.zeros(nu), 0])
                        a[0] += np.array(v)
                        a[1] += n
                olo, ohi = lmfao.owner_range(ncell, rank, world)
                ks = np.array(sorted(got), dtype=np.int64)
                assert ((ks >= olo) & (ks < ohi)).all()
                mine = (ks, np.array([got[k][0] for k in ks]).reshape(len(ks), nu),
                        np.array([got[k][1] for k in ks], dtype=np.int64))
            # lmfao_gather_result: ranks' groups concatenated in rank order on rank 0
            allp = [None] * world
            dist.all_gather_object(allp, (mine[0].tolist(), mine[1].tolist(), mine[2].tolist()))
            if rank == 0:
                f = full[qi]
                if replicated:
                    allp = allp[:1]  # rank 0 alone is complete
                ck = np.concatenate([np.asarray(p[0], dtype=np.int64) for p in allp])
                cv = np.concatenate([np.asarray(p[1], dtype=np.float64).reshape(-1, nu) for p in allp])
                cc = np.concatenate([np.asarray(p[2], dtype=np.int64) for p in allp])
                assert np.array_equal(ck, _cells(f.keys, doms)), qi  # canonical order
                assert np.array_equal(cc, f.counts.astype(np.int64)), qi
                assert np.allclose(cv, f.vals, rtol=1e-9, atol=1e-9 * max(1.0, float(np.abs(f.vals).max()))), qi
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, repr(e) + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_and_combine_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


def test_partition_functions_host_only():
    """lmfao_shard_range / lmfao_owner_range (no device): shards tile the rows, owner ranges
    tile the cells, both ascend with the rank."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1906_08687_b200 import lmfao
    for n in (0, 1, 7, 100, 10_000_019):
        for g in (1, 2, 3, 8):
            s = [lmfao.shard_range(n, r, g) for r in range(g)]
            o = [lmfao.owner_range(n, r, g) for r in range(g)]
            for rng in (s, o):
                assert rng[0][0] == 0 and rng[-1][1] == n
                assert all(a[1] == b[0] and a[0] <= a[1] for a, b in zip(rng, rng[1:]))
            assert max(hi - lo for lo, hi in s) - min(hi - lo for lo, hi in s) <= 1
