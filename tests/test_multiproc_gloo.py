"""World-size-2 tests of the multi-GPU host logic on CPU (gloo): unique-id
broadcast, max-over-ranks timing, and the partition + combine semantics of the
row-sharded root — each rank evaluates its contiguous shard (lmfao_prepare's
formula), partial aggregates are all-reduced over a rank-independent dense cell
layout, and the result equals the whole-root oracle."""
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


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1906_08687_b200.parallel import broadcast_bytes, max_over_ranks, shard_range
        uid = broadcast_bytes(dist, bytes(range(128)) if rank == 0 else None, 128, rank)
        assert uid == bytes(range(128))
        mx = max_over_ranks(dist, [float(rank + 1), 10.0 - rank])
        assert mx == [float(world), 10.0]
        w = synth.config4(fact_rows=9_001, dim_rows=(20, 60, 200))
        batch = [q for q in w.batch if len(q.groupby) <= 1][:6] + [w.batch[0]]
        N = w.db.rel("F").nrows
        lo, hi = shard_range(N, rank, world)
        part = oracle.evaluate(w.db, batch, root_range=(lo, hi))
        full = oracle.evaluate(w.db, batch) if rank == 0 else None
        for qi, (qq, r) in enumerate(zip(batch, part)):
            # rank-independent dense layout: the global value domain of each group attribute
            doms = [int(max(rel.cols[a].max() for rel in w.db.relations if a in rel.cols)) + 1 for a in qq.groupby]
            ncell = int(np.prod(doms)) if doms else 1
            vals = torch.zeros(ncell, dtype=torch.float64)
            cnts = torch.zeros(ncell, dtype=torch.int64)
            for k, v, c in zip(r.keys, r.vals[:, 0], r.counts):
                cell = 0
                for a, d in zip(k, doms):
                    cell = cell * d + int(a)
                vals[cell] += v
                cnts[cell] += int(c)
            dist.all_reduce(vals)
            dist.all_reduce(cnts)
            if rank == 0:
                f = full[qi]
                present = torch.nonzero(cnts).flatten().numpy()
                assert len(present) == len(f.keys)
                for (k, v, c) in zip(f.keys, f.vals[:, 0], f.counts):
                    cell = 0
                    for a, d in zip(k, doms):
                        cell = cell * d + int(a)
                    assert int(cnts[cell]) == int(c)
                    assert abs(float(vals[cell]) - v) <= 1e-9 * max(1.0, abs(v))
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
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
