"""World-size-2 gloo tests of the multi-GPU host logic (CPU only)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch.distributed as dist

    from oracle_lib import Oracle
    from paper_1607_02925_b200.replicas import column_shard, max_over_ranks, sum_partials
    from problems import planted_dense

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    o.nthreads = 1
    X, _, _ = planted_dense(40, 130, seed=7)
    W = np.random.default_rng(1).standard_normal((40, 5))
    j0, j1 = column_shard(130, rank, world)
    _, zpart, _ = o.gram_block(o.dense(X[:, j0:j1]), W)
    z = sum_partials(zpart)
    m = max_over_ranks([float(rank), 10.0 - rank])
    q.put((rank, z, m, (j0, j1)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_column_sharded_gram_pass_and_max_reduction(world, oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    from problems import planted_dense

    X, _, _ = planted_dense(40, 130, seed=7)
    W = np.random.default_rng(1).standard_normal((40, 5))
    _, zfull, _ = oracle.gram_block(oracle.dense(X), W)
    shards = sorted(r[3] for r in res)
    assert shards[0][0] == 0 and shards[-1][1] == 130 and shards[0][1] == shards[1][0]
    for rank, z, m, _ in res:
        assert np.allclose(z, zfull, rtol=1e-12, atol=1e-12)
        assert m == [1.0, 10.0]
    # deterministic ordered sum: every rank holds the identical bytes
    assert np.array_equal(res[0][1], res[1][1])


def test_column_shard_balanced():
    from paper_1607_02925_b200.replicas import column_shard

    for n, w in [(10, 3), (5, 8), (100000, 8)]:
        rngs = [column_shard(n, r, w) for r in range(w)]
        assert rngs[0][0] == 0 and rngs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
        assert max(b - a for a, b in rngs) - min(b - a for a, b in rngs) <= 1
