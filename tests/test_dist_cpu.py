"""Multi-process host logic of the sharded path on CPU (gloo, world_size 2): the row partition
covers [0, n) with contiguous blocks in rank order, and the handle exchange returns every rank's
blob in rank order on every rank (what svm_shard_connect requires)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1706_05544_b200.dist import shard_bounds


def test_shard_bounds_cover_rows():
    for n in (2, 7, 50000, 2000001):
        for world in (1, 2, 3, 8):
            blocks = [shard_bounds(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (a, b), (c, _) in zip(blocks, blocks[1:]):
                assert b == c and a <= b
            assert max(b - a for a, b in blocks) - min(b - a for a, b in blocks) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_1706_05544_b200.dist import all_gather_bytes, shard_bounds
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank]) * 1024                       # SVM_SHARD_HANDLE_BYTES
    got = all_gather_bytes(blob)
    r0, r1 = shard_bounds(1001, world, rank)
    q.put((rank, [g[:4] for g in got], len(b"".join(got)), (r0, r1)))
    dist.barrier()
    dist.destroy_process_group()


def test_handle_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, heads, total, (r0, r1) in res:
        assert heads == [bytes([0]) * 4, bytes([1]) * 4]
        assert total == 2 * 1024
    assert res[0][3] == (0, 500) and res[1][3] == (500, 1001)


def test_kfold_split_sizes_and_stratification():
    """SPEC kfold_split: union = all rows, sizes differ by at most one, stratified per class."""
    import numpy as np
    from paper_1706_05544_b200 import binding
    f = binding.kfold_split(10, 5, seed=1)
    assert sorted(np.bincount(f).tolist()) == [2, 2, 2, 2, 2]
    f = binding.kfold_split(7, 3, seed=2)
    assert sorted(np.bincount(f).tolist()) == [2, 2, 3]
    lab = np.array([0] * 6 + [1] * 4)
    f = binding.kfold_split(10, 2, seed=3, labels=lab)
    for k in range(2):
        assert (lab[f == k] == 0).sum() == 3 and (lab[f == k] == 1).sum() == 2
