"""Multi-rank host logic on CPU with gloo, world_size 2: shard planning,
sharding invariance of the counter-based RNG (via the oracle's identical
draws), count all-reduce and rank-ordered gather."""

import os
import socket

import numpy as np
import pytest

from paper_2103_02202_b200.parallel import shard


def test_shard_partitions_tiles():
    for total, world, T in [(1000, 3, 64), (1 << 20, 8, 512), (33, 4, 32), (5, 2, 32)]:
        ranges = [shard(total, world, r, T) for r in range(world)]
        covered = []
        for off, cnt in ranges:
            assert off % T == 0
            covered += list(range(off, off + cnt))
        assert covered == list(range(total))
    assert shard(100, 4, 3, 32, weak=True) == (3 * 128, 100)
    with pytest.raises(ValueError):
        shard(10, 2, 2, 32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, text, total, T, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2103_02202_b200.parallel import all_reduce_counts, gather_shards
        from paper_2103_02202_b200.program import flatten

        prog = flatten(text)
        off, cnt = shard(total, world, rank, T)
        _, ev = O.sample(prog, cnt, T, seed=77, tile_offset=off // T, flips=False)
        b8 = O.rows_to_b8(ev, cnt)
        counts = np.unpackbits(b8, axis=1, bitorder="little")[:, :prog.num_columns].sum(0)
        tot = all_reduce_counts(counts.astype(np.uint64))
        full = gather_shards(b8)
        if rank == 0:
            q.put((tot, full))
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_gloo_two_ranks_match_single_run(oracle_lib):
    import torch.multiprocessing as mp

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.program import flatten

    text = gen.surface_code_memory(5, 5, 5e-3)
    total, T = 4 * 256 + 100, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, text, total, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    tot, full = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    prog = flatten(text)
    _, ev = oracle_lib.sample(prog, total, T, seed=77, flips=False)
    ref = oracle_lib.rows_to_b8(ev, total)
    assert np.array_equal(full, ref)  # sharding invariance + gather order
    assert np.array_equal(tot, np.unpackbits(ref, axis=1, bitorder="little")
                          [:, :prog.num_columns].sum(0).astype(np.uint64))
