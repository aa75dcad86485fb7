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
        from tests._util import rule_chunk_lengths

        prog = flatten(text)
        off, cnt = shard(total, world, rank, T)
        _, ev = O.sample(prog, cnt, T, seed=77, tile_offset=off // T, flips=False,
                         chunk_L=rule_chunk_lengths(prog, T))
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
    from tests._util import rule_chunk_lengths

    prog = flatten(text)
    _, ev = oracle_lib.sample(prog, total, T, seed=77, flips=False, chunk_L=rule_chunk_lengths(prog, T))
    ref = oracle_lib.rows_to_b8(ev, total)
    assert np.array_equal(full, ref)  # sharding invariance + gather order
    assert np.array_equal(tot, np.unpackbits(ref, axis=1, bitorder="little")
                          [:, :prog.num_columns].sum(0).astype(np.uint64))


def _bench_worker(rank, world, port, text, shots, T, steps, q):
    """Runs bench.py's own config-3 helper (parallel.counts_steps) with the
    oracle standing in for the GPU sampler."""
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_2103_02202_b200.parallel import counts_steps, rank_offset, reduce_max
        from paper_2103_02202_b200.program import flatten
        from tests._util import rule_chunk_lengths

        prog = flatten(text)
        L = rule_chunk_lengths(prog, T)

        def sample_counts(n, seed, off, out):
            _, ev = O.sample(prog, n, T, seed=seed, tile_offset=off // T, flips=False, chunk_L=L)
            bits = np.unpackbits(O.rows_to_b8(ev, n), axis=1, bitorder="little")[:, :prog.num_columns]
            out.copy_(torch.from_numpy(bits.sum(0).astype(np.int64)))

        counts = torch.zeros(prog.num_columns, dtype=torch.int64)
        counts_steps(sample_counts, counts, shots, T, world, rank, steps, 7)
        el = reduce_max(0.5 + rank)  # bench.py's max-over-ranks timing reduction
        q.put((rank, counts.numpy().copy(), el, rank_offset(shots, world, rank, T)))
    finally:
        dist.destroy_process_group()


@pytest.mark.slow
def test_gloo_two_ranks_bench_counts_helper(oracle_lib):
    """bench.py's multi-rank config-3 path (weak-scaled offsets, per-step counts,
    one sum over ranks, max-over-ranks timing) on world_size 2 with gloo."""
    import torch.multiprocessing as mp

    from paper_2103_02202_b200 import generators as gen
    from paper_2103_02202_b200.program import flatten
    from tests._util import rule_chunk_lengths

    text = gen.surface_code_memory(5, 5, 5e-3)
    shots, T, steps = 3 * 256 + 40, 256, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, text, shots, T, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][2] == res[1][2] == 1.5
    offs = [r[3] for r in res]
    assert offs == [0, 4 * 256]
    prog = flatten(text)
    L = rule_chunk_lengths(prog, T)
    ref = np.zeros(prog.num_columns, dtype=np.int64)
    for off in offs:  # the last step (seed 7 + steps - 1) on each rank's own shots
        _, ev = oracle_lib.sample(prog, shots, T, seed=7 + steps - 1, tile_offset=off // T, flips=False, chunk_L=L)
        ref += np.unpackbits(oracle_lib.rows_to_b8(ev, shots), axis=1, bitorder="little")[:, :prog.num_columns].sum(0, dtype=np.int64)
    assert np.array_equal(res[0][1], ref) and np.array_equal(res[1][1], ref)
