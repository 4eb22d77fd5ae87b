"""Multi-rank host logic on CPU (gloo, world size 2) -- -m "not gpu".

The N-GPU path shards the unit list with Algorithm 1 (PAPER.md:235-251,
the library's lnorm_partition) and combines ranks with ONE max all-reduce of
the 8-byte key (value biased to unsigned order in the high word, ~unit in the
low word: the library's lnorm_reduction_key, the kernels' make_key).  Here each
rank evaluates its slice's per-prefix maxima with the CPU oracle (the GPU is not
needed for the decomposition logic), packs them with the LIBRARY's key (checked
against the documented layout), and the gloo all-reduce must yield the global
maximum and the SMALLEST unit attaining it -- the unit that holds the
lexicographically smallest optimum.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def pack_key(v, unit):
    return ((((v & 0xFFFFFFFF) ^ 0x80000000) << 32) | (0xFFFFFFFF - unit))


def unpack_key(k):
    hi = (k >> 32) ^ 0x80000000
    v = hi - (1 << 32) if hi >= (1 << 31) else hi
    return v, 0xFFFFFFFF - (k & 0xFFFFFFFF)


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import paper_2503_21596_b200 as L
    from paper_2503_21596_b200 import synth
    n, m, k, marg, seed = case
    M = synth.random_matrix(n, m, seed, -3, 3)
    units = 1 << k
    lo, hi = L.partition(units, world, rank)
    best = None
    for u in range(lo, hi + 1):
        prefix = [0] + [(u >> (k - x)) & 1 for x in range(1, k + 1)]
        v, _ = oracle.prefix_max(M, prefix, d=1, with_marginals=marg)
        key = L.reduction_key(v, u)          # the library's own key (csrc/common.cuh make_key)
        assert key == pack_key(v, u)         # ... equal to the documented layout
        best = key if best is None or key > best else best
    # order-preserving u64 -> i64 map (flip the top bit) so gloo's int64 MAX reduces the key
    t = torch.tensor([best - (1 << 63)], dtype=torch.int64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    key = t.item() + (1 << 63)
    assert L.key_decode(key) == unpack_key(key)
    if rank == 0:
        q.put((unpack_key(key), (lo, hi)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [(9, 7, 4, False, 1), (10, 6, 5, True, 2), (8, 8, 3, False, 3)])
def test_two_rank_partition_and_key_reduction(case):
    import oracle
    from paper_2503_21596_b200 import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    (v, unit), _ = q.get(timeout=10)
    n, m, k, marg, seed = case
    M = synth.random_matrix(n, m, seed, -3, 3)
    ov, oarg = (oracle.marg(M) if marg else oracle.l1(M))
    assert v == ov
    # the winning unit is the prefix (rows 1..k) of the lexicographically smallest optimum
    digits = [0 if a == 1 else 1 for a in oarg]
    assert unit == int("".join(map(str, digits[1:k + 1])), 2)


def test_partition_covers_units_for_every_world_size():
    import paper_2503_21596_b200 as L
    for units in (1, 7, 1 << 10, (1 << 24) + 3):
        for world in (1, 2, 3, 4, 8):
            rngs = [L.partition(units, world, r) for r in range(world)]
            assert rngs[0][0] == 0 and rngs[-1][1] == units - 1
            for (a, b), (c, d) in zip(rngs, rngs[1:]):
                assert c == b + 1
            sizes = [b - a + 1 for a, b in rngs]
            assert max(sizes) - min(sizes) <= 1


def test_library_reduction_key_order():
    """lnorm_reduction_key (the kernels' make_key, host side): unsigned key order = (value, then the
    SMALLER unit) for negative and positive values; lnorm_key_decode inverts it."""
    import paper_2503_21596_b200 as L
    vals = [-(2 ** 31), -5, -1, 0, 1, 17, 2 ** 31 - 1]
    units = [0, 1, 7, 2 ** 32 - 1]
    keys = {(v, u): L.reduction_key(v, u) for v in vals for u in units}
    for (v, u), k in keys.items():
        assert L.key_decode(k) == (v, u)
        assert k == pack_key(v, u)
    order = sorted(keys, key=lambda vu: keys[vu])
    assert order == sorted(keys, key=lambda vu: (vu[0], -vu[1]))
