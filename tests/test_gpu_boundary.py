"""GPU: the C-ABI boundary's contracts (include/lnorm.h) -- stream ordering, device-side
guard statistics, the recovery self-check, and the batched path at any batch size."""
import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu


def test_compute_device_honours_caller_stream(lib):
    """M is produced on a side stream behind a ~30 ms spin; the search is enqueued on that
    stream (no host sync in between) and must read the produced matrix, not the zeros."""
    import torch
    M = synth.random_matrix(20, 22, 12_345)
    ov, oarg = oracle.l1(M)
    src = torch.from_numpy(M).cuda()
    Md = torch.zeros_like(src)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(60_000_000)
        Md.copy_(src)
    v, arg = lib.compute_device(Md, stream=side)
    assert v == ov and list(arg) == list(oarg)
    # the same through the rank entry point with the caller's stream
    torch.cuda.synchronize()
    Md.zero_()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(60_000_000)
        Md.copy_(src)
    v2, arg2 = lib.compute_rank_device(Md, None, 0, 1, stream=side)
    assert v2 == ov and list(arg2) == list(oarg)


@pytest.mark.parametrize("d,marg,W", [(1, False, 127), (1, False, 128), (2, False, 255), (2, False, 256),
                                      (3, False, 255), (3, False, 256)])
def test_device_guard_stats_match_host(lib, d, marg, W):
    """Guard statistics computed on the device (lnorm_compute_device) pick the same kernel and
    split as the host's (lnorm_compute) at the byte guard's boundary, with the oracle's result."""
    import torch
    g = synth.SplitMix64(70_000 + W + d)
    n, m = 9, 12
    M = np.array(synth.random_matrix(n, m, 70_100 + W, -6, 6), dtype=np.int64)
    rows = 7 if d <= 2 else n
    base, extra = divmod(W, rows)
    for i in range(rows):
        M[n - rows + i, 0] = (base + (1 if i < extra else 0)) * (1 if g.next() & 1 else -1)
    M = M.astype(np.int32)
    v, arg = lib.compute(M, d=d, with_marginals=marg)
    sh = lib.last_stats()
    vd, argd = lib.compute_device(torch.from_numpy(M).cuda(), d=d, with_marginals=marg)
    sd = lib.last_stats()
    assert (sd["variant"], sd["prefix_digits"], sd["suffix_digits"]) == (sh["variant"], sh["prefix_digits"], sh["suffix_digits"])
    ov, oarg = oracle.norm(M, d=d, with_marginals=marg)
    assert v == vd == ov and list(arg) == list(argd) == list(oarg)


def test_device_input_errors(lib):
    import torch
    from paper_2503_21596_b200 import LNormError
    with pytest.raises(LNormError) as e:
        lib.compute_device(torch.full((3, 3), 2 ** 29, dtype=torch.int32, device="cuda"))
    assert e.value.name == "EOVERFLOW"
    with pytest.raises(LNormError) as e:
        lib.compute_device(torch.ones((64, 64), dtype=torch.int32, device="cuda"))
    assert e.value.name == "ETOOLARGE"


@pytest.mark.parametrize("family,d,marg,n,m", [
    ("auto", 1, False, 16, 18),      # byte walk
    ("auto", 1, True, 15, 16),       # byte walk, L_marg
    ("auto", 3, False, 11, 12),      # byte d-ary walk
    ("pair16", 1, False, 14, 15),
    ("generic", 2, False, 9, 8),
])
@pytest.mark.parametrize("delta", [1, -1, 1000])
def test_recovery_self_check_catches_a_corrupted_key(lib, monkeypatch, family, d, marg, n, m, delta):
    """A reduced key that no strategy of the winning unit attains (delta > 0), or that a strategy
    of the unit exceeds (delta < 0), makes the call fail with EINTERNAL instead of returning a
    garbage argmax; without the hook the same input is exact."""
    from paper_2503_21596_b200 import LNormError
    M = synth.random_matrix(n, m, 71_000 + n + d)
    monkeypatch.setenv("LNORM_KERNEL", family)
    v, arg = lib.compute(M, d=d, with_marginals=marg)
    assert v == oracle.norm(M, d=d, with_marginals=marg)[0]
    monkeypatch.setenv("LNORM_TEST_CORRUPT_KEY", str(delta))
    with pytest.raises(LNormError) as e:
        lib.compute(M, d=d, with_marginals=marg)
    assert e.value.name == "EINTERNAL"
    monkeypatch.delenv("LNORM_TEST_CORRUPT_KEY")
    assert lib.compute(M, d=d, with_marginals=marg)[0] == v


def test_batch_beyond_65535_matrices(lib):
    """The batched call takes any batch size (orientation and recovery loop over the matrix index
    instead of one grid row per matrix); spot-checked against the oracle."""
    b = 70_001
    g = synth.SplitMix64(72_000)
    Ms = np.array([(g.next() % 7) - 3 for _ in range(b * 6)], dtype=np.int32).reshape(b, 2, 3)
    vals, args = lib.compute_batch(Ms)
    for i in list(range(0, b, 997)) + [b - 1, 65_535, 65_536]:
        ov, oarg = oracle.l1(Ms[i], threads=1)
        assert vals[i] == ov and list(args[i]) == list(oarg), i
    vals3, args3 = lib.compute_batch(Ms.reshape(b, 3, 2), d=3)
    for i in list(range(0, b, 1301)) + [b - 1, 65_535]:
        ov, oarg = oracle.ld(Ms[i].reshape(3, 2), 3, threads=1)
        assert vals3[i] == ov and list(args3[i]) == list(oarg), i


@pytest.mark.parametrize("d", [3, 4])
def test_batch_ld_one_launch(lib, d):
    """L_3 / L_4 batches of small matrices run as one batched launch (no per-matrix loop)."""
    Ms = np.stack([synth.random_matrix(7, 6, 73_000 + i) for i in range(300)])
    vals, args = lib.compute_batch(Ms, d=d)
    assert lib.last_stats()["units"] >= 300
    for i in range(0, 300, 7):
        ov, oarg = oracle.ld(Ms[i], d)
        assert vals[i] == ov and list(args[i]) == list(oarg)
