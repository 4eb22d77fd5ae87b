"""GPU: checkpoint / resume of long searches: the resumed result equals the ORACLE's
value and lexicographically smallest argmax, and every partial best is a value some strategy
attains (it never exceeds the oracle's norm)."""
import os

import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,marg,n,m", [(1, False, 24, 26), (1, True, 22, 20), (3, False, 14, 12), (2, False, 20, 18)])
def test_resume_in_chunks_matches_one_shot(lib, tmp_path, d, marg, n, m):
    M = synth.random_matrix(n, m, 90_000 + n + d)
    ref_v, ref_a = oracle.norm(M, d=d, with_marginals=marg)
    units = lib.plan(M, d=d, with_marginals=marg)["units"]
    chunk = max(1, units // 7)
    path = str(tmp_path / "ck.bin")
    calls, prev = 0, -1
    while True:
        done, v, arg, udone = lib.compute_checkpointed(M, path, d=d, with_marginals=marg,
                                                       chunk_units=chunk, max_chunks=2)
        calls += 1
        assert udone > prev
        prev = udone
        if done:
            break
        assert v <= ref_v                       # best so far never exceeds the norm
        assert os.path.exists(path)
    assert calls >= 3
    assert v == ref_v and list(arg) == list(ref_a)
    # a finished checkpoint returns the result immediately
    done, v2, arg2, udone = lib.compute_checkpointed(M, path, d=d, with_marginals=marg, chunk_units=chunk)
    assert done and v2 == ref_v and list(arg2) == list(ref_a) and udone == units


def test_fingerprint_mismatch_restarts(lib, tmp_path):
    A = synth.random_matrix(20, 20, 91_000)
    B = synth.random_matrix(20, 20, 91_001)
    path = str(tmp_path / "ck.bin")
    units = lib.plan(A)["units"]
    done, _, _, udone = lib.compute_checkpointed(A, path, chunk_units=units // 4, max_chunks=1)
    assert not done and udone == units // 4
    done, v, arg, udone = lib.compute_checkpointed(B, path)          # different matrix: starts over, one chunk
    ov, oarg = oracle.l1(B)
    assert done and v == ov and list(arg) == list(oarg)
