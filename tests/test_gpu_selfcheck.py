"""GPU: the self-check build -- the byte binary walk compiled with -G and
LN_SELFCHECK=1 compares every Gray step's strategy values of one unit per lane with a
from-scratch evaluation (Eqs. 1, 2, 6 over all rows; walk_u8_impl.cuh) and fails the call with
LNORM_EINTERNAL on any difference.  Clean inputs pass with the oracle's value and argmax; an
injected offset (LNORM_SELFCHECK_INJECT) must be caught."""
import ctypes
import os

import numpy as np
import pytest

import oracle
import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import build as B
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sclib():
    path = B.SELFCHECK_OUT
    if not os.path.exists(path):
        B.build_selfcheck()
    lib = ctypes.CDLL(path)
    P = ctypes.POINTER
    lib.lnorm_compute.argtypes = [P(ctypes.c_int32), ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                  P(ctypes.c_int64), P(ctypes.c_int8)]
    lib.lnorm_compute.restype = ctypes.c_int
    lib.lnorm_last_stats.argtypes = [P(L.Stats)]
    return lib


def run(lib, M, d=1, marg=False):
    A = np.ascontiguousarray(M, dtype=np.int32)
    v = ctypes.c_int64()
    arg = np.zeros(A.shape[0], dtype=np.int8)
    rc = lib.lnorm_compute(A.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), A.shape[0], A.shape[1], d, int(marg),
                           ctypes.byref(v), arg.ctypes.data_as(ctypes.POINTER(ctypes.c_int8)))
    st = L.Stats()
    lib.lnorm_last_stats(ctypes.byref(st))
    return rc, int(v.value), arg, st.variant


@pytest.mark.parametrize("n,m,d,marg", [(13, 14, 1, False), (12, 16, 1, True), (11, 13, 2, False), (15, 15, 1, False),
                                        (14, 13, 2, False)])
def test_selfcheck_build_every_step_matches_scratch(sclib, n, m, d, marg):
    M = synth.random_matrix(n, m, 97_000 + 31 * n + m + d)
    P = L.plan(M, d=d, with_marginals=marg)
    assert P["variant_name"] == "bin_u8" and P["words"] == 4, P          # the self-checked instance
    rc, v, arg, variant = run(sclib, M, d, marg)
    assert rc == 0 and variant == 7
    ov, oa = oracle.norm(M, d=d, with_marginals=marg)
    assert v == ov and list(arg) == list(oa)


def test_selfcheck_catches_an_injected_difference(sclib):
    M = synth.random_matrix(13, 14, 97_500)
    os.environ["LNORM_SELFCHECK_INJECT"] = "1"
    try:
        rc = run(sclib, M)[0]
    finally:
        del os.environ["LNORM_SELFCHECK_INJECT"]
    assert rc == 8                                                      # LNORM_EINTERNAL
    assert run(sclib, M)[0] == 0
