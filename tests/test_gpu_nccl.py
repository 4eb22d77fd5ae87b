"""GPU: the multi-GPU code path executes on one device: real NCCL communicators
(library-made, ncclCommInitRank at world 1; torch.distributed's own; ncclCommInitAll), the
rank slice walk, the ONE ncclAllReduce(max) of {key, error flag}, and recovery -- against the
oracle.  The driver's 2/4/8-GPU runs execute the same code with world > 1."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2503_21596_b200 import synth

pytestmark = pytest.mark.gpu

CASES = [(synth.random_matrix(18, 20, 74_001), 1, False), (synth.random_matrix(16, 17, 74_002), 1, True),
         (synth.random_matrix(12, 11, 74_003), 3, False), (synth.random_matrix(20, 21, 74_004), 2, False)]


def test_library_comm_world1_runs_the_allreduce(lib):
    import torch
    dev = torch.cuda.current_device()
    c = lib.Comm(lib.Comm.unique_id(), 0, 1, dev)
    assert c.nccl != 0
    try:
        for M, d, marg in CASES:
            ov, oarg = oracle.norm(M, d=d, with_marginals=marg)
            v, arg = c.compute(M, d=d, with_marginals=marg)
            assert v == ov and list(arg) == list(oarg)
            vd, argd = c.compute_device(torch.from_numpy(M).cuda(), d=d, with_marginals=marg)
            assert vd == ov and list(argd) == list(oarg)
    finally:
        c.close()


def test_multi_single_device_uses_nccl(lib):
    for M, d, marg in CASES:
        ov, oarg = oracle.norm(M, d=d, with_marginals=marg)
        v, arg = lib.compute_multi(M, d=d, with_marginals=marg, devices=[0])
        assert v == ov and list(arg) == list(oarg)


def test_comm_rank_mismatch_rejected(lib):
    import torch
    from paper_2503_21596_b200 import LNormError
    c = lib.Comm(lib.Comm.unique_id(), 0, 1, torch.cuda.current_device())
    M = synth.random_matrix(8, 9, 74_010)
    try:
        with pytest.raises(LNormError) as e:
            lib.compute_rank(M, c.nccl, 0, 2)           # the communicator has 1 rank, not 2
        assert e.value.name == "EINVAL"
    finally:
        c.close()
    with pytest.raises(LNormError):
        lib.compute_rank(M, None, 1, 2)                 # world > 1 needs a communicator


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_torch_process_group_comm(lib):
    """The caller-owned communicator of a torch.distributed NCCL group (world 1), on the
    caller's stream: the library all-reduces through torch's ncclComm_t and never destroys it."""
    import torch
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group already exists")
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", torch.cuda.current_device())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        t = torch.ones(1, device=dev)
        dist.all_reduce(t)                              # make sure the communicator exists
        comm = lib.torch_nccl_comm()
        assert comm != 0
        stream = torch.cuda.Stream()
        for M, d, marg in CASES:
            ov, oarg = oracle.norm(M, d=d, with_marginals=marg)
            v, arg = lib.compute_rank(M, comm, 0, 1, d=d, with_marginals=marg, stream=stream)
            assert v == ov and list(arg) == list(oarg)
        dist.all_reduce(t)                              # torch's communicator is still alive
        torch.cuda.synchronize()
        assert t.item() == 1.0
    finally:
        dist.destroy_process_group()
