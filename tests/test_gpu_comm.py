"""libspx NCCL collectives (spx_comm_* / spx_gather / spx_reduce_rows, comm.py)
on one B200: one-rank communicators, so the results are checkable exactly
(NCCL refuses two ranks on one GPU; the N>1 host logic is covered by
tests/test_multirank.py over gloo)."""

from __future__ import annotations

import ctypes
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2001_00532_b200 import _lib, comm  # noqa: E402
from paper_2001_00532_b200.partition import gather_rows, reduce_partials  # noqa: E402


@pytest.fixture(scope="module")
def one():
    assert torch.cuda.is_available()
    assert comm.available(), "libnccl.so.2 not found on the GPU box"
    c = comm.Comm.single()
    yield c
    c.close()


def test_info(one):
    assert one.info() == (1, 0)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32, torch.int32])
def test_all_gather_and_reduce(one, dtype):
    g = torch.Generator(device="cpu").manual_seed(5)
    x = (torch.rand(1000, generator=g) * 100).to(dtype).cuda()
    out = torch.empty_like(x)
    one.all_gather(x, out)
    torch.cuda.synchronize()
    assert torch.equal(out, x)
    y = x.clone()
    one.all_reduce(y)
    torch.cuda.synchronize()
    assert torch.equal(y, x)


def test_gather_rows_and_reduce_partials_route_through_comm(one):
    local = torch.randn(37, 128, device="cuda", dtype=torch.float32)
    before = _lib.load()
    full = gather_rows(local, [37], comm=one)
    assert torch.equal(full, local)
    p = torch.randn(2048, 32, device="cuda", dtype=torch.float64)
    assert torch.equal(reduce_partials(p.clone(), comm=one), p)
    assert before is _lib.load()


def test_gather_rows_empty_shard(one):
    local = torch.empty(0, 8, device="cuda")
    assert gather_rows(local, [0], comm=one).shape == (0, 8)


def test_argument_errors(one):
    with pytest.raises(TypeError):
        one.all_reduce(torch.zeros(4, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        one.all_gather(torch.zeros(4, device="cuda"), torch.zeros(5, device="cuda"))
    with pytest.raises(ValueError):
        comm.Comm.init(1, 0, b"short")


def test_init_all_one_device():
    lib = _lib.load()
    comms = (ctypes.c_void_p * 1)()
    devs = (ctypes.c_int * 1)(torch.cuda.current_device())
    _lib.check(lib.spx_comm_init_all(1, devs, comms), "spx_comm_init_all")
    c = comm.Comm(comms[0], 1, 0)
    assert c.info() == (1, 0)
    x = torch.arange(10, dtype=torch.float32, device="cuda")
    _lib.check(lib.spx_comm_group(1))
    c.all_reduce(x)
    _lib.check(lib.spx_comm_group(0))
    torch.cuda.synchronize()
    assert np.array_equal(x.cpu().numpy(), np.arange(10, dtype=np.float32))
    c.close()


def test_from_process_group_single_rank():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        with comm.Comm.from_process_group() as c:
            assert (c.nranks, c.rank) == (1, 0)
            v = torch.ones(3, device="cuda")
            c.all_reduce(v)
            torch.cuda.synchronize()
            assert v.tolist() == [1.0, 1.0, 1.0]
    finally:
        dist.destroy_process_group()
