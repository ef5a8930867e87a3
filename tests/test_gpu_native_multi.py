"""The multi-device C-ABI entry points on one B200:
* bgx_contract_sharded (through shard.contract_devices): every slab a plain
  GEMM -> one C call launching all slabs; bit-identical to one device;
* bgx_nccl_* + bgx_ksplit_reduce (shard.NcclComm, ksplit_contract(comm=)):
  the library's own NCCL communicator at world 1 (NCCL refuses two ranks on
  one GPU; world > 1 is the same code path over NVLink), reduce-scatter and
  all-reduce forms, c0 added and cast;
* bgx_shutdown refuses while a communicator is alive."""

import pytest
import torch

import oracle
from paper_2503_04771_b200 import _lib, contract, executor, shard

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("spec,shapes,dt", [
    ("(i,k),(k,j)->(i,j)", [(1000, 320), (320, 272)], torch.bfloat16),
    ("(b,i,k),(b,k,j)->(b,i,j)", [(5, 256, 128), (5, 128, 192)], torch.bfloat16),
    ("(i,k),(k,j)->(i,j)", [(333, 70), (70, 90)], torch.float32),
    ("(k,j),(i,k)->(i,j)", [(64, 96), (500, 64)], torch.float32)])
def test_contract_devices_uses_sharded_entry(dev, spec, shapes, dt):
    g = torch.Generator(device=dev).manual_seed(3)
    ops = [torch.randn(s, generator=g, device=dev).to(dt) for s in shapes]
    want = contract(spec, *ops)
    executor.reset_launch_log()
    got = contract(spec, *ops, devices=[0, 0, 0])
    torch.cuda.synchronize()
    assert "sharded" in executor.launch_log()
    assert torch.equal(got, want)


def test_contract_devices_falls_back_for_permutations(dev):
    x = torch.randn(300, 200, device=dev)
    executor.reset_launch_log()
    y = contract("(i,j)->(j,i)", x, devices=[0, 0])
    assert "sharded" not in executor.launch_log()
    assert torch.equal(y, x.t())


def test_contract_sharded_rejects_bad_device(dev):
    lib = _lib.load()
    arr = (_lib.BgxContractDesc * 1)()
    devs = (_lib._i32 * 1)(99)
    rc = lib.bgx_contract_sharded(arr, devs, None, 1)
    assert rc == _lib.ERR_INVALID
    assert b"device 99" in lib.bgx_last_error()


@pytest.mark.parametrize("scatter", [False, True])
@pytest.mark.parametrize("out_dtype,with_c0", [(torch.float32, False), (torch.bfloat16, True),
                                               (torch.float32, True)])
def test_native_nccl_ksplit_world1(dev, scatter, out_dtype, with_c0):
    comm = shard.NcclComm()
    try:
        assert comm.world == 1 and comm.rank == 0
        g = torch.Generator(device=dev).manual_seed(7)
        a = torch.randn(256, 2048, device=dev, generator=g).bfloat16()
        b = torch.randn(2048, 384, device=dev, generator=g).bfloat16()
        c0 = torch.randn(256, 384, device=dev, generator=g).to(out_dtype) if with_c0 else None
        executor.reset_launch_log()
        y = shard.ksplit_contract("(i,k),(k,j)->(i,j)", a, b, c0=c0, out_dtype=out_dtype,
                                  scatter=scatter, comm=comm)
        torch.cuda.synchronize()
        assert "ksplit-reduce" in executor.launch_log()
        want = oracle.gemm_kseq(a.float().cpu().numpy(), b.float().cpu().numpy(),
                                c0.float().cpu().numpy() if c0 is not None else None)
        tol = 1e-5 if out_dtype == torch.float32 else 1e-2
        assert y.shape == (256, 384) and y.dtype == out_dtype
        assert oracle.rel_frobenius(y.float().cpu().numpy(), want) <= tol
    finally:
        comm.close()


def test_shutdown_waits_for_communicators(dev):
    lib = _lib.load()
    comm = shard.NcclComm()
    assert lib.bgx_shutdown() == _lib.ERR_INVALID
    comm.close()
    assert lib.bgx_shutdown() == _lib.OK
