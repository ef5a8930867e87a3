"""C ABI checks that need no GPU: libbgx.so loads and exports exactly the
functions include/bgx.h declares; the ctypes structs match the C layout; the
UMMA shared-memory / instruction descriptor encodings match the sm_100 field
layout (restated here independently from the CUTLASS bitfield definitions in
cute/arch/mma_sm100_desc.hpp: SmemDescriptor, InstrDescriptor)."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2503_04771_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bgx.h")


def header_functions():
    text = open(HEADER).read()
    return set(re.findall(r"BGX_API\s+[\w\s\*]+?\b(bgx_\w+)\s*\(", text))


def test_header_and_binding_agree():
    assert header_functions() == set(_lib.SIGNATURES)


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (bgx_\w+)", out))
    assert exported == header_functions()
    assert lib.bgx_version() == 1


def test_error_paths_without_gpu():
    lib = _lib.load()
    d = _lib.BgxContractDesc()
    d.batch = d.M = d.N = d.K = 1
    d.in_dtype = d.out_dtype = 7  # bad dtype -> validated before any CUDA call
    assert lib.bgx_contract_kernel(d) == _lib.ERR_INVALID
    assert b"dtype" in lib.bgx_last_error()
    t = _lib.BgxTensor()
    t.rank = 2
    u = _lib.BgxTensor()
    u.rank = 3
    assert lib.bgx_permute(t, u, (_lib._i32 * 3)(0, 1, 2), None) == _lib.ERR_INVALID
    assert b"rank mismatch" in lib.bgx_last_error()
    g = _lib.BgxGenericDesc()
    g.n_in = 9
    assert lib.bgx_generic(g, None) == _lib.ERR_INVALID
    d.in_dtype = d.out_dtype = _lib.BF16
    pl = _lib.BgxRsPlan()
    assert lib.bgx_contract_rs_plan(d, 9, pl) == _lib.ERR_INVALID
    assert b"world 9" in lib.bgx_last_error()
    rs = _lib.BgxReduceScatter()
    rs.plan.world, rs.plan.rank = 2, 2
    assert lib.bgx_contract_reduce_scatter(d, rs, None) == _lib.ERR_INVALID
    assert b"null operand" in lib.bgx_last_error()


@pytest.fixture(scope="module")
def probe(tmp_path_factory):
    exe = tmp_path_factory.mktemp("abi") / "probe"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-o", str(exe),
                    os.path.join(ROOT, "tests", "abi_probe.cu")], check=True,
                   capture_output=True)
    lines = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    return {ln.split()[0]: [int(x) for x in ln.split()[1:]] for ln in lines.splitlines()}


def test_struct_layouts(probe):
    T, G, C = _lib.BgxTensor, _lib.BgxGenericDesc, _lib.BgxContractDesc
    assert probe["bgx_tensor"] == [ctypes.sizeof(T), T.shape.offset, T.stride.offset]
    assert probe["bgx_generic_desc"] == [ctypes.sizeof(G), G.ins.offset, G.c0.offset, G.out.offset]
    assert probe["bgx_contract_desc"] == [ctypes.sizeof(C), C.c0.offset, C.in_dtype.offset,
                                          C.sched.offset]
    P, R = _lib.BgxRsPlan, _lib.BgxReduceScatter
    assert probe["bgx_rs_plan"] == [ctypes.sizeof(P), P.rows_per_owner.offset, P.ws_bytes.offset]
    assert probe["bgx_reduce_scatter"] == [ctypes.sizeof(R), R.slots.offset, R.out.offset,
                                           R.ws.offset, R.ws_counters.offset]


def sdesc(addr, lbo, sbo):
    # start_address [0,14) lbo [16,30) sbo [32,46) version [46,48)=1 layout [61,64)=2 (SW128)
    return ((addr >> 4) & 0x3FFF) | (((lbo >> 4) & 0x3FFF) << 16) | \
        (((sbo >> 4) & 0x3FFF) << 32) | (1 << 46) | (2 << 61)


def idesc(bf16, a_mn, b_mn, m, n):
    # c_format [4,6)=F32; a/b format [7,10)/[10,13); a/b major [15]/[16];
    # n_dim [17,23) = N>>3; m_dim [24,29) = M>>4
    f = 1 if bf16 else 0
    return (1 << 4) | (f << 7) | (f << 10) | (a_mn << 15) | (b_mn << 16) | \
        ((n >> 3) << 17) | ((m >> 4) << 24)


def test_umma_descriptor_encodings(probe):
    assert probe["sdesc"] == [sdesc(0x12400, 16, 1024), sdesc(0x3F800, 8192, 1024)]
    assert probe["idesc"] == [idesc(1, 0, 1, 128, 256), idesc(0, 1, 0, 128, 64),
                              idesc(1, 1, 1, 256, 128)]


def test_rs_plan_sizes_follow_mode_and_split():
    """shard._finish_plan: deferred slots hold world x local_splits partial
    planes and need no local workspace; in-kernel slots hold one plane per
    rank plus a local split workspace (bgx.h bgx_rs_plan)."""
    from paper_2503_04771_b200 import shard
    pl = _lib.BgxRsPlan()
    pl.world, pl.rows_per_owner = 8, 128
    shard._finish_plan(pl, 1024, 512, 4, _lib.RS_DEFERRED)
    assert (pl.mode, pl.local_splits, pl.ws_bytes) == (_lib.RS_DEFERRED, 4, 0)
    assert pl.slot_bytes == 8 * 4 * 128 * 512 * 4
    shard._finish_plan(pl, 1024, 512, 3, _lib.RS_IN_KERNEL)
    assert pl.slot_bytes == 8 * 128 * 512 * 4 and pl.ws_bytes == 3 * 1024 * 512 * 4
    shard._finish_plan(pl, 1024, 512, 0, None)          # clamps to one slice
    assert pl.local_splits == 1 and pl.ws_bytes == 0
