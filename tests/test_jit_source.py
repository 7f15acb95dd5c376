"""K1c source (jit.cpp) without a GPU: the CUDA C++ the library generates
for a program and run shape compiles with NVRTC for sm_100a in every mode
(write records into the bucket regions or into the record planes,
fuel-checked, direct commit, every read logged), for the workload
kernels, the opcode corpus and random kernels.  Semantics are checked on the
GPU (tests/test_gpu_parity.py runs every parity test under K1 and K1c)."""
import ctypes
import os

import numpy as np
import pytest

from workloads import kernels as K

NVRTC = None
for name in ("libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12"):
    try:
        NVRTC = ctypes.CDLL(name)
        break
    except OSError:
        pass


@pytest.fixture(scope="module")
def rc():
    import paper_1308_3203_b200 as pkg
    pkg.lib()
    return pkg


def nvrtc_compile(src: str) -> tuple[int, str, int]:
    prog = ctypes.c_void_p()
    assert NVRTC.nvrtcCreateProgram(ctypes.byref(prog), src.encode(), b"k1c.cu", 0, None, None) == 0
    opts = [b"--gpu-architecture=sm_100a", b"--std=c++17", b"-w"]
    arr = (ctypes.c_char_p * len(opts))(*opts)
    r = NVRTC.nvrtcCompileProgram(prog, len(opts), arr)
    n = ctypes.c_size_t()
    NVRTC.nvrtcGetProgramLogSize(prog, ctypes.byref(n))
    log = ctypes.create_string_buffer(n.value + 1)
    NVRTC.nvrtcGetProgramLog(prog, log)
    nb = ctypes.c_size_t(0)
    if r == 0:
        NVRTC.nvrtcGetCUBINSize(prog, ctypes.byref(nb))
    NVRTC.nvrtcDestroyProgram(ctypes.byref(prog))
    return r, log.value.decode(errors="replace"), nb.value


def programs():
    out = [("stencil", K.program(K.STENCIL), 1 << 20, [(1 << 20) + 2] * 2),
           ("tree", K.program(K.TREE), 1024, [1024]),
           ("fig1", K.program(K.FIG1), 8, None),
           ("cfg4", K.random_stencil_kernel(0), 65536, None),
           ("cfg4_full", K.random_stencil_kernel(3, isa="full"), 4096, None)]
    for name, src in list(K.BENIGN.items())[:3]:
        out.append((name, K.program(src), 32, None))
    rng = np.random.default_rng(7)
    for i in range(3):
        out.append((f"tiny{i}", K.random_tiny_kernel(rng), 4, None))
    return out


@pytest.mark.skipif(NVRTC is None, reason="libnvrtc not found")
@pytest.mark.parametrize("name,p,n,sizes", programs(), ids=[x[0] for x in programs()])
def test_k1c_source_compiles(rc, name, p, n, sizes):
    prog = rc.rc_load_program(p.bytecode)
    sizes = sizes or [n + 16] * prog.n_arrays
    modes = [dict(wbucket=True, narrow=True), dict(), dict(fuel=True), dict(direct=True, narrow=True),
             dict(ro_skip=False, wbucket=True)]
    for m in modes[: 5 if name in ("stencil", "tree", "tiny0") else 2]:
        src = prog.jit_source(n, sizes, **m)
        assert 'extern "C" __global__' in src and "rc_k1c" in src
        r, log, nb = nvrtc_compile(src)
        assert r == 0 and nb > 0, f"{name} {m}: {log[:2000]}"


def test_k1c_source_shape_constants(rc):
    """Operands and array geometry are immediates: the stencil's B array
    starts at cell size(A) and its bounds check is against size(B)."""
    prog = rc.rc_load_program(K.program(K.STENCIL).bytecode)
    src = prog.jit_source(1000, [1002, 1002])
    assert "cb + 1002u + (u32)idx" in src and ">= 1002u" in src
    assert "switch (pc)" in src and "case 0u:" in src
    # the first loads of an interval search no overlay (nothing stored yet)
    first_ld = src.index("pc 4\n")
    assert "oc0 == cell" not in src[first_ld:src.index("pc 5\n")]
